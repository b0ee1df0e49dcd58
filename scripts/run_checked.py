"""Run the GPU test-suite on the PDD_CHECKED build of libpdd (bounds checks of the kernels' own
making on every shared-memory address of the sweeps and on tile / queue indices; the pool has no
compute-sanitizer) and report the number of violations counted on the device."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import pytest
from paper_1502_01629_b200 import _native

_native.use_library(os.path.join(ROOT, "build", "ab", "checked", "libpdd.so"))
# negative control: a deliberately failing check must be counted (and an in-range one must not)
L0 = _native.lib()
o0 = (ctypes.c_ulonglong * 2)()
L0.pdd_dev_faults(o0)
L0.pdd_dev_fault_selftest()
L0.pdd_dev_faults(o0)
assert (o0[0], o0[1]) == (1, 99), ("the checked build does not count violations", o0[0], o0[1])
print("negative control ok: 1 violation counted (code 99)")
args = sys.argv[1:] or ["tests", "-m", "gpu", "-q", "-x", "-k", "not fullsize"]
rc = pytest.main(args)
L = _native.lib()
out = (ctypes.c_ulonglong * 2)()
L.pdd_dev_faults(out)
print(f"pytest rc={int(rc)}; bounds violations counted by the checked kernels: {out[0]} (first code {out[1]})")
sys.exit(int(rc) or (1 if out[0] else 0))
