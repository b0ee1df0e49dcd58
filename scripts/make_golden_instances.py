"""Write tests/golden/instances.txt: per BASELINE config, the target-node count and the SHA-256
fingerprint of the instance built by pdd_inputs (problem data only; no oracle, no CUDA path).
The counts are also pinned independently in tests/test_oracle_labels.py by the lattice-point
count of the disc (reading R7)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import pdd_inputs as I  # noqa: E402

lines = ["# instance pins written by scripts/make_golden_instances.py (pdd_inputs only)",
         "# targets_<cfg>: target nodes of the full-size config (reading R7, lattice rule)",
         "# fingerprint_<cfg>: Instance.fingerprint() of make_config(<cfg>) (SHA-256 of every array)"]
for cfg in ("C1", "C2", "C3", "C4", "C5"):
    t = time.time()
    inst = I.make_config(cfg)
    lines.append(f"targets_{cfg} {int(np.count_nonzero(inst.kind == I.KIND_TARGET))}")
    lines.append(f"fingerprint_{cfg} {inst.fingerprint()}")
    print(cfg, f"{time.time() - t:.1f} s", file=sys.stderr)
with open(os.path.join(ROOT, "tests", "golden", "instances.txt"), "w") as f:
    f.write("\n".join(lines) + "\n")
