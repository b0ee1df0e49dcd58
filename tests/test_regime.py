"""The upwind diffusion ball analysis exposed by libpdd (pdd_regime_analyse), pinned
to what the paper prints: the eps thresholds dx/4 and dx/120 and the bold / non-bold pattern of
its Tables 1 and 2 (tests/golden/paper_regime_tables.txt), plus the closed-form properties the
text states (alpha = 1/(1+Upsilon) lies strictly between the two bounds exactly when the
condition holds).  Host arithmetic only: no GPU."""
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_regime_tables.txt")
DXS = (0.02, 0.01, 0.005, 0.0025)
FMINMAX = {"T1": (1.0, 1.0), "T2": (1.0 / 6.0, 1.5)}


@pytest.fixture(scope="module")
def ra():
    from paper_1502_01629_b200 import build as B
    B.build()
    from paper_1502_01629_b200 import regime_analyse
    return regime_analyse


def _rows():
    thr, cells = {}, []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        t = line.split()
        if t[0] == "thr":
            thr[t[1]] = [float(v) for v in t[2:]]
        else:
            cells.append((t[0], float(t[1]), [int(v) for v in t[2:]]))
    return thr, cells


def test_thresholds_printed_in_the_paper(ra):
    thr, _ = _rows()
    for tab, (fmin, fmax) in FMINMAX.items():
        for dx, want in zip(DXS, thr[tab]):
            r = ra(fmin, fmax, 0.0, dx)
            assert math.isclose(r["eps_threshold"], want, rel_tol=1e-12)
    assert ra(1 / 6, 1.5, 0.0, 0.02)["upsilon"] == pytest.approx(9.0, rel=1e-15)


def test_bold_pattern_of_tables_1_and_2(ra):
    _, cells = _rows()
    assert len(cells) == 22
    for tab, eps, bold in cells:
        fmin, fmax = FMINMAX[tab]
        got = [int(ra(fmin, fmax, math.sqrt(2.0 * eps), dx)["hyperbolic"]) for dx in DXS]
        assert got == bold, (tab, eps, got, bold)


@pytest.mark.parametrize("ups", [1.0, 2.5, 9.0])
def test_alpha_window(ra, ups):
    """Condition (hyperbolicity) <=> alpha_lo < alpha_hi, and alpha = 1/(1+Upsilon) is inside the
    window whenever it holds; the window closes at 1/(omega dx) = 1/(1+Upsilon)."""
    dx, fmin = 0.01, 1.0
    for s in np.linspace(0.02, 0.98, 25) / (1.0 + ups):      # s = 1/(omega dx) below threshold
        sig = math.sqrt(s * dx * fmin)
        r = ra(fmin, ups * fmin, sig, dx)
        assert r["hyperbolic"]
        assert r["alpha_lo"] < r["alpha"] < r["alpha_hi"]
        assert r["alpha"] == pytest.approx(1.0 / (1.0 + ups))
        assert r["h"] == pytest.approx(dx / ((1.0 + ups) * fmin))
        # both bounds of the text hold with h = alpha dx / f_min (Eqs. upper-bound, lower-bound)
        h = r["h"]
        assert h * ups * fmin + sig * math.sqrt(h) < dx
        assert h * fmin - sig * math.sqrt(h) > 0.0
    for s in np.linspace(1.05, 4.0, 12) / (1.0 + ups):       # above threshold
        sig = math.sqrt(s * dx * fmin)
        r = ra(fmin, ups * fmin, sig, dx)
        assert not r["hyperbolic"]
        assert r["alpha_hi"] <= r["alpha_lo"] * (1 + 1e-12)
        h = r["h"]
        assert h * ups * fmin + sig * math.sqrt(h) < dx       # the upper bound is kept
    # at the threshold the two bounds meet at 1/(1+Upsilon)
    s = 1.0 / (1.0 + ups)
    r = ra(fmin, ups * fmin, math.sqrt(s * dx * fmin), dx)
    assert r["alpha_hi"] == pytest.approx(1.0 / (1.0 + ups), rel=1e-9)
    assert r["alpha_lo"] == pytest.approx(1.0 / (1.0 + ups), rel=1e-12)


def test_no_diffusion_is_hyperbolic(ra):
    r = ra(0.5, 2.0, 0.0, 0.01)
    assert r["hyperbolic"] and r["alpha_lo"] == 0.0 and r["alpha_hi"] == pytest.approx(0.25)
    assert r["alpha"] == pytest.approx(0.2)


def test_invalid_arguments(ra):
    from paper_1502_01629_b200 import PddError
    with pytest.raises(PddError):
        ra(0.0, 1.0, 0.1, 0.01)
    with pytest.raises(PddError):
        ra(2.0, 1.0, 0.1, 0.01)


def test_generator_time_step_matches_analyser(ra):
    """pdd_inputs.paper_time_step (problem data, written independently) and the library's
    pdd_regime_analyse give the same h = alpha dx / f_min on both sides of the threshold."""
    import pdd_inputs as I
    for problem, (fmin, fmax) in I.PAPER_FMINMAX.items():
        for dx in (0.02, 0.005):
            for eps in (0.0, 1e-6, 1e-4, 2.5e-3, 1e-2):
                h = I.paper_time_step(dx, eps, fmin, fmax)
                r = ra(fmin, fmax, math.sqrt(2.0 * eps), dx)
                assert h == pytest.approx(r["h"], rel=1e-12), (problem, dx, eps)
