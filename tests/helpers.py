"""Shared helpers for the parity tests."""

import numpy as np

#: north-star tolerance for the fp32 path (BASELINE.json north_star)
REL_L2_TOL = 1e-5


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def top2_margin(values):
    """Relative gap between the best and second-best value of a map."""
    v = np.sort(np.asarray(values, dtype=np.float64))[::-1]
    scale = max(np.max(np.abs(v)), 1e-300)
    return float((v[0] - v[1]) / scale) if v.size > 1 else np.inf


#: reference top-2 gaps below this (relative to the map scale) are ties at
#: fp64 rounding (e.g. mirror-symmetric candidates); an fp32 map cannot order
#: them, so only there may the argmax differ
TIE_REL = 1e-9


def assert_maps_match(gpu, ref, argmax_gpu, tol=REL_L2_TOL, what=""):
    """Per-frame rel-L2 <= tol and identical argmax (lowest index on ties,
    BASELINE north_star).  The only argmax difference accepted is between
    candidates the reference itself scores equal to fp64 rounding
    (gap <= TIE_REL of the map scale).  Returns the worst rel-L2."""
    gpu = np.atleast_2d(np.asarray(gpu, dtype=np.float64))
    ref = np.atleast_2d(np.asarray(ref, dtype=np.float64))
    assert gpu.shape == ref.shape, (gpu.shape, ref.shape)
    worst = 0.0
    for f in range(ref.shape[0]):
        e = rel_l2(gpu[f], ref[f])
        worst = max(worst, e)
        assert e <= tol, f"{what} frame {f}: rel-L2 {e:.3e} > {tol:.0e}"
        ra = int(np.argmax(ref[f]))
        ga = int(argmax_gpu[f])
        if ga != ra:
            gap = (ref[f][ra] - ref[f][ga]) / max(np.max(np.abs(ref[f])), 1e-300)
            assert gap <= TIE_REL, (
                f"{what} frame {f}: argmax {ga} != reference {ra} (reference gap {gap:.3e}, "
                f"top-2 margin {top2_margin(ref[f]):.3e})"
            )
    return worst
