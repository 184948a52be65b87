"""Device-side map metrics.

``approximation_error_db`` restates ``metrics.approximation_error_db``
(``pkg/src/srpfast/metrics.py:22-41``): ``10 log10(sum (ref - approx)^2 /
sum ref^2)``, floored at :data:`APPROX_ERROR_FLOOR_DB`, with the reference's
validation errors.  The energies are reduced on the GPU by ``srpb_map_error``
(fp64 accumulation, fixed order), so whole [F, J] batches of device maps --
e.g. approximate vs conventional at full C2-C5 scale -- are scored without
copying them to the host.  Only the per-frame scalar ratio is finished here.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N

__all__ = ["APPROX_ERROR_FLOOR_DB", "approximation_error_db", "map_error_energy"]

#: reported instead of -inf when the approximation is numerically exact
APPROX_ERROR_FLOOR_DB = -300.0

_SCRATCH_PER_FRAME = 128  # SRPB_MAP_ERROR_SCRATCH (include/srpb.h)


def _as_device_map(x, dev):
    """SrpMap / tensor / array -> contiguous fp32 or fp64 device tensor."""
    if hasattr(x, "device_values"):
        row = x.device_values()
        x = row if row is not None else x.values
    elif hasattr(x, "values") and not isinstance(x, (np.ndarray, torch.Tensor)):
        x = x.values
    if isinstance(x, torch.Tensor):
        t = x.to(dev)
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        return t.contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)), device=dev)


def map_error_energy(reference, approximate):
    """Per-frame ``(sum (ref - app)^2, sum ref^2)`` as fp64 device tensors
    [F] for maps of shape [J] or [F, J]."""
    dev = N.require_cuda()
    ref = _as_device_map(reference, dev)
    app = _as_device_map(approximate, dev)
    if tuple(ref.shape) != tuple(app.shape):
        raise ValueError(f"map sizes differ: {tuple(ref.shape)} vs {tuple(app.shape)}")
    if ref.dim() == 1:
        ref, app = ref[None], app[None]
    if ref.dim() != 2 or ref.shape[1] == 0:
        raise ValueError(f"maps must be [J] or [F, J] with J >= 1, got {tuple(ref.shape)}")
    F, J = ref.shape
    scratch = torch.empty(max(F, 1) * _SCRATCH_PER_FRAME, dtype=torch.float64, device=dev)
    num = torch.empty(F, dtype=torch.float64, device=dev)
    den = torch.empty(F, dtype=torch.float64, device=dev)
    N.call("srpb_map_error", N.ptr(ref), int(ref.dtype == torch.float64), N.ptr(app),
           int(app.dtype == torch.float64), F, J, N.ptr(scratch), N.ptr(num), N.ptr(den),
           N.stream_handle(dev))
    return num, den


def _db(num: float, den: float) -> float:
    if den == 0.0:
        raise ValueError("reference map is identically zero")
    if num == 0.0:
        return APPROX_ERROR_FLOOR_DB
    return max(APPROX_ERROR_FLOOR_DB, 10.0 * math.log10(num / den))


def approximation_error_db(reference, approximate):
    """Relative energy of the map error in dB (``metrics.py:22-41``).

    One map (SrpMap or vector) returns a float like the reference; a batch
    ``[F, J]`` returns a float64 array of per-frame values.
    """
    batched = getattr(getattr(reference, "shape", ()), "__len__", lambda: 0)() == 2
    num, den = map_error_energy(reference, approximate)
    num, den = num.cpu().numpy(), den.cpu().numpy()
    out = np.array([_db(float(a), float(b)) for a, b in zip(num, den)])
    return out if batched else float(out[0])
