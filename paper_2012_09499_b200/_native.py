"""ctypes binding of ``libsrpb.so`` (the C ABI declared in ``include/srpb.h``).

There is deliberately no CPU fallback: if the library is missing or no CUDA
device is present, every hot-path call raises.  Tensors are passed as raw
device pointers (``tensor.data_ptr()``) and the current torch CUDA stream.
"""

from __future__ import annotations

import ctypes
import os

import torch

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsrpb.so")
_lib = None

#: the C ABI revision these signatures describe (include/srpb.h); load()
#: refuses a library of another revision instead of calling it with
#: mismatched arguments
ABI_VERSION = 13

c_int, c_double, c_void_p = ctypes.c_int, ctypes.c_double, ctypes.c_void_p

# name -> argtypes (restype int unless listed in _RESTYPES)
_SIGNATURES = {
    "srpb_abi_version": [],
    "srpb_last_error": [],
    "srpb_last_gcc_kernels": [],
    "srpb_tdoa_split": [c_void_p, c_int, c_void_p, c_int, c_void_p, c_void_p, c_int, c_int,
                        c_double, c_double, c_int, c_double, c_void_p, c_double, c_void_p,
                        c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "srpb_stft": [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p],
    "srpb_gcc_phat": [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_int,
                      c_double, c_double, c_void_p, c_void_p, c_void_p],
    "srpb_conventional": [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_int,
                          c_void_p, c_void_p, c_void_p],
    "srpb_conventional_general": [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int,
                                  c_void_p, c_void_p, c_void_p],
    "srpb_lattice_twiddles": [c_void_p, c_int, c_double, c_int, c_void_p, c_void_p],
    "srpb_lattice": [c_void_p, c_int, c_int, c_int, c_void_p, c_int, c_void_p, c_void_p, c_int,
                     c_void_p, c_void_p],
    "srpb_gcc_phat_split16": [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_int,
                              c_double, c_double, c_void_p, c_void_p, c_void_p, ctypes.c_float,
                              c_void_p, c_void_p],
    "srpb_gcc_floor": [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_double,
                       c_void_p, c_void_p, c_void_p],
    "srpb_lattice_from_spectra": [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_int,
                                  c_void_p, c_double, c_void_p, c_void_p, c_int, c_void_p,
                                  c_void_p, c_int, c_void_p, c_void_p, c_void_p, ctypes.c_float,
                                  c_double, c_void_p, c_void_p],
    "srpb_lattice_tc_cols": [c_int],
    "srpb_lattice_tc_supported": [c_int, c_int, c_int, c_int, c_int],
    "srpb_lattice_tc_twiddles": [c_void_p, c_int, c_double, c_int, c_void_p, c_void_p, c_void_p],
    "srpb_lattice_from_spectra_tc": [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int,
                                     c_int, c_void_p, c_double, c_void_p, c_void_p, c_int,
                                     c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                     ctypes.c_float, c_double, c_void_p, c_void_p, c_void_p,
                                     c_void_p, c_void_p],
    "srpb_sinc_table": [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_int, c_void_p,
                        c_void_p],
    "srpb_interp": [c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p],
    "srpb_interp_onthefly": [c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_int,
                             c_int, c_int, c_void_p, c_void_p, c_void_p],
    "srpb_tf32_split": [c_void_p, ctypes.c_size_t, c_void_p, c_void_p, c_void_p],
    "srpb_conventional_tc": [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                             c_int, c_void_p, c_void_p, c_int, c_void_p],
    "srpb_interp_tc": [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p,
                       c_void_p, c_int, c_void_p],
    "srpb_f16_split": [c_void_p, ctypes.c_size_t, ctypes.c_float, c_void_p, c_void_p, c_void_p],
    "srpb_conventional_tc16": [c_void_p, c_void_p, ctypes.c_float, c_int, c_int, c_int, c_int,
                               c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_int, c_void_p,
                               c_void_p, c_void_p],
    "srpb_interp_tc16": [c_void_p, c_void_p, ctypes.c_float, c_void_p, c_void_p, ctypes.c_float,
                         c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                         c_void_p],
    "srpb_interp_tc16_onthefly": [c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                  c_void_p, ctypes.c_float, c_int, c_int, c_int, c_void_p,
                                  c_void_p, c_int, c_void_p, c_void_p, c_void_p],
    "srpb_argmax": [c_void_p, c_int, c_int, c_void_p, c_void_p],
    "srpb_argmax_f64": [c_void_p, c_int, c_int, c_void_p, c_void_p],
    "srpb_argmax_keys_reset": [c_void_p, c_int, c_void_p],
    "srpb_keys_to_index": [c_void_p, c_int, c_void_p, c_void_p],
    "srpb_copy_rows_h2d": [c_void_p, ctypes.c_size_t, c_void_p, ctypes.c_size_t,
                           ctypes.c_size_t, c_int, c_void_p],
    "srpb_srp_quadform": [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_int,
                          c_void_p, c_void_p, c_void_p, c_void_p],
    "srpb_map_error": [c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p,
                       c_void_p, c_void_p],
}
_RESTYPES = {"srpb_last_error": ctypes.c_char_p}


class NativeError(RuntimeError):
    """A CUDA launch or runtime failure reported by libsrpb."""


def lib_path() -> str:
    return _LIB_PATH


def load(path: str | None = None):
    """Load and type the library (idempotent).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    # SRPB_LIB: an alternative build of the same ABI (tuning experiments)
    path = path or os.environ.get("SRPB_LIB") or _LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"libsrpb.so not found at {path}; build it with `make` or "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
        )
    lib = ctypes.CDLL(path)
    lib.srpb_abi_version.argtypes = []
    lib.srpb_abi_version.restype = c_int
    got = int(lib.srpb_abi_version())
    if got != ABI_VERSION:
        raise ImportError(f"{path} implements C ABI v{got}, this package binds v{ABI_VERSION}; "
                          "rebuild it (make)")
    for name, argtypes in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, c_int)
    _lib = lib
    return lib


def exported_symbols():
    return tuple(_SIGNATURES)


def ptr(t):
    """Device pointer of a tensor (or 0 for None)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("hot-path tensors must live on a CUDA device")
    if not t.is_contiguous():
        raise ValueError("hot-path tensors must be contiguous (row-major)")
    return t.data_ptr()


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle(device=None):
    """``cudaStream_t`` of torch's current stream on ``device`` (an int).
    The raw getter skips the Stream object the public call builds (several
    lookups per frame on the per-frame drop-in path)."""
    if _raw_stream is not None:
        idx = getattr(device, "index", None) if device is not None else None
        if isinstance(device, int):
            idx = device
        if idx is None:
            if device is not None and not isinstance(device, torch.device):
                return torch.cuda.current_stream(device).cuda_stream
            idx = torch.cuda.current_device()
        return _raw_stream(idx)
    return torch.cuda.current_stream(device).cuda_stream


_LAUNCHING = {n for n in _SIGNATURES if n not in ("srpb_abi_version", "srpb_last_error",
                                                   "srpb_last_gcc_kernels",
                                                   "srpb_lattice_tc_cols",
                                                   "srpb_lattice_tc_supported",
                                                   "srpb_copy_rows_h2d")}
# entry points that launch more than one kernel (speculative-floor lattice +
# its fix-up pass); the GCC-PHAT entries report theirs (srpb_last_gcc_kernels)
_KERNELS_PER_CALL = {"srpb_lattice_from_spectra": 2, "srpb_lattice_from_spectra_tc": 2,
                     "srpb_map_error": 2}
_GCC = ("srpb_gcc_phat", "srpb_gcc_phat_split16")
_launches = 0


def launch_count() -> int:
    """Kernel launches issued through the C ABI by this process so far."""
    return _launches


def note_launches(n: int) -> None:
    """Correct the launch tally for an entry whose kernel count depends on
    its arguments (added to the per-call default)."""
    global _launches
    _launches += int(n)


def query(name, *args) -> int:
    """Call a non-launching query entry and return its integer result."""
    return int(getattr(load(), name)(*args))


def call(name, *args):
    """Invoke ``name`` and translate its status code.

    <0 -> ValueError (invalid argument, nothing launched);
    >0 -> NativeError (CUDA error from the launch).
    """
    global _launches
    lib = load()
    rc = getattr(lib, name)(*args)
    if name in _GCC:
        _launches += int(lib.srpb_last_gcc_kernels()) if rc == 0 else 0
    elif name in _LAUNCHING:
        _launches += _KERNELS_PER_CALL.get(name, 1)
    if rc != 0:
        msg = lib.srpb_last_error().decode(errors="replace")
        if rc < 0:
            raise ValueError(msg)
        raise NativeError(msg)
    return rc


def on_device(device):
    """Context in which launches go to ``device``: libsrpb launches on the
    current CUDA device with the stream passed in, so a plan living on a
    non-current GPU switches to it for its calls."""
    return torch.cuda.device(device)


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2012_09499_b200 needs a CUDA device (B200); there is no CPU fallback"
        )
    load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    return dev
