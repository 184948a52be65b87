"""B200-native SRP-map hot path of arXiv 2012.09499 (drop-in for ``srpfast``).

GCC-PHAT cross-spectra -> {conventional SRP | Nyquist lattice IDFT + sinc
interpolation} -> per-frame argmax, as hand-written sm_100a CUDA kernels in
``libsrpb.so`` (C ABI: ``include/srpb.h``) driven from PyTorch host code.

The public names mirror the reference's hot-path API
(``pkg/src/srpfast/__init__.py:13-66``: geometry inputs, spectral and srp
functions and types); :class:`SrpPlan` is the batched device-resident entry.
There is no CPU fallback: without the library and a CUDA device the compute
functions raise.
"""

from .geometry import (
    CandidateGrid,
    MicArray,
    MicPair,
    build_tdoa_table,
    circular_array,
    enumerate_pairs,
    tdoa_farfield,
    tdoa_nearfield,
)
from .distributed import ShardedRunner, run_candidate_sharded, run_frame_sharded
from .metrics import APPROX_ERROR_FLOOR_DB, approximation_error_db, map_error_energy
from .pipeline import ChunkedRunner, chunk_bounds
from .plan import CapturedStep, SrpPlan, lattice_layout, standalone_argmax
from .spectral import (
    DEFAULT_PHAT_FLOOR_REL,
    CrossSpectra,
    FrameSpec,
    SpectralFrame,
    cross_spectrum,
    cross_spectrum_frames,
    stft_analyze,
    stft_frames,
)
from .srp import (
    ComplexityReport,
    GccLattice,
    MultCounter,
    SincTable,
    SrpMap,
    argmax_candidate,
    build_gcc_lattice,
    build_gcc_lattice_frames,
    complexity_report,
    gcc_at_lag,
    lattice_half_counts,
    precompute_sinc_table,
    srp_approx,
    srp_approx_frames,
    srp_conventional,
    srp_conventional_frames,
    srp_oracle,
    srp_oracle_frames,
)

__version__ = "0.1.0"

__all__ = [
    "CapturedStep",
    "ChunkedRunner",
    "ShardedRunner", "run_frame_sharded", "run_candidate_sharded",
    "chunk_bounds",
    "CandidateGrid", "MicArray", "MicPair", "build_tdoa_table", "circular_array",
    "enumerate_pairs", "tdoa_farfield", "tdoa_nearfield",
    "SrpPlan", "lattice_layout", "standalone_argmax",
    "DEFAULT_PHAT_FLOOR_REL", "CrossSpectra", "FrameSpec", "SpectralFrame", "cross_spectrum",
    "cross_spectrum_frames", "stft_analyze", "stft_frames",
    "ComplexityReport", "GccLattice", "MultCounter", "SincTable", "SrpMap",
    "argmax_candidate", "build_gcc_lattice", "build_gcc_lattice_frames", "complexity_report",
    "gcc_at_lag", "lattice_half_counts", "precompute_sinc_table", "srp_approx",
    "srp_approx_frames", "srp_conventional", "srp_conventional_frames", "srp_oracle",
    "srp_oracle_frames", "APPROX_ERROR_FLOOR_DB", "approximation_error_db", "map_error_energy",
    "__version__",
]
