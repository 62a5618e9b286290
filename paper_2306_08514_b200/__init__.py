"""B200-native SRP-map engine (arXiv 2306.08514 hot path) -- drop-in for `srpmap`.

The reference's hot-path entry points keep their names and argument lists and
run on hand-written sm_100a kernels (libsrpgpu.so, C-ABI in include/srpgpu.h):

    stft_frame, fd_gcc                     (srpmap/frontend.py)
    td_gcc_samples                         (srpmap/sampling.py)
    srp_map_exact, locate                  (srpmap/srp.py)
    lr_map                                 (srpmap/lowrank.py)
    si_map, slri_map, sspi_map             (srpmap/interpolation.py)
    evaluate_map                           (srpmap/cli.py:170-180)

Each accepts a leading frame axis and returns device tensors.  Host-side
geometry and operator fitting (float64 NumPy, uploaded once) mirror the
reference builders.  Fused chains: `gcc_frames` (samples -> cross-spectra) and
`frames_to_samples` (samples -> TD-GCC samples).  Operator caches in the
reference's SRPM format load straight into device layouts (`load_operator`).
There is no CPU fallback.
"""

from .errors import (CacheFormatError, CapacityError, ConfigError, DimensionError,
                     InvalidGeometryError, InvalidGridError, NativeLibraryError, SrpMapError)
from .cache import CacheBundle, load_cache, load_operator, operator_from_bundle, params_hash, save_cache
from .frontend import FdGcc, FrameSpec, fd_gcc, frame_window, gcc_frames, num_frames, stft_frame
from .maps import (decode_keys, evaluate_map, locate, lr_map, map_argmax, si_map, slri_map,
                   sspi_map, srp_map_exact)
from .operators import (DEFAULT_MATRIX_CAP_BYTES, FixedNnzInterp, InterpMatrix, LowRankInterp,
                        LowRankSrp, SteeringTdoa, sparse_interp_fixed, steering_operator,
                        SparseInterp, SrpMatrix, build_interp_matrix, build_srp_matrix,
                        check_capacity, low_rank_interp_from_svd, low_rank_srp_from_svd,
                        resolve_sparsity, srp_matrix_shape, truncate_low_rank, truncate_sparse,
                        truncate_sparse_fixed, truncate_sparse_streamed, truncate_srp_matrix)
from .sampling import (SampleSpec, TdGccSamples, frames_to_samples, sample_spec,
                       spectra_to_samples, td_gcc_samples)
from .scene import (CandidateGrid, MicrophoneArray, PairTable, TdoaTable, build_ff_grid,
                    build_nf_grid, enumerate_pairs, tdoa_table)

__version__ = "0.1.0"
