"""B200-native dashSVD hot path (arXiv 2404.09276): randomized truncated SVD of
sparse CSR matrices with dynamically shifted power iteration and PVE accuracy
control, computed by sm_100a kernels behind the C ABI in include/dashsvd_b200.h.

The public surface mirrors the reference library's dashsvd:: namespace; see
``api`` for the mapping.
"""
from . import errors
from .api import (Algorithm, assemble, eps_sigma, load_dense_array, load_reference_spectrum, write_dense_array,
                  write_reference_spectrum, load_cache, load_matrix_market, read_matrix_market_triplets, save_cache, write_matrix_market, Device, DeviceMatrix, EigenPair, IterationState, Orthonormalizer,
                  ShiftTrace, SolveResult, SolverConfig, SparseMatrix, StopReason, TruncatedSvd,
                  basic_rsvd, comm_unique_id, dash_svd, default_device, eig_svd, eps_pve, eps_res,
                  eps_spec, finalize_row_basis, gaussian_matrix, gaussian_rows, gram, LoopbackGroup, matmul, max_triplet_residual,
                  pin, powerlaw, pve_stop_check, rmat,
                  shifted_rsvd, solve, sparse_random, splitmix64_at, spmm, spmm_shift, sym_eig,
                  transpose, unpin, update_shift, validate_config)
from .errors import (ConfigError, DegenerateReference, DeviceError, Error, NumericalError, RankDeficient,
                     ParseError, ShapeError, UnsupportedFormat, UnsupportedOnDevice)

__all__ = [n for n in dir() if not n.startswith("_")]
