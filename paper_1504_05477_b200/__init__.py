"""B200-native randomized block-Krylov / simultaneous-iteration partial SVD.

Drop-in for the hot path of rsvdkit 0.1.0 (Musco & Musco, arXiv 1504.05477):
the names below keep the reference's signatures and semantics
(rsvdkit/__init__.py:59-70 for the algorithms, matrix.py for the containers,
errors.py for the exception types). Compute runs in librsvd_b200.so
(hand-written sm_100a CUDA behind the C ABI in include/rsvd_b200.h); there is
no CPU fallback.
"""

import warnings as _warnings

# The reference's containers hand out read-only arrays (DenseMatrix.data,
# SparseMatrixCSR.values ...); this package only ever uploads them, so torch's
# one-time "array is not writable" warning on torch.from_numpy is noise here.
_warnings.filterwarnings("ignore", message="The given NumPy array is not writable", category=UserWarning)

from . import metrics  # noqa: F401,E402  (GPU parity metrics)
from .backend import active_backend  # backend.py:31-36
from .experiment import ExperimentSpec, OracleSpectrum, oracle_spectrum, rows_to_csv, run_experiment  # f4
from .io import load_dense_csv, load_matrix_market, write_dense_csv, write_matrix_market  # f3
from .metrics import (AdditiveSpectralCheck, ErrorReport, additive_spectral_check, compute_error_report, error_function, frob_error_ratio, per_vector_errors,
                      spectral_error_ratio)
from .errors import ConvergenceError, ParseError
from .factor import (EigResult, SvdResult, dense_svd_reference, qr_orthonormalize,  # factor.py's entry points
                     spectral_norm_est, spectral_norm_max_restarts, symmetric_eig)
from .matrix import (DenseMatrix, MatrixOperator, SeededRng, SparseMatrixCSR, as_dense_array, as_operator,
                     frobenius_norm_sq, gaussian, matmul, spmm)
from .synth import SyntheticSpec, synth_matrix
from .rsvd import (
    PartialSvdResult,
    RsvdConfig,
    Variant,
    block_krylov,
    derive_q,
    derive_q_gap,
    factorize,
    post_process,
    simultaneous_iteration,
    sketch_and_solve,
)

__version__ = "0.1.0"

__all__ = [
    "active_backend",
    "ExperimentSpec",
    "OracleSpectrum",
    "oracle_spectrum",
    "rows_to_csv",
    "run_experiment",
    "load_dense_csv",
    "load_matrix_market",
    "write_matrix_market",
    "write_dense_csv",
    "ErrorReport",
    "compute_error_report",
    "AdditiveSpectralCheck",
    "additive_spectral_check",
    "error_function",
    "frob_error_ratio",
    "per_vector_errors",
    "spectral_error_ratio",
    "SyntheticSpec",
    "synth_matrix",
    "ConvergenceError",
    "EigResult",
    "SvdResult",
    "dense_svd_reference",
    "spectral_norm_est",
    "spectral_norm_max_restarts",
    "qr_orthonormalize",
    "symmetric_eig",
    "ParseError",
    "DenseMatrix",
    "SparseMatrixCSR",
    "SeededRng",
    "as_dense_array",
    "MatrixOperator",
    "as_operator",
    "matmul",
    "spmm",
    "frobenius_norm_sq",
    "gaussian",
    "PartialSvdResult",
    "RsvdConfig",
    "Variant",
    "block_krylov",
    "derive_q",
    "derive_q_gap",
    "factorize",
    "post_process",
    "simultaneous_iteration",
    "sketch_and_solve",
]
