"""B200-native dense integer polynomial multiplication (arXiv 1612.05778).

Drop-in for the reference package `twoconv`'s multiply path: the same public
names (tc/__init__.py:10-54) -- `IntPolynomial`, `MulRequest`, `multiply`,
`multiply_with_stats`, `StageTimings`, the planning API and the error types --
with the arithmetic in hand-written sm_100a CUDA kernels (libtcgpu.so, C-ABI in
include/tc_api.h) called through ctypes.  No CPU fallback exists.
"""

from .errors import (BenchMismatchError, CorruptedConvolutionError, DeviceError, EmptyInputError,
                     EncodingError, ParityError, PolynomialParseError, PrimeCapacityError,
                     RootOrderError, TransformLengthError)
from .multiplier import MulRequest, StageTimings, multiply, multiply_with_plan, multiply_with_stats
from .params import (FermatPrimeEntry, GpuPlan, MulPlan, PrimeSpec, build_plan, determine_base,
                     fermat_prime_table, fourier_prime_table, gpu_prime_table, plan_for,
                     plan_from_shape, plan_gpu, recovery_primes)
from .zpoly import IntPolynomial, format_polynomial, parse_polynomial, product_bit_width

__version__ = "0.1.0"

__all__ = [
    "BenchMismatchError", "CorruptedConvolutionError", "DeviceError", "EmptyInputError",
    "EncodingError", "FermatPrimeEntry", "GpuPlan", "IntPolynomial", "MulPlan", "MulRequest",
    "ParityError", "PolynomialParseError", "PrimeCapacityError", "PrimeSpec", "RootOrderError",
    "StageTimings", "TransformLengthError", "build_plan", "determine_base", "fermat_prime_table",
    "format_polynomial", "fourier_prime_table", "gpu_prime_table", "multiply", "multiply_with_plan",
    "multiply_with_stats", "parse_polynomial", "plan_for", "plan_from_shape", "plan_gpu",
    "product_bit_width", "recovery_primes", "__version__",
]
