"""B200-native full / low / high integer products (arxiv 1703.00640).

The hot path is the reference's float pipeline (products_f64.cpp) rebuilt as
sm_100a CUDA kernels behind the C ABI in include/truncmul_b200.h; this
package is the host-side mirror of the reference's product API.
"""
from .products import (  # noqa: F401
    Backend,
    Context,
    ConvolutionPrecisionFailure,
    CudaError,
    Error,
    InputOutOfRange,
    Mode,
    NoValidParams,
    Params,
    PlanMismatch,
    Policy,
    Stats,
    Unsupported,
    UnsupportedLength,
    cyclic_convolve_f64,
    default_context,
    default_lambda,
    from_limbs,
    full_product,
    full_product_limbs,
    high_product,
    high_product_limbs,
    low_product,
    low_product_limbs,
    manual_params,
    multiply,
    output_limbs,
    predicted_sigma,
    required_precision,
    select_params,
    split_high_i64,
    split_low_i64,
    to_limbs,
    validate_params,
)
