"""B200-native activation compressors of Adacc (arXiv 2508.00806).

A drop-in for the reference package's codec path (``actplan.codec``): the
same public names, backed by hand-written sm_100a kernels behind a C-ABI
(``include/adacc.h``).  Importing the package does not touch the GPU; the
first codec call loads ``_lib/libadacc.so`` and fails loudly if it is absent.
"""

from .codec import (
    DEFAULT_GROUP_SIZE,
    DEFAULT_Z_THRESHOLD,
    MAGIC,
    PER_CHANNEL,
    SERIALIZED_HEADER_BYTES,
    CodecReport,
    CompressedTensor,
    Int4F32Tensor,
    Int8Tensor,
    Scheme,
    SchemeSpec,
    channel_abs_sums,
    compress,
    compress_async,
    compress_outlier_separated,
    decompress,
    decompress_into,
    dequantize,
    dequantize_int4_f32,
    dequantize_int8,
    deserialize,
    detect_outlier_channels,
    measure_codec,
    outlier_separated_rate,
    pack_bitmask,
    packed_payload_bytes,
    quantize_asymmetric,
    quantize_int4_f32,
    quantize_int8,
    quantize_symmetric,
    scheme_for,
    serialize,
    serialize_device,
    unpack_bitmask,
)
from .errors import (
    ActplanError,
    CorruptPayloadError,
    NonBinaryMaskError,
    NonFiniteInputError,
    ParseError,
    TooManyOutliersError,
    ValidationError,
)
from .profiles import LayerKind, ModelProfile, OperatorProfile, load_profile, save_profile

__version__ = "0.1.0"
