"""B200-native EDPC compression hot path (arXiv 2507.18969).

Drop-in for the reference package's compress/decompress path
(`pkg/src/edpc/__init__.py:24-41`): same public names and signatures, with
the predictor, its online backward + Adam update, the quantizer and the
arithmetic coder running as hand-written sm_100a CUDA kernels behind the C
ABI in ``include/edpc_b200.h`` (library: ``_edpc_b200.so``).  There is no CPU
fallback: compute calls fail loudly without the library or a GPU.
"""

from .coder import (ArithmeticDecoder, ArithmeticEncoder, CoderError, QuantizedDistribution,
                    TOTAL, quantize, quantize_rows, uniform_distribution)
from .config import (ModelConfig, dense_mixer_param_count, lte_param_count, model_param_count,
                     model_param_count_dense_mixer, param_layout)
from .container import (BadMagicError, BadVersionError, ChecksumError, ContainerError,
                        EdpcContainer, FORMAT_VERSION, Header, InvalidHeaderError,
                        TruncatedError, header_size, read_container, write_container)
from .archive import (ArchiveHeader, compress_chunked, decompress_chunked, is_archive,
                      read_archive, write_archive)
from .lanes import LaneSplit, join_lanes, split_lanes
from .model import EdpcModel
from .pipeline import compress, decompress

__version__ = "0.1.0"

__all__ = [
    "ArithmeticDecoder", "ArithmeticEncoder", "CoderError", "QuantizedDistribution", "TOTAL",
    "quantize", "quantize_rows", "uniform_distribution",
    "ModelConfig", "model_param_count", "lte_param_count", "dense_mixer_param_count",
    "model_param_count_dense_mixer", "param_layout",
    "ContainerError", "BadMagicError", "BadVersionError", "ChecksumError", "TruncatedError",
    "InvalidHeaderError", "EdpcContainer", "Header", "FORMAT_VERSION", "header_size",
    "read_container", "write_container",
    "LaneSplit", "split_lanes", "join_lanes", "EdpcModel", "compress", "decompress",
    "ArchiveHeader", "compress_chunked", "decompress_chunked", "is_archive", "read_archive",
    "write_archive",
]
