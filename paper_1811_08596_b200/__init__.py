"""B200-native SuperNeurons gradient compression (arXiv 1811.08596).

A drop-in for the reference package ``fgc``'s hot path
(pkg/src/fgc/__init__.py:3-61): the same names, signatures, defaults and
error classes for the codec (FFT sparsification + range-float quantization +
stream compaction + FGC1 wire format) and the compressed gradient average,
executed by hand-written sm_100a CUDA kernels behind a C ABI
(include/fgc_b200.h, libfgc_b200.so).  There is no CPU fallback: without a
CUDA device every data-path call raises.
"""

from ._lib import (BitmapMismatchError, CodecFormatError, CorruptHeaderError, NativeError,
                   TruncatedPayloadError, kernel_launches)
from .quantizer import (QuantizerConfig, tune_eps, encode, decode, encode_array, decode_array,
                        encode_block, decode_block, pack_codes, unpack_codes)
from .spectral import (Spectrum, SparsificationSpec, dft_forward, dft_inverse, truncate,
                       half_round_trip, bin_weights, spectrum_energy)
from .packer import PackedSparse, pack, unpack, prefix_sum, bitmap_to_bytes, bitmap_from_bytes
from .codec import (CodecConfig, ChunkPayload, CompressedMessage, compress, decompress, reconstruct,
                    reconstruct_rows, serialize, deserialize, calibrate, compression_ratio)
from .comm import GradientAverager, NcclComm, PeerExchange, allgather_average, message_layout, shard_weights
from .simulator import (QuadraticProblem, LogisticProblem, MlpProblem, make_problem, LrSchedule, ThetaSchedule,
                        TrainConfig, ConvergenceTrace, sub_gradient, step, run, gradient_stats)

__version__ = "0.1.0"
