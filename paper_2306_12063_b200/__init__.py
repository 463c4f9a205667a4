"""paper_2306_12063_b200 -- B200-native batched QC-LDPC codec (sm_100a).

Drop-in for the reference package `qcldpc` on its hot path (layered
single-scan min-sum decoding, float32 and wrap-around int16, plus the packed
direct encoder) for the IEEE 802.11 (Wi-Fi) and 802.16 (WiMAX) codes.  The
host side keeps the reference API; the work runs in libqcb200.so
(csrc/*.cu, C ABI in include/qcb200.h) with no CPU fallback.
"""

from .codebook import (NB, WIFI_RATES, WIFI_Z, WIMAX_Z, ModelMatrix, Rate,
                       SparseParityCheck, Standard, expand, get_model_matrix,
                       parse_rate, parse_standard, scale_model_matrix,
                       supported_codes)
from .decoder import (Arithmetic, DecodeResult, DecoderConfig, DecoderState,
                      LlrBlock, code_handle, decode, decode_batch, decode_block,
                      decode_grouped, init_state, quantize_llr, row_parities,
                      syndrome_check, tier_update)
from .encoder import (EncoderPlan, EncoderVariant, bytes_to_words,
                      cyclic_shift_inverse, cyclic_shift_packed,
                      default_word_bits, encode, encode_array, encode_bits, encode_packed,
                      find_y, make_plan, pack_bits, unpack_bits, words_to_bytes)
from .errors import (ArithmeticMismatch, BadZ, CodecError, CorruptFile,
                     DeviceError, DivByZeroSigma, MalformedHb,
                     NativeLibraryError, SizeMismatch, UnsupportedCode,
                     UnsupportedZ)

from . import channel, llrio  # noqa: E402  (device channel / waterfall, LLR0 + records)
from .channel import (ChannelConfig, ThroughputReport, WaterfallPoint,
                      WaterfallTable, ebn0_to_sigma2, run_throughput_bench,
                      run_waterfall)
from .llrio import decode_llr_file, read_llr_file, write_llr_file

__version__ = "0.2.0"
