/*
 * fgc_b200 -- C ABI of the B200-native SuperNeurons gradient codec
 * (FFT sparsification + range-float quantization + compressed allgather
 * average, arXiv 1811.08596).
 *
 * The reference (`fgc`, /root/reference/pkg/src/fgc) is a pure Python/numpy
 * package with no FFI layer; its drop-in boundary is the Python API of
 * pkg/src/fgc/__init__.py:3-61.  Every entry point below is what a binding of
 * that API needs underneath: plain pointers (device pointers unless noted),
 * sizes, scalars and a cudaStream_t / ncclComm_t passed as `void*`.  No torch
 * types appear here.  Each function cites the reference interface it replaces.
 *
 * Conventions
 *   - Functions return an fgc_status (0 = ok).  Data-dependent failures that
 *     the reference raises as ValueError (non-finite gradient, binary16
 *     overflow) are reported through a device `uint32_t* flags` word that the
 *     caller reads after synchronising the stream (FGC_FLAG_*).
 *   - Device pointers must stay valid until the stream work completes.
 *   - A plan owns device scratch and is NOT safe for concurrent use on two
 *     streams at once.  Plans are otherwise immutable and thread-agnostic.
 *   - No function allocates device memory except fgc_plan_create.
 */
#ifndef FGC_B200_H
#define FGC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fgc_status {
  FGC_OK = 0,
  FGC_ERR_INVALID = 1,      /* bad argument / config (ValueError)                 */
  FGC_ERR_UNSUPPORTED = 2,  /* valid for the reference, not implemented on GPU   */
  FGC_ERR_CUDA = 3,         /* CUDA runtime error (see fgc_last_error)            */
  FGC_ERR_NCCL = 4,         /* NCCL error                                         */
  FGC_ERR_HEADER = 5,       /* CorruptHeaderError      (codec.py:80-81)           */
  FGC_ERR_TRUNCATED = 6,    /* TruncatedPayloadError   (codec.py:84-85)           */
  FGC_ERR_BITMAP = 7,       /* BitmapMismatchError     (codec.py:88-89)           */
  FGC_ERR_FORMAT = 8,       /* CodecFormatError, e.g. trailing bytes (codec.py:76)*/
  FGC_ERR_NO_CONFIG = 9     /* tune_eps found no valid configuration              */
} fgc_status;

/* device flag bits written by data-path kernels */
#define FGC_FLAG_NONFINITE     0x1u  /* "gradient must be finite"       codec.py:225-226 */
#define FGC_FLAG_HALF_OVERFLOW 0x2u  /* binary16 overflow               codec.py:213-214 */
#define FGC_FLAG_F32_RANGE     0x4u  /* f64 input outside float32 range (GPU computes in f32) */
#define FGC_FLAG_CAPACITY      0x8u  /* internal: message exceeded capacity (never expected) */

#define FGC_MODE_COUNT  0            /* SparsificationSpec.mode (spectral.py:366) */
#define FGC_MODE_ENERGY 1

#define FGC_DTYPE_F32 0
#define FGC_DTYPE_F64 1

#define FGC_HEADER_BYTES 36          /* struct "<4sBBQIffffBB" (codec.py:67-70) */
#define FGC_MAX_WORKERS 256

/* QuantizerConfig primitives and derived lattice (quantizer.py:71-151). */
typedef struct fgc_quantizer {
  float    min;            /* float32(min)                                  */
  float    max;            /* float32(max)                                  */
  float    eps;            /* lattice-snapped eps                           */
  int32_t  n_bits;         /* N in [2,16]                                   */
  int32_t  mantissa_bits;  /* m in [1,N)                                    */
  uint32_t pbase;          /* bits(eps) >> (23-m)                           */
  uint32_t pos_count;      /* P                                             */
  uint32_t neg_count;      /* 2^N - 1 - P                                   */
  float    actual_min;     /* most negative representable value             */
  float    actual_max;     /* decoded value of code P                       */
} fgc_quantizer;

/* QuantizerConfig.from_params (quantizer.py:108-135) incl. __post_init__
 * validation (quantizer.py:89-106).  Host-only, no GPU needed. */
fgc_status fgc_quantizer_from_params(double min, double max, int n_bits, int mantissa_bits,
                                     double eps, fgc_quantizer* out);

/* QuantizerConfig.__post_init__ (quantizer.py:89-106) on given fields
 * (min, max, n_bits, mantissa_bits, eps, pbase, pos_count); fills
 * neg_count, actual_min, actual_max.  Host-only. */
fgc_status fgc_quantizer_validate(fgc_quantizer* q);

/* tune_eps (quantizer.py:154-214).  Host-only. */
fgc_status fgc_tune_eps(double min, double max, int n_bits, int mantissa_bits, double eps_init,
                        fgc_quantizer* out);

/* CodecConfig + message length (codec.py:92-109, 133). */
typedef struct fgc_codec_desc {
  uint64_t n;              /* gradient length (original_len)                */
  uint32_t chunk_size;     /* >= 16                                         */
  int32_t  mode;           /* FGC_MODE_COUNT or FGC_MODE_ENERGY             */
  double   theta;          /* DROP ratio in [0,1] (float64, spectral.py:131);
                              count mode: also the capacity theta -- the
                              plan accepts any runtime theta >= it         */
  int32_t  half_pass;      /* half_precision_pass                           */
  int32_t  passthrough;    /* 1: quantizer None, codes are raw f32 bits     */
  int32_t  full_capacity;  /* 1: size segments for every slot (messages not
                              produced by this plan, e.g. deserialized)     */
  fgc_quantizer quant;     /* ignored when passthrough                      */
} fgc_codec_desc;

typedef struct fgc_plan fgc_plan;

typedef struct fgc_plan_info {
  uint64_t n;
  uint32_t n_chunks;
  uint32_t chunk_size;
  uint32_t tail_len;           /* 0 when n is a multiple of chunk_size          */
  uint32_t n_bits;             /* 32 in passthrough                             */
  uint64_t message_bytes;      /* fixed device-message capacity (allgather unit)*/
  uint64_t wire_bytes_max;     /* upper bound of serialize() output            */
  uint64_t spectrum_bins;      /* sum over chunks of (len//2+1)                 */
  uint32_t fused_chunks;       /* chunks taken by the fused sm_100a kernels     */
  uint32_t max_slots;          /* largest per-chunk slot count                  */
  uint64_t total_slots;        /* sum over chunks of slots                      */
} fgc_plan_info;

/* Host-only: number of chunks, fixed device-message bytes and (optionally,
 * n_chunks+1 entries) the segment byte offsets for a config -- what every
 * rank of an allgather must agree on.  No GPU needed. */
fgc_status fgc_message_layout(const fgc_codec_desc* desc, uint32_t* n_chunks, uint64_t* message_bytes,
                              uint64_t* segment_offsets);

/* Create / destroy a plan for one CodecConfig and gradient length.
 * Allocates device tables and scratch once (not on any hot path). */
fgc_status fgc_plan_create(const fgc_codec_desc* desc, fgc_plan** out);
void       fgc_plan_destroy(fgc_plan* plan);
fgc_status fgc_plan_get_info(const fgc_plan* plan, fgc_plan_info* out);
/* Host array of n_chunks+1 byte offsets of each chunk segment in the device
 * message (same on every rank: count mode has a-priori capacity). */
fgc_status fgc_plan_segment_offsets(const fgc_plan* plan, uint64_t* offsets_host);
/* Host array of n_chunks+1 bin offsets into a chunk-major spectrum. */
fgc_status fgc_plan_bin_offsets(const fgc_plan* plan, uint64_t* offsets_host);

/* Runtime theta: the drop ratio of the next compress calls on `stream`
 * (the reference rebuilds its SparsificationSpec whenever the schedule moves
 * theta, simulator.py:333-341, 522-528; here the plan, its message layout
 * and any peer exchange stay).  Count mode: theta must not be below the
 * plan's capacity theta (desc.theta at creation) unless the plan was
 * created with full_capacity; energy mode: any theta in [0, 1].  The new
 * per-chunk drop counts min(ceil(theta*bins), bins) (spectral.py:131) are
 * written to the device chunk table on `stream` when they change. */
fgc_status fgc_plan_set_theta(fgc_plan* plan, double theta, void* stream);

/* ---- compress side (codec.compress, codec.py:220-243) ------------------ */

/* grad (device, n values of `dtype`) -> device message (message_bytes).
 * Replaces compress(): chunked rfft (spectral.py:95), count-mode truncate
 * (spectral.py:142-156), quantize (quantizer.py:217-236) and pack
 * (packer.py:49-58).  flags: device uint32 OR-ed with FGC_FLAG_*. */
fgc_status fgc_compress(fgc_plan* plan, const void* grad, int dtype, uint8_t* message,
                        uint32_t* flags, void* stream);

/* Stage injection: a given chunk-major float2 spectrum (spectrum_bins)
 * -> device message.  Replaces truncate + _interleave + _quantize_parts +
 * pack (codec.py:215-217, 232) for identical coefficients.  Optionally
 * writes the truncate kept-mask (uint8 per bin, may be NULL). */
fgc_status fgc_encode_spectrum(fgc_plan* plan, const void* spectrum, uint8_t* message,
                               uint8_t* kept_mask, uint32_t* flags, void* stream);

/* The forward coefficients compress() quantizes (debug hook for parity):
 * grad -> chunk-major float2 spectrum.  Replaces dft_forward per chunk
 * (spectral.py:88-95, codec.py:215). */
fgc_status fgc_forward_spectrum(fgc_plan* plan, const void* grad, int dtype, void* spectrum,
                                uint32_t* flags, void* stream);

/* ---- decompress / average side ----------------------------------------- */

/* out[n] (float32, device) = sum_w weights[w] * decompress(message_w),
 * accumulated in worker order in the frequency domain, then one C2R iFFT
 * per chunk.  messages: W device messages at stride `message_stride` bytes.
 * Replaces decompress (codec.py:246-270) and the simulator's
 * `shard_weights @ recon` (simulator.py:547).  weights: host array. */
fgc_status fgc_decode_average(fgc_plan* plan, const uint8_t* messages, int W,
                              uint64_t message_stride, const double* weights, float* out,
                              void* stream);

/* Sender-side reconstruction error by Parseval (the simulator's err_ratio,
 * simulator.py:538-542, without a decode): given a chunk-major float2
 * spectrum (fgc_forward_spectrum) and the message compress() made from it,
 * err_norm[2c], err_norm[2c+1] (device doubles) = ||x - decompress(m)||^2 and
 * ||x||^2 of chunk c, from (1/L) sum_k w_k |X_k - Xhat_k|^2 and
 * (1/L) sum_k w_k |X_k|^2 (Parseval weights, spectral.py:109-115). */
fgc_status fgc_spectrum_error(fgc_plan* plan, const void* spectrum, const uint8_t* message, double* err_norm,
                              void* stream);

/* Debug hook: the averaged spectrum before the inverse FFT (float2). */
fgc_status fgc_decode_spectrum(fgc_plan* plan, const uint8_t* messages, int W,
                               uint64_t message_stride, const double* weights, void* spectrum,
                               void* stream);

/* C2R of a chunk-major float2 spectrum (dft_inverse per chunk,
 * spectral.py:98-106; imag of DC/Nyquist ignored like numpy's irfft). */
fgc_status fgc_inverse_spectrum(fgc_plan* plan, const void* spectrum, float* out, void* stream);

/* ---- wire format (codec.serialize / deserialize, codec.py:340-441) ------ */

/* Device message -> FGC1 bytes (header + per chunk u32, bitmap, codes) at
 * `wire` (device, >= wire_bytes_max).  The byte length is written to the
 * device uint64 `wire_len`. */
fgc_status fgc_serialize(fgc_plan* plan, const uint8_t* message, uint8_t* wire,
                         uint64_t* wire_len, void* stream);

/* Parse + validate an FGC1 header (codec.py:379-405).  Host memory.
 * Fills desc (n, chunk_size, mode, theta as stored (f32), flags, quantizer). */
fgc_status fgc_parse_header(const uint8_t* wire_host, uint64_t len, fgc_codec_desc* desc);

/* Walk the chunk framing of a host FGC1 buffer (codec.py:415-440): per chunk
 * byte offset of its u32 kept-count and the count.  Returns TRUNCATED /
 * FORMAT like the reference; on TRUNCATED, *n_valid = chunks fully present. */
fgc_status fgc_wire_index(const uint8_t* wire_host, uint64_t len, const fgc_codec_desc* desc,
                          uint64_t* chunk_offsets_host, uint32_t* nnz_host, uint32_t* n_valid);

/* FGC1 bytes (device copy) + chunk offsets (device) -> device message, and
 * the bitmap popcount of each chunk (device uint32[n_chunks]) so the caller
 * can raise BitmapMismatchError (codec.py:427-430). */
fgc_status fgc_deserialize(fgc_plan* plan, const uint8_t* wire, const uint64_t* chunk_offsets,
                           uint8_t* message, uint32_t* popcounts, void* stream);

/* Per-chunk non-zero code counts of a device message (device uint32). */
fgc_status fgc_message_counts(fgc_plan* plan, const uint8_t* message, uint32_t* nnz, void* stream);

/* Materialize ChunkPayload arrays (codec.py:112-125): bitmap as uint8 0/1
 * per slot (chunk-major, sum of slots) and codes as uint32 (chunk-major at
 * code_offsets[c], device uint64[n_chunks]). */
fgc_status fgc_message_unpack(fgc_plan* plan, const uint8_t* message, const uint64_t* code_offsets,
                              uint8_t* bitmap_flags, uint32_t* codes, void* stream);

/* Build a device message from ChunkPayload arrays (inverse of the above);
 * popcounts (device uint32[n_chunks]) let the caller check bitmap/codes
 * agreement (codec.py:261-265).  flags gets FGC_FLAG_CAPACITY if a chunk
 * does not fit the plan's fixed capacity. */
fgc_status fgc_message_pack(fgc_plan* plan, const uint8_t* bitmap_flags, const uint32_t* codes,
                            const uint64_t* code_offsets, uint8_t* message, uint32_t* popcounts,
                            uint32_t* flags, void* stream);

/* ---- primitives (quantizer.py / packer.py / spectral.py) ---------------- */

/* encode_array (quantizer.py:217-236); values float32 or float64 (rounded
 * to f32 like np.asarray(values, float32)).  first_nan: device int64, set to
 * the lowest NaN index (initialise to INT64_MAX). */
fgc_status fgc_quantize(const fgc_quantizer* q, const void* values, int dtype, uint64_t count,
                        uint32_t* codes, int64_t* first_nan, void* stream);
/* decode_array (quantizer.py:239-253); bad: device uint32 set if a code is
 * negative or >= 2^N (the reference's ValueError). */
fgc_status fgc_dequantize(const fgc_quantizer* q, const int64_t* codes, uint64_t count,
                          float* values, uint32_t* bad, void* stream);
/* pack_codes / unpack_codes: LSB-first width-bit fields (quantizer.py:266-285). */
fgc_status fgc_pack_bits(const uint32_t* codes, uint64_t count, int width, uint8_t* out, void* stream);
fgc_status fgc_unpack_bits(const uint8_t* data, uint64_t count, int width, uint32_t* codes, void* stream);
/* bitmap_to_bytes / bitmap_from_bytes: MSB-first (packer.py:73-84). */
fgc_status fgc_flags_to_bitmap(const uint8_t* flags01, uint64_t count, uint8_t* out, void* stream);
fgc_status fgc_bitmap_to_flags(const uint8_t* bitmap, uint64_t count, uint8_t* flags01, void* stream);
/* prefix_sum (packer.py:41-46): inclusive int64 scan of 0/1 values; bad
 * (device uint32) set if an entry is not 0/1; scratch: device uint64 of
 * ceil(count/4096)+1 entries. */
fgc_status fgc_prefix_sum(const uint8_t* status01, uint64_t count, int64_t* out, uint32_t* bad,
                          uint64_t* scratch, void* stream);
/* pack's scatter (packer.py:55-57): dense[loc[i] - 1] = values[i] where
 * status01[i], loc = the inclusive prefix_sum above; elem_bytes 1/2/4/8. */
fgc_status fgc_compact(const void* values, const uint8_t* status01, const int64_t* loc, uint64_t count,
                       int elem_bytes, void* dense, void* stream);
/* unpack's gather (packer.py:67-69): out[i] = status01[i] ? dense[loc[i] - 1]
 * : 0. */
fgc_status fgc_expand(const void* dense, const uint8_t* status01, const int64_t* loc, uint64_t count,
                      int elem_bytes, void* out, void* stream);

/* dft_forward / dft_inverse of ONE length-L real signal (spectral.py:88-106)
 * in float64 like the reference: any L >= 1, float32/float64 input,
 * complex128 half spectrum (L//2+1 bins).  Allocates temporary tables
 * (not a hot path).  flags: device uint32 (FGC_FLAG_NONFINITE). */
fgc_status fgc_rfft(const void* signal, int dtype, uint64_t L, void* spectrum_c128, uint32_t* flags, void* stream);
fgc_status fgc_irfft(const void* spectrum_c128, uint64_t L, double* signal, void* stream);

/* truncate (spectral.py:142-156), count mode, on a complex128 half spectrum:
 * numpy's exact magnitude key and the stable index tie-break.  Writes the
 * zeroed spectrum (may alias the input) and the kept mask (uint8/bin). */
fgc_status fgc_truncate(const void* spectrum_c128, uint64_t bins, double theta, void* out_c128, uint8_t* kept_mask,
                        void* stream);
/* truncate for either mode (spectral.py:124-156) of the half spectrum of an
 * n-sample signal (bins = n/2 + 1; n's parity sets the Nyquist weight of
 * the energy rule, bin_weights spectral.py:109-115). */
fgc_status fgc_truncate_mode(const void* spectrum_c128, uint64_t bins, uint64_t n, double theta, int mode,
                             void* out_c128, uint8_t* kept_mask, void* stream);

/* calibrate's range reduction (codec.py:463-464): max over |Re|, |Im| of the
 * float64 rfft of one sample, max-accumulated into the device double *peak
 * (initialise to 0). */
fgc_status fgc_spectrum_peak(const void* signal, int dtype, uint64_t L, double* peak, uint32_t* flags, void* stream);

/* half_round_trip (spectral.py:189-196): float64 -> binary16 (RNE) -> float64. */
fgc_status fgc_half_round_trip(const double* in, uint64_t count, double* out, void* stream);

/* ---- multi-GPU exchange (the simulated channel of simulator.py:529-535) - */

/* NCCL bootstrap: rank 0 calls fgc_nccl_unique_id, the caller broadcasts the
 * 128 bytes by any means, every rank calls fgc_nccl_comm_create. */
fgc_status fgc_nccl_unique_id(uint8_t id_out[128]);
fgc_status fgc_nccl_comm_create(const uint8_t id[128], int nranks, int rank, void** comm_out);
fgc_status fgc_nccl_comm_destroy(void* comm);

/* Allgather of fixed-capacity device messages: recv holds nranks messages
 * of `bytes` each, rank-major. */
fgc_status fgc_allgather(void* comm, const uint8_t* send, uint8_t* recv, uint64_t bytes,
                         void* stream);
/* Uncompressed baseline: in-place float32 sum allreduce. */
fgc_status fgc_allreduce_sum_f32(void* comm, float* data, uint64_t count, void* stream);

/* One step of the compressed average for this rank (simulator.py:520-547):
 * compress(grad) -> allgather -> decode_average(weights) -> out, pipelined
 * in pieces of consecutive chunks (whole waves of the fused kernels;
 * FGC_PIPELINE_WAVES per piece; default 0 = one piece): piece i
 * is allgathered on an internal high-priority stream while piece i+1
 * compresses, and decoded when its exchange completes.  gathered must hold
 * nranks * message_bytes; its layout is piece-major (piece i of every rank
 * contiguous), i.e. internal.  comm may be NULL for W=1.  Work is ordered
 * after prior work on `stream` and everything it launches is joined back
 * into `stream`. */
fgc_status fgc_allgather_average(fgc_plan* plan, void* comm, int nranks, const void* grad,
                                 int dtype, const double* weights, uint8_t* message,
                                 uint8_t* gathered, float* out, uint32_t* flags, void* stream);

/* ---- peer-memory exchange (copy engines over NVLink, CUDA IPC) ---------- */
/* The allgather of simulator.py:529-535 without collective kernels: each
 * rank pushes its message pieces into every peer's gather buffer with
 * peer-to-peer copies and signals them with stream memory operations, so
 * the exchange overlaps the codec kernels without taking SMs.  Setup:
 * create on every rank, exchange the 128-byte handles (e.g. through
 * torch.distributed), open with all ranks' handles (rank-major). */
typedef struct fgc_exchange fgc_exchange;
fgc_status fgc_exchange_create(int nranks, int rank, uint64_t message_bytes, fgc_exchange** out);
fgc_status fgc_exchange_handles(fgc_exchange* x, uint8_t handles_out[128]);
fgc_status fgc_exchange_open(fgc_exchange* x, const uint8_t* all_handles /* nranks * 128 */);
void       fgc_exchange_destroy(fgc_exchange* x);   /* all ranks: after a barrier */
/* This rank's message slot / the gather buffer of step parity `parity`. */
fgc_status fgc_exchange_message(fgc_exchange* x, int parity, uint8_t** message, uint8_t** gathered);
/* One averaging step over the exchange (same result as
 * fgc_allgather_average): compress into this rank's slot piece by piece,
 * push each piece to every peer as soon as it is compressed, decode each
 * piece once every peer's copy of it has landed.  Steps alternate between
 * two gather buffers; every rank must call it the same number of times. */
fgc_status fgc_exchange_average(fgc_plan* plan, fgc_exchange* x, const void* grad, int dtype,
                                const double* weights, float* out, uint32_t* flags, void* stream);

/* The averaging step from and to HOST memory (pinned for overlap): the
 * host->device copy of the gradient and the device->host copy of the
 * average run on copy streams in pieces of consecutive chunks, overlapped
 * with the codec kernels.  x = NULL: single rank (message is this rank's
 * device message buffer); otherwise the peer exchange (message ignored).
 * dev_grad (n values of dtype) and dev_out (n floats) are device scratch.
 * dev_grad belongs to this plan's host steps: a call's host->device copy of
 * a piece waits only until the previous call's compress has read that
 * piece (not for other work on `stream`), so back-to-back calls overlap one
 * step's copy-out with the next step's copy-in (FGC_HOST_SERIAL=1: wait for
 * everything earlier on `stream`).  host_out is complete once `stream` is. */
fgc_status fgc_average_host(fgc_plan* plan, fgc_exchange* x, const void* host_grad, int dtype,
                            const double* weights, void* dev_grad, uint8_t* message, float* dev_out,
                            float* host_out, uint32_t* flags, void* stream);

/* ---- misc -------------------------------------------------------------- */
const char* fgc_last_error(void);   /* thread-local message of the last failure */
int         fgc_version(void);      /* 0xMMmmpp                                  */
/* Count of device kernels launched by this process (instrumentation). */
uint64_t    fgc_kernel_launches(void);
/* Instrumentation for the roofline: launch ONLY the fused compress kernel of
 * the plan's 65536-sample chunks (no tail chunk, no exchange) on `stream`;
 * *alg_bytes = that launch's algorithmic bytes (signal read + segments
 * written).  Not a codec entry point: the tail chunks' segments are left
 * untouched. */
fgc_status  fgc_profile_fused_compress(fgc_plan* plan, const void* grad, int dtype, uint8_t* message,
                                       uint32_t* flags, void* stream, uint64_t* alg_bytes);

#ifdef __cplusplus
}
#endif
#endif /* FGC_B200_H */
