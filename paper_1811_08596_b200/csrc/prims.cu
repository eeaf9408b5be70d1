// Device implementations of the reference's element-wise primitives, so the
// drop-in module functions run on the GPU too:
//   encode_array / decode_array        quantizer.py:217-253
//   pack_codes / unpack_codes          quantizer.py:266-285
//   bitmap_to_bytes / bitmap_from_bytes packer.py:73-84
//   prefix_sum                          packer.py:41-46
//   dft_forward / dft_inverse           spectral.py:88-106 (float64 engine)
//   truncate (count mode)               spectral.py:124-156
//   half_round_trip                     spectral.py:189-196
//   calibrate's peak reduction          codec.py:455-465
// These are library conveniences, not the hot path: the whole-signal
// transforms allocate their tables per call.
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <vector>

#include <algorithm>

#include "fgc_device.cuh"
#include "fgc_internal.h"

namespace fgc {
namespace {

inline uint32_t cdiv(uint64_t a, uint32_t b) { return (uint32_t)((a + b - 1) / b); }

QuantParams qparams(const fgc_quantizer& q) {
  QuantParams p{};
  p.n_bits = q.n_bits;
  p.shift = 23 - q.mantissa_bits;
  p.pbase = q.pbase;
  p.npos = q.pos_count;
  p.nneg = q.neg_count;
  p.eps = q.eps;
  p.pos_cap = q.max;
  p.neg_cap = -q.actual_min;
  return p;
}

template <class T>
__global__ void k_quantize(QuantParams q, const T* v, uint64_t n, uint32_t* codes, long long* first_nan) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float x = (float)v[i];          // np.asarray(values, float32)
  if (isnan(x)) {
    atomicMin(first_nan, (long long)i);
    codes[i] = 0;
    return;
  }
  codes[i] = encode_code(q, x);
}

__global__ void k_dequantize(QuantParams q, const long long* c, uint64_t n, float* out, uint32_t* bad) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long v = c[i];
  if (v < 0 || v >= (1ll << q.n_bits)) {
    atomicOr(bad, 1u);
    out[i] = 0.f;
    return;
  }
  out[i] = decode_code(q, (uint32_t)v);
}

// byte b of the LSB-first stream gathers the codes overlapping bits [8b, 8b+8)
__global__ void k_pack_bits(const uint32_t* codes, uint64_t n, int w, uint8_t* out, uint64_t nbytes) {
  const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbytes) return;
  const uint64_t b0 = 8 * b, b1 = b0 + 8;
  const uint32_t mask = w == 32 ? ~0u : ((1u << w) - 1u);
  uint32_t v = 0;
  for (uint64_t j = b0 / w; j < n && j * w < b1; ++j) {
    const uint64_t pos = j * w;
    const uint64_t code = codes[j] & mask;
    if (pos >= b0) v |= (uint32_t)(code << (pos - b0));
    else v |= (uint32_t)(code >> (b0 - pos));
  }
  out[b] = (uint8_t)(v & 0xFFu);
}

__global__ void k_unpack_bits(const uint8_t* d, uint64_t n, int w, uint32_t* codes) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint64_t pos = j * w;
  uint64_t acc = 0;
  const uint64_t first = pos >> 3;
  const uint32_t nb = (uint32_t)(((pos & 7) + w + 7) >> 3);
  for (uint32_t k = 0; k < nb; ++k) acc |= (uint64_t)d[first + k] << (8 * k);
  acc >>= (pos & 7);
  codes[j] = (uint32_t)(w == 32 ? acc : (acc & ((1ull << w) - 1ull)));
}

__global__ void k_flags_to_bitmap(const uint8_t* f, uint64_t n, uint8_t* out) {
  const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (8 * b >= n) return;
  uint32_t v = 0;
  for (int k = 0; k < 8; ++k) {
    const uint64_t s = 8 * b + k;
    if (s < n && f[s]) v |= 0x80u >> k;
  }
  out[b] = (uint8_t)v;
}

__global__ void k_bitmap_to_flags(const uint8_t* bm, uint64_t n, uint8_t* f) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  f[s] = (bm[s >> 3] >> (7 - (s & 7))) & 1u;
}

constexpr int kScanThreads = 1024;
constexpr uint32_t kScanTile = kScanThreads * 4;

__global__ void k_tile_sums(const uint8_t* st, uint64_t n, uint64_t* sums, uint32_t* bad) {
  __shared__ uint32_t scan[40];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint32_t local = 0;
  for (uint32_t k = 0; k < 4; ++k) {
    const uint64_t i = base + threadIdx.x * 4 + k;
    if (i < n) {
      const uint8_t v = st[i];
      if (v > 1) atomicOr(bad, 1u);
      local += v ? 1u : 0u;
    }
  }
  const uint32_t tot = block_sum<kScanThreads>(local, scan);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void k_tile_apply(const uint8_t* st, uint64_t n, const uint64_t* offs, long long* out) {
  __shared__ uint32_t scan[40];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint32_t v[4], local = 0;
  for (uint32_t k = 0; k < 4; ++k) {
    const uint64_t i = base + threadIdx.x * 4 + k;
    v[k] = (i < n && st[i]) ? 1u : 0u;
    local += v[k];
  }
  uint32_t tot;
  uint32_t pre = block_exclusive_scan<kScanThreads>(local, scan, tot);
  uint64_t run = offs[blockIdx.x] + pre;
  for (uint32_t k = 0; k < 4; ++k) {
    const uint64_t i = base + threadIdx.x * 4 + k;
    run += v[k];
    if (i < n) out[i] = (long long)run;
  }
}

__global__ void k_zero_dropped(const double2* in, const uint8_t* mask, uint64_t n, double2* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = mask[i] ? in[i] : make_double2(0.0, 0.0);
}

__global__ void k_peak(const double2* sp, uint64_t n, unsigned long long* peak) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double m = 0.0;
  if (i < n) m = fmax(fabs(sp[i].x), fabs(sp[i].y));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(peak, (unsigned long long)__double_as_longlong(m));
}

__global__ void k_half_rt(const double* in, uint64_t n, double* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = (double)__half2float(__double2half(in[i]));
}

// One temporary single-chunk layout for whole-signal transforms.
struct OneChunk {
  ChunkInfo* d = nullptr;
  fgc_status make(uint64_t L) {
    if (L > 0xFFFFFFFFull) { set_error("signal too long"); return FGC_ERR_UNSUPPORTED; }
    ChunkInfo ci{};
    ci.len = (uint32_t)L;
    ci.bins = (uint32_t)(L / 2 + 1);
    ci.slots = 2 * ci.bins;
    FGC_CUDA(cudaMalloc(&d, sizeof(ChunkInfo)));
    FGC_CUDA(cudaMemcpy(d, &ci, sizeof(ChunkInfo), cudaMemcpyHostToDevice));
    return FGC_OK;
  }
  ~OneChunk() { cudaFree(d); }
};

}  // namespace
}  // namespace fgc

using namespace fgc;

extern "C" fgc_status fgc_quantize(const fgc_quantizer* q, const void* values, int dtype, uint64_t count,
                                   uint32_t* codes, int64_t* first_nan, void* stream) {
  if (!q || (!values && count) || (!codes && count) || !first_nan) return FGC_ERR_INVALID;
  if (!count) return FGC_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const QuantParams p = qparams(*q);
  if (dtype == FGC_DTYPE_F64)
    k_quantize<double><<<cdiv(count, 256), 256, 0, s>>>(p, static_cast<const double*>(values), count, codes,
                                                        reinterpret_cast<long long*>(first_nan));
  else
    k_quantize<float><<<cdiv(count, 256), 256, 0, s>>>(p, static_cast<const float*>(values), count, codes,
                                                       reinterpret_cast<long long*>(first_nan));
  FGC_LAUNCHED(1);
  return FGC_OK;
}

extern "C" fgc_status fgc_dequantize(const fgc_quantizer* q, const int64_t* codes, uint64_t count, float* values,
                                     uint32_t* bad, void* stream) {
  if (!q || !bad) return FGC_ERR_INVALID;
  if (!count) return FGC_OK;
  k_dequantize<<<cdiv(count, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      qparams(*q), reinterpret_cast<const long long*>(codes), count, values, bad);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

extern "C" fgc_status fgc_pack_bits(const uint32_t* codes, uint64_t count, int width, uint8_t* out, void* stream) {
  if (width < 1 || width > 32) return FGC_ERR_INVALID;
  const uint64_t nbytes = (count * width + 7) / 8;
  if (!nbytes) return FGC_OK;
  k_pack_bits<<<cdiv(nbytes, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(codes, count, width, out, nbytes);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

extern "C" fgc_status fgc_unpack_bits(const uint8_t* data, uint64_t count, int width, uint32_t* codes, void* stream) {
  if (width < 1 || width > 32) return FGC_ERR_INVALID;
  if (!count) return FGC_OK;
  k_unpack_bits<<<cdiv(count, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(data, count, width, codes);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

extern "C" fgc_status fgc_flags_to_bitmap(const uint8_t* flags01, uint64_t count, uint8_t* out, void* stream) {
  if (!count) return FGC_OK;
  k_flags_to_bitmap<<<cdiv((count + 7) / 8, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(flags01, count, out);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

extern "C" fgc_status fgc_bitmap_to_flags(const uint8_t* bitmap, uint64_t count, uint8_t* flags01, void* stream) {
  if (!count) return FGC_OK;
  k_bitmap_to_flags<<<cdiv(count, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(bitmap, count, flags01);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

extern "C" fgc_status fgc_prefix_sum(const uint8_t* status01, uint64_t count, int64_t* out, uint32_t* bad,
                                     uint64_t* scratch, void* stream) {
  if (!count) return FGC_OK;
  if (!bad || !scratch) return FGC_ERR_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t tiles = (count + kScanTile - 1) / kScanTile;
  if (tiles > 0xFFFFFFFFull) return FGC_ERR_UNSUPPORTED;
  k_tile_sums<<<(uint32_t)tiles, kScanThreads, 0, s>>>(status01, count, scratch, bad);
  FGC_LAUNCHED(1);
  FGC_TRY(launch_scan_u64(scratch, (uint32_t)tiles, scratch + tiles, 0, s));
  k_tile_apply<<<(uint32_t)tiles, kScanThreads, 0, s>>>(status01, count, scratch, reinterpret_cast<long long*>(out));
  FGC_LAUNCHED(1);
  return FGC_OK;
}

template <class E>
__global__ void k_compact(const E* v, const uint8_t* st, const long long* loc, uint64_t n, E* dense) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (st[i]) dense[loc[i] - 1] = v[i];
}
template <class E>
__global__ void k_expand(const E* dense, const uint8_t* st, const long long* loc, uint64_t n, E* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = st[i] ? dense[loc[i] - 1] : E(0);
}

template <template <class> class K, class... A>
static fgc_status launch_by_size(int elem_bytes, uint64_t n, cudaStream_t s, const void* a, const uint8_t* st,
                                 const int64_t* loc, void* b) {
  const uint32_t grid = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  const long long* l = reinterpret_cast<const long long*>(loc);
  switch (elem_bytes) {
    case 1: K<uint8_t>::run(grid, s, a, st, l, n, b); break;
    case 2: K<uint16_t>::run(grid, s, a, st, l, n, b); break;
    case 4: K<uint32_t>::run(grid, s, a, st, l, n, b); break;
    case 8: K<unsigned long long>::run(grid, s, a, st, l, n, b); break;
    default: set_error("elem_bytes must be 1, 2, 4 or 8"); return FGC_ERR_INVALID;
  }
  FGC_LAUNCHED(1);
  return FGC_OK;
}
template <class E> struct CompactK {
  static void run(uint32_t g, cudaStream_t s, const void* a, const uint8_t* st, const long long* l, uint64_t n,
                  void* b) {
    k_compact<E><<<g, 256, 0, s>>>(static_cast<const E*>(a), st, l, n, static_cast<E*>(b));
  }
};
template <class E> struct ExpandK {
  static void run(uint32_t g, cudaStream_t s, const void* a, const uint8_t* st, const long long* l, uint64_t n,
                  void* b) {
    k_expand<E><<<g, 256, 0, s>>>(static_cast<const E*>(a), st, l, n, static_cast<E*>(b));
  }
};

extern "C" fgc_status fgc_compact(const void* values, const uint8_t* status01, const int64_t* loc, uint64_t count,
                                  int elem_bytes, void* dense, void* stream) {
  if (!count) return FGC_OK;
  if (!values || !status01 || !loc || !dense) { set_error("null argument"); return FGC_ERR_INVALID; }
  return launch_by_size<CompactK>(elem_bytes, count, static_cast<cudaStream_t>(stream), values, status01, loc, dense);
}

extern "C" fgc_status fgc_expand(const void* dense, const uint8_t* status01, const int64_t* loc, uint64_t count,
                                 int elem_bytes, void* out, void* stream) {
  if (!count) return FGC_OK;
  if (!dense || !status01 || !loc || !out) { set_error("null argument"); return FGC_ERR_INVALID; }
  return launch_by_size<ExpandK>(elem_bytes, count, static_cast<cudaStream_t>(stream), dense, status01, loc, out);
}

extern "C" fgc_status fgc_rfft(const void* signal, int dtype, uint64_t L, void* spectrum, uint32_t* flags,
                               void* stream) {
  if (!signal || !spectrum || !flags || L < 1) return FGC_ERR_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  OneChunk oc;
  FGC_TRY(oc.make(L));
  RealClassT<double> rc;
  rc.L = (uint32_t)L;
  rc.bins = (uint32_t)(L / 2 + 1);
  rc.first = 0;
  rc.count = 1;
  fgc_status st = rc.init(s);
  if (st == FGC_OK) st = real_forward<double>(rc, oc.d, signal, dtype, 0, flags, static_cast<double2*>(spectrum), s);
  cudaError_t e = cudaStreamSynchronize(s);
  rc.free_all();
  if (st != FGC_OK) return st;
  if (e != cudaSuccess) return cuda_check(e, "rfft");
  return FGC_OK;
}

extern "C" fgc_status fgc_irfft(const void* spectrum, uint64_t L, double* signal, void* stream) {
  if (!signal || !spectrum || L < 1) return FGC_ERR_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  OneChunk oc;
  FGC_TRY(oc.make(L));
  RealClassT<double> rc;
  rc.L = (uint32_t)L;
  rc.bins = (uint32_t)(L / 2 + 1);
  rc.first = 0;
  rc.count = 1;
  fgc_status st = rc.init(s);
  if (st == FGC_OK) st = real_inverse<double>(rc, oc.d, static_cast<const double2*>(spectrum), signal, s);
  cudaError_t e = cudaStreamSynchronize(s);
  rc.free_all();
  if (st != FGC_OK) return st;
  if (e != cudaSuccess) return cuda_check(e, "irfft");
  return FGC_OK;
}

namespace fgc {
__global__ void k_set_drop(ChunkInfo* chunks, uint32_t n, double theta) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const uint32_t bins = chunks[c].bins;
  const double kd = ceil(theta * (double)bins);             // IEEE-RN product, exact ceil: as on the host
  chunks[c].drop = kd >= (double)bins ? bins : (uint32_t)kd;
}

fgc_status launch_set_drop(ChunkInfo* d_chunks, uint32_t n_chunks, double theta, cudaStream_t s) {
  if (!n_chunks) return FGC_OK;
  k_set_drop<<<(n_chunks + 255) / 256, 256, 0, s>>>(d_chunks, n_chunks, theta);
  FGC_LAUNCHED(1);
  return FGC_OK;
}
}  // namespace fgc

static fgc_status truncate_impl(const void* spectrum, uint64_t bins, uint64_t n, double theta, int mode, void* out,
                                uint8_t* kept_mask, void* stream) {
  if (!spectrum || !out || !kept_mask || bins < 1 || bins > 0x7FFFFFFFull) return FGC_ERR_INVALID;
  if (!(theta >= 0.0 && theta <= 1.0)) { set_error("theta must be in [0, 1]"); return FGC_ERR_INVALID; }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // one passthrough "chunk" whose bins are the given spectrum
  ChunkInfo ci{};
  ci.bins = (uint32_t)bins;
  ci.slots = 2 * ci.bins;
  ci.len = (uint32_t)n;
  ci.drop = (uint32_t)ceil(theta * (double)bins);
  if (ci.drop > bins) ci.drop = (uint32_t)bins;
  const uint64_t bm_words = (ci.slots + 31) / 32;
  ci.code_off = (uint32_t)(kSegHeader + ((4 * bm_words + 15) & ~15ull));
  ci.code_cap = ci.slots;
  const uint64_t msg = ci.code_off + 4ull * ci.code_cap;
  ChunkInfo* d_ci = nullptr;
  uint8_t* d_msg = nullptr;
  uint32_t* d_flags = nullptr;
  EnergyScratch es;
  fgc_status st = FGC_OK;
  cudaError_t e;
  if ((e = cudaMalloc(&d_ci, sizeof(ChunkInfo))) != cudaSuccess) st = cuda_check(e, "cudaMalloc");
  if (st == FGC_OK && (e = cudaMalloc(&d_msg, msg)) != cudaSuccess) st = cuda_check(e, "cudaMalloc");
  if (st == FGC_OK && (e = cudaMalloc(&d_flags, 4)) != cudaSuccess) st = cuda_check(e, "cudaMalloc");
  if (st == FGC_OK && (e = cudaMemcpyAsync(d_ci, &ci, sizeof(ci), cudaMemcpyHostToDevice, s)) != cudaSuccess)
    st = cuda_check(e, "cudaMemcpyAsync");
  const uint8_t* drop = nullptr;
  if (st == FGC_OK && mode == FGC_MODE_ENERGY)
    st = energy_drop_mask(es, d_ci, 0, 1, 0, bins, (uint32_t)bins, spectrum, 1, theta, s, &drop);
  if (st == FGC_OK) {
    QuantParams q{};
    q.n_bits = 32;
    st = launch_select_pack(d_ci, 0, 1, spectrum, 1, q, d_msg, kept_mask, d_flags, s, nullptr, PieceCounter(),
                            drop);
  }
  if (st == FGC_OK) {
    k_zero_dropped<<<cdiv(bins, 256), 256, 0, s>>>(static_cast<const double2*>(spectrum), kept_mask, bins,
                                                   static_cast<double2*>(out));
    count_launch(1);
  }
  e = cudaStreamSynchronize(s);
  if (st == FGC_OK && e != cudaSuccess) st = cuda_check(e, "truncate");
  cudaFree(d_ci);
  cudaFree(d_msg);
  cudaFree(d_flags);
  es.free_all();
  return st;
}

extern "C" fgc_status fgc_truncate(const void* spectrum, uint64_t bins, double theta, void* out, uint8_t* kept_mask,
                                   void* stream) {
  return truncate_impl(spectrum, bins, 2 * (bins - 1), theta, FGC_MODE_COUNT, out, kept_mask, stream);
}

extern "C" fgc_status fgc_truncate_mode(const void* spectrum, uint64_t bins, uint64_t n, double theta, int mode,
                                        void* out, uint8_t* kept_mask, void* stream) {
  if (mode != FGC_MODE_COUNT && mode != FGC_MODE_ENERGY) { set_error("unknown mode"); return FGC_ERR_INVALID; }
  if (n / 2 + 1 != bins) { set_error("bins must be n // 2 + 1"); return FGC_ERR_INVALID; }
  return truncate_impl(spectrum, bins, n, theta, mode, out, kept_mask, stream);
}

extern "C" fgc_status fgc_spectrum_peak(const void* signal, int dtype, uint64_t L, double* peak, uint32_t* flags,
                                        void* stream) {
  if (!signal || !peak || !flags || L < 1) return FGC_ERR_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t bins = L / 2 + 1;
  double2* sp = nullptr;
  FGC_CUDA(cudaMalloc(&sp, sizeof(double2) * bins));
  fgc_status st = fgc_rfft(signal, dtype, L, sp, flags, stream);
  if (st == FGC_OK) {
    k_peak<<<cdiv(bins, 256), 256, 0, s>>>(sp, bins, reinterpret_cast<unsigned long long*>(peak));
    count_launch(1);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_check(e, "peak");
  }
  cudaFree(sp);
  return st;
}

extern "C" fgc_status fgc_half_round_trip(const double* in, uint64_t count, double* out, void* stream) {
  if (!count) return FGC_OK;
  k_half_rt<<<cdiv(count, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(in, count, out);
  FGC_LAUNCHED(1);
  return FGC_OK;
}
