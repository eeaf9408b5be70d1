// Real-signal glue around the generic complex DFT engine (fft_generic.cu):
// numpy's rfft / irfft semantics (spectral.py:88-106) for a batch of equal
// length chunks, in float32 (codec) or float64 (primitives).
//
//   even L: z[n] = x[2n] + i x[2n+1], Z = DFT_{L/2}(z),
//           X[k] = (Z[k] + conj Z[L/2-k])/2 - i W_L^k (Z[k] - conj Z[L/2-k])/2
//   odd  L: Z = DFT_L(x + 0i), X[k] = Z[k]
//   inverse: the algebraic inverse of the above; Im X[0] (and Im X[L/2] for
//   even L) are ignored exactly like numpy's irfft.
// The forward load applies the codec's input checks: non-finite values
// (codec.py:225-226) and the optional binary16 round trip with overflow
// detection (spectral.py:189-196, codec.py:211-214).
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <math.h>

#include <algorithm>

#include "decode_acc.cuh"
#include "fgc_device.cuh"
#include "fgc_internal.h"
#include "generic_dev.cuh"
#include "select_pack.cuh"

namespace fgc {

namespace {

inline uint32_t cdiv(uint64_t a, uint32_t b) { return (uint32_t)((a + b - 1) / b); }

__device__ __forceinline__ float2 mk2(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ double2 mk2(double x, double y) { return make_double2(x, y); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return cmul(a, b); }
__device__ __forceinline__ double2 mul2(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
template <class T2> __device__ __forceinline__ T2 cj(T2 a) { return mk2(a.x, -a.y); }

// ------------------------------------------------------------- input loads

template <class R, class In> struct Loader;
template <> struct Loader<float, float> {
  __device__ static float get(const float* g, uint64_t i, int half, uint32_t* flags) {
    float x = g[i];
    if (!isfinite(x)) { atomicOr(flags, FGC_FLAG_NONFINITE); return 0.0f; }
    if (half) {
      x = __half2float(__float2half_rn(x));
      if (isinf(x)) atomicOr(flags, FGC_FLAG_HALF_OVERFLOW);
    }
    return x;
  }
};
template <> struct Loader<float, double> {
  __device__ static float get(const double* g, uint64_t i, int half, uint32_t* flags) {
    const double d = g[i];
    if (!isfinite(d)) { atomicOr(flags, FGC_FLAG_NONFINITE); return 0.0f; }
    float x;
    if (half) {
      x = __half2float(__double2half(d));     // f64 -> f16 directly, like numpy
      if (isinf(x)) atomicOr(flags, FGC_FLAG_HALF_OVERFLOW);
    } else {
      x = (float)d;
      if (isinf(x)) atomicOr(flags, FGC_FLAG_F32_RANGE);
    }
    return x;
  }
};
template <> struct Loader<double, double> {
  __device__ static double get(const double* g, uint64_t i, int, uint32_t* flags) {
    const double d = g[i];
    if (!isfinite(d)) { atomicOr(flags, FGC_FLAG_NONFINITE); return 0.0; }
    return d;
  }
};
template <> struct Loader<double, float> {
  __device__ static double get(const float* g, uint64_t i, int, uint32_t* flags) {
    const float x = g[i];
    if (!isfinite(x)) { atomicOr(flags, FGC_FLAG_NONFINITE); return 0.0; }
    return (double)x;
  }
};

template <class R>
struct Args {
  using T2 = typename Vec2<R>::T;
  const ChunkInfo* chunks;
  uint32_t first, L, Lc, Pw, P, A, B, bins, cap;
  int kind;
  T2* work;
  const T2* chirp;
  const T2* rtw;
  R invP;
};

template <class R, class In>
__device__ __forceinline__ void prep_elem(const Args<R>& a, const In* in, int half, uint32_t* flags, uint32_t j,
                                          const ChunkInfo& ci, uint32_t n) {
  using T2 = typename Vec2<R>::T;
  T2 v = mk2((R)0, (R)0);
  if (n < a.Lc) {
    if ((a.L & 1u) == 0) {
      v.x = Loader<R, In>::get(in, ci.in_off + 2ull * n, half, flags);
      v.y = Loader<R, In>::get(in, ci.in_off + 2ull * n + 1, half, flags);
    } else {
      v.x = Loader<R, In>::get(in, ci.in_off + n, half, flags);
    }
    if (a.kind == (int)DftKind::Bluestein) v = mul2(v, a.chirp[n]);
  }
  a.work[(uint64_t)j * a.Pw + n] = v;
}

template <class R, class In>
__global__ void k_prep(Args<R> a, const In* in, int half, uint32_t* flags) {
  const uint32_t j = blockIdx.y;
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= a.Pw) return;
  const ChunkInfo ci = a.chunks[a.first + j];
  prep_elem(a, in, half, flags, j, ci, n);
}

template <class R>
struct Res {
  const typename Vec2<R>::T* base;
  uint64_t stride;
  int layout, chirp;
};

template <class R>
__device__ __forceinline__ typename Vec2<R>::T res_get(const Args<R>& a, const Res<R>& r, uint32_t j, uint64_t k) {
  const uint64_t pos = result_pos(r.layout, a.P, a.A, a.B, a.cap, k);
  typename Vec2<R>::T v = r.base[(uint64_t)j * r.stride + pos];
  if (r.chirp) {
    v = mul2(v, a.chirp[k]);
    v.x *= a.invP;
    v.y *= a.invP;
  }
  return v;
}

template <class R>
__device__ __forceinline__ void post_elem(const Args<R>& a, const Res<R>& r, typename Vec2<R>::T* spectrum, uint32_t j,
                                          const ChunkInfo& ci, uint32_t k) {
  using T2 = typename Vec2<R>::T;
  T2 X;
  if ((a.L & 1u) == 0) {
    const uint32_t Lc = a.Lc;
    const T2 zk = res_get(a, r, j, k == Lc ? 0 : k);
    const T2 zm = res_get(a, r, j, k == 0 ? 0 : Lc - k);
    const T2 A = mk2(zk.x + zm.x, zk.y - zm.y);   // Z[k] + conj Z[Lc-k]
    const T2 B = mk2(zk.x - zm.x, zk.y + zm.y);   // Z[k] - conj Z[Lc-k]
    const T2 t = mul2(a.rtw[k], mk2(B.y, -B.x));  // W^k (-i B)
    X = mk2((R)0.5 * (A.x + t.x), (R)0.5 * (A.y + t.y));
    if (k == 0 || k == Lc) X.y = (R)0;
  } else {
    X = res_get(a, r, j, k);
    if (k == 0) X.y = (R)0;
  }
  spectrum[ci.bin_off + k] = X;
}

template <class R>
__global__ void k_post(Args<R> a, Res<R> r, typename Vec2<R>::T* spectrum) {
  const uint32_t j = blockIdx.y;
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.bins) return;
  const ChunkInfo ci = a.chunks[a.first + j];
  post_elem(a, r, spectrum, j, ci, k);
}

template <class R>
__device__ __forceinline__ void iprep_elem(const Args<R>& a, const typename Vec2<R>::T* spectrum, uint32_t j,
                                           const ChunkInfo& ci, uint32_t k) {
  using T2 = typename Vec2<R>::T;
  const T2* X = spectrum + ci.bin_off;
  T2 Z = mk2((R)0, (R)0);
  if (k < a.Lc) {
    if ((a.L & 1u) == 0) {
      const uint32_t Lc = a.Lc;
      T2 xk = X[k], xm = X[Lc - k];
      if (k == 0) { xk.y = (R)0; xm.y = (R)0; }   // DC and Nyquist imag ignored
      const T2 E = mk2((R)0.5 * (xk.x + xm.x), (R)0.5 * (xk.y - xm.y));
      const T2 D = mk2((R)0.5 * (xk.x - xm.x), (R)0.5 * (xk.y + xm.y));
      const T2 O = mul2(D, cj(a.rtw[k]));         // W^{-k} D
      Z = mk2(E.x - O.y, E.y + O.x);              // E + i O
    } else {
      const uint32_t h = (a.L - 1) / 2;
      if (k <= h) {
        Z = X[k];
        if (k == 0) Z.y = (R)0;
      } else {
        Z = cj(X[a.L - k]);
      }
    }
  }
  uint64_t pos = k;
  if (a.kind == (int)DftKind::Bluestein) {
    if (k < a.Lc) Z = mul2(cj(Z), a.chirp[k]);
  } else if (a.kind == (int)DftKind::Pow2) {
    pos = engine_pos(a.P, a.cap, k);
  } else if (a.kind == (int)DftKind::Mixed) {
    pos = result_pos(2, a.P, a.A, a.B, a.cap, k);
  }
  a.work[(uint64_t)j * a.Pw + pos] = Z;
}

template <class R>
__global__ void k_iprep(Args<R> a, const typename Vec2<R>::T* spectrum) {
  const uint32_t j = blockIdx.y;
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.Pw) return;
  const ChunkInfo ci = a.chunks[a.first + j];
  iprep_elem(a, spectrum, j, ci, k);
}

template <class R>
__device__ __forceinline__ void ipost_elem(const Args<R>& a, const Res<R>& r, R* out, R scale, uint32_t j,
                                           const ChunkInfo& ci, uint32_t n) {
  using T2 = typename Vec2<R>::T;
  T2 v = res_get(a, r, j, n);
  if (a.kind == (int)DftKind::Bluestein) v = cj(v);
  if ((a.L & 1u) == 0) {
    out[ci.in_off + 2ull * n] = v.x * scale;
    out[ci.in_off + 2ull * n + 1] = v.y * scale;
  } else {
    out[ci.in_off + n] = v.x * scale;
  }
}

template <class R>
__global__ void k_ipost(Args<R> a, Res<R> r, R* out, R scale) {
  const uint32_t j = blockIdx.y;
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= a.Lc) return;
  const ChunkInfo ci = a.chunks[a.first + j];
  ipost_elem(a, r, out, scale, j, ci, n);
}

template <class R>
Args<R> make_args(const RealClassT<R>& rc, const ChunkInfo* d_chunks) {
  Args<R> a;
  const DftPlanT<R>& d = rc.dft;
  a.chunks = d_chunks;
  a.first = rc.first;
  a.L = rc.L;
  a.Lc = d.Lc;
  a.Pw = d.P;
  a.P = d.P;
  a.A = d.A;
  a.B = d.B;
  a.bins = rc.bins;
  a.cap = smem_points(sizeof(R));
  a.kind = (int)d.kind;
  a.work = d.work;
  a.chirp = d.chirp;
  a.rtw = d.rtw;
  a.invP = (R)1 / (R)d.P;
  return a;
}

// ---------------------------------------------------------- single-CTA tail chains
//
// A plan's tail chunk runs on the side stream beside the fused grid.  As a
// chain of small kernels each launch waits for SMs the fused grid frees only
// at its CTAs' ends, and the chain costs ~12 us of step at 25.6M floats (the
// same for a 4096- as for a 40960-sample tail); a single CTA spinning for
// 100 us per direction costs only ~2 us.  One 1024-thread CTA here runs the
// whole chain per direction, the same device code in the same order (so the
// same bits): forward = prep, mixed outer pass, row FFTs, real
// post-processing, select + pack; inverse = weighted decode of the W
// messages, pre-processing, row FFTs, mixed outer pass, real
// post-processing.  Pow2 (P <= 4096) and Mixed (B <= 4096) only.  Measured
// at C2 (tools/tail_phase_probe.py, us): forward prep 15, mixed 28, rows 69,
// post 26, select + pack 44 (183); inverse decode 16, pre 14, rows 71, mixed
// 26, post 4 (131) -- too long: the chain lands on the critical path, so it
// is opt-in (FGC_TAIL_CHAIN=1) until its phases are made latency-tolerant.

constexpr int kTailThreads = 1024;
__device__ unsigned long long g_tail_ts[32];     // phase stamps of the last tail chains (diagnostics)
__device__ __forceinline__ void tail_ts(int k) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tail_ts[k] = t;
  }
}
constexpr size_t kTailSmem = 200 * 1024;

__device__ __forceinline__ void tail_rows(float2* rows, uint32_t nrows, uint32_t S, const float2* tw, int dir,
                                          unsigned char* sm) {
  float2* x = reinterpret_cast<float2*>(sm);
  float2* y = x + S;
  float2* stw = y + S;
  gdev::load_stage_twiddles(stw, S, tw, S);
  for (uint32_t r = 0; r < nrows; ++r) {
    float2* g = rows + (uint64_t)r * S;
    for (uint32_t e = threadIdx.x; e < S; e += blockDim.x) x[e] = g[e];
    __syncthreads();
    const float2* res = gdev::smem_stockham(x, y, S, 1, stw, dir);
    for (uint32_t e = threadIdx.x; e < S; e += blockDim.x) g[e] = res[e];
    __syncthreads();
  }
}

__device__ __forceinline__ void tail_mixed(const float2* in, float2* out, const float2* mtw, uint32_t A, uint32_t B,
                                           uint32_t cols, int dir, unsigned char* sm) {
  for (uint32_t bx = 0; bx * cols < B; ++bx) {
    gdev::mixed_tile(in, out, mtw, A, B, cols, A, dir, bx, 0, 0, sm);
    __syncthreads();
  }
}

template <class In>
__global__ void __launch_bounds__(kTailThreads, 1) k_tail_forward(Args<float> a, const In* in, int half,
                                                                  uint32_t* flags, float2* spectrum, const float2* tw,
                                                                  const float2* mtw, float2* work2, uint32_t cols,
                                                                  QuantParams q, uint8_t* message) {
  extern __shared__ __align__(16) unsigned char sm[];
  const ChunkInfo ci = a.chunks[a.first];
  tail_ts(0);
  for (uint32_t n = threadIdx.x; n < a.Pw; n += blockDim.x) prep_elem(a, in, half, flags, 0, ci, n);
  __syncthreads();
  tail_ts(1);
  const bool mixed = a.kind == (int)DftKind::Mixed;
  if (mixed) tail_mixed(a.work, work2, mtw, a.A, a.B, cols, -1, sm);
  tail_ts(2);
  tail_rows(mixed ? work2 : a.work, mixed ? a.A : 1u, mixed ? a.B : a.P, tw, -1, sm);
  tail_ts(3);
  const Res<float> rr = mixed ? Res<float>{work2, a.Lc, 2, 0} : Res<float>{a.work, a.P, 1, 0};
  for (uint32_t k = threadIdx.x; k < a.bins; k += blockDim.x) post_elem(a, rr, spectrum, 0, ci, k);
  __syncthreads();
  tail_ts(4);
  sel::select_pack_chunk<float2, kTailThreads>(*reinterpret_cast<sel::SelectSharedT<kTailThreads>*>(sm), ci,
                                               sel::Coeffs<float2>{spectrum + ci.bin_off}, 0, q, message, nullptr,
                                               flags, nullptr);
  tail_ts(5);
}

__global__ void __launch_bounds__(kTailThreads, 1) k_tail_inverse(Args<float> a, const uint8_t* messages, int W,
                                                                  int G, uint64_t stride, Weights wts, QuantParams q,
                                                                  float2* spectrum, const float2* tw,
                                                                  const float2* mtw, float2* work2, uint32_t cols,
                                                                  float* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint32_t scan[40];
  const ChunkInfo ci = a.chunks[a.first];
  tail_ts(10);
  for (int w0 = 0; w0 < W; w0 += G) {
    decode_accumulate_chunk<kTailThreads>(ci, messages, W, w0, G, stride, wts, q, spectrum,
                                          reinterpret_cast<uint32_t*>(sm), scan);
    __syncthreads();
  }
  tail_ts(11);
  for (uint32_t k = threadIdx.x; k < a.Pw; k += blockDim.x) iprep_elem(a, spectrum, 0, ci, k);
  __syncthreads();
  tail_ts(12);
  const bool mixed = a.kind == (int)DftKind::Mixed;
  tail_rows(a.work, mixed ? a.A : 1u, mixed ? a.B : a.P, tw, +1, sm);
  tail_ts(13);
  if (mixed) tail_mixed(a.work, work2, mtw, a.A, a.B, cols, +1, sm);
  tail_ts(14);
  const Res<float> rr = mixed ? Res<float>{work2, a.Lc, 0, 0} : Res<float>{a.work, a.P, 0, 0};
  for (uint32_t n = threadIdx.x; n < a.Lc; n += blockDim.x) ipost_elem(a, rr, out, 1.0f / (float)a.Lc, 0, ci, n);
  __syncthreads();
  tail_ts(15);
}

// columns of the mixed outer pass per tile within the shared-memory budget
uint32_t tail_cols(uint32_t A, uint32_t B) {
  uint32_t cols = B;
  while (cols > 1 && (uint64_t)(A + A * cols) * sizeof(float2) > kTailSmem) cols >>= 1;
  return cols;
}

}  // namespace

template <class R>
fgc_status RealClassT<R>::init(cudaStream_t s) {
  using T2 = typename Vec2<R>::T;
  const uint32_t Lc = (L % 2 == 0) ? L / 2 : L;
  FGC_TRY(dft.init(Lc, count, s));
  if (L % 2 == 0) {
    std::vector<T2> h(Lc + 1);
    for (uint32_t k = 0; k <= Lc; ++k) {
      const double ang = -2.0 * M_PI * (double)k / (double)L;
      h[k].x = (R)cos(ang);
      h[k].y = (R)sin(ang);
    }
    FGC_CUDA(cudaMalloc(&dft.rtw, sizeof(T2) * (Lc + 1)));
    FGC_CUDA(cudaMemcpy(dft.rtw, h.data(), sizeof(T2) * (Lc + 1), cudaMemcpyHostToDevice));
  }
  return FGC_OK;
}

template <class R>
fgc_status real_forward(RealClassT<R>& rc, const ChunkInfo* d_chunks, const void* in, int in_dtype, int half_pass,
                        uint32_t* flags, typename Vec2<R>::T* spectrum, cudaStream_t s) {
  if (!rc.count) return FGC_OK;
  Args<R> a = make_args(rc, d_chunks);
  dim3 grid(cdiv(a.Pw, 256), rc.count);
  if (in_dtype == FGC_DTYPE_F64)
    k_prep<R, double><<<grid, 256, 0, s>>>(a, static_cast<const double*>(in), half_pass, flags);
  else
    k_prep<R, float><<<grid, 256, 0, s>>>(a, static_cast<const float*>(in), half_pass, flags);
  FGC_LAUNCHED(1);
  DftResultT<R> r;
  FGC_TRY(rc.dft.run(-1, r, s));
  Res<R> rr{r.base, r.stride, r.layout, r.chirp};
  k_post<R><<<dim3(cdiv(a.bins, 256), rc.count), 256, 0, s>>>(a, rr, spectrum);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

template <class R>
fgc_status real_inverse(RealClassT<R>& rc, const ChunkInfo* d_chunks, const typename Vec2<R>::T* spectrum, R* out,
                        cudaStream_t s) {
  if (!rc.count) return FGC_OK;
  Args<R> a = make_args(rc, d_chunks);
  k_iprep<R><<<dim3(cdiv(a.Pw, 256), rc.count), 256, 0, s>>>(a, spectrum);
  FGC_LAUNCHED(1);
  DftResultT<R> r;
  FGC_TRY(rc.dft.run(+1, r, s));
  Res<R> rr{r.base, r.stride, r.layout, r.chirp};
  k_ipost<R><<<dim3(cdiv(a.Lc, 256), rc.count), 256, 0, s>>>(a, rr, out, (R)1 / (R)a.Lc);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

bool tail_chain_ok(const RealClassT<float>& rc) {
  if (rc.count != 1 || !rc.dft.batch) return false;
  const uint32_t cap = smem_points(sizeof(float));
  if (rc.dft.kind == DftKind::Pow2) return rc.dft.P <= cap && rc.dft.P >= 2;
  if (rc.dft.kind == DftKind::Mixed) return rc.dft.B <= cap && rc.dft.B >= 2;
  return false;
}

static fgc_status tail_attrs() {
  static bool done = false;
  if (done) return FGC_OK;
  FGC_CUDA(cudaFuncSetAttribute(k_tail_forward<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailSmem));
  FGC_CUDA(cudaFuncSetAttribute(k_tail_forward<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailSmem));
  FGC_CUDA(cudaFuncSetAttribute(k_tail_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailSmem));
  done = true;
  return FGC_OK;
}

fgc_status tail_forward_chain(RealClassT<float>& rc, const ChunkInfo* d_chunks, const void* in, int in_dtype,
                              int half_pass, uint32_t* flags, float2* spectrum, const QuantParams& q, uint8_t* message,
                              cudaStream_t s) {
  FGC_TRY(tail_attrs());
  Args<float> a = make_args(rc, d_chunks);
  const uint32_t cols = tail_cols(a.A, a.B);
  if (in_dtype == FGC_DTYPE_F64)
    k_tail_forward<double><<<1, kTailThreads, kTailSmem, s>>>(a, static_cast<const double*>(in), half_pass, flags,
                                                              spectrum, rc.dft.tw, rc.dft.mtw, rc.dft.work2, cols, q,
                                                              message);
  else
    k_tail_forward<float><<<1, kTailThreads, kTailSmem, s>>>(a, static_cast<const float*>(in), half_pass, flags,
                                                             spectrum, rc.dft.tw, rc.dft.mtw, rc.dft.work2, cols, q,
                                                             message);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

fgc_status tail_inverse_chain(RealClassT<float>& rc, const ChunkInfo* d_chunks, const uint8_t* messages, int W,
                              uint64_t stride, const Weights& wts, const QuantParams& q, float2* spectrum, float* out,
                              uint32_t max_slots, cudaStream_t s) {
  FGC_TRY(tail_attrs());
  Args<float> a = make_args(rc, d_chunks);
  const uint32_t bm_words = (max_slots + 31) / 32;
  const int G = (int)std::max<size_t>(1, std::min<size_t>((size_t)W, kTailSmem / (bm_words * 4ull)));
  if ((size_t)bm_words * 4 > kTailSmem) { set_error("tail chunk too large for the prefix tables"); return FGC_ERR_UNSUPPORTED; }
  const uint32_t cols = tail_cols(a.A, a.B);
  k_tail_inverse<<<1, kTailThreads, kTailSmem, s>>>(a, messages, W, G, stride, wts, q, spectrum, rc.dft.tw,
                                                    rc.dft.mtw, rc.dft.work2, cols, out);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

}  // namespace fgc
extern "C" int fgc_debug_tail_timestamps(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, fgc::g_tail_ts, 32 * sizeof(unsigned long long)) == cudaSuccess ? 0 : 1;
}
namespace fgc {

template struct RealClassT<float>;
template struct RealClassT<double>;
template fgc_status real_forward<float>(RealClassT<float>&, const ChunkInfo*, const void*, int, int, uint32_t*, float2*,
                                        cudaStream_t);
template fgc_status real_forward<double>(RealClassT<double>&, const ChunkInfo*, const void*, int, int, uint32_t*,
                                         double2*, cudaStream_t);
template fgc_status real_inverse<float>(RealClassT<float>&, const ChunkInfo*, const float2*, float*, cudaStream_t);
template fgc_status real_inverse<double>(RealClassT<double>&, const ChunkInfo*, const double2*, double*, cudaStream_t);

}  // namespace fgc
