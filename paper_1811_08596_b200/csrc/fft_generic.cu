// Generic batched complex DFT engine, float32 or float64.  It takes every
// transform the fused kernels do not: tail chunks, non-power-of-two chunk
// sizes, and the whole-signal primitives (dft_forward / dft_inverse /
// calibrate, which the reference computes in float64 with numpy's pocketfft:
// spectral.py:95,106, codec.py:463).
//
//   Direct     Lc <= 64            O(Lc^2) per signal, exact-reduced twiddles
//   Pow2       Lc = 2^k            Stockham radix-4 in shared memory (<= 4096
//                                  points), larger sizes by a four-step split
//                                  through global memory (recursive on rows)
//   Mixed      Lc = A 2^e, A odd    one direct pass over the odd factor (A <=
//              <= kMixedMaxA       kMixedMaxA, twiddles folded in) + A Pow2
//                                  rows of B = 2^e points (Cooley-Tukey)
//   Bluestein  anything else        chirp-z convolution on a Pow2 engine of
//                                  size P >= 2 Lc - 1
//
// Twiddles/chirps are evaluated in float64 with the angle reduced exactly in
// integers, then stored in the engine precision.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "fgc_device.cuh"
#include "fgc_internal.h"
#include "generic_dev.cuh"

namespace fgc {

namespace {

using namespace gdev;

constexpr int kFftThreads = 256;

template <class R>
__global__ void k_init_twiddles(typename V2<R>::T* tw, uint32_t P) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P) return;
  double s, c;
  sincospi(-2.0 * (double)j / (double)P, &s, &c);
  tw[j] = mk((R)c, (R)s);
}

template <class R>
__global__ void k_init_chirp(typename V2<R>::T* chirp, uint32_t Lc) {
  uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= Lc) return;
  const uint64_t m = ((uint64_t)n * n) % (2ull * Lc);       // exact angle reduction
  double s, c;
  sincospi(-(double)m / (double)Lc, &s, &c);
  chirp[n] = mk((R)c, (R)s);
}

template <class R>
__global__ void k_init_bluestein_b(typename V2<R>::T* b, const typename V2<R>::T* chirp, uint32_t P, uint32_t Lc) {
  uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P) return;
  typename V2<R>::T v = mk((R)0, (R)0);
  if (e < Lc) v = zconj(chirp[e]);
  else if (P - e < Lc) v = zconj(chirp[P - e]);
  b[e] = v;
}

// Batched transforms of size S <= kSmemFftMax stored contiguously.  NT
// threads: 1024 when the batch is too small to fill the GPU (a tail chunk's
// sub-transforms), where every radix-2 stage is latency-bound per thread.
template <class T2, int NT>
__global__ void __launch_bounds__(NT) k_smem_fft(T2* data, uint32_t S, uint32_t per_cta, uint64_t total,
                                                 const T2* tw, uint32_t twP, int dir) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T2* sm = reinterpret_cast<T2*>(smraw);
  const uint64_t first = (uint64_t)blockIdx.x * per_cta;
  if (first >= total) return;
  const uint32_t nt = (uint32_t)min((uint64_t)per_cta, total - first);
  T2* x = sm;
  T2* y = sm + (size_t)per_cta * S;
  T2* stw = y + (size_t)per_cta * S;
  T2* g = data + first * S;
  load_stage_twiddles(stw, S, tw, twP);
  for (uint32_t e = threadIdx.x; e < nt * S; e += blockDim.x) x[e] = g[e];
  __syncthreads();
  T2* r = smem_stockham(x, y, S, nt, stw, dir);
  for (uint32_t e = threadIdx.x; e < nt * S; e += blockDim.x) g[e] = r[e];
}

// Four-step column pass over an R x C matrix per item (item stride R*C):
// G columns per CTA, a length-R FFT down each, with the inter-step twiddle
// W_{RC}^{c k1} after (forward) or before (inverse) the column transform.
template <class T2>
__global__ void __launch_bounds__(kFftThreads) k_col_fft(T2* data, uint32_t Rr, uint32_t C, uint32_t G, const T2* tw,
                                                         uint32_t twP, int dir) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T2* sm = reinterpret_cast<T2*>(smraw);
  const uint32_t groups = C / G;
  const uint64_t P = (uint64_t)Rr * C;
  const uint64_t item = blockIdx.x / groups;
  const uint32_t c0 = (blockIdx.x % groups) * G;
  const uint32_t tws = (uint32_t)(twP / P);   // table is for twP >= P
  T2* g = data + item * P;
  T2* x = sm;
  T2* y = sm + (size_t)G * Rr;
  T2* stw = y + (size_t)G * Rr;
  load_stage_twiddles(stw, Rr, tw, twP);
  for (uint32_t e = threadIdx.x; e < G * Rr; e += blockDim.x) {
    const uint32_t r = e / G, cg = e % G;            // coalesced along columns
    T2 v = g[(uint64_t)r * C + c0 + cg];
    if (dir > 0) {
      T2 w = tw[(((uint64_t)(c0 + cg) * r) % P) * tws];
      w.y = -w.y;
      v = zmul(v, w);
    }
    x[cg * Rr + r] = v;
  }
  __syncthreads();
  T2* res = smem_stockham(x, y, Rr, G, stw, dir);
  for (uint32_t e = threadIdx.x; e < G * Rr; e += blockDim.x) {
    const uint32_t r = e / G, cg = e % G;
    T2 v = res[cg * Rr + r];
    if (dir < 0) v = zmul(v, tw[(((uint64_t)(c0 + cg) * r) % P) * tws]);
    g[(uint64_t)r * C + c0 + cg] = v;
  }
}

// Direct DFT for Lc <= 64: out[k] = sum_n in[n] exp(dir * 2 pi i n k / Lc).
template <class R>
__global__ void k_direct_dft(const typename V2<R>::T* in, typename V2<R>::T* out, uint32_t Lc, int dir) {
  using T2 = typename V2<R>::T;
  __shared__ T2 z[64];
  __shared__ T2 w[64];
  const T2* src = in + (uint64_t)blockIdx.x * Lc;
  T2* dst = out + (uint64_t)blockIdx.x * Lc;
  for (uint32_t n = threadIdx.x; n < Lc; n += blockDim.x) {
    z[n] = src[n];
    double s, c;
    sincospi((double)dir * 2.0 * (double)n / (double)Lc, &s, &c);
    w[n] = mk((R)c, (R)s);
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < Lc; k += blockDim.x) {
    T2 acc = mk((R)0, (R)0);
    uint32_t idx = 0;
    for (uint32_t n = 0; n < Lc; ++n) {
      acc = zadd(acc, zmul(z[n], w[idx]));
      idx += k;
      if (idx >= Lc) idx -= Lc;
    }
    dst[k] = acc;
  }
}

template <class T2>
__global__ void __launch_bounds__(256) k_mixed_pass(const T2* in, T2* out, const T2* mtw, uint32_t A, uint32_t B,
                                                    uint32_t cols, uint32_t kg, int dir) {
  extern __shared__ __align__(16) unsigned char smraw[];
  mixed_tile(in, out, mtw, A, B, cols, kg, dir, blockIdx.x, blockIdx.y, blockIdx.z, smraw);
}

template <class T2>
__global__ void k_pointwise_mul(T2* data, const T2* f, uint32_t P, uint64_t total) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  data[e] = zmul(data[e], f[e % P]);
}

inline uint32_t ceil_div(uint64_t a, uint32_t b) { return (uint32_t)((a + b - 1) / b); }

template <class R>
fgc_status mixed_pass(const typename V2<R>::T* in, typename V2<R>::T* out, const typename V2<R>::T* mtw, uint32_t A,
                      uint32_t B, uint32_t batch, int dir, cudaStream_t s) {
  using T2 = typename V2<R>::T;
  // columns per CTA: up to 32, within ~96 KB of tile; rows so a CTA has ~256 outputs
  uint32_t cols = 32;
  while (cols > 1 && (uint64_t)(A + A * cols) * sizeof(T2) > 96 * 1024) cols >>= 1;
  cols = std::min(cols, B);
  // ~64 outputs per CTA: the A-term sums are latency-bound, so spread them wide
  const uint32_t kg = std::max(1u, 64u / cols);
  const size_t smem = (size_t)(A + A * cols) * sizeof(T2);
  static bool attr = false;
  if (!attr) {
    FGC_CUDA(cudaFuncSetAttribute(k_mixed_pass<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    FGC_CUDA(cudaFuncSetAttribute(k_mixed_pass<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    attr = true;
  }
  const dim3 grid(ceil_div(B, cols), ceil_div(A, kg), batch);
  k_mixed_pass<T2><<<grid, 256, smem, s>>>(in, out, mtw, A, B, cols, kg, dir);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

template <class R>
fgc_status pow2_rec(typename V2<R>::T* data, uint64_t batch, uint32_t P, const typename V2<R>::T* tw, uint32_t twP,
                    int dir, cudaStream_t s) {
  using T2 = typename V2<R>::T;
  if (P <= 1 || batch == 0) return FGC_OK;
  const uint32_t cap = smem_points(sizeof(R));   // points per CTA, held twice in 64 KB
  if (P <= cap) {
    // transforms per CTA: up to a full shared-memory tile, but small batches
    // are spread over the SMs (latency, not throughput, rules there)
    const uint32_t per = max(1u, min(cap / P, (uint32_t)((batch + 295) / 296)));
    const size_t smem = (2ull * per * P + stage_twiddles(P)) * sizeof(T2);
    const uint32_t ctas = ceil_div(batch, per);
    if (ctas < 148 && P * per >= 4096)
      k_smem_fft<T2, 1024><<<ctas, 1024, smem, s>>>(data, P, per, batch, tw, twP, dir);
    else
      k_smem_fft<T2, kFftThreads><<<ctas, kFftThreads, smem, s>>>(data, P, per, batch, tw, twP, dir);
    FGC_LAUNCHED(1);
    return FGC_OK;
  }
  uint32_t Rr, C;
  fft_split(P, cap, Rr, C);
  const uint32_t G = max(1u, min(C, cap / Rr));
  const size_t col_smem = (2ull * G * Rr + stage_twiddles(Rr)) * sizeof(T2);
  const uint64_t cols = batch * (C / G);
  if (cols > 0x7FFFFFFFull) { set_error("transform batch too large"); return FGC_ERR_UNSUPPORTED; }
  if (dir < 0) {
    k_col_fft<T2><<<(uint32_t)cols, kFftThreads, col_smem, s>>>(data, Rr, C, G, tw, twP, dir);
    FGC_LAUNCHED(1);
    FGC_TRY(pow2_rec<R>(data, batch * Rr, C, tw, twP, dir, s));
  } else {
    FGC_TRY(pow2_rec<R>(data, batch * Rr, C, tw, twP, dir, s));
    k_col_fft<T2><<<(uint32_t)cols, kFftThreads, col_smem, s>>>(data, Rr, C, G, tw, twP, dir);
    FGC_LAUNCHED(1);
  }
  return FGC_OK;
}

uint32_t next_pow2(uint64_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

template <class R>
fgc_status set_attrs() {
  using T2 = typename V2<R>::T;
  static bool done = false;
  if (done) return FGC_OK;
  const int bytes = (int)((2 * smem_points(sizeof(R)) + stage_twiddles(smem_points(sizeof(R)))) * sizeof(T2));
  FGC_CUDA(cudaFuncSetAttribute(k_smem_fft<T2, kFftThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  FGC_CUDA(cudaFuncSetAttribute(k_smem_fft<T2, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  FGC_CUDA(cudaFuncSetAttribute(k_col_fft<T2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done = true;
  return FGC_OK;
}

}  // namespace

template <class R>
fgc_status DftPlanT<R>::init(uint32_t Lc_, uint32_t batch_, cudaStream_t s) {
  FGC_TRY(set_attrs<R>());
  Lc = Lc_;
  batch = batch_;
  if (Lc <= 64) {
    kind = DftKind::Direct;
    P = Lc;
  } else if ((Lc & (Lc - 1)) == 0) {
    kind = DftKind::Pow2;
    P = Lc;
  } else if ((Lc >> __builtin_ctz(Lc)) <= kMixedMaxA) {
    kind = DftKind::Mixed;
    B = 1u << __builtin_ctz(Lc);
    A = Lc / B;
    P = Lc;
  } else {
    kind = DftKind::Bluestein;
    if (2ull * Lc - 1 > (1ull << 31)) { set_error("DFT length too large"); return FGC_ERR_UNSUPPORTED; }
    P = next_pow2(2ull * Lc - 1);
  }
  if (kind == DftKind::Mixed) {
    FGC_CUDA(cudaMalloc(&mtw, sizeof(T2) * Lc));
    k_init_twiddles<R><<<ceil_div(Lc, 256), 256, 0, s>>>(mtw, Lc);
    FGC_LAUNCHED(1);
    if (B > 1) {
      FGC_CUDA(cudaMalloc(&tw, sizeof(T2) * B));
      k_init_twiddles<R><<<ceil_div(B, 256), 256, 0, s>>>(tw, B);
      FGC_LAUNCHED(1);
    }
  } else if (kind != DftKind::Direct) {
    FGC_CUDA(cudaMalloc(&tw, sizeof(T2) * P));
    k_init_twiddles<R><<<ceil_div(P, 256), 256, 0, s>>>(tw, P);
    FGC_LAUNCHED(1);
  }
  if (batch) {
    FGC_CUDA(cudaMalloc(&work, sizeof(T2) * (uint64_t)P * batch));
    if (kind == DftKind::Direct || kind == DftKind::Mixed)
      FGC_CUDA(cudaMalloc(&work2, sizeof(T2) * (uint64_t)P * batch));
  }
  if (kind == DftKind::Bluestein) {
    FGC_CUDA(cudaMalloc(&chirp, sizeof(T2) * Lc));
    FGC_CUDA(cudaMalloc(&bf, sizeof(T2) * P));
    k_init_chirp<R><<<ceil_div(Lc, 256), 256, 0, s>>>(chirp, Lc);
    FGC_LAUNCHED(1);
    k_init_bluestein_b<R><<<ceil_div(P, 256), 256, 0, s>>>(bf, chirp, P, Lc);
    FGC_LAUNCHED(1);
    FGC_TRY(pow2_rec<R>(bf, 1, P, tw, P, -1, s));
  }
  return FGC_OK;
}

template <class R>
void DftPlanT<R>::free_all() {
  cudaFree(tw);
  cudaFree(chirp);
  cudaFree(bf);
  cudaFree(work);
  cudaFree(work2);
  cudaFree(rtw);
  cudaFree(mtw);
  tw = chirp = bf = work = work2 = rtw = mtw = nullptr;
}

template <class R>
fgc_status DftPlanT<R>::run(int dir, DftResultT<R>& res, cudaStream_t s) {
  switch (kind) {
    case DftKind::Direct:
      if (batch) {
        k_direct_dft<R><<<batch, 64, 0, s>>>(work, work2, Lc, dir > 0 ? 1 : -1);
        FGC_LAUNCHED(1);
      }
      res = DftResultT<R>{work2, Lc, 0, 0};
      return FGC_OK;
    case DftKind::Pow2:
      FGC_TRY(pow2_rec<R>(work, batch, P, tw, P, dir, s));
      res = DftResultT<R>{work, P, dir < 0 ? 1 : 0, 0};
      return FGC_OK;
    case DftKind::Mixed: {
      const uint64_t total = (uint64_t)batch * Lc;
      if (dir < 0) {                                 // natural work -> rows in work2 (engine layout)
        if (total) FGC_TRY(mixed_pass<R>(work, work2, mtw, A, B, batch, -1, s));
        FGC_TRY(pow2_rec<R>(work2, (uint64_t)batch * A, B, tw, B, -1, s));
        res = DftResultT<R>{work2, Lc, 2, 0};
      } else {                                       // rows (engine layout) in work -> natural work2
        FGC_TRY(pow2_rec<R>(work, (uint64_t)batch * A, B, tw, B, +1, s));
        if (total) FGC_TRY(mixed_pass<R>(work, work2, mtw, A, B, batch, +1, s));
        res = DftResultT<R>{work2, Lc, 0, 0};
      }
      return FGC_OK;
    }
    case DftKind::Bluestein: {
      FGC_TRY(pow2_rec<R>(work, batch, P, tw, P, -1, s));
      const uint64_t total = (uint64_t)batch * P;
      if (total) {
        k_pointwise_mul<T2><<<ceil_div(total, 256), 256, 0, s>>>(work, bf, P, total);
        FGC_LAUNCHED(1);
      }
      FGC_TRY(pow2_rec<R>(work, batch, P, tw, P, +1, s));
      res = DftResultT<R>{work, P, 0, 1};
      return FGC_OK;
    }
  }
  return FGC_ERR_INVALID;
}

template struct DftPlanT<float>;
template struct DftPlanT<double>;

}  // namespace fgc
