// Compress of 65536-sample chunks by 2-CTA clusters of 1024 threads: the
// k_fused_compress design (fused.cu) with every radix-32 column split over a
// lane pair, so an SM holds 32 warps instead of 16 and each thread keeps 16
// of the chunk's values (64 registers) instead of 32.
//
// Thread t is half h = (t >> 4) & 1 of pair i = 16 (t >> 5) + (t & 15); its
// partner is lane ^ 16.  A 32-point DFT over j (x[i + 512 j]) becomes one
// radix-2 DIF stage across the pair (shuffle) and a 16-point DFT per half:
// half 0 ends with the even outputs X[2k], half 1 with the odd X[2k + 1].
// Pass 3 gives each half one of the pair's two columns (k, 1024 - k) /
// (k, 1023 - k); the real-FFT post-processing exchanges the columns once.
// From there each thread holds the 16 bins of one column, and the
// selection, emit and pack phases -- latency-bound chains per thread in
// fused.cu -- do half the work per thread with twice the warps to overlap.
// The message is bit-identical to k_fused_compress's.
#include <cooperative_groups.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>

#include <type_traits>

#include "fgc_device.cuh"
#include "fgc_internal.h"
#include "fused_fft.cuh"
#include "select_pack.cuh"

namespace cg = cooperative_groups;

namespace fgc {
namespace {

using ff::bitrev;
using ff::dft;
using ff::kL;
using ff::kM;
using ff::kN;
using ff::kPadded;
using ff::kT1024Padded;
using ff::kTloPadded;
using ff::pad;
using ff::tpad;
using ff::tw;
using ff::twc;
using ff::w32mul;
using ff::w64mul;

constexpr int kTW = 1024;                              // threads per CTA
constexpr int kCand = 512;
constexpr uint32_t kBins = kN + 1;                     // 32769
constexpr uint32_t kBmWords = (2 * kBins + 31) / 32;   // 2049
constexpr uint32_t kHalfBins = kN / 2;                 // 16384: pack split point
constexpr uint32_t kStageOff = 16900;                  // u32 offset of the code-stream staging in buf
constexpr uint32_t kEmitStageOff = 16904;              // emit strips: per warp 128 bins + 128 float2
constexpr uint32_t kEmitStageWords = 384;
static_assert(kEmitStageOff % 2 == 0 && kEmitStageOff >= kHalfBins + kHalfBins / 32 &&
              kEmitStageOff + 32 * kEmitStageWords <= 2 * (kPadded + 64), "emit strips fit in buf");

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

template <class T> struct InW;
template <> struct InW<float> {
  template <bool HALF>
  __device__ static float2 get(const float* g, uint64_t e, uint32_t& bad) {
    float2 v = __ldg(reinterpret_cast<const float2*>(g + e));
    bad |= (isfinite(v.x) && isfinite(v.y)) ? 0u : FGC_FLAG_NONFINITE;
    if (HALF) {
      v.x = __half2float(__float2half_rn(v.x));
      v.y = __half2float(__float2half_rn(v.y));
      bad |= (isinf(v.x) || isinf(v.y)) ? FGC_FLAG_HALF_OVERFLOW : 0u;
    }
    return v;
  }
};
template <> struct InW<double> {
  template <bool HALF>
  __device__ static float2 get(const double* g, uint64_t e, uint32_t& bad) {
    const double2 d = __ldg(reinterpret_cast<const double2*>(g + e));
    if (!isfinite(d.x) || !isfinite(d.y)) { bad |= FGC_FLAG_NONFINITE; return make_float2(0.f, 0.f); }
    float2 v;
    if (HALF) {
      v = make_float2(__half2float(__double2half(d.x)), __half2float(__double2half(d.y)));
      if (isinf(v.x) || isinf(v.y)) bad |= FGC_FLAG_HALF_OVERFLOW;
    } else {
      v = make_float2((float)d.x, (float)d.y);
      if (isinf(v.x) || isinf(v.y)) bad |= FGC_FLAG_F32_RANGE;
    }
    return v;
  }
};

__device__ __forceinline__ uint32_t enc16(const QuantParams& q, float x) {
  const float a = fabsf(x);
  const bool pos = x > 0.0f;
  const uint32_t off = (__float_as_uint(fminf(a, pos ? q.pos_cap : q.neg_cap)) >> q.shift) - q.pbase + 1u;
  const uint32_t c = pos ? min(off, q.npos) : q.npos + min(off, q.nneg);
  return (a < q.eps) ? 0u : c;
}

__device__ __forceinline__ float2 shfl16(float2 v) {
  return make_float2(__shfl_xor_sync(0xffffffffu, v.x, 16), __shfl_xor_sync(0xffffffffu, v.y, 16));
}

// 32-point DFT over j of a lane pair: v holds j = 16 h + jj (jj < 16); on
// exit v[bitrev4(k)] = X[2 k + h].
template <bool INV>
__device__ __forceinline__ void pair_dft32(float2 (&v)[16], uint32_t h) {
  // first radix-2 DIF stage across the pair: half 0 keeps x_j + x_{j+16},
  // half 1 keeps (x_j - x_{j+16}) W_32^j
  static_for<0, 16>([&](auto J) {
    constexpr int j = decltype(J)::value;
    const float2 o = shfl16(v[j]);
    if (h == 0) {
      v[j] = make_float2(v[j].x + o.x, v[j].y + o.y);
    } else {
      v[j] = ff::tw32<j, INV>(make_float2(o.x - v[j].x, o.y - v[j].y));
    }
  });
  dft<16, INV>(v);
}

struct CWArgs {
  const ChunkInfo* chunks;
  uint32_t first;
  const void* grad;
  QuantParams q;
  uint8_t* message;
  uint32_t* flags;
  const float2* thi;
  const float2* tlo;
  const float2* t1024;
  float2* fb_spec;
  float2* dbg_spec;
  uint32_t count;
  uint32_t ahead;
  PieceCounter pc;
  uint32_t dbg;                      // instrumentation knobs (128: phase stamps into ts)
  unsigned long long* ts;
};

__device__ __forceinline__ unsigned long long globaltimer_w() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define FGC_TS(k)                                                                     \
  do {                                                                                \
    if ((a.dbg & 128u) && threadIdx.x == 0 && blockIdx.x < 2048)                       \
      a.ts[blockIdx.x * 16 + (k)] = globaltimer_w();                                   \
  } while (0)

struct __align__(16) ShW {
  float2 buf[kPadded + 64];          // FFT transposes / 4 sub-histograms / bin-ordered code half + staging
  float2 thi[256], tlo[kTloPadded];
  float2 t1024[kT1024Padded];
  uint32_t hbm[1024 + 4];            // bitmap of this CTA's half (natural slot order), set during emit
  uint32_t hist[2048];
  uint32_t hist2[2048];
  uint32_t scan[40];
  unsigned long long ckey[kCand];    // CTA 0: undecided bins (exact key, bin), pushed by both CTAs
  uint32_t cidx[kCand];
  unsigned long long lkey[kCand];    // each CTA's own copy of CTA 0's list, sorted locally
  uint32_t lidx[kCand];
  uint32_t ccount, below, anynz, rcount[2], fbin, fbelow;
};
static_assert(sizeof(sel::SelectSharedT<kTW>) <= sizeof(ShW::buf), "fallback select scratch fits in buf");

enum : int { kModeKeepAll = 0, kModeDropAll = 1, kModeList = 2, kModeFallback = 3 };

__device__ void merged_bucket_w(ShW& sh, const uint32_t* own, const uint32_t* peer, uint32_t r, uint32_t& bucket,
                                uint32_t& below) {
  const uint32_t t = threadIdx.x;
  const uint2 a = reinterpret_cast<const uint2*>(own)[t];
  const uint2 b = peer ? reinterpret_cast<const uint2*>(peer)[t] : make_uint2(0, 0);
  const uint32_t h0 = a.x + b.x, h1 = a.y + b.y;
  const uint32_t local = h0 + h1;
  uint32_t total;
  const uint32_t before = block_exclusive_scan<kTW>(local, sh.scan, total);
  if (r >= before && r < before + local) {
    if (r < before + h0) { sh.fbin = 2 * t; sh.fbelow = before; }
    else { sh.fbin = 2 * t + 1; sh.fbelow = before + h0; }
  }
  __syncthreads();
  bucket = sh.fbin;
  below = sh.fbelow;
}

__device__ __noinline__ bool inband_dropped_w(const ShW* sh, uint32_t mcount, uint32_t bin) {
  uint32_t lo = 0, hi = mcount;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((sh->lidx[mid] & 0x7FFFFFFFu) < bin) lo = mid + 1; else hi = mid;
  }
  return lo < mcount && (sh->lidx[lo] & 0x7FFFFFFFu) == bin && (sh->lidx[lo] & 0x80000000u);
}

__device__ __noinline__ void push_candidate_w(ShW* sh0, uint32_t bin, float re, float im) {
  const uint32_t s = atomicAdd(&sh0->ccount, 1u);
  FGC_CHECK(bin <= kN);
  if (s < (uint32_t)kCand) {
    sh0->cidx[s] = bin;
    sh0->ckey[s] = (unsigned long long)__double_as_longlong(cabs_key((double)re, (double)im));
  }
}

__device__ __noinline__ void resolve_w(ShW& sh, uint32_t m, uint32_t need) {
  const uint32_t tid = threadIdx.x;
  uint32_t M2 = 1;
  while (M2 < m) M2 <<= 1;
  for (uint32_t s = m + tid; s < M2; s += kTW) {
    sh.lkey[s] = ~0ull;
    sh.lidx[s] = 0x7FFFFFFFu;
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    for (uint32_t k = 2; k <= M2; k <<= 1) {
      for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
        for (uint32_t t = tid; t < M2; t += kTW) {
          const uint32_t u = t ^ jj;
          if (u > t) {
            const bool asc = (t & k) == 0;
            bool gt;
            if (pass == 0) {
              gt = sh.lkey[t] > sh.lkey[u] ||
                   (sh.lkey[t] == sh.lkey[u] && (sh.lidx[t] & 0x7FFFFFFFu) > (sh.lidx[u] & 0x7FFFFFFFu));
            } else {
              gt = (sh.lidx[t] & 0x7FFFFFFFu) > (sh.lidx[u] & 0x7FFFFFFFu);
            }
            if (gt == asc) {
              const unsigned long long tk = sh.lkey[t]; sh.lkey[t] = sh.lkey[u]; sh.lkey[u] = tk;
              const uint32_t ti = sh.lidx[t]; sh.lidx[t] = sh.lidx[u]; sh.lidx[u] = ti;
            }
          }
        }
        __syncthreads();
      }
    }
    if (pass == 0) {
      for (uint32_t s = tid; s < need && s < m; s += kTW) sh.lidx[s] |= 0x80000000u;
      __syncthreads();
    }
  }
}

template <class T, bool DEBUG, bool HALF>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTW, 1) k_fused_compress_w(CWArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ShW& sh = *reinterpret_cast<ShW*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t r = cluster.block_rank();
  const uint32_t tid = threadIdx.x;
  const uint32_t h = (tid >> 4) & 1u;                  // half of the lane pair
  const uint32_t i = (tid >> 5) * 16u + (tid & 15u);   // pair index (a 512-thread kernel's thread)
  const uint32_t chunk = a.first + blockIdx.x / 2;
  const ChunkInfo ci = a.chunks[chunk];
  ShW& sh0 = *cluster.map_shared_rank(&sh, 0);
  ShW& shp = *cluster.map_shared_rank(&sh, r ^ 1);
  const QuantParams q = a.q;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const T* g = static_cast<const T*>(a.grad) + ci.in_off;

  if (tid == 0) {
    const uint32_t half_bytes = (uint32_t)(kL / 2 * sizeof(T));
    const char* base = reinterpret_cast<const char*>(g) + (uint64_t)r * half_bytes;
    for (uint32_t off = 0; off < half_bytes; off += 32768u)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(32768u) : "memory");
  }
  if (tid < 256) {
    sh.thi[tid] = a.thi[tid];
    sh.tlo[tpad(tid)] = a.tlo[tid];
  }
  sh.t1024[tpad(tid)] = a.t1024[tid];
  reinterpret_cast<uint2*>(sh.hist2)[tid] = make_uint2(0, 0);
  sh.hbm[tid] = 0u;
  if (tid < 4) sh.hbm[1024 + tid] = 0u;
  if (tid == 0) { sh.ccount = 0; sh.below = 0; sh.anynz = 0; sh.rcount[0] = 0; sh.rcount[1] = 0; }
  uint32_t* codes_g = DEBUG ? nullptr : reinterpret_cast<uint32_t*>(a.message + ci.seg_off + ci.code_off);
  __syncthreads();

  FGC_TS(0);
  // ---- 1. load + decimation-in-frequency split: v[jj] = x-index i + 512 (16 h + jj)
  float2 v[16];
  {
    uint32_t bad = 0;
    const float2 wi = tw(sh.thi, sh.tlo, 2u * i);          // W_N^i
    static_for<0, 16>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      const uint32_t n = i + 512u * (16u * h + jj);
      const float2 z0 = InW<T>::template get<HALF>(g, 2ull * n, bad);
      const float2 z1 = InW<T>::template get<HALF>(g, 2ull * (n + kM), bad);
      if (r == 0) {
        v[jj] = make_float2(z0.x + z1.x, z0.y + z1.y);
      } else {                                              // (z0 - z1) W_N^(i + 512 j), j = 16 h + jj
        const float2 d = cmul(make_float2(z0.x - z1.x, z0.y - z1.y), wi);
        if constexpr (jj == 0) {
          v[jj] = h ? make_float2(d.y, -d.x) : d;           // w64mul<0> / w64mul<16>
        } else {                                            // w64mul<16 h + jj>, same arithmetic
          const float c = h ? ff::kC64[16 + jj] : ff::kC64[jj];
          const float s = h ? -ff::kS64[16 + jj] : -ff::kS64[jj];
          v[jj] = make_float2(__fmaf_rn(d.x, c, -d.y * s), __fmaf_rn(d.x, s, d.y * c));
        }
      }
    });
    if (bad && r == 0) atomicOr(a.flags, bad);
  }
  if (tid == 0 && blockIdx.x / 2 + a.ahead < a.count) {
    const ChunkInfo cn = a.chunks[chunk + a.ahead];
    const uint32_t half_bytes = (uint32_t)(kL / 2 * sizeof(T));
    const char* base = reinterpret_cast<const char*>(static_cast<const T*>(a.grad) + cn.in_off) + (uint64_t)r * half_bytes;
    for (uint32_t off = 0; off < half_bytes; off += 32768u)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(32768u) : "memory");
  }

  FGC_TS(1);
  // ---- 2. 16384-point FFT (32 x 32 x 16, as fused_fft.cuh) over lane pairs
  {
    // pass 1: the pair's 32-point DFT; X[m] to buf[33 i + m]
    pair_dft32<false>(v, h);
    float2* w1 = sh.buf + 33u * i;
#pragma unroll
    for (int k = 0; k < 16; ++k) w1[2 * k + h] = v[bitrev(k, 4)];
    __syncthreads();
    // pass 2: column i reads x[i + 512 j] at pad(i + 512 j) = i + i/32 + 528 j
    const float2* r2 = sh.buf + i + (i >> 5);
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) v[jj] = r2[528u * (16u * h + jj)];
    const uint32_t k = i & 31u;
    // W_1024^{jk}, j = 16 h + jj: odd j from the table, even j as W^{(j-1)k} W^k
    // (the products fft_pass12 forms, so the values are bit-identical)
    const float2 wk = sh.t1024[tpad(k)];
    float2 wprev = wk;
    static_for<0, 16>([&](auto J) {
      constexpr int jj = decltype(J)::value;
      if constexpr (jj == 0) {
        if (h) v[0] = cmul(v[0], cmul(sh.t1024[tpad(15u * k)], wk));   // j = 16; j = 0 has no twiddle
      } else if constexpr (jj & 1) {
        wprev = sh.t1024[tpad((16u * h + jj) * k)];
        v[jj] = cmul(v[jj], wprev);
      } else {
        v[jj] = cmul(v[jj], cmul(wprev, wk));
      }
    });
    pair_dft32<false>(v, h);
    float2* w2 = sh.buf + (i >> 5) * 1056u + k;
    __syncthreads();                                        // every pass-2 read is done before the writes
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) w2[33u * (2 * kk + h)] = v[bitrev(kk, 4)];
    __syncthreads();
  }
  FGC_TS(2);
  // pass 3: the pair's columns (ka, kb); half h takes one
  const bool special = (r == 0 && i == 0);
  const uint32_t ka = i;
  const uint32_t kb = (r == 0) ? (i == 0 ? 512u : 1024u - i) : 1023u - i;
  const uint32_t col = h ? kb : ka;
  ff::fft_pass3<false>(col, sh.buf, v, sh.thi, sh.tlo);    // v[m] = Z-half[col + 1024 m]

  // ---- 3. real-FFT post-processing: X_own[j] = r2c(own[j], other[15 - j], W_L^{bin})
  auto r2c = [](float2 P, float2 Q, float2 w) -> float2 {
    const float2 A = make_float2(P.x + Q.x, P.y - Q.y);
    const float2 B = make_float2(P.x - Q.x, P.y + Q.y);
    const float2 t = cmul(w, make_float2(B.y, -B.x));
    return make_float2(0.5f * (A.x + t.x), 0.5f * (A.y + t.y));
  };
  float2 xn = make_float2(0.f, 0.f);                       // X[N] (CTA 0, pair 0, half 0)
  {
    // the partner's column, two values at a time (j and 15 - j are consumed
    // together, so no more than four extra floats are live)
    const float2 wc = tw(sh.thi, sh.tlo, 2u * col + r);
    static_for<0, 8>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 pj = shfl16(v[j]), pk = shfl16(v[15 - j]);
      if (!special) {
        v[j] = r2c(v[j], pk, w32mul<j>(wc));
        v[15 - j] = r2c(v[15 - j], pj, w32mul<15 - j>(wc));
      }
    });
    if (special && h == 0) {
      // column 0: pairs j <-> 16-j; self pairs j = 0 (X[0], X[N]) and j = 8 (X[M])
      const float2 a0 = v[0];
      static_for<1, 8>([&](auto J) {
        constexpr int j = decltype(J)::value;
        const float2 P = v[j], Q = v[16 - j];
        v[j] = r2c(P, Q, w32mul<j>(make_float2(1.f, 0.f)));
        v[16 - j] = r2c(Q, P, w32mul<16 - j>(make_float2(1.f, 0.f)));
      });
      v[8] = r2c(v[8], v[8], w32mul<8>(make_float2(1.f, 0.f)));
      v[0] = make_float2(a0.x + a0.y, 0.f);
      xn = make_float2(a0.x - a0.y, 0.f);
    } else if (special) {
      // column 512: bins 1024 + 2048 j, pairs j <-> 15-j; W_L^1024 = W_64^1
      const float2 w1 = w64mul<1>(make_float2(1.f, 0.f));
      static_for<0, 8>([&](auto J) {
        constexpr int j = decltype(J)::value;
        const float2 P = v[j], Q = v[15 - j];
        v[j] = r2c(P, Q, w32mul<j>(w1));
        v[15 - j] = r2c(Q, P, w32mul<15 - j>(w1));
      });
    }
  }
  const bool hasN = special && h == 0;
#define BIN(j) (2u * (col + 1024u * (j)) + r)

  if (DEBUG) {
    float2* out = a.dbg_spec + ci.bin_off;
#pragma unroll
    for (int j = 0; j < 16; ++j) out[BIN(j)] = v[j];
    if (hasN) out[kN] = xn;
    return;
  }

  FGC_TS(3);
  // ---- 4. count-mode selection, cluster-wide (cluster barriers A-C)
  const uint32_t kdrop = ci.drop;
  int mode = kModeList;
  if (kdrop == 0) mode = kModeKeepAll;
  else if (kdrop >= kBins) mode = kModeDropAll;
  float band_lo = 0.f, band_hi = INFINITY;
  uint32_t mcount = 0;
  __syncthreads();                                          // pass-3 reads of buf are done
  if (mode == kModeList) {
    uint32_t* sub = reinterpret_cast<uint32_t*>(sh.buf) + 2048u * ((tid >> 5) & 3u);
    {
      uint4* z = reinterpret_cast<uint4*>(sh.buf);
      for (uint32_t e = tid; e < 2048; e += kTW) z[e] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    uint32_t nz = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t p = __float_as_uint(proxy_key(v[j].x, v[j].y));
      nz |= __float_as_uint(v[j].x) | __float_as_uint(v[j].y);
      atomicAdd(&sub[p >> 20], 1u);
    }
    if (hasN) {
      nz |= __float_as_uint(xn.x) | __float_as_uint(xn.y);
      atomicAdd(&sub[__float_as_uint(proxy_key(xn.x, xn.y)) >> 20], 1u);
    }
    nz &= 0x7FFFFFFFu;
    if (__any_sync(0xffffffffu, nz != 0) && (tid & 31) == 0) atomicOr(&sh.anynz, 1u);
    __syncthreads();
    {
      const uint2* s2 = reinterpret_cast<const uint2*>(sh.buf);
      const uint2 x0 = s2[tid], x1 = s2[1024 + tid], x2 = s2[2048 + tid], x3 = s2[3072 + tid];
      reinterpret_cast<uint2*>(sh.hist)[tid] = make_uint2(x0.x + x1.x + x2.x + x3.x, x0.y + x1.y + x2.y + x3.y);
    }
    FGC_TS(7);
    cluster.sync();                                         // A: pass-1 histograms visible
    const bool anynz = (sh.anynz | shp.anynz) != 0;
    uint32_t b1, below1;
    merged_bucket_w(sh, sh.hist, shp.hist, kdrop - 1, b1, below1);
    if (!anynz) {
      mode = kModeDropAll;
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t p = __float_as_uint(proxy_key(v[j].x, v[j].y));
        if ((p >> 20) == b1) atomicAdd(&sh.hist2[(p >> 9) & 0x7FFu], 1u);
      }
      if (hasN) {
        const uint32_t pn = __float_as_uint(proxy_key(xn.x, xn.y));
        if ((pn >> 20) == b1) atomicAdd(&sh.hist2[(pn >> 9) & 0x7FFu], 1u);
      }
      __syncthreads();
    }
    FGC_TS(8);
    cluster.sync();                                         // B: pass-2 histograms visible
    if (mode == kModeList) {
      uint32_t b2, below2;
      merged_bucket_w(sh, sh.hist2, shp.hist2, kdrop - 1 - below1, b2, below2);
      const uint32_t lo_pat = (b1 << 20) | (b2 << 9);
      const float lo_f = __uint_as_float(lo_pat);
      const float hi_f = __uint_as_float(lo_pat + 512u);
      if (lo_f < 0x1p-100f || hi_f > 0x1p100f) {
        mode = kModeFallback;
      } else {
        band_lo = lo_f * (1.0f - 0x1p-16f);
        band_hi = hi_f * (1.0f + 0x1p-16f);
        uint32_t below_l = 0;
        auto collect = [&](float2 x, uint32_t bin) {
          const float p = proxy_key(x.x, x.y);
          below_l += (p < band_lo) ? 1u : 0u;
          if (p >= band_lo && p < band_hi) push_candidate_w(&sh0, bin, x.x, x.y);
        };
#pragma unroll
        for (int j = 0; j < 16; ++j) collect(v[j], BIN(j));
        if (hasN) collect(xn, kN);
        const uint32_t bl = block_sum<kTW>(below_l, sh.scan);
        if (tid == 0) sh.below = bl;
      }
    }
    FGC_TS(9);
    cluster.sync();                                         // C: candidates and counts visible
    {
      const uint32_t m = sh0.ccount;
      const uint32_t below = sh.below + shp.below;
      if (mode == kModeList && (m > (uint32_t)kCand || below > kdrop || below + m < kdrop)) mode = kModeFallback;
      if (mode == kModeList) {
        for (uint32_t s = tid; s < m; s += kTW) {
          sh.lkey[s] = sh0.ckey[s];
          sh.lidx[s] = sh0.cidx[s];
        }
        __syncthreads();
        resolve_w(sh, m, kdrop - below);
        mcount = m;
      }
    }
    FGC_TS(10);
  } else {
    cluster.sync();                                         // D': both bitmaps zeroed (peer atomics follow)
  }

  FGC_TS(4);
  if (mode == kModeFallback) {
    float2* out = a.fb_spec + ci.bin_off;
#pragma unroll
    for (int j = 0; j < 16; ++j) out[BIN(j)] = v[j];
    if (hasN) out[kN] = xn;
    __threadfence();
    cluster.sync();                                         // both halves written; CTA 0's list read
    if (r == 1) return;
    sel::select_pack_chunk<float2, kTW>(*reinterpret_cast<sel::SelectSharedT<kTW>*>(sh.buf), ci,
                                        sel::Coeffs<float2>{a.fb_spec + ci.bin_off}, 0, q, a.message, nullptr,
                                        a.flags, nullptr);
    if (a.pc.cnt || a.pc.done) {
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        if (a.pc.cnt) atomicAdd(&a.pc.cnt[(chunk - a.pc.first) / a.pc.per], 1u);
        if (a.pc.done) release_tag(a.pc.done + chunk, a.pc.tag, a.pc.sys);
      }
    }
    return;
  }

  // ---- 5. codes -> two bin-ordered halves (CTA 0: bins [0, 16384), CTA 1:
  //         [16384, 32768]); bin (2 col + r) + 2048 j lands in half j >= 8
  float lo_b = band_lo, hi_b = band_hi;
  if (mode == kModeKeepAll) { lo_b = -1.0f; hi_b = -1.0f; }
  if (mode == kModeDropAll) { lo_b = INFINITY; hi_b = INFINITY; }
  uint32_t* arr_own = reinterpret_cast<uint32_t*>(sh.buf);
  uint32_t* arr_peer = reinterpret_cast<uint32_t*>(shp.buf);
  uint32_t rc0 = 0, rc1 = 0;
  uint32_t keep = 0, band = 0;                              // bit j: v[j]
  static_for<0, 16>([&](auto J) {
    constexpr int j = decltype(J)::value;
    const float p = proxy_key(v[j].x, v[j].y);
    keep |= (p >= hi_b ? 1u : 0u) << j;
    band |= (p >= lo_b && p < hi_b ? 1u : 0u) << j;
  });
  while (band) {
    const uint32_t b = __ffs(band) - 1u;
    band &= band - 1u;
    if (!inband_dropped_w(&sh, mcount, BIN(b))) keep |= 1u << b;
  }
  {
    const uint32_t lane = tid & 31u;
    uint32_t* wmeta = arr_own + kEmitStageOff + (tid >> 5) * kEmitStageWords;
    float2* wval = reinterpret_cast<float2*>(wmeta + 128);
    static_for<0, 4>([&](auto R) {
      constexpr int j0 = 4 * decltype(R)::value;
      constexpr uint32_t d = j0 >= 8 ? 1u : 0u;
      const uint32_t m4 = (keep >> j0) & 0xFu;
      const uint32_t cnt = __popc(m4);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += t;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      uint32_t pos = incl - cnt;
      static_for<0, 4>([&](auto K) {
        constexpr int k = decltype(K)::value;
        constexpr int j = j0 + k;
        if ((m4 >> k) & 1u) {
          FGC_CHECK(pos < 128u);
          wmeta[pos] = BIN(j);
          wval[pos] = v[j];
          ++pos;
        }
      });
      __syncwarp();
      for (uint32_t e = lane; e < total; e += 32) {
        const uint32_t bin = wmeta[e];
        const float2 x = wval[e];
        const uint32_t cre = enc16(q, x.x), cim = enc16(q, x.y);
        const uint32_t pc = cre | (cim << 16);
        if (pc) {
          const uint32_t c = (cre ? 1u : 0u) + (cim ? 1u : 0u);
          if (d) rc1 += c; else rc0 += c;
          const uint32_t lb = bin - d * kHalfBins;
          FGC_CHECK(lb <= kHalfBins && pad(lb) < kStageOff);
          const uint32_t bits = ((cre ? 1u : 0u) | (cim ? 2u : 0u)) << (2u * (lb & 15u));
          if (d == r) {
            arr_own[pad(lb)] = pc;
            atomicOr(&sh.hbm[lb >> 4], bits);
          } else {
            arr_peer[pad(lb)] = pc;
            atomicOr(&shp.hbm[lb >> 4], bits);
          }
        }
      }
      __syncwarp();
    });
  }
  if (hasN) {                                               // bin N: half 1 (CTA 1), local bin 16384
    const float p = proxy_key(xn.x, xn.y);
    bool kp = p >= lo_b;
    if (kp && p < hi_b) kp = !inband_dropped_w(&sh, mcount, kN);
    if (kp) {
      const uint32_t cre = enc16(q, xn.x), cim = enc16(q, xn.y);
      const uint32_t pc = cre | (cim << 16);
      if (pc) {
        rc1 += (cre ? 1u : 0u) + (cim ? 1u : 0u);
        uint32_t* dst = (r == 1) ? arr_own : arr_peer;
        uint32_t* hb = (r == 1) ? sh.hbm : shp.hbm;
        dst[pad(kHalfBins)] = pc;
        atomicOr(&hb[kHalfBins >> 4], (cre ? 1u : 0u) | (cim ? 2u : 0u));
      }
    }
  }
#undef BIN
  {
    const uint32_t s0 = __reduce_add_sync(0xffffffffu, rc0), s1 = __reduce_add_sync(0xffffffffu, rc1);
    if ((tid & 31) == 0) {
      if (s0) atomicAdd(&sh.rcount[0], s0);
      if (s1) atomicAdd(&sh.rcount[1], s1);
    }
  }
  FGC_TS(11);
  cluster.sync();                                           // E: both halves complete, per-half counts visible
  FGC_TS(5);
  const uint32_t t0 = sh.rcount[0] + shp.rcount[0];
  const uint32_t all = t0 + sh.rcount[1] + shp.rcount[1];
  const int N = q.n_bits;
  const uint64_t s1bits = (uint64_t)t0 * N;
  const bool fold = (s1bits & 7u) != 0;
  if (!fold) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");

  // ---- 6. pack: thread t of CTA d owns bins d*16384 + [16t, 16t+16) (+ bin N)
  const bool nb33 = (r == 1 && tid == kTW - 1);
  const uint32_t w0 = sh.hbm[tid], w2 = nb33 ? sh.hbm[1024] : 0u;
  const uint32_t cnt = __popc(w0) + __popc(w2);
  uint32_t* seg = reinterpret_cast<uint32_t*>(a.message + ci.seg_off);
  uint32_t* bm = seg + kSegHeader / 4;
  {
    const uint32_t wb = r * (kHalfBins / 16) + tid;
    bm[wb] = ballot_to_wire(w0);
    if (nb33) {
      bm[wb + 1] = ballot_to_wire(w2);
      const uint32_t pad_words = (ci.code_off - kSegHeader) / 4;
      for (uint32_t w = kBmWords; w < pad_words; ++w) bm[w] = 0u;
    }
  }
  uint32_t total;
  const uint32_t base = block_exclusive_scan<kTW>(cnt, sh.scan, total);
  const uint64_t S = r ? s1bits : 0ull;
  const uint32_t wstart = (uint32_t)(S >> 5), o = (uint32_t)(S & 31u);
  const uint32_t nwords = (uint32_t)((o + (uint64_t)total * N + 31) / 32);
  uint32_t* stg = arr_own + kStageOff;
  FGC_CHECK(kStageOff + nwords + 1 <= 2 * (kPadded + 64));
  for (uint32_t k = tid; k < nwords; k += kTW) stg[k] = 0u;
  __syncthreads();
  {
    uint32_t lbit = o + base * (uint32_t)N;
    const uint32_t* row = arr_own + pad(16u * tid);         // my 16 bins (pad(16t + j) = pad(16t) + j)
    uint8_t* stg8 = reinterpret_cast<uint8_t*>(stg);
    auto emit_slots = [&](uint32_t m, const uint32_t* src) {
      while (m) {
        const uint32_t pos = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t pc = src[pos >> 1];
        const uint32_t code = (pos & 1) ? (pc >> 16) : (pc & 0xFFFFu);
        FGC_CHECK((lbit >> 5) < nwords);
        if (N == 8) {
          stg8[lbit >> 3] = (uint8_t)code;
        } else {
          const uint32_t wi = lbit >> 5, sb = lbit & 31u;
          atomicOr(&stg[wi], code << sb);
          if (sb + N > 32u) atomicOr(&stg[wi + 1], code >> (32u - sb));
        }
        lbit += N;
      }
    };
    emit_slots(w0, row);
    if (w2) emit_slots(w2, arr_own + pad(16u * tid + 16u));
  }
  __syncthreads();
  if (fold) {
    cluster.sync();                                         // F: CTA 1's staging complete
    if (r == 0 && tid == 0) stg[s1bits >> 5] |= (reinterpret_cast<const uint32_t*>(shp.buf) + kStageOff)[0];
    __syncthreads();
  }
  const uint32_t shared_w = (uint32_t)(s1bits >> 5);
  const bool split = (s1bits & 31u) != 0 && !fold;
  for (uint32_t k = tid; k < nwords; k += kTW) {
    const uint32_t w = wstart + k;
    if (w >= ci.code_cap) continue;
    if (r == 1 && fold && k == 0) continue;
    if (split && w == shared_w) {
      uint8_t* p = reinterpret_cast<uint8_t*>(codes_g + w);
      const uint32_t bb = (uint32_t)(s1bits & 31u) >> 3;
      const uint32_t val = stg[k];
      for (uint32_t b = (r ? bb : 0u); b < (r ? 4u : bb); ++b) p[b] = (uint8_t)(val >> (8 * b));
      continue;
    }
    codes_g[w] = stg[k];
  }
  const uint32_t used = (uint32_t)(((uint64_t)all * N + 31) / 32);
  const uint32_t cap_padded = (ci.code_cap + 3u) & ~3u;
  if (r == 1)
    for (uint32_t w = used + tid; w < cap_padded; w += kTW) codes_g[w] = 0u;
  if (r == 0 && tid == 0) {
    seg[0] = all;
    seg[1] = 0; seg[2] = 0; seg[3] = 0;
    if (used > ci.code_cap) atomicOr(a.flags, FGC_FLAG_CAPACITY);
  }
  if (a.pc.cnt || a.pc.done) {
    __threadfence();
    if (!fold) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    cluster.sync();
    if (r == 0 && tid == 0) {
      if (a.pc.cnt) atomicAdd(&a.pc.cnt[(chunk - a.pc.first) / a.pc.per], 1u);
      if (a.pc.done) release_tag(a.pc.done + chunk, a.pc.tag, a.pc.sys);
    }
  } else if (fold) {
    cluster.sync();
  } else {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  FGC_TS(6);
}

template <class K>
fgc_status set_smem_w(K kernel, size_t bytes) {
  FGC_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return FGC_OK;
}

}  // namespace

fgc_status launch_compress_w(const float2* thi, const float2* tlo, const float2* t1024, uint32_t ahead,
                             const ChunkInfo* d_chunks, uint32_t first, uint32_t count, const void* grad, int dtype,
                             int half_pass, const QuantParams& q, uint8_t* message, uint32_t* flags, float2* fb_spec,
                             float2* dbg, cudaStream_t s, PieceCounter pc) {
  if (!count) return FGC_OK;
  static bool attrs = false;
  const size_t smem = sizeof(ShW);
  if (!attrs) {
    FGC_TRY(set_smem_w(k_fused_compress_w<float, false, false>, smem));
    FGC_TRY(set_smem_w(k_fused_compress_w<double, false, false>, smem));
    FGC_TRY(set_smem_w(k_fused_compress_w<float, true, false>, smem));
    FGC_TRY(set_smem_w(k_fused_compress_w<double, true, false>, smem));
    FGC_TRY(set_smem_w(k_fused_compress_w<float, false, true>, smem));
    FGC_TRY(set_smem_w(k_fused_compress_w<double, false, true>, smem));
    FGC_TRY(set_smem_w(k_fused_compress_w<float, true, true>, smem));
    FGC_TRY(set_smem_w(k_fused_compress_w<double, true, true>, smem));
    attrs = true;
  }
  CWArgs a{d_chunks, first, grad, q, message, flags, thi, tlo, t1024, fb_spec, dbg, count, ahead, pc, 0, nullptr};
  fused_debug_state(a.dbg, a.ts);
  const dim3 grid(2 * count), block(kTW);
  const bool f64 = dtype == FGC_DTYPE_F64, hp = half_pass != 0;
#define FGC_LAUNCH_CW(T, D, H) k_fused_compress_w<T, D, H><<<grid, block, smem, s>>>(a)
  if (dbg) {
    if (f64) { if (hp) FGC_LAUNCH_CW(double, true, true); else FGC_LAUNCH_CW(double, true, false); }
    else { if (hp) FGC_LAUNCH_CW(float, true, true); else FGC_LAUNCH_CW(float, true, false); }
  } else {
    if (f64) { if (hp) FGC_LAUNCH_CW(double, false, true); else FGC_LAUNCH_CW(double, false, false); }
    else { if (hp) FGC_LAUNCH_CW(float, false, true); else FGC_LAUNCH_CW(float, false, false); }
  }
#undef FGC_LAUNCH_CW
  FGC_LAUNCHED(1);
  return FGC_OK;
}

}  // namespace fgc
