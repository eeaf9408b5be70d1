// Compress of 65536-sample chunks by 4-CTA clusters, two CTAs per SM.
//
// Same message as k_fused_compress (fused.cu) -- count-mode truncate
// (spectral.py:124-156), quantize (quantizer.py:217-236), pack
// (packer.py:41-58) of the chunk's real FFT (spectral.py:88-95) -- laid out
// so that two chunks' CTAs share every SM: 256 threads x 128 registers and
// ~99 KB of shared memory per CTA.  While one CTA waits at a barrier (the
// selection and pack phases are barrier- and latency-bound), the other
// computes; the 2-CTA kernel of fused.cu holds a whole SM per CTA.
//
// Transform: z[n] = x[2n] + i x[2n+1], N = 32768.  A radix-8 decimation in
// frequency splits Z into 8 residue classes Z[8m + q] = FFT_4096(a_q)[m],
//   a_q[n] = W_N^{nq} sum_p z[n + 4096 p] W_8^{pq},   n < 4096.
// CTA r takes the classes (q, 8 - q): (0, 4), (1, 7), (2, 6), (3, 5), so the
// real-FFT post-processing pair Z[k], Z[N - k] (k = 8m + q -> N - k =
// 8(4095 - m) + 8 - q) never leaves the CTA: with each 4096-point FFT done as
// 16 x 16 x 16 (two padded shared-memory transposes), pass 3 leaves column c
// of a class in one thread (X[c + 256 j], j < 16) and the thread that owns
// column c of class q also owns column 255 - c of class 8 - q.
// Every CTA reads the whole chunk (one HBM read, three L2 hits); the two
// class outputs of one radix-8 row share their sums (b_q = P + T,
// b_{8-q} = P - T).
//
// Selection is a cluster-wide radix select on the fp32 proxy |X|^2
// (histograms merged over DSMEM, exact numpy cabs keys for the undecided
// band, collected in CTA 0), as in fused.cu.  Bin b is packed by CTA b / 8192:
// the owner of bin 8(c + 256 j) + q is CTA j / 4 for every thread, so each
// emit round stores to one owner; each owner writes its quarter of the
// bitmap and its run of the LSB-first code stream.
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
using ff::kTloPadded;
using ff::pad;
using ff::tpad;
using ff::tw;
using ff::w32mul;
using ff::w64mul;

constexpr int kT = 256;                              // threads per CTA
constexpr uint32_t kN = 32768;                       // complex points per chunk
constexpr uint32_t kL = 65536;                       // chunk length
constexpr uint32_t kRow = 17;                        // padded 16-value row
constexpr uint32_t kFft = 256 * kRow;                // float2 per class buffer
constexpr uint32_t kOwn = 8192;                      // bins packed per CTA (CTA 3: + bin N)
constexpr uint32_t kBins = kN + 1;
constexpr uint32_t kBmWords = (2 * kBins + 31) / 32; // 2049
constexpr int kCand = 512;
constexpr uint32_t kBufWords = 4 * kFft;             // buf as u32 words (17408)
constexpr uint32_t kUpper = 8456;                    // u32 offset of the emit strips / pack staging
constexpr uint32_t kStripWords = 768;                // per warp: 256 bins + 256 float2
static_assert(kUpper >= kOwn + kOwn / 32 + 1 && kUpper % 4 == 0, "code array below the strips");
static_assert(kUpper + (kT / 32) * kStripWords <= kBufWords, "emit strips fit");
static_assert(kUpper + (2 * (kOwn + 1) * 16 + 31) / 32 + 2 <= kBufWords, "pack staging fits (N <= 16)");
static_assert(4 * 2048 <= kBufWords, "pass-1 sub-histograms fit");

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

struct C4Args {
  const ChunkInfo* chunks;
  uint32_t first;
  const void* grad;
  QuantParams q;
  uint8_t* message;
  uint32_t* flags;
  const float2* thi;
  const float2* tlo;
  float2* fb_spec;       // chunk-major spectrum scratch for degenerate chunks
  float2* dbg_spec;      // debug hook: write the spectrum and stop
  uint32_t count;        // chunks in this launch
  uint32_t ahead;        // L2 prefetch distance in chunks (one wave)
  PieceCounter pc;
};

struct __align__(16) Sh4 {
  float2 buf[2 * kFft];               // 2 class buffers; later histograms / code array / strips / staging
  float2 thi[256];
  float2 tlo[kTloPadded];
  uint32_t hist[2048];               // pass-1 histogram (read by the peers)
  uint32_t hist2[2048];              // pass-2 histogram (read by the peers)
  uint32_t hbm[kOwn / 16 + 4];       // bitmap of the owned bins, natural slot order (peers OR into it)
  unsigned long long ckey[kCand];    // CTA 0: undecided bins (exact key, bin)
  uint32_t cidx[kCand];
  uint32_t scan[40];
  uint32_t rcount[4];                // my non-zero codes per owner
  uint32_t S[5];                     // bit offset of each owner's codes; S[4] = total bits
  uint32_t ccount, below, anynz, fbin, fbelow, need;
  int mode;
};
static_assert(sizeof(Sh4::buf) == 4 * kFft * 4, "buf size");
static_assert(sizeof(sel::SelectSharedT<kT>) <= sizeof(Sh4::buf), "fallback select scratch fits in buf");

enum : int { kModeKeepAll = 0, kModeDropAll = 1, kModeList = 2, kModeFallback = 3 };

template <class T> struct In4;
template <> struct In4<float> {
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
template <> struct In4<double> {
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

// Bucket holding rank `rk` in the cluster-merged histogram h[0..3].
__device__ void merged_bucket4(Sh4& sh, uint32_t* const (&h)[4], uint32_t rk, uint32_t& bucket, uint32_t& below) {
  const uint32_t t = threadIdx.x;
  uint32_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 x = reinterpret_cast<const uint4*>(h[c])[2 * t];
    const uint4 y = reinterpret_cast<const uint4*>(h[c])[2 * t + 1];
    v[0] += x.x; v[1] += x.y; v[2] += x.z; v[3] += x.w;
    v[4] += y.x; v[5] += y.y; v[6] += y.z; v[7] += y.w;
  }
  uint32_t local = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) local += v[k];
  uint32_t total;
  const uint32_t before = block_exclusive_scan<kT>(local, sh.scan, total);
  if (rk >= before && rk < before + local) {
    uint32_t acc = before;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (rk >= acc && rk < acc + v[k]) {
        sh.fbin = 8 * t + k;
        sh.fbelow = acc;
      }
      acc += v[k];
    }
  }
  __syncthreads();
  bucket = sh.fbin;
  below = sh.fbelow;
}

__device__ __noinline__ bool inband_dropped4(const Sh4* sh0, uint32_t mcount, uint32_t bin) {
  uint32_t lo = 0, hi = mcount;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((sh0->cidx[mid] & 0x7FFFFFFFu) < bin) lo = mid + 1; else hi = mid;
  }
  return lo < mcount && (sh0->cidx[lo] & 0x7FFFFFFFu) == bin && (sh0->cidx[lo] & 0x80000000u);
}

__device__ __noinline__ void push_candidate4(Sh4* sh0, uint32_t bin, float re, float im) {
  const uint32_t s = atomicAdd(&sh0->ccount, 1u);
  if (s < (uint32_t)kCand) {
    sh0->cidx[s] = bin;
    sh0->ckey[s] = (unsigned long long)__double_as_longlong(cabs_key((double)re, (double)im));
  }
}

// CTA 0: sort the undecided bins by (exact key, bin) -- stable argsort ties
// drop the lower index first -- mark the `need` smallest dropped, re-sort by bin.
__device__ __noinline__ void resolve4(Sh4& sh, uint32_t m, uint32_t need) {
  const uint32_t tid = threadIdx.x;
  uint32_t M2 = 1;
  while (M2 < m) M2 <<= 1;
  for (uint32_t s = m + tid; s < M2; s += kT) {
    sh.ckey[s] = ~0ull;
    sh.cidx[s] = 0x7FFFFFFFu;
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    for (uint32_t k = 2; k <= M2; k <<= 1) {
      for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
        for (uint32_t t = tid; t < M2; t += kT) {
          const uint32_t u = t ^ jj;
          if (u > t) {
            const bool asc = (t & k) == 0;
            bool gt;
            if (pass == 0) {
              gt = sh.ckey[t] > sh.ckey[u] ||
                   (sh.ckey[t] == sh.ckey[u] && (sh.cidx[t] & 0x7FFFFFFFu) > (sh.cidx[u] & 0x7FFFFFFFu));
            } else {
              gt = (sh.cidx[t] & 0x7FFFFFFFu) > (sh.cidx[u] & 0x7FFFFFFFu);
            }
            if (gt == asc) {
              const unsigned long long tk = sh.ckey[t]; sh.ckey[t] = sh.ckey[u]; sh.ckey[u] = tk;
              const uint32_t ti = sh.cidx[t]; sh.cidx[t] = sh.cidx[u]; sh.cidx[u] = ti;
            }
          }
        }
        __syncthreads();
      }
    }
    if (pass == 0) {
      for (uint32_t s = tid; s < need && s < m; s += kT) sh.cidx[s] |= 0x80000000u;
      __syncthreads();
    }
  }
}

template <class T, bool DEBUG, bool HALF>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(kT, 2) k_fused_compress4(C4Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Sh4& sh = *reinterpret_cast<Sh4*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t r = cluster.block_rank();
  const uint32_t tid = threadIdx.x;
  const uint32_t chunk = a.first + blockIdx.x / 4;
  const ChunkInfo ci = a.chunks[chunk];
  Sh4& sh0 = *cluster.map_shared_rank(&sh, 0);
  const QuantParams q = a.q;
  // every CTA of the grid is resident or done from here on: the dependent
  // decode grid may start filling SMs as they free up (it waits per chunk)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const T* g = static_cast<const T*>(a.grad) + ci.in_off;

  if (tid == 0) {
    // quarter r of the chunk into L2 while the tables load (every CTA reads all of it)
    const uint32_t qb = (uint32_t)(kL / 4 * sizeof(T));
    const char* base = reinterpret_cast<const char*>(g) + (uint64_t)r * qb;
    for (uint32_t off = 0; off < qb; off += 32768u)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(32768u) : "memory");
  }
  sh.thi[tid] = a.thi[tid];
  sh.tlo[tpad(tid)] = a.tlo[tid];
  reinterpret_cast<uint4*>(sh.hist2)[2 * tid] = make_uint4(0, 0, 0, 0);
  reinterpret_cast<uint4*>(sh.hist2)[2 * tid + 1] = make_uint4(0, 0, 0, 0);
  sh.hbm[tid] = 0u;
  sh.hbm[tid + 256] = 0u;
  if (tid < 4) { sh.hbm[512 + tid] = 0u; sh.rcount[tid] = 0u; }
  if (tid == 0) { sh.ccount = 0; sh.below = 0; sh.anynz = 0; }
  __syncthreads();

  // ---- 1. load + radix-8 DIF: classes c0 (FFT 0) and c1 (FFT 1) of rows n = tid + 256 j
  const uint32_t c0 = r == 0 ? 0u : r, c1 = r == 0 ? 4u : 8u - r;
  float2 v0[16], v1[16];
  {
    // b_c0 = P + T, b_c1 = P - T with e_p = z_p +- z_{p+4}:
    //   r = 0: P = e0 + e2,        T = e1 + e3
    //   r = 2: P = e0 - e2,        T = -i (e1 - e3)
    //   r = 1, 3 (s = +-1): P = e0 + s h (e1 - e3),  T = -i (s e2 + h (e1 + e3))
    const float h = 0.70710678118654752f;
    const float se = (r & 1) ? -1.0f : 1.0f;
    const float sg = (r == 3) ? -1.0f : 1.0f;
    const float kA = r == 0 ? 1.0f : (r == 2 ? -1.0f : 0.0f);     // P = e0 + kA e2 + kB (e1 - e3)
    const float kB = (r & 1) ? sg * h : 0.0f;
    const float kC = (r & 1) ? sg : 0.0f;                         // T' = kC e2 + kD e1 + kE e3
    const float kD = (r & 1) ? h : 1.0f;
    const float kE = (r & 1) ? h : (r == 2 ? -1.0f : 1.0f);
    const bool rot = r != 0;                                      // T = -i T'
    const float2 w0t = tw(sh.thi, sh.tlo, 2u * tid * c0);         // W_N^{t c0}
    const float2 w1t = tw(sh.thi, sh.tlo, 2u * tid * c1);         // W_N^{t c1}
    uint32_t bad = 0;
    static_for<0, 16>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const uint32_t n = tid + 256u * j;
      float2 z[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) z[p] = In4<T>::template get<HALF>(g, 2ull * (n + 4096u * p), bad);
      float2 e[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) e[p] = make_float2(__fmaf_rn(se, z[p + 4].x, z[p].x), __fmaf_rn(se, z[p + 4].y, z[p].y));
      const float2 d = make_float2(e[1].x - e[3].x, e[1].y - e[3].y);
      const float2 P = make_float2(__fmaf_rn(kB, d.x, __fmaf_rn(kA, e[2].x, e[0].x)),
                                   __fmaf_rn(kB, d.y, __fmaf_rn(kA, e[2].y, e[0].y)));
      const float2 Tp = make_float2(__fmaf_rn(kC, e[2].x, __fmaf_rn(kD, e[1].x, kE * e[3].x)),
                                    __fmaf_rn(kC, e[2].y, __fmaf_rn(kD, e[1].y, kE * e[3].y)));
      const float2 Tt = rot ? make_float2(Tp.y, -Tp.x) : Tp;
      const float2 b0 = make_float2(P.x + Tt.x, P.y + Tt.y);
      const float2 b1 = make_float2(P.x - Tt.x, P.y - Tt.y);
      // W_N^{n c} = W_N^{t c} W_128^{j c}, W_128^m = thi[2m mod 256] (a broadcast load)
      v0[j] = cmul(cmul(b0, sh.thi[(2u * j * c0) & 255u]), w0t);
      v1[j] = cmul(cmul(b1, sh.thi[(2u * j * c1) & 255u]), w1t);
    });
    if (bad && r == 0) atomicOr(a.flags, bad);
  }
  if (tid == 0 && blockIdx.x / 4 + a.ahead < a.count) {
    // the chunk the next wave runs here: its HBM read overlaps this wave's compute
    const ChunkInfo cn = a.chunks[chunk + a.ahead];
    const uint32_t qb = (uint32_t)(kL / 4 * sizeof(T));
    const char* base = reinterpret_cast<const char*>(static_cast<const T*>(a.grad) + cn.in_off) + (uint64_t)r * qb;
    for (uint32_t off = 0; off < qb; off += 32768u)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(32768u) : "memory");
  }

  // ---- 2. two 4096-point FFTs, 16 x 16 x 16
  {
    // pass 1: column t of each class, twiddle W_4096^{t k1}; (t, k1) at t*17 + k1
    const float2 wk = tw(sh.thi, sh.tlo, 16u * tid);
    auto pass1 = [&](float2 (&v)[16], float2* b) {
      dft<16, false>(v);
      float2* row = b + tid * kRow;
      float2 wprev = wk;
      static_for<0, 16>([&](auto K) {
        constexpr int k1 = decltype(K)::value;
        const float2 y = v[bitrev(k1, 4)];
        if constexpr (k1 == 0) {
          row[0] = y;
        } else {
          float2 w;
          if constexpr (k1 == 1) w = wk;
          else if constexpr (k1 & 1) w = tw(sh.thi, sh.tlo, 16u * tid * k1);
          else w = cmul(wprev, wk);
          if constexpr (k1 & 1) wprev = w;
          row[k1] = cmul(y, w);
        }
      });
    };
    pass1(v0, sh.buf);
    pass1(v1, sh.buf + kFft);
    __syncthreads();
    // pass 2: (k1, u) = (t / 16, t % 16); reads (u + 16 v, k1), twiddle W_256^{u k2},
    // writes (k1 + 16 k2, u) at (k1 + 16 k2)*17 + u
    const uint32_t k1 = tid >> 4, u = tid & 15u;
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) {
      v0[vv] = sh.buf[(u + 16u * vv) * kRow + k1];
      v1[vv] = sh.buf[kFft + (u + 16u * vv) * kRow + k1];
    }
    const float2 wu = sh.thi[u];                                  // W_256^u
    auto pass2 = [&](float2 (&v)[16]) {
      dft<16, false>(v);
      float2 o[16];
      float2 wprev = wu;
      static_for<0, 16>([&](auto K) {
        constexpr int k2 = decltype(K)::value;
        const float2 y = v[bitrev(k2, 4)];
        if constexpr (k2 == 0) {
          o[0] = y;
        } else {
          float2 w;
          if constexpr (k2 == 1) w = wu;
          else if constexpr (k2 & 1) w = sh.thi[u * k2];
          else w = cmul(wprev, wu);
          if constexpr (k2 & 1) wprev = w;
          o[k2] = cmul(y, w);
        }
      });
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = o[k];
    };
    pass2(v0);
    pass2(v1);
    __syncthreads();                     // every pass-2 read is done before the writes
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
      sh.buf[(k1 + 16u * k2) * kRow + u] = v0[k2];
      sh.buf[kFft + (k1 + 16u * k2) * kRow + u] = v1[k2];
    }
    __syncthreads();
  }
  // pass 3: two columns per thread, X[c + 256 j] in natural order
  uint32_t fa, ca, fb, cb, qa, qbb;
  if (r != 0) { fa = 0; ca = tid; fb = 1; cb = 255u - tid; qa = c0; qbb = c1; }
  else if (tid < 128) { fa = fb = 0; ca = tid; cb = tid == 0 ? 128u : 256u - tid; qa = qbb = 0; }
  else { fa = fb = 1; ca = tid - 128u; cb = 383u - tid; qa = qbb = 4; }
  const bool special = (r == 0 && tid == 0);
  float2 va[16], vb[16];
  {
    const float2* pa = sh.buf + fa * kFft + ca * kRow;
    const float2* pb = sh.buf + fb * kFft + cb * kRow;
    float2 ta[16], tb[16];
#pragma unroll
    for (int uu = 0; uu < 16; ++uu) { ta[uu] = pa[uu]; tb[uu] = pb[uu]; }
    dft<16, false>(ta);
    dft<16, false>(tb);
#pragma unroll
    for (int m = 0; m < 16; ++m) { va[m] = ta[bitrev(m, 4)]; vb[m] = tb[bitrev(m, 4)]; }
  }

  // ---- 3. real-FFT post-processing in registers: X[k] = (P + conj Q)/2 - i W_L^k (P - conj Q)/2
  auto r2c = [](float2 P, float2 Q, float2 w) -> float2 {
    const float2 A = make_float2(P.x + Q.x, P.y - Q.y);
    const float2 B = make_float2(P.x - Q.x, P.y + Q.y);
    const float2 t = cmul(w, make_float2(B.y, -B.x));
    return make_float2(0.5f * (A.x + t.x), 0.5f * (A.y + t.y));
  };
  float2 xn = make_float2(0.f, 0.f);      // X[N] (CTA 0, thread 0 only)
  if (!special) {
    // bins 8(c + 256 j) + q: W_L^{8c + q} W_32^j
    const float2 wA = tw(sh.thi, sh.tlo, 8u * ca + qa);
    const float2 wB = tw(sh.thi, sh.tlo, 8u * cb + qbb);
    static_for<0, 16>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 P = va[j], Q = vb[15 - j];
      va[j] = r2c(P, Q, w32mul<j>(wA));
      vb[15 - j] = r2c(Q, P, w32mul<15 - j>(wB));
    });
  } else {
    // column 0 of class 0: pairs j <-> 16-j; self pairs j = 0 (X[0], X[N]) and j = 8 (X[N/2])
    const float2 a0 = va[0];
    static_for<1, 8>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 P = va[j], Q = va[16 - j];
      va[j] = r2c(P, Q, w32mul<j>(make_float2(1.f, 0.f)));
      va[16 - j] = r2c(Q, P, w32mul<16 - j>(make_float2(1.f, 0.f)));
    });
    va[8] = r2c(va[8], va[8], w32mul<8>(make_float2(1.f, 0.f)));
    va[0] = make_float2(a0.x + a0.y, 0.f);
    xn = make_float2(a0.x - a0.y, 0.f);
    // column 128 of class 0: bins 1024 + 2048 j, pairs j <-> 15-j; W_L^1024 = W_64^1
    const float2 w1 = w64mul<1>(make_float2(1.f, 0.f));
    static_for<0, 8>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 P = vb[j], Q = vb[15 - j];
      vb[j] = r2c(P, Q, w32mul<j>(w1));
      vb[15 - j] = r2c(Q, P, w32mul<15 - j>(w1));
    });
  }
#define BIN_A(j) (8u * (ca + 256u * (j)) + qa)
#define BIN_B(j) (8u * (cb + 256u * (j)) + qbb)

  if (DEBUG) {
    float2* out = a.dbg_spec + ci.bin_off;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      out[BIN_A(j)] = va[j];
      out[BIN_B(j)] = vb[j];
    }
    if (special) out[kN] = xn;
    return;
  }

  // ---- 4. count-mode selection, cluster-wide (cluster barriers A-D)
  const uint32_t kdrop = ci.drop;
  int mode = kModeList;
  if (kdrop == 0) mode = kModeKeepAll;
  else if (kdrop >= kBins) mode = kModeDropAll;
  float band_lo = 0.f, band_hi = INFINITY;
  uint32_t mcount = 0;
  __syncthreads();                                // pass-3 reads of buf are done
  if (mode == kModeList) {
    uint32_t* hp[4];
    uint32_t* hp2[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      hp[c] = cluster.map_shared_rank(sh.hist, c);
      hp2[c] = cluster.map_shared_rank(sh.hist2, c);
    }
    // pass 1: proxy bits [30:20] into four sub-histograms (in buf)
    uint32_t* sub = reinterpret_cast<uint32_t*>(sh.buf) + 2048u * ((tid >> 5) & 3u);
    {
      uint4* z = reinterpret_cast<uint4*>(sh.buf);
      for (uint32_t e = tid; e < 2048; e += kT) z[e] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    uint32_t nz = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t pa = __float_as_uint(proxy_key(va[j].x, va[j].y));
      const uint32_t pb = __float_as_uint(proxy_key(vb[j].x, vb[j].y));
      nz |= __float_as_uint(va[j].x) | __float_as_uint(va[j].y) | __float_as_uint(vb[j].x) |
            __float_as_uint(vb[j].y);
      atomicAdd(&sub[pa >> 20], 1u);
      atomicAdd(&sub[pb >> 20], 1u);
    }
    if (special) {
      nz |= __float_as_uint(xn.x) | __float_as_uint(xn.y);
      atomicAdd(&sub[__float_as_uint(proxy_key(xn.x, xn.y)) >> 20], 1u);
    }
    nz &= 0x7FFFFFFFu;                            // -0.0 is zero
    if (__any_sync(0xffffffffu, nz != 0) && (tid & 31) == 0) atomicOr(&sh.anynz, 1u);
    __syncthreads();
    {
      const uint4* s4 = reinterpret_cast<const uint4*>(sh.buf);
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const uint32_t e = 2 * tid + h2;
        const uint4 x0 = s4[e], x1 = s4[512 + e], x2 = s4[1024 + e], x3 = s4[1536 + e];
        reinterpret_cast<uint4*>(sh.hist)[e] =
            make_uint4(x0.x + x1.x + x2.x + x3.x, x0.y + x1.y + x2.y + x3.y, x0.z + x1.z + x2.z + x3.z,
                       x0.w + x1.w + x2.w + x3.w);
      }
    }
    cluster.sync();                               // A: pass-1 histograms visible
    bool anynz = false;
#pragma unroll
    for (int c = 0; c < 4; ++c) anynz |= cluster.map_shared_rank(&sh, c)->anynz != 0;
    uint32_t b1, below1;
    merged_bucket4(sh, hp, kdrop - 1, b1, below1);
    if (!anynz) {
      mode = kModeDropAll;                        // every coefficient is exactly zero: all codes 0
    } else {
      // pass 2: proxy bits [19:9] of the bins inside bucket b1 (few: direct atomics)
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t pa = __float_as_uint(proxy_key(va[j].x, va[j].y));
        const uint32_t pb = __float_as_uint(proxy_key(vb[j].x, vb[j].y));
        if ((pa >> 20) == b1) atomicAdd(&sh.hist2[(pa >> 9) & 0x7FFu], 1u);
        if ((pb >> 20) == b1) atomicAdd(&sh.hist2[(pb >> 9) & 0x7FFu], 1u);
      }
      if (special) {
        const uint32_t pn = __float_as_uint(proxy_key(xn.x, xn.y));
        if ((pn >> 20) == b1) atomicAdd(&sh.hist2[(pn >> 9) & 0x7FFu], 1u);
      }
    }
    cluster.sync();                               // B: pass-2 histograms visible
    if (mode == kModeList) {
      uint32_t b2, below2;
      merged_bucket4(sh, hp2, kdrop - 1 - below1, b2, below2);
      const uint32_t lo_pat = (b1 << 20) | (b2 << 9);
      const float lo_f = __uint_as_float(lo_pat);
      const float hi_f = __uint_as_float(lo_pat + 512u);
      if (lo_f < 0x1p-100f || hi_f > 0x1p100f) {
        mode = kModeFallback;
      } else {
        band_lo = lo_f * (1.0f - 0x1p-16f);
        band_hi = hi_f * (1.0f + 0x1p-16f);
        // collect undecided bins into CTA 0's list; count the certainly dropped
        uint32_t below_l = 0;
        auto collect = [&](float2 x, uint32_t bin) {
          const float p = proxy_key(x.x, x.y);
          below_l += (p < band_lo) ? 1u : 0u;
          if (p >= band_lo && p < band_hi) push_candidate4(&sh0, bin, x.x, x.y);
        };
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          collect(va[j], BIN_A(j));
          collect(vb[j], BIN_B(j));
        }
        if (special) collect(xn, kN);
        const uint32_t bl = block_sum<kT>(below_l, sh.scan);
        if (tid == 0) sh.below = bl;
      }
    }
    cluster.sync();                               // C: candidates and counts visible
    if (r == 0) {
      if (tid == 0) {
        int md = mode;
        const uint32_t m = sh.ccount;
        uint32_t below = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) below += cluster.map_shared_rank(&sh, c)->below;
        if (md == kModeList && (m > (uint32_t)kCand || below > kdrop || below + m < kdrop)) md = kModeFallback;
        sh.need = kdrop - below;
        sh.mode = md;
      }
      __syncthreads();
      if (sh.mode == kModeList) resolve4(sh, sh.ccount, sh.need);
    }
    cluster.sync();                               // D: decisions visible
    mode = sh0.mode;
    mcount = (mode == kModeList) ? sh0.ccount : 0u;
  } else {
    cluster.sync();                               // D': every bitmap zeroed (peer atomics follow)
  }

  if (mode == kModeFallback) {
    float2* out = a.fb_spec + ci.bin_off;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      out[BIN_A(j)] = va[j];
      out[BIN_B(j)] = vb[j];
    }
    if (special) out[kN] = xn;
    __threadfence();
    cluster.sync();          // every part written; the peers finished reading sh0.mode
    if (r != 0) return;
    // CTA 0 selects and packs the chunk with the generic single-CTA code,
    // its scratch in the (now free) class buffers
    sel::select_pack_chunk<float2, kT>(*reinterpret_cast<sel::SelectSharedT<kT>*>(sh.buf), ci,
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

  // ---- 5. emit: non-zero (re | im << 16) codes of kept bins into their owner's
  //         bin-ordered array; owner of BIN_A(j) / BIN_B(j) is CTA j / 4.
  float lo_b = band_lo, hi_b = band_hi;           // KeepAll / DropAll as degenerate bands
  if (mode == kModeKeepAll) { lo_b = -1.0f; hi_b = -1.0f; }
  if (mode == kModeDropAll) { lo_b = INFINITY; hi_b = INFINITY; }
  uint32_t* arr_own = reinterpret_cast<uint32_t*>(sh.buf);
  uint32_t keep = 0, band = 0;                    // bit 2j: va[j], 2j+1: vb[j]
  static_for<0, 16>([&](auto J) {
    constexpr int j = decltype(J)::value;
    const float pa = proxy_key(va[j].x, va[j].y), pb = proxy_key(vb[j].x, vb[j].y);
    keep |= ((pa >= hi_b ? 1u : 0u) << (2 * j)) | ((pb >= hi_b ? 1u : 0u) << (2 * j + 1));
    band |= ((pa >= lo_b && pa < hi_b ? 1u : 0u) << (2 * j)) | ((pb >= lo_b && pb < hi_b ? 1u : 0u) << (2 * j + 1));
  });
  while (band) {                                  // undecided bins: the resolved list decides
    const uint32_t b = __ffs(band) - 1u;
    band &= band - 1u;
    const uint32_t bin = 8u * (((b & 1u) ? cb : ca) + 256u * (b >> 1)) + ((b & 1u) ? qbb : qa);
    if (!inband_dropped4(&sh0, mcount, bin)) keep |= 1u << b;
  }
  uint32_t rc[4] = {0, 0, 0, 0};                  // my non-zero codes per owner
  {
    const uint32_t lane = tid & 31u;
    uint32_t* wmeta = arr_own + kUpper + (tid >> 5) * kStripWords;
    float2* wval = reinterpret_cast<float2*>(wmeta + 256);
    static_for<0, 4>([&](auto R) {
      constexpr int d = decltype(R)::value;        // owner of this round's bins
      constexpr int j0 = 4 * d;
      uint32_t* arr_d = reinterpret_cast<uint32_t*>(cluster.map_shared_rank(sh.buf, d));
      uint32_t* hbm_d = cluster.map_shared_rank(sh.hbm, d);
      const uint32_t m8 = (keep >> (2 * j0)) & 0xFFu;
      const uint32_t cnt = __popc(m8);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += t;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      uint32_t pos = incl - cnt;
      static_for<0, 8>([&](auto K) {
        constexpr int k = decltype(K)::value;
        constexpr int j = j0 + k / 2;
        if ((m8 >> k) & 1u) {
          wmeta[pos] = (k & 1) ? BIN_B(j) : BIN_A(j);
          wval[pos] = (k & 1) ? vb[j] : va[j];
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
          rc[d] += (cre ? 1u : 0u) + (cim ? 1u : 0u);
          const uint32_t lb = bin - (uint32_t)d * kOwn;
          arr_d[pad(lb)] = pc;
          atomicOr(&hbm_d[lb >> 4], ((cre ? 1u : 0u) | (cim ? 2u : 0u)) << (2u * (lb & 15u)));
        }
      }
      __syncwarp();                               // strip reused by the next round
    });
  }
  if (special) {                                  // bin N -> CTA 3, local bin 8192
    const float p = proxy_key(xn.x, xn.y);
    bool kp = p >= lo_b;
    if (kp && p < hi_b) kp = !inband_dropped4(&sh0, mcount, kN);
    if (kp) {
      const uint32_t cre = enc16(q, xn.x), cim = enc16(q, xn.y);
      const uint32_t pc = cre | (cim << 16);
      if (pc) {
        rc[3] += (cre ? 1u : 0u) + (cim ? 1u : 0u);
        reinterpret_cast<uint32_t*>(cluster.map_shared_rank(sh.buf, 3))[pad(kOwn)] = pc;
        atomicOr(&cluster.map_shared_rank(sh.hbm, 3)[kOwn >> 4], (cre ? 1u : 0u) | (cim ? 2u : 0u));
      }
    }
  }
#undef BIN_A
#undef BIN_B
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    const uint32_t sd = __reduce_add_sync(0xffffffffu, rc[d]);
    if ((tid & 31) == 0 && sd) atomicAdd(&sh.rcount[d], sd);
  }
  cluster.sync();                                 // E: owners' arrays, bitmaps and counts complete
  if (tid == 0) {
    uint32_t tot[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const Sh4* pcs = cluster.map_shared_rank(&sh, c);
#pragma unroll
      for (int d = 0; d < 4; ++d) tot[d] += pcs->rcount[d];
    }
    sh.S[0] = 0;
#pragma unroll
    for (int d = 0; d < 4; ++d) sh.S[d + 1] = sh.S[d] + tot[d] * (uint32_t)q.n_bits;
  }
  __syncthreads();
  const int N = q.n_bits;
  const uint32_t Sb = sh.S[r], Se = sh.S[r + 1], Stot = sh.S[4];
  // a boundary between two owners' code runs that splits a byte needs the
  // owners' staged words merged (fold, cluster barrier F); byte-aligned
  // boundaries are written bytewise by each owner
  bool fold = false;
  if (N != 8 && N != 16) {
#pragma unroll
    for (int d = 1; d < 4; ++d) fold |= (sh.S[d] & 7u) != 0;
  }
  // Without a fold the rcount reads were the last remote access: arrive now,
  // wait before exiting (a CTA's shared memory must outlive its peers' accesses).
  if (!fold) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");

  // ---- 6. pack: thread t of CTA r owns bins 8192 r + [32t, 32t+32) (+ bin N)
  const uint32_t nb = (r == 3 && tid == kT - 1) ? 33u : 32u;
  const uint32_t w0 = sh.hbm[2 * tid], w1 = sh.hbm[2 * tid + 1], w2 = (nb == 33) ? sh.hbm[kOwn >> 4] : 0u;
  const uint32_t cnt = __popc(w0) + __popc(w1) + __popc(w2);
  uint32_t* seg = reinterpret_cast<uint32_t*>(a.message + ci.seg_off);
  uint32_t* bm = seg + kSegHeader / 4;
  {
    const uint32_t wb = r * (kOwn / 16) + 2u * tid;
    bm[wb] = ballot_to_wire(w0);
    bm[wb + 1] = ballot_to_wire(w1);
    if (nb == 33) {
      bm[wb + 2] = ballot_to_wire(w2);
      const uint32_t pad_words = (ci.code_off - kSegHeader) / 4;
      for (uint32_t w = kBmWords; w < pad_words; ++w) bm[w] = 0u;
    }
  }
  uint32_t total;
  const uint32_t base = block_exclusive_scan<kT>(cnt, sh.scan, total);
  // this CTA's run starts at global bit Sb; staged in shared memory:
  // local word k <-> global word (Sb >> 5) + k
  const uint32_t wstart = Sb >> 5, o = Sb & 31u;
  const uint32_t nwords = total ? (uint32_t)((o + (uint64_t)total * N + 31) / 32) : 0u;
  uint32_t* stg = arr_own + kUpper;
  for (uint32_t k = tid; k <= nwords; k += kT) stg[k] = 0u;
  __syncthreads();
  {
    uint32_t lbit = o + base * (uint32_t)N;               // local bit of my first code
    uint8_t* stg8 = reinterpret_cast<uint8_t*>(stg);
    // slot s of my bins: bin s / 2, re (s even) / im (s odd)
    auto emit_slots = [&](uint32_t m, const uint32_t* src) {
      while (m) {
        const uint32_t pos = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t pc = src[pos >> 1];
        const uint32_t code = (pos & 1) ? (pc >> 16) : (pc & 0xFFFFu);
        if (N == 8) {
          stg8[lbit >> 3] = (uint8_t)code;                // byte-aligned codes: plain stores
        } else {
          const uint32_t wi = lbit >> 5, sb = lbit & 31u;
          atomicOr(&stg[wi], code << sb);
          if (sb + N > 32u) atomicOr(&stg[wi + 1], code >> (32u - sb));
        }
        lbit += N;
      }
    };
    const uint32_t* row = arr_own + pad(32u * tid);       // my 32 bins (pad(32t + j) = pad(32t) + j)
    emit_slots(w0, row);
    emit_slots(w1, row + 16);
    if (w2) emit_slots(w2, arr_own + pad(kOwn));
  }
  __syncthreads();
  if (fold) cluster.sync();                       // F: every owner's staging complete
  uint32_t* codes_g = reinterpret_cast<uint32_t*>(a.message + ci.seg_off + ci.code_off);
  const bool tail_shared = (Se & 31u) != 0 && Se < Stot;   // later owners' bits follow in my last word
  for (uint32_t k = tid; k < nwords; k += kT) {
    const uint32_t w = wstart + k;
    if (w >= ci.code_cap) continue;
    const bool first = k == 0 && o != 0;          // word shared with earlier owners
    const bool last = k + 1 == nwords && tail_shared;
    if (!first && !last) {
      codes_g[w] = stg[k];
    } else if (!fold) {
      const uint32_t lo = first ? (o >> 3) : 0u, hi = last ? ((Se & 31u) >> 3) : 4u;
      uint8_t* p = reinterpret_cast<uint8_t*>(codes_g + w);
      const uint32_t val = stg[k];
      for (uint32_t b = lo; b < hi; ++b) p[b] = (uint8_t)(val >> (8 * b));
    } else if (!first) {
      // I own bit 32w: merge the staged first words of the later owners starting in it
      uint32_t val = stg[k];
#pragma unroll
      for (int e = 1; e < 4; ++e) {
        if (e > (int)r && sh.S[e + 1] > sh.S[e] && (sh.S[e] >> 5) == w)
          val |= reinterpret_cast<const uint32_t*>(cluster.map_shared_rank(sh.buf, e))[kUpper];
      }
      codes_g[w] = val;
    }
  }
  const uint32_t used = (uint32_t)(((uint64_t)Stot + 31) / 32);
  const uint32_t cap_padded = (ci.code_cap + 3u) & ~3u;
  if (r == 3)
    for (uint32_t w = used + tid; w < cap_padded; w += kT) codes_g[w] = 0u;
  if (r == 0 && tid == 0) {
    seg[0] = Stot / (uint32_t)N;
    seg[1] = 0; seg[2] = 0; seg[3] = 0;
    if (used > ci.code_cap) atomicOr(a.flags, FGC_FLAG_CAPACITY);
  }
  if (a.pc.cnt || a.pc.done) {
    // the segment is complete once every CTA's writes are visible device-wide
    __threadfence();
    if (!fold) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // the early arrive's phase
    cluster.sync();                               // (G) every thread of the cluster has fenced
    if (r == 0 && tid == 0) {
      if (a.pc.cnt) atomicAdd(&a.pc.cnt[(chunk - a.pc.first) / a.pc.per], 1u);
      if (a.pc.done) release_tag(a.pc.done + chunk, a.pc.tag, a.pc.sys);
    }
  } else if (fold) {
    cluster.sync();                               // G: owners finished reading the peers' staging
  } else {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

template <class K>
fgc_status set_smem4(K kernel, size_t bytes) {
  FGC_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return FGC_OK;
}

}  // namespace
}  // namespace fgc

namespace fgc {

fgc_status compress4_init() {
  static bool done = false;
  if (done) return FGC_OK;
  const size_t b = sizeof(Sh4);
  FGC_TRY(set_smem4(k_fused_compress4<float, false, false>, b));
  FGC_TRY(set_smem4(k_fused_compress4<double, false, false>, b));
  FGC_TRY(set_smem4(k_fused_compress4<float, true, false>, b));
  FGC_TRY(set_smem4(k_fused_compress4<double, true, false>, b));
  FGC_TRY(set_smem4(k_fused_compress4<float, false, true>, b));
  FGC_TRY(set_smem4(k_fused_compress4<double, false, true>, b));
  FGC_TRY(set_smem4(k_fused_compress4<float, true, true>, b));
  FGC_TRY(set_smem4(k_fused_compress4<double, true, true>, b));
  done = true;
  return FGC_OK;
}

fgc_status launch_compress4(const float2* thi, const float2* tlo, uint32_t ahead, const ChunkInfo* d_chunks,
                            uint32_t first, uint32_t count, const void* grad, int dtype, int half_pass,
                            const QuantParams& q, uint8_t* message, uint32_t* flags, float2* fb_spec, float2* dbg,
                            cudaStream_t s, PieceCounter pc) {
  if (!count) return FGC_OK;
  FGC_TRY(compress4_init());
  C4Args a{d_chunks, first, grad, q, message, flags, thi, tlo, fb_spec, dbg, count, ahead, pc};
  const size_t smem = sizeof(Sh4);
  const dim3 grid(4 * count), block(kT);
  const bool f64 = dtype == FGC_DTYPE_F64, h = half_pass != 0;
#define FGC_LAUNCH_C4(T, D, H) k_fused_compress4<T, D, H><<<grid, block, smem, s>>>(a)
  if (dbg) {
    if (f64) { if (h) FGC_LAUNCH_C4(double, true, true); else FGC_LAUNCH_C4(double, true, false); }
    else { if (h) FGC_LAUNCH_C4(float, true, true); else FGC_LAUNCH_C4(float, true, false); }
  } else {
    if (f64) { if (h) FGC_LAUNCH_C4(double, false, true); else FGC_LAUNCH_C4(double, false, false); }
    else { if (h) FGC_LAUNCH_C4(float, false, true); else FGC_LAUNCH_C4(float, false, false); }
  }
#undef FGC_LAUNCH_C4
  FGC_LAUNCHED(1);
  return FGC_OK;
}

}  // namespace fgc
