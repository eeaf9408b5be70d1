// Host-side internal interfaces between the plan (plan.cpp) and the kernel
// translation units.  Not part of the public C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "fgc_types.h"
#include "../../include/fgc_b200.h"

namespace fgc {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
const std::string& last_error();
fgc_status cuda_check(cudaError_t e, const char* what);
void count_launch(uint64_t n = 1);
#define FGC_CUDA(call)                                                  \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) return ::fgc::cuda_check(e_, #call);         \
  } while (0)
#define FGC_STR2(x) #x
#define FGC_STR(x) FGC_STR2(x)
#define FGC_LAUNCHED(n)                                                                       \
  do {                                                                                        \
    ::fgc::count_launch(n);                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                      \
    if (e_ != cudaSuccess) return ::fgc::cuda_check(e_, "kernel launch " __FILE__ ":" FGC_STR(__LINE__)); \
  } while (0)
#define FGC_TRY(expr)                                                   \
  do {                                                                  \
    fgc_status s_ = (expr);                                             \
    if (s_ != FGC_OK) return s_;                                        \
  } while (0)

// ---------------------------------------------------------------- generic DFT
// Complex DFT of length Lc for a batch of signals (fft_generic.cu), in
// float32 (codec tails) or float64 (whole-signal primitives, calibrate).
enum class DftKind : int { Direct = 0, Pow2 = 1, Bluestein = 2, Mixed = 3 };

// Mixed: Lc = A * B, B = 2^e, A odd <= kMixedMaxA (one direct pass + Pow2 rows).
constexpr uint32_t kMixedMaxA = 512;

template <class R> struct Vec2;
template <> struct Vec2<float> { using T = float2; };
template <> struct Vec2<double> { using T = double2; };

// Points one CTA transforms in shared memory (two 64 KB ping-pong halves).
__host__ __device__ inline uint32_t smem_points(uint32_t real_bytes) { return real_bytes == 4 ? 4096u : 2048u; }

__host__ __device__ inline void fft_split(uint32_t P, uint32_t cap, uint32_t& Rr, uint32_t& C) {
  uint32_t lg = 0;
  while ((1u << lg) < P) ++lg;
  uint32_t lr = lg / 2;
  while ((1u << lr) > cap) --lr;
  Rr = 1u << lr;
  C = P / Rr;
}

// Position of frequency k in the four-step engine layout of a size-P pow2
// transform (natural when P fits one CTA).
__host__ __device__ inline uint64_t engine_pos(uint32_t P, uint32_t cap, uint64_t k) {
  uint64_t base = 0;
  while (P > cap) {
    uint32_t Rr, C;
    fft_split(P, cap, Rr, C);
    base += (k % Rr) * C;
    k /= Rr;
    P = C;
  }
  return base + k;
}

// Where frequency k of a DFT result lives: layout 0 natural, 1 Pow2 engine
// layout of size P, 2 Mixed rows (k % A) of B points in engine layout.
__host__ __device__ inline uint64_t result_pos(int layout, uint32_t P, uint32_t A, uint32_t B, uint32_t cap,
                                               uint64_t k) {
  if (layout == 1) return engine_pos(P, cap, k);
  if (layout == 2) return (k % A) * B + engine_pos(B, cap, k / A);
  return k;
}

template <class R>
struct DftResultT {
  const typename Vec2<R>::T* base;  // buffer
  uint64_t stride;                  // per batch item
  int layout;                       // 0 natural, 1 engine layout, 2 mixed rows (result_pos)
  int chirp;                        // 1: multiply by chirp[k] / P (Bluestein)
};

template <class R>
struct DftPlanT {
  using T2 = typename Vec2<R>::T;
  DftKind kind = DftKind::Direct;
  uint32_t Lc = 1;        // DFT length
  uint32_t P = 1;         // pow2 transform size (Pow2 / Bluestein); Lc for Direct / Mixed
  uint32_t A = 1, B = 1;  // Mixed factors (Lc = A * B)
  uint32_t batch = 0;
  T2* tw = nullptr;       // P twiddles exp(-2 pi i j / P)
  T2* chirp = nullptr;    // Bluestein chirp exp(-i pi n^2 / Lc), n < Lc
  T2* bf = nullptr;       // Bluestein kernel spectrum, engine layout
  T2* mtw = nullptr;      // Mixed: exp(-2 pi i m / Lc), m < Lc
  T2* work = nullptr;     // batch * P
  T2* work2 = nullptr;    // Direct output buffer
  T2* rtw = nullptr;      // real-signal twiddles exp(-2 pi i k / L), k <= L/2 (even L)
  fgc_status init(uint32_t Lc, uint32_t batch, cudaStream_t s);
  void free_all();
  // dir=-1 forward (natural input in work), dir=+1 unscaled inverse (Pow2:
  // engine-layout input).  Bluestein always runs the forward chirp-z on the
  // chirped, zero-padded input; inverse callers conjugate around it.
  fgc_status run(int dir, DftResultT<R>& res, cudaStream_t s);
};

// Real-signal transforms of a batch of equal-length chunks described by
// ChunkInfo entries [first, first+count) (real_fft.cu).
template <class R>
struct RealClassT {
  uint32_t L = 0, bins = 0, first = 0, count = 0;
  bool fused = false;
  DftPlanT<R> dft;
  fgc_status init(cudaStream_t s);   // needs L, count
  void free_all() { dft.free_all(); }
};

// in_dtype: FGC_DTYPE_F32 / F64 input; spectrum and out in precision R.
template <class R>
fgc_status real_forward(RealClassT<R>& rc, const ChunkInfo* d_chunks, const void* in, int in_dtype, int half_pass,
                        uint32_t* flags, typename Vec2<R>::T* spectrum, cudaStream_t s);
template <class R>
fgc_status real_inverse(RealClassT<R>& rc, const ChunkInfo* d_chunks, const typename Vec2<R>::T* spectrum, R* out,
                        cudaStream_t s);

// The whole chain of one tail chunk in one 1024-thread CTA per direction
// (real_fft.cu): forward transform + select + pack into `message`, and the
// weighted decode of W messages + inverse transform into `out`.  Float
// plans, one chunk, Pow2 (P <= 4096) or Mixed (B <= 4096) only.
bool tail_chain_ok(const RealClassT<float>& rc);
fgc_status tail_forward_chain(RealClassT<float>& rc, const ChunkInfo* d_chunks, const void* in, int in_dtype,
                              int half_pass, uint32_t* flags, float2* spectrum, const QuantParams& q, uint8_t* message,
                              cudaStream_t s);
struct Weights;
fgc_status tail_inverse_chain(RealClassT<float>& rc, const ChunkInfo* d_chunks, const uint8_t* messages, int W,
                              uint64_t stride, const Weights& wts, const QuantParams& q, float2* spectrum, float* out,
                              uint32_t max_slots, cudaStream_t s);

// ---------------------------------------------------------------- codec kernels

// Select (count mode) + quantize + pack from a chunk-major spectrum.
// Chunks [first, first+count).  coeff_f64: spectrum is double2.
// only_if (may be null): skip chunk c unless only_if[c] != 0.
// Per-piece completion counters for the peer exchange: chunk c adds one to
// cnt[(c - first) / per] once its message segment is globally visible.
struct PieceCounter {
  uint32_t* cnt = nullptr;
  uint32_t first = 0, per = 1;
  uint32_t* done = nullptr;           // per chunk id: set to `tag` (release) once the segment is written
  uint32_t tag = 0;
  uint32_t sys = 0;                   // release `done` at system scope (peers on other GPUs read it)
  // kernel pushes (exchange_kpush): CTA r of chunk c's cluster stores its half
  // of the segment at pdst[p] + seg_off and then releases ptag[p][2c + r] =
  // pval (system scope) for each of the npeers peers
  uint8_t* const* pdst = nullptr;
  uint32_t* const* ptag = nullptr;
  uint32_t npeers = 0, pval = 0;
};

// Decode-side wait of the peer exchange: before reading chunk c, every peer
// b != me must have set flags[b * stride + (c - first) / per] >= target.
struct PieceWait {
  const uint32_t* flags = nullptr;
  uint32_t stride = 0, first = 0, per = 1, target = 0;
  int nranks = 0, me = 0;
  // this rank's own segment: done[c] == tag (the compress kernel of the same
  // step runs concurrently; the decode is launched as its programmatic dependent)
  const uint32_t* done = nullptr;
  uint32_t tag = 0;
  // in-kernel transports: before reading chunk c, dtab[b][c * tstride + j]
  // >= target for every peer b != me and j < tstride (tags its compress
  // kernel released); message w starts at mtab[w] when set (direct reads of
  // the peers' own buffers), else in the local gathered stack
  const uint8_t* const* mtab = nullptr;
  const uint32_t* const* dtab = nullptr;
  uint32_t tstride = 1;
};

// drop_mask (may be null): 1 byte per bin of the chunk-major spectrum; when
// given it replaces the count-mode selection (energy mode).
fgc_status launch_select_pack(const ChunkInfo* d_chunks, uint32_t first, uint32_t count, const void* spectrum,
                              int coeff_f64, const QuantParams& q, uint8_t* message, uint8_t* kept_mask,
                              uint32_t* flags, cudaStream_t s, const uint32_t* only_if = nullptr,
                              PieceCounter pc = PieceCounter(), const uint8_t* drop_mask = nullptr);

// Energy-mode drop sets (energy.cu).
struct EnergyScratch {
  double* keys = nullptr;            // per bin: numpy cabs key (sorted in place by the exact fallback)
  uint32_t* idx = nullptr;           // per bin: bin index (exact fallback)
  uint32_t* kcut = nullptr;          // per chunk: 1 = redo with the exact fallback
  uint8_t* drop = nullptr;           // per bin: 1 = dropped
  uint64_t cap_bins = 0;
  uint32_t cap_chunks = 0;
  fgc_status ensure(uint64_t bins, uint32_t chunks);
  void free_all();
};
fgc_status energy_drop_mask(EnergyScratch& e, const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                            uint64_t bin0, uint64_t nbins, uint32_t max_bins, const void* spectrum, int f64,
                            double theta, cudaStream_t s, const uint8_t** drop_out);

// Decode + weighted accumulate of W messages into a chunk-major spectrum.
struct Weights {
  float w[FGC_MAX_WORKERS];
};
fgc_status launch_decode_accumulate(const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                                    const uint8_t* messages, int W, uint64_t stride, const Weights& wts,
                                    const QuantParams& q, float2* spectrum, uint32_t max_slots, cudaStream_t s);

// Parseval reconstruction error per chunk: out[c] = (err, norm) of chunk c.
fgc_status launch_spectrum_error(const ChunkInfo* d_chunks, uint32_t n_chunks, uint32_t max_slots,
                                 const float2* spectrum, const uint8_t* message, const QuantParams& q, double2* out,
                                 cudaStream_t s);

// Wire format kernels (wire.cu).
fgc_status launch_serialize(const ChunkInfo* d_chunks, uint32_t n_chunks, const uint8_t* message, int n_bits,
                            const uint8_t header[FGC_HEADER_BYTES], uint8_t* wire, uint64_t* wire_len,
                            uint64_t* scratch, cudaStream_t s);
fgc_status launch_deserialize(const ChunkInfo* d_chunks, uint32_t n_chunks, const uint8_t* wire,
                              const uint64_t* chunk_offsets, int n_bits, uint8_t* message, uint32_t* popcounts,
                              cudaStream_t s);
fgc_status launch_message_counts(const ChunkInfo* d_chunks, uint32_t n_chunks, const uint8_t* message, uint32_t* nnz,
                                 cudaStream_t s);
fgc_status launch_message_unpack(const ChunkInfo* d_chunks, uint32_t n_chunks, const uint8_t* message, int n_bits,
                                 const uint64_t* code_offsets, uint8_t* flags01, uint32_t* codes, cudaStream_t s);
fgc_status launch_message_pack(const ChunkInfo* d_chunks, uint32_t n_chunks, const uint8_t* flags01,
                               const uint32_t* codes, const uint64_t* code_offsets, int n_bits, uint8_t* message,
                               uint32_t* popcounts, uint32_t* flags, cudaStream_t s);
// Runtime theta (fgc_plan_set_theta): chunk c's drop count becomes
// min(ceil(theta * bins), bins) in float64 (spectral.py:131), on the stream.
fgc_status launch_set_drop(ChunkInfo* d_chunks, uint32_t n_chunks, double theta, cudaStream_t s);
fgc_status launch_scan_u64(uint64_t* v, uint32_t n, uint64_t* total, uint64_t add, cudaStream_t s);

// Fused sm_100a kernels for 65536-sample chunks (fused.cu).
struct FusedTables;
bool fused_available();
fgc_status fused_tables_init(FusedTables** t, cudaStream_t s);
void fused_tables_free(FusedTables* t);
// fb_spec: chunk-major spectrum scratch; a degenerate chunk's spectrum goes
// there and CTA 0 selects it with the generic code in place.
fgc_status launch_fused_compress(const FusedTables* t, const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                                 const void* grad, int dtype, int half_pass, const QuantParams& q, uint8_t* message,
                                 uint32_t* flags, float2* fb_spec, cudaStream_t s,
                                 PieceCounter pc = PieceCounter());
fgc_status launch_fused_decode(const FusedTables* t, const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                               const uint8_t* messages, int W, uint64_t stride, const Weights& wts,
                               const QuantParams& q, float* out, cudaStream_t s, PieceWait pw = PieceWait());
// 4-CTA-cluster compress, two CTAs per SM (fused4.cu); thi / tlo are the
// fused kernels' twiddle tables, `ahead` the L2 prefetch distance in chunks.
fgc_status launch_compress4(const float2* thi, const float2* tlo, uint32_t ahead, const ChunkInfo* d_chunks,
                            uint32_t first, uint32_t count, const void* grad, int dtype, int half_pass,
                            const QuantParams& q, uint8_t* message, uint32_t* flags, float2* fb_spec, float2* dbg,
                            cudaStream_t s, PieceCounter pc);
// 2-CTA-cluster compress with 1024 threads per CTA (fused_w.cu): the
// radix-32 columns split over lane pairs; t1024 is W_1024^m.
fgc_status launch_compress_w(const float2* thi, const float2* tlo, const float2* t1024, uint32_t ahead,
                             const ChunkInfo* d_chunks, uint32_t first, uint32_t count, const void* grad, int dtype,
                             int half_pass, const QuantParams& q, uint8_t* message, uint32_t* flags, float2* fb_spec,
                             float2* dbg, cudaStream_t s, PieceCounter pc);
// Instrumentation knobs (fgc_debug_set_fused_knobs) and the per-CTA phase
// timestamp buffer, for fused kernels outside fused.cu (knobs 0: none).
void fused_debug_state(uint32_t& knobs, unsigned long long*& ts);
// Debug hooks: the fused kernels' own forward coefficients / inverse.
fgc_status launch_fused_spectrum(const FusedTables* t, const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                                 const void* grad, int dtype, int half_pass, float2* spectrum, uint32_t* flags,
                                 cudaStream_t s);
fgc_status launch_fused_inverse(const FusedTables* t, const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                                const float2* spectrum, float* out, cudaStream_t s);

// Peer exchange internals (xchg.cu).
fgc_status exchange_publish_event(fgc_exchange* x, int k, uint64_t lo, uint64_t bytes, cudaEvent_t ready,
                                  uint32_t value, int fi = -1);
fgc_status exchange_publish_piece(fgc_exchange* x, int k, uint32_t i, uint64_t lo, uint64_t bytes,
                                  uint32_t count_target, uint32_t value);
fgc_status exchange_publish_used(fgc_exchange* x, int k, const ChunkInfo* d_chunks, uint32_t n_chunks, int n_bits,
                                 cudaEvent_t ready, uint32_t value, int fi = -1);
fgc_status exchange_wait(fgc_exchange* x, cudaStream_t s, int fi, uint32_t value);
PieceCounter exchange_counter(fgc_exchange* x, uint32_t first, uint32_t per);
PieceWait exchange_piece_wait(fgc_exchange* x, uint32_t first, uint32_t per, uint32_t target);
// Transport of the fused chunks (FGC_EXCHANGE_DIRECT): 0 copy-engine pushes
// in pieces (default), 1 direct reads -- the decode reads every peer's
// segments in the peer's own buffer over NVLink, 2 kernel pushes -- the
// compress kernel stores each finished segment into the peers' buffers.
// Both in-kernel transports signal per chunk.
int exchange_transport(const fgc_exchange* x, uint32_t chunk_end);
void exchange_direct(fgc_exchange* x, int k, uint32_t tag, PieceCounter& pc, PieceWait& pw);
void exchange_kpush(fgc_exchange* x, int k, uint32_t tag, PieceCounter& pc, PieceWait& pw);
uint32_t exchange_max_pieces();
uint32_t exchange_piece_target(fgc_exchange* x, uint32_t i, uint32_t chunks);
fgc_status exchange_join(fgc_exchange* x, cudaStream_t s);
fgc_status exchange_events(fgc_exchange* x, uint32_t P, std::vector<cudaEvent_t>** ev);
void exchange_counters(fgc_exchange* x, uint32_t** counter, uint64_t** step, int* nranks, int* rank,
                       uint64_t* msg_bytes);
bool exchange_ready(const fgc_exchange* x);
// A step that failed after it began enqueueing pushes / flag writes leaves the
// peers' counters out of step with ours: poison the exchange so every later
// call fails fast instead of waiting forever.
void exchange_poison(fgc_exchange* x);
bool exchange_poisoned(const fgc_exchange* x);
void exchange_trace(cudaStream_t s, const char* tag);

}  // namespace fgc
