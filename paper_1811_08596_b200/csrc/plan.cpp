// The C ABI (include/fgc_b200.h): plans, the compress / decode-average hot
// path, wire-format entry points.  Host logic only; kernels live in *.cu.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <vector>

#include "fgc_internal.h"

namespace fgc {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
fgc_status cuda_check(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return FGC_ERR_CUDA;
}
void count_launch(uint64_t n) { g_launches += n; }

const std::string& last_error() { return g_last_error; }
using RealClass = RealClassT<float>;

static uint64_t a16(uint64_t x) { return (x + 15) & ~15ull; }

// The transform kernels load the signal two samples at a time (float2 /
// double2), so a device gradient must be 8-byte (f32) or 16-byte (f64)
// aligned.
static fgc_status check_signal(const void* g, int dtype) {
  if (dtype != FGC_DTYPE_F32 && dtype != FGC_DTYPE_F64) {
    set_error("unknown dtype");
    return FGC_ERR_INVALID;
  }
  const uintptr_t need = dtype == FGC_DTYPE_F64 ? 16 : 8;
  if (reinterpret_cast<uintptr_t>(g) % need) {
    set_error(dtype == FGC_DTYPE_F64 ? "float64 gradient must be 16-byte aligned"
                                     : "float32 gradient must be 8-byte aligned");
    return FGC_ERR_INVALID;
  }
  return FGC_OK;
}

// The decode kernels load message segments 16 bytes at a time.
static fgc_status check_messages(const uint8_t* m, uint64_t stride) {
  if (reinterpret_cast<uintptr_t>(m) % 16 || stride % 16) {
    set_error("device messages must be 16-byte aligned with a 16-byte multiple stride");
    return FGC_ERR_INVALID;
  }
  return FGC_OK;
}

// The decode kernels store two output samples at a time (float2).
static fgc_status check_out(const float* out) {
  if (reinterpret_cast<uintptr_t>(out) % 8) {
    set_error("float32 output must be 8-byte aligned");
    return FGC_ERR_INVALID;
  }
  return FGC_OK;
}

}  // namespace fgc

using namespace fgc;

struct fgc_plan {
  fgc_codec_desc desc{};
  double theta_cap = 0.0;            // count mode: the theta message capacity is sized for
  QuantParams q{};
  uint32_t n_chunks = 0;
  std::vector<ChunkInfo> chunks;
  std::vector<RealClass> classes;
  std::vector<uint64_t> seg_off, bin_off;
  uint64_t msg_bytes = 0, spec_bins = 0, wire_max = 0, total_slots = 0;
  uint32_t max_slots = 0;
  ChunkInfo* d_chunks = nullptr;
  float2* d_spec = nullptr;
  uint64_t* d_scratch = nullptr;
  uint32_t* d_done = nullptr;        // per chunk: tag of the last compress that wrote its segment
  uint32_t tag = 0;                  // last tag handed out
  cudaStream_t side = nullptr;       // generic (tail) classes overlap the fused kernels here
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  FusedTables* fused = nullptr;
  uint32_t fused_first = 0, fused_count = 0;     // chunk range taken by fused kernels
  EnergyScratch energy;              // energy-mode selection scratch (allocated on first use)
  // host-buffer averaging: copy streams and per-piece events (created on first use)
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev_h, ev_c2, ev_d;
  // host step: piece i of dev_grad fully read by the last call's compress
  // (the next call's host->device copy of piece i waits only for that)
  std::vector<cudaEvent_t> ev_cin;
  cudaEvent_t ev_step = nullptr;
  // pipelined allgather-average: exchange stream + per-piece events (created on first use)
  cudaStream_t xstream = nullptr;
  std::vector<cudaEvent_t> ev_comp, ev_gath;
};

static QuantParams make_qparams(const fgc_codec_desc& d) {
  QuantParams q{};
  if (d.passthrough) {
    q.n_bits = 32;
    return q;
  }
  q.n_bits = d.quant.n_bits;
  q.shift = 23 - d.quant.mantissa_bits;
  q.pbase = d.quant.pbase;
  q.npos = d.quant.pos_count;
  q.nneg = d.quant.neg_count;
  q.eps = d.quant.eps;
  q.pos_cap = d.quant.max;
  q.neg_cap = -d.quant.actual_min;
  return q;
}

// Decode overlapped with the compress grid's last wave (programmatic
// dependent launch + per-chunk done tags); FGC_NO_OVERLAP=1 serialises them.
static bool overlap_enabled() {
  const char* e = getenv("FGC_NO_OVERLAP");
  return !(e && e[0] == '1');
}

static bool fused_enabled() {
  const char* e = getenv("FGC_DISABLE_FUSED");
  return !(e && e[0] == '1');
}

extern "C" fgc_status fgc_message_layout(const fgc_codec_desc* d, uint32_t* n_chunks, uint64_t* message_bytes,
                                         uint64_t* offs) {
  if (!d || !n_chunks || !message_bytes) return FGC_ERR_INVALID;
  if (d->n < 1 || d->chunk_size < 16 || !(d->theta >= 0.0 && d->theta <= 1.0)) {
    set_error("invalid codec description");
    return FGC_ERR_INVALID;
  }
  const int N = d->passthrough ? 32 : d->quant.n_bits;
  const uint64_t full = d->n / d->chunk_size;
  const uint64_t tail = d->n % d->chunk_size;
  const uint64_t count = full + (tail ? 1 : 0);
  uint64_t seg = 0;
  for (uint64_t c = 0; c < count; ++c) {
    const uint64_t L = c < full ? d->chunk_size : tail;
    const uint64_t bins = L / 2 + 1, slots = 2 * bins;
    uint64_t drop = (uint64_t)ceil(d->theta * (double)bins);
    if (drop > bins) drop = bins;
    const uint64_t maxnz = (d->mode == FGC_MODE_COUNT && !d->full_capacity) ? 2 * (bins - drop) : slots;
    if (offs) offs[c] = seg;
    seg += kSegHeader + a16(4 * ((slots + 31) / 32)) + a16(4 * ((maxnz * N + 31) / 32));
  }
  if (offs) offs[count] = seg;
  *n_chunks = (uint32_t)count;
  *message_bytes = seg;
  return FGC_OK;
}

extern "C" fgc_status fgc_plan_create(const fgc_codec_desc* desc, fgc_plan** out) {
  if (!desc || !out) { set_error("null argument"); return FGC_ERR_INVALID; }
  *out = nullptr;
  const fgc_codec_desc& d = *desc;
  if (d.n < 1) { set_error("gradient must be a non-empty 1D sequence"); return FGC_ERR_INVALID; }
  if (d.chunk_size < 16) { set_error("chunk_size must be >= 16"); return FGC_ERR_INVALID; }
  if (!(d.theta >= 0.0 && d.theta <= 1.0)) { set_error("theta must be in [0, 1]"); return FGC_ERR_INVALID; }
  if (d.mode != FGC_MODE_COUNT && d.mode != FGC_MODE_ENERGY) { set_error("unknown mode"); return FGC_ERR_INVALID; }
  if (d.chunk_size > (1u << 20)) {
    set_error("chunk_size above 2^20 is not supported by the GPU codec");
    return FGC_ERR_UNSUPPORTED;
  }
  fgc_codec_desc dd = d;
  if (!d.passthrough) {
    fgc_status st = fgc_quantizer_validate(&dd.quant);
    if (st != FGC_OK) return st;
  }
  fgc_plan* p = new fgc_plan();
  p->desc = dd;
  p->theta_cap = dd.theta;
  p->q = make_qparams(p->desc);
  const int N = p->q.n_bits;
  const uint64_t full = d.n / d.chunk_size;
  const uint32_t tail = (uint32_t)(d.n % d.chunk_size);
  p->n_chunks = (uint32_t)(full + (tail ? 1 : 0));
  if (full) {
    RealClass c;
    c.L = d.chunk_size;
    c.bins = c.L / 2 + 1;
    c.first = 0;
    c.count = (uint32_t)full;
    // 65536-sample chunks run the fused kernels: the fused compress in count
    // mode; in energy mode the fused forward transform and the fused decode
    // around the energy selection
    c.fused = fused_available() && fused_enabled() && c.L == 65536 && !d.passthrough && d.quant.n_bits <= 16;
    p->classes.push_back(c);
  }
  if (tail) {
    RealClass c;
    c.L = tail;
    c.bins = tail / 2 + 1;
    c.first = (uint32_t)full;
    c.count = 1;
    c.fused = false;
    p->classes.push_back(c);
  }
  p->chunks.resize(p->n_chunks);
  p->seg_off.resize(p->n_chunks + 1);
  p->bin_off.resize(p->n_chunks + 1);
  uint64_t seg = 0, bin = 0, slot = 0, in = 0;
  for (uint32_t cls = 0; cls < p->classes.size(); ++cls) {
    const RealClass& rc = p->classes[cls];
    for (uint32_t j = 0; j < rc.count; ++j) {
      const uint32_t c = rc.first + j;
      ChunkInfo ci{};
      ci.in_off = in;
      ci.seg_off = seg;
      ci.bin_off = bin;
      ci.slot_off = slot;
      ci.len = rc.L;
      ci.bins = rc.bins;
      ci.slots = 2 * rc.bins;
      // k = ceil(theta * bins) in float64 (spectral.py:131)
      const double kd = ceil(d.theta * (double)rc.bins);
      ci.drop = (uint32_t)std::min<double>(kd, (double)rc.bins);
      uint64_t maxnz = ci.slots;
      if (d.mode == FGC_MODE_COUNT && !d.full_capacity) maxnz = 2ull * (rc.bins - ci.drop);
      const uint64_t bm_words = (ci.slots + 31) / 32;
      ci.code_off = (uint32_t)(kSegHeader + a16(4 * bm_words));
      ci.code_cap = (uint32_t)((maxnz * N + 31) / 32);
      ci.cls = cls;
      ci.idx_in_cls = j;
      p->chunks[c] = ci;
      p->seg_off[c] = seg;
      p->bin_off[c] = bin;
      seg += ci.code_off + a16(4ull * ci.code_cap);
      bin += ci.bins;
      slot += ci.slots;
      in += rc.L;
      p->wire_max += 4 + (ci.slots + 7) / 8 + (maxnz * N + 7) / 8;
      p->max_slots = std::max(p->max_slots, ci.slots);
    }
  }
  p->seg_off[p->n_chunks] = seg;
  p->bin_off[p->n_chunks] = bin;
  p->msg_bytes = seg;
  p->spec_bins = bin;
  p->total_slots = slot;
  p->wire_max += FGC_HEADER_BYTES;

  auto fail = [&](fgc_status st) {
    fgc_plan_destroy(p);
    return st;
  };
  cudaStream_t s = 0;
  cudaError_t e;
  if ((e = cudaMalloc(&p->d_chunks, sizeof(ChunkInfo) * p->n_chunks)) != cudaSuccess) return fail(cuda_check(e, "cudaMalloc"));
  if ((e = cudaMemcpy(p->d_chunks, p->chunks.data(), sizeof(ChunkInfo) * p->n_chunks, cudaMemcpyHostToDevice)) != cudaSuccess)
    return fail(cuda_check(e, "cudaMemcpy"));
  if ((e = cudaMalloc(&p->d_spec, sizeof(float2) * p->spec_bins)) != cudaSuccess) return fail(cuda_check(e, "cudaMalloc"));
  if ((e = cudaMalloc(&p->d_scratch, sizeof(uint64_t) * (p->n_chunks + 1))) != cudaSuccess)
    return fail(cuda_check(e, "cudaMalloc"));
  if ((e = cudaMalloc(&p->d_done, sizeof(uint32_t) * p->n_chunks)) != cudaSuccess)
    return fail(cuda_check(e, "cudaMalloc"));
  if ((e = cudaMemset(p->d_done, 0, sizeof(uint32_t) * p->n_chunks)) != cudaSuccess)
    return fail(cuda_check(e, "cudaMemset"));
  {
    // the side stream carries the small tail-chunk kernels: give them priority
    // so they take SMs as soon as the wide fused kernels release any
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if ((e = cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, greatest)) != cudaSuccess)
      return fail(cuda_check(e, "cudaStreamCreate"));
  }
  if ((e = cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming)) != cudaSuccess)
    return fail(cuda_check(e, "cudaEventCreate"));
  if ((e = cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming)) != cudaSuccess)
    return fail(cuda_check(e, "cudaEventCreate"));
  for (RealClass& rc : p->classes) {
    if (rc.fused) {
      fgc_status st = fused_tables_init(&p->fused, s);
      if (st != FGC_OK) return fail(st);
      p->fused_first = rc.first;
      p->fused_count = rc.count;
      continue;
    }
    fgc_status st = rc.init(s);
    if (st != FGC_OK) return fail(st);
  }
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return fail(cuda_check(e, "plan init"));
  *out = p;
  return FGC_OK;
}

extern "C" void fgc_plan_destroy(fgc_plan* p) {
  if (!p) return;
  for (RealClass& rc : p->classes) rc.free_all();
  p->energy.free_all();
  if (p->fused) fused_tables_free(p->fused);
  cudaFree(p->d_chunks);
  cudaFree(p->d_spec);
  cudaFree(p->d_scratch);
  cudaFree(p->d_done);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  if (p->side) cudaStreamDestroy(p->side);
  for (cudaEvent_t e : p->ev_h) cudaEventDestroy(e);
  for (cudaEvent_t e : p->ev_c2) cudaEventDestroy(e);
  for (cudaEvent_t e : p->ev_d) cudaEventDestroy(e);
  for (cudaEvent_t e : p->ev_cin) cudaEventDestroy(e);
  if (p->ev_step) cudaEventDestroy(p->ev_step);
  if (p->h2d) cudaStreamDestroy(p->h2d);
  if (p->d2h) cudaStreamDestroy(p->d2h);
  for (cudaEvent_t e : p->ev_comp) cudaEventDestroy(e);
  for (cudaEvent_t e : p->ev_gath) cudaEventDestroy(e);
  if (p->xstream) cudaStreamDestroy(p->xstream);
  delete p;
}

extern "C" fgc_status fgc_plan_set_theta(fgc_plan* p, double theta, void* stream) {
  if (!p) { set_error("null argument"); return FGC_ERR_INVALID; }
  if (!(theta >= 0.0 && theta <= 1.0)) { set_error("theta must be in [0, 1]"); return FGC_ERR_INVALID; }
  if (p->desc.mode == FGC_MODE_COUNT && !p->desc.full_capacity && theta < p->theta_cap) {
    set_error("theta " + std::to_string(theta) + " is below the plan's capacity theta " +
              std::to_string(p->theta_cap));
    return FGC_ERR_INVALID;
  }
  if (theta == p->desc.theta) return FGC_OK;
  p->desc.theta = theta;
  bool changed = false;
  for (ChunkInfo& ci : p->chunks) {
    const double kd = ceil(theta * (double)ci.bins);
    const uint32_t drop = (uint32_t)std::min<double>(kd, (double)ci.bins);
    changed |= drop != ci.drop;
    ci.drop = drop;
  }
  if (!changed) return FGC_OK;
  return launch_set_drop(p->d_chunks, p->n_chunks, theta, static_cast<cudaStream_t>(stream));
}

extern "C" fgc_status fgc_plan_get_info(const fgc_plan* p, fgc_plan_info* out) {
  if (!p || !out) return FGC_ERR_INVALID;
  out->n = p->desc.n;
  out->n_chunks = p->n_chunks;
  out->chunk_size = p->desc.chunk_size;
  out->tail_len = (uint32_t)(p->desc.n % p->desc.chunk_size);
  out->n_bits = (uint32_t)p->q.n_bits;
  out->message_bytes = p->msg_bytes;
  out->wire_bytes_max = p->wire_max;
  out->spectrum_bins = p->spec_bins;
  out->fused_chunks = p->fused_count;
  out->max_slots = p->max_slots;
  out->total_slots = p->total_slots;
  return FGC_OK;
}

extern "C" fgc_status fgc_plan_segment_offsets(const fgc_plan* p, uint64_t* o) {
  if (!p || !o) return FGC_ERR_INVALID;
  memcpy(o, p->seg_off.data(), sizeof(uint64_t) * (p->n_chunks + 1));
  return FGC_OK;
}

extern "C" fgc_status fgc_plan_bin_offsets(const fgc_plan* p, uint64_t* o) {
  if (!p || !o) return FGC_ERR_INVALID;
  memcpy(o, p->bin_off.data(), sizeof(uint64_t) * (p->n_chunks + 1));
  return FGC_OK;
}

// Forward transform of every non-fused class into `spectrum`.
static fgc_status forward_generic(fgc_plan* p, const void* grad, int dtype, float2* spectrum, uint32_t* flags,
                                  cudaStream_t s, bool include_fused_classes) {
  for (RealClass& rc : p->classes) {
    if (rc.fused && !include_fused_classes) continue;
    if (rc.fused) {
      set_error("fused class has no generic plan");
      return FGC_ERR_UNSUPPORTED;
    }
    FGC_TRY(real_forward<float>(rc, p->d_chunks, grad, dtype, p->desc.half_pass, flags, spectrum, s));
  }
  return FGC_OK;
}

// FGC_TAIL_CHAIN=1: the tail class beside the fused grid runs as one
// single-CTA chain per direction (real_fft.cu) when every generic class
// qualifies.  Bit-identical to the multi-kernel chain but measured slower
// (0.363 vs 0.300 ms per step: its 183 / 131 us of latency per direction
// end up on the critical path), so off by default.
static bool tail_chain(const fgc_plan* p) {
  static const bool on = [] { const char* e = getenv("FGC_TAIL_CHAIN"); return e && e[0] == '1'; }();
  if (!on || !p->fused_count) return false;
  for (const RealClass& rc : p->classes)
    if (!rc.fused && !tail_chain_ok(rc)) return false;
  return true;
}

static fgc_status check_mode(const fgc_plan* p) {
  if (p->desc.mode != FGC_MODE_COUNT && p->desc.mode != FGC_MODE_ENERGY) {
    set_error("unknown sparsification mode");
    return FGC_ERR_INVALID;
  }
  return FGC_OK;
}

// Energy mode (spectral.py:134-139): the forward transform (the fused
// kernel's for 65536-sample chunks, the generic engine otherwise), the exact
// energy drop set, then the common quantize + pack with the drop mask.
// spectrum_in (chunk-major float2) replaces the forward transform when given
// (stage injection).
static fgc_status energy_compress(fgc_plan* p, const void* grad, int dtype, const float2* spectrum_in,
                                  uint8_t* message, uint8_t* kept_mask, uint32_t* flags, cudaStream_t s) {
  const float2* spec = spectrum_in;
  if (!spec) {
    for (RealClass& rc : p->classes)
      if (rc.fused)
        FGC_TRY(launch_fused_spectrum(p->fused, p->d_chunks, rc.first, rc.count, grad, dtype, p->desc.half_pass,
                                      p->d_spec, flags, s));
    FGC_TRY(forward_generic(p, grad, dtype, p->d_spec, flags, s, false));
    spec = p->d_spec;
  }
  uint32_t max_bins = 1;
  for (const ChunkInfo& ci : p->chunks) max_bins = std::max(max_bins, ci.bins);
  const uint8_t* drop = nullptr;
  FGC_TRY(energy_drop_mask(p->energy, p->d_chunks, 0, p->n_chunks, 0, p->spec_bins, max_bins, spec, 0,
                           p->desc.theta, s, &drop));
  return launch_select_pack(p->d_chunks, 0, p->n_chunks, spec, 0, p->q, message, kept_mask, flags, s, nullptr,
                            PieceCounter(), drop);
}

// Compress the fused chunks [f0, f0 + fc) and, when `generic`, every generic
// (tail) class -- those on the high-priority side stream, joined back into s.
static fgc_status compress_range(fgc_plan* p, const void* grad, int dtype, uint8_t* message, uint32_t* flags,
                                 cudaStream_t s, uint32_t f0, uint32_t fc, bool generic) {
  const bool fork = generic && fc && p->classes.size() > 1;
  cudaStream_t g = fork ? p->side : s;
  if (fork) {
    FGC_CUDA(cudaEventRecord(p->ev_fork, s));
    FGC_CUDA(cudaStreamWaitEvent(g, p->ev_fork, 0));
  }
  if (generic && tail_chain(p)) {
    for (RealClass& rc : p->classes)
      if (!rc.fused)
        FGC_TRY(tail_forward_chain(rc, p->d_chunks, grad, dtype, p->desc.half_pass, flags, p->d_spec, p->q, message, g));
  } else if (generic) {
    FGC_TRY(forward_generic(p, grad, dtype, p->d_spec, flags, g, false));
    for (RealClass& rc : p->classes) {
      if (rc.fused) continue;
      FGC_TRY(launch_select_pack(p->d_chunks, rc.first, rc.count, p->d_spec, 0, p->q, message, nullptr, flags, g));
    }
  }
  if (fc) {
    // (degenerate chunks are selected in place by the generic code, spectrum in d_spec)
    FGC_TRY(launch_fused_compress(p->fused, p->d_chunks, f0, fc, grad, dtype, p->desc.half_pass, p->q, message,
                                  flags, p->d_spec, s));
  }
  if (fork) {
    FGC_CUDA(cudaEventRecord(p->ev_join, g));
    FGC_CUDA(cudaStreamWaitEvent(s, p->ev_join, 0));
  }
  return FGC_OK;
}

extern "C" fgc_status fgc_compress(fgc_plan* p, const void* grad, int dtype, uint8_t* message, uint32_t* flags,
                                   void* stream) {
  if (!p || !grad || !message || !flags) { set_error("null argument"); return FGC_ERR_INVALID; }
  FGC_TRY(check_mode(p));
  FGC_TRY(check_signal(grad, dtype));
  if (p->desc.mode == FGC_MODE_ENERGY)
    return energy_compress(p, grad, dtype, nullptr, message, nullptr, flags, static_cast<cudaStream_t>(stream));
  return compress_range(p, grad, dtype, message, flags, static_cast<cudaStream_t>(stream), p->fused_first,
                        p->fused_count, true);
}

extern "C" fgc_status fgc_encode_spectrum(fgc_plan* p, const void* spectrum, uint8_t* message, uint8_t* kept_mask,
                                          uint32_t* flags, void* stream) {
  if (!p || !spectrum || !message || !flags) { set_error("null argument"); return FGC_ERR_INVALID; }
  FGC_TRY(check_mode(p));
  if (p->desc.mode == FGC_MODE_ENERGY)
    return energy_compress(p, nullptr, 0, static_cast<const float2*>(spectrum), message, kept_mask, flags,
                           static_cast<cudaStream_t>(stream));
  return launch_select_pack(p->d_chunks, 0, p->n_chunks, spectrum, 0, p->q, message, kept_mask, flags,
                            static_cast<cudaStream_t>(stream));
}

extern "C" fgc_status fgc_forward_spectrum(fgc_plan* p, const void* grad, int dtype, void* spectrum, uint32_t* flags,
                                           void* stream) {
  if (!p || !grad || !spectrum || !flags) { set_error("null argument"); return FGC_ERR_INVALID; }
  FGC_TRY(check_signal(grad, dtype));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (RealClass& rc : p->classes) {
    if (!rc.fused) continue;
    FGC_TRY(launch_fused_spectrum(p->fused, p->d_chunks, rc.first, rc.count, grad, dtype, p->desc.half_pass,
                                  static_cast<float2*>(spectrum), flags, s));
  }
  return forward_generic(p, grad, dtype, static_cast<float2*>(spectrum), flags, s, false);
}

static fgc_status fill_weights(const double* weights, int W, Weights& w) {
  if (W < 1 || W > FGC_MAX_WORKERS) {
    set_error("worker count out of range");
    return FGC_ERR_INVALID;
  }
  for (int i = 0; i < W; ++i) w.w[i] = weights ? (float)weights[i] : 1.0f;
  return FGC_OK;
}

static fgc_status inverse_generic(fgc_plan* p, const float2* spectrum, float* out, cudaStream_t s) {
  for (RealClass& rc : p->classes) {
    if (rc.fused) continue;
    FGC_TRY(real_inverse<float>(rc, p->d_chunks, spectrum, out, s));
  }
  return FGC_OK;
}

// Decode-average the fused chunks [f0, f0 + fc) (and the generic classes when
// `generic`).  Message w's chunk c lives at messages + w * stride + seg_off(c).
static fgc_status decode_range(fgc_plan* p, const uint8_t* messages, int W, uint64_t stride, const Weights& w,
                               float* out, cudaStream_t s, uint32_t f0, uint32_t fc, bool generic) {
  const bool fork = generic && fc && p->classes.size() > 1;
  cudaStream_t g = fork ? p->side : s;
  if (fork) {
    FGC_CUDA(cudaEventRecord(p->ev_fork, s));
    FGC_CUDA(cudaStreamWaitEvent(g, p->ev_fork, 0));
  }
  if (generic && tail_chain(p)) {
    for (RealClass& rc : p->classes)
      if (!rc.fused)
        FGC_TRY(tail_inverse_chain(rc, p->d_chunks, messages, W, stride, w, p->q, p->d_spec, out, p->max_slots, g));
  } else if (generic) {
    for (RealClass& rc : p->classes) {
      if (rc.fused) continue;
      FGC_TRY(launch_decode_accumulate(p->d_chunks, rc.first, rc.count, messages, W, stride, w, p->q, p->d_spec,
                                       p->max_slots, g));
    }
    FGC_TRY(inverse_generic(p, p->d_spec, out, g));
  }
  if (fc) FGC_TRY(launch_fused_decode(p->fused, p->d_chunks, f0, fc, messages, W, stride, w, p->q, out, s));
  if (fork) {
    FGC_CUDA(cudaEventRecord(p->ev_join, g));
    FGC_CUDA(cudaStreamWaitEvent(s, p->ev_join, 0));
  }
  return FGC_OK;
}

extern "C" fgc_status fgc_decode_average(fgc_plan* p, const uint8_t* messages, int W, uint64_t stride,
                                         const double* weights, float* out, void* stream) {
  if (!p || !messages || !out) { set_error("null argument"); return FGC_ERR_INVALID; }
  FGC_TRY(check_out(out));
  FGC_TRY(check_messages(messages, stride));
  Weights w;
  FGC_TRY(fill_weights(weights, W, w));
  return decode_range(p, messages, W, stride, w, out, static_cast<cudaStream_t>(stream), p->fused_first,
                      p->fused_count, true);
}

extern "C" fgc_status fgc_decode_spectrum(fgc_plan* p, const uint8_t* messages, int W, uint64_t stride,
                                          const double* weights, void* spectrum, void* stream) {
  if (!p || !messages || !spectrum) { set_error("null argument"); return FGC_ERR_INVALID; }
  FGC_TRY(check_messages(messages, stride));
  Weights w;
  FGC_TRY(fill_weights(weights, W, w));
  return launch_decode_accumulate(p->d_chunks, 0, p->n_chunks, messages, W, stride, w, p->q,
                                  static_cast<float2*>(spectrum), p->max_slots, static_cast<cudaStream_t>(stream));
}

extern "C" fgc_status fgc_spectrum_error(fgc_plan* p, const void* spectrum, const uint8_t* message,
                                         double* err_norm, void* stream) {
  if (!p || !spectrum || !message || !err_norm) { set_error("null argument"); return FGC_ERR_INVALID; }
  FGC_TRY(check_messages(message, 16));
  if (p->q.n_bits == 32) {
    set_error("the Parseval error needs a quantizer (passthrough codes are the coefficients)");
    return FGC_ERR_UNSUPPORTED;
  }
  return launch_spectrum_error(p->d_chunks, p->n_chunks, p->max_slots, static_cast<const float2*>(spectrum),
                               message, p->q, reinterpret_cast<double2*>(err_norm),
                               static_cast<cudaStream_t>(stream));
}

extern "C" fgc_status fgc_inverse_spectrum(fgc_plan* p, const void* spectrum, float* out, void* stream) {
  if (!p || !spectrum || !out) { set_error("null argument"); return FGC_ERR_INVALID; }
  FGC_TRY(check_out(out));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (RealClass& rc : p->classes) {
    if (!rc.fused) continue;
    FGC_TRY(launch_fused_inverse(p->fused, p->d_chunks, rc.first, rc.count, static_cast<const float2*>(spectrum),
                                 out, s));
  }
  return inverse_generic(p, static_cast<const float2*>(spectrum), out, s);
}

// ------------------------------------------------------------------ wire

static void build_header(const fgc_plan* p, uint8_t h[FGC_HEADER_BYTES]) {
  const fgc_codec_desc& d = p->desc;
  uint8_t flags = 0;
  if (d.half_pass) flags |= 1;
  if (d.mode == FGC_MODE_ENERGY) flags |= 2;
  if (d.passthrough) flags |= 4;
  const float theta = (float)d.theta;
  const float qmin = d.passthrough ? 0.0f : d.quant.min;
  const float qmax = d.passthrough ? 0.0f : d.quant.max;
  const float qeps = d.passthrough ? 0.0f : d.quant.eps;
  const uint8_t nb = d.passthrough ? 32 : (uint8_t)d.quant.n_bits;
  const uint8_t mb = d.passthrough ? 0 : (uint8_t)d.quant.mantissa_bits;
  memcpy(h, "FGC1", 4);
  h[4] = 1;
  h[5] = flags;
  memcpy(h + 6, &d.n, 8);
  memcpy(h + 14, &d.chunk_size, 4);
  memcpy(h + 18, &theta, 4);
  memcpy(h + 22, &qmin, 4);
  memcpy(h + 26, &qmax, 4);
  memcpy(h + 30, &qeps, 4);
  h[34] = nb;
  h[35] = mb;
}

extern "C" fgc_status fgc_serialize(fgc_plan* p, const uint8_t* message, uint8_t* wire, uint64_t* wire_len,
                                    void* stream) {
  if (!p || !message || !wire || !wire_len) { set_error("null argument"); return FGC_ERR_INVALID; }
  uint8_t h[FGC_HEADER_BYTES];
  build_header(p, h);
  return launch_serialize(p->d_chunks, p->n_chunks, message, p->q.n_bits, h, wire, wire_len, p->d_scratch,
                          static_cast<cudaStream_t>(stream));
}

extern "C" fgc_status fgc_parse_header(const uint8_t* w, uint64_t len, fgc_codec_desc* d) {
  if (!w || !d) return FGC_ERR_INVALID;
  if (len < FGC_HEADER_BYTES) { set_error("buffer is shorter than the header"); return FGC_ERR_TRUNCATED; }
  if (memcmp(w, "FGC1", 4) != 0) { set_error("bad magic"); return FGC_ERR_HEADER; }
  if (w[4] != 1) { set_error("unsupported version"); return FGC_ERR_HEADER; }
  const uint8_t flags = w[5];
  if (flags & ~0x07) { set_error("unknown flag bits"); return FGC_ERR_HEADER; }
  uint64_t n;
  uint32_t chunk;
  float theta, qmin, qmax, qeps;
  memcpy(&n, w + 6, 8);
  memcpy(&chunk, w + 14, 4);
  memcpy(&theta, w + 18, 4);
  memcpy(&qmin, w + 22, 4);
  memcpy(&qmax, w + 26, 4);
  memcpy(&qeps, w + 30, 4);
  const int nb = w[34], mb = w[35];
  if (n < 1) { set_error("original_len must be >= 1"); return FGC_ERR_HEADER; }
  if (chunk < 16) { set_error("chunk_size below minimum 16"); return FGC_ERR_HEADER; }
  if (!(isfinite(theta) && theta >= 0.0f && theta <= 1.0f)) { set_error("theta outside [0, 1]"); return FGC_ERR_HEADER; }
  memset(d, 0, sizeof(*d));
  d->n = n;
  d->chunk_size = chunk;
  d->theta = (double)theta;
  d->mode = (flags & 2) ? FGC_MODE_ENERGY : FGC_MODE_COUNT;
  d->half_pass = (flags & 1) ? 1 : 0;
  d->passthrough = (flags & 4) ? 1 : 0;
  if (d->passthrough) {
    if (nb != 32) { set_error("passthrough flag requires N=32"); return FGC_ERR_HEADER; }
  } else {
    fgc_status st = fgc_quantizer_from_params(qmin, qmax, nb, mb, qeps, &d->quant);
    if (st != FGC_OK) {
      set_error("invalid quantizer parameters: " + last_error());
      return FGC_ERR_HEADER;
    }
  }
  return FGC_OK;
}

extern "C" fgc_status fgc_wire_index(const uint8_t* w, uint64_t len, const fgc_codec_desc* d, uint64_t* offsets,
                                     uint32_t* nnz, uint32_t* n_valid) {
  if (!w || !d || !offsets || !nnz || !n_valid) return FGC_ERR_INVALID;
  const int N = d->passthrough ? 32 : d->quant.n_bits;
  uint64_t pos = FGC_HEADER_BYTES;
  const uint64_t full = d->n / d->chunk_size;
  const uint64_t tail = d->n % d->chunk_size;
  const uint64_t count = full + (tail ? 1 : 0);
  *n_valid = 0;
  for (uint64_t c = 0; c < count; ++c) {
    const uint64_t L = c < full ? d->chunk_size : tail;
    const uint64_t slots = 2 * (L / 2 + 1);
    if (pos + 4 > len) { set_error("buffer ended before chunk header"); return FGC_ERR_TRUNCATED; }
    uint32_t k;
    memcpy(&k, w + pos, 4);
    offsets[c] = pos;
    nnz[c] = k;
    pos += 4;
    const uint64_t bmb = (slots + 7) / 8;
    if (pos + bmb > len) { set_error("buffer ended inside the bitmap"); return FGC_ERR_TRUNCATED; }
    pos += bmb;
    const uint64_t cb = ((uint64_t)k * N + 7) / 8;
    if (pos + cb > len) {
      *n_valid = (uint32_t)c;   // bitmap of chunk c is present; its codes are not
      // the reference checks the bitmap popcount against `kept` before the
      // code bytes (codec.py:424-433): chunk c's bitmap decides the error class
      uint64_t pop = 0;
      const uint8_t* b = w + pos - bmb;
      for (uint64_t i = 0; i < slots / 8; ++i) pop += (uint64_t)__builtin_popcount(b[i]);
      if (slots % 8) pop += (uint64_t)__builtin_popcount(b[slots / 8] >> (8 - slots % 8));
      if (pop != k) {
        set_error("bitmap marks " + std::to_string(pop) + " slots, header says " + std::to_string(k));
        return FGC_ERR_BITMAP;
      }
      set_error("buffer ended inside the packed codes");
      return FGC_ERR_TRUNCATED;
    }
    pos += cb;
    *n_valid = (uint32_t)(c + 1);
  }
  if (pos != len) {
    set_error(std::to_string(len - pos) + " unexpected trailing bytes");
    return FGC_ERR_FORMAT;
  }
  return FGC_OK;
}

extern "C" fgc_status fgc_deserialize(fgc_plan* p, const uint8_t* wire, const uint64_t* chunk_offsets,
                                      uint8_t* message, uint32_t* popcounts, void* stream) {
  if (!p || !wire || !chunk_offsets || !message || !popcounts) { set_error("null argument"); return FGC_ERR_INVALID; }
  return launch_deserialize(p->d_chunks, p->n_chunks, wire, chunk_offsets, p->q.n_bits, message, popcounts,
                            static_cast<cudaStream_t>(stream));
}

extern "C" fgc_status fgc_message_counts(fgc_plan* p, const uint8_t* message, uint32_t* nnz, void* stream) {
  if (!p || !message || !nnz) return FGC_ERR_INVALID;
  return launch_message_counts(p->d_chunks, p->n_chunks, message, nnz, static_cast<cudaStream_t>(stream));
}

extern "C" fgc_status fgc_message_unpack(fgc_plan* p, const uint8_t* message, const uint64_t* code_offsets,
                                         uint8_t* flags01, uint32_t* codes, void* stream) {
  if (!p || !message || !code_offsets || !flags01 || !codes) return FGC_ERR_INVALID;
  return launch_message_unpack(p->d_chunks, p->n_chunks, message, p->q.n_bits, code_offsets, flags01, codes,
                               static_cast<cudaStream_t>(stream));
}

extern "C" fgc_status fgc_message_pack(fgc_plan* p, const uint8_t* flags01, const uint32_t* codes,
                                       const uint64_t* code_offsets, uint8_t* message, uint32_t* popcounts,
                                       uint32_t* flags, void* stream) {
  if (!p || !flags01 || !code_offsets || !message || !popcounts || !flags) return FGC_ERR_INVALID;
  return launch_message_pack(p->d_chunks, p->n_chunks, flags01, codes, code_offsets, p->q.n_bits, message,
                             popcounts, flags, static_cast<cudaStream_t>(stream));
}

extern "C" fgc_status fgc_allgather_average(fgc_plan* p, void* comm, int nranks, const void* grad, int dtype,
                                            const double* weights, uint8_t* message, uint8_t* gathered, float* out,
                                            uint32_t* flags, void* stream) {
  if (!p || !grad || !message || !out || !flags) { set_error("null argument"); return FGC_ERR_INVALID; }
  FGC_TRY(check_out(out));
  if (nranks <= 1) {
    if (!p->fused_count || p->desc.mode != FGC_MODE_COUNT || !overlap_enabled()) {
      FGC_TRY(fgc_compress(p, grad, dtype, message, flags, stream));
      return fgc_decode_average(p, message, 1, p->msg_bytes, weights, out, stream);
    }
    // one rank: generic chunks compress + decode on the side stream; the fused
    // decode runs as the fused compress grid's programmatic dependent, each
    // chunk's CTAs waiting for that chunk's segment (done tag)
    FGC_TRY(check_mode(p));
    FGC_TRY(check_signal(grad, dtype));
    Weights w;
    FGC_TRY(fill_weights(weights, 1, w));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool generic = p->classes.size() > 1;
    if (generic) {
      FGC_CUDA(cudaEventRecord(p->ev_fork, s));
      FGC_CUDA(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
      FGC_TRY(compress_range(p, grad, dtype, message, flags, p->side, 0, 0, true));
      FGC_TRY(decode_range(p, message, 1, p->msg_bytes, w, out, p->side, 0, 0, true));
      FGC_CUDA(cudaEventRecord(p->ev_join, p->side));
    }
    PieceCounter pc;
    pc.done = p->d_done;
    pc.tag = ++p->tag;
    FGC_TRY(launch_fused_compress(p->fused, p->d_chunks, p->fused_first, p->fused_count, grad, dtype,
                                  p->desc.half_pass, p->q, message, flags, p->d_spec, s, pc));
    PieceWait pw;
    pw.done = p->d_done;
    pw.tag = pc.tag;
    FGC_TRY(launch_fused_decode(p->fused, p->d_chunks, p->fused_first, p->fused_count, message, 1, p->msg_bytes, w,
                                p->q, out, s, pw));
    if (generic) FGC_CUDA(cudaStreamWaitEvent(s, p->ev_join, 0));
    return FGC_OK;
  }
  if (!comm || !gathered) { set_error("multi-rank average needs a communicator and a gather buffer"); return FGC_ERR_INVALID; }
  FGC_TRY(check_mode(p));
  FGC_TRY(check_signal(grad, dtype));
  Weights w;
  FGC_TRY(fill_weights(weights, nranks, w));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t wpp = 0;
  if (const char* e = getenv("FGC_PIPELINE_WAVES")) wpp = (uint32_t)std::max(0, atoi(e));
  if (wpp == 0 || p->desc.mode != FGC_MODE_COUNT || !p->fused_count) {
    // one piece: compress, one allgather, decode
    FGC_TRY(fgc_compress(p, grad, dtype, message, flags, stream));
    FGC_TRY(fgc_allgather(comm, message, gathered, p->msg_bytes, stream));
    return decode_range(p, gathered, nranks, p->msg_bytes, w, out, s, p->fused_first, p->fused_count, true);
  }
  // Pipeline in P pieces of consecutive chunks (their segments are contiguous):
  // piece i is allgathered on the exchange stream while piece i+1 compresses,
  // and decoded once its exchange is done.  The gather buffer holds piece i of
  // all ranks contiguously at W * seg_off(first chunk of i).
  // Pieces are whole waves of fused clusters (one 2-CTA cluster per 2 SMs), so
  // splitting the launches adds no partial waves; a short remainder joins the
  // last piece.  FGC_PIPELINE_WAVES sets the waves per piece (default 0 = one piece:
  // measured on 4 B200s, NCCL's allgather kernels competing for SMs cost more
  // than the overlap gains).
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t per = std::max(1u, wpp * (uint32_t)(sms / 2));
  uint32_t P = wpp ? std::max(1u, p->fused_count / per) : 1u;
  std::vector<uint32_t> f(P + 1);
  for (uint32_t i = 0; i < P; ++i) f[i] = p->fused_first + i * per;
  f[P] = p->fused_first + p->fused_count;                // the remainder (< 2 pieces) joins the last
  if (!p->xstream) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    FGC_CUDA(cudaStreamCreateWithPriority(&p->xstream, cudaStreamNonBlocking, greatest));
  }
  while (p->ev_comp.size() < P) {
    cudaEvent_t a, b;
    FGC_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    FGC_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    p->ev_comp.push_back(a);
    p->ev_gath.push_back(b);
  }
  // the generic (tail) chunks ride with the last piece
  auto piece_lo = [&](uint32_t i) -> uint64_t { return i == 0 ? 0 : p->seg_off[f[i]]; };
  auto piece_hi = [&](uint32_t i) -> uint64_t { return i + 1 == P ? p->msg_bytes : p->seg_off[f[i + 1]]; };
  for (uint32_t i = 0; i < P; ++i) {
    FGC_TRY(compress_range(p, grad, dtype, message, flags, s, f[i], f[i + 1] - f[i], i + 1 == P));
    FGC_CUDA(cudaEventRecord(p->ev_comp[i], s));
    FGC_CUDA(cudaStreamWaitEvent(p->xstream, p->ev_comp[i], 0));
    const uint64_t lo = piece_lo(i), bytes = piece_hi(i) - lo;
    FGC_TRY(fgc_allgather(comm, message + lo, gathered + (uint64_t)nranks * lo, bytes, p->xstream));
    FGC_CUDA(cudaEventRecord(p->ev_gath[i], p->xstream));
  }
  for (uint32_t i = 0; i < P; ++i) {
    FGC_CUDA(cudaStreamWaitEvent(s, p->ev_gath[i], 0));
    const uint64_t lo = piece_lo(i), bytes = piece_hi(i) - lo;
    FGC_TRY(decode_range(p, gathered + (uint64_t)nranks * lo - lo, nranks, bytes, w, out, s, f[i], f[i + 1] - f[i],
                         i + 1 == P));
  }
  return FGC_OK;
}

static fgc_status exchange_not_ready(const fgc_exchange* x) {
  set_error(exchange_poisoned(x) ? "exchange poisoned: an earlier step failed after it began publishing"
                                 : "exchange not opened");
  return FGC_ERR_INVALID;
}

static fgc_status exchange_average_impl(fgc_plan* p, fgc_exchange* x, const void* grad, int dtype,
                                        const double* weights, float* out, uint32_t* flags, void* stream,
                                        bool* started);

extern "C" fgc_status fgc_exchange_average(fgc_plan* p, fgc_exchange* x, const void* grad, int dtype,
                                           const double* weights, float* out, uint32_t* flags, void* stream) {
  bool started = false;
  const fgc_status st = exchange_average_impl(p, x, grad, dtype, weights, out, flags, stream, &started);
  if (st != FGC_OK && started) exchange_poison(x);
  return st;
}

static fgc_status exchange_average_impl(fgc_plan* p, fgc_exchange* x, const void* grad, int dtype,
                                        const double* weights, float* out, uint32_t* flags, void* stream,
                                        bool* started) {
  if (!p || !x || !grad || !out || !flags) { set_error("null argument"); return FGC_ERR_INVALID; }
  FGC_TRY(check_out(out));
  if (!exchange_ready(x)) return exchange_not_ready(x);
  FGC_TRY(check_mode(p));
  FGC_TRY(check_signal(grad, dtype));
  uint32_t* counter;
  uint64_t* step;
  int W, me;
  uint64_t mb;
  exchange_counters(x, &counter, &step, &W, &me, &mb);
  if (mb != p->msg_bytes) { set_error("exchange sized for another plan"); return FGC_ERR_INVALID; }
  Weights w;
  FGC_TRY(fill_weights(weights, W, w));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<cudaEvent_t>* ev;
  FGC_TRY(exchange_events(x, 1, &ev));
  cudaEvent_t ev_start = (*ev)[0], ev_tail = (*ev)[1], ev_side = (*ev)[2];
  const int k = (int)(*step & 1);
  const uint32_t tval = (uint32_t)(*step + 1);          // this step's flag value
  const uint32_t Pmax = exchange_max_pieces();
  uint8_t *message, *gathered;
  FGC_TRY(fgc_exchange_message(x, k, &message, &gathered));
  *started = true;
  exchange_trace(s, "start");
  if (p->desc.mode == FGC_MODE_ENERGY) {
    // energy mode: no fused chunks; the whole message is one piece
    FGC_TRY(energy_compress(p, grad, dtype, nullptr, message, nullptr, flags, s));
    FGC_CUDA(cudaEventRecord(ev_tail, s));
    // energy messages are sized for every slot: push each segment's used bytes only
    FGC_TRY(exchange_publish_used(x, k, p->d_chunks, p->n_chunks, p->q.n_bits, ev_tail, tval));
    FGC_TRY(exchange_wait(x, s, (int)Pmax, tval));
    FGC_TRY(decode_range(p, gathered, W, p->msg_bytes, w, out, s, p->fused_first, p->fused_count, true));
    FGC_TRY(exchange_join(x, s));
    *step += 1;
    return FGC_OK;
  }
  // generic (tail) chunks on the side stream from the start of the step:
  // compress -> push (copy stream) -> wait for the peers' -> decode
  const bool generic = p->classes.size() > (p->fused_count ? 1u : 0u);
  const uint64_t fused_end = p->fused_count ? p->seg_off[p->fused_first + p->fused_count] : 0;
  if (generic) {
    FGC_CUDA(cudaEventRecord(ev_start, s));
    FGC_CUDA(cudaStreamWaitEvent(p->side, ev_start, 0));
    FGC_TRY(compress_range(p, grad, dtype, message, flags, p->side, 0, 0, true));
    FGC_CUDA(cudaEventRecord(ev_tail, p->side));
    exchange_trace(p->side, "tail-compressed");
    FGC_TRY(exchange_publish_event(x, k, fused_end, p->msg_bytes - fused_end, ev_tail, tval));
    FGC_TRY(exchange_wait(x, p->side, (int)Pmax, tval));
    exchange_trace(p->side, "tail-arrived");
    FGC_TRY(decode_range(p, gathered, W, p->msg_bytes, w, out, p->side, 0, 0, true));
    exchange_trace(p->side, "tail-decoded");
    FGC_CUDA(cudaEventRecord(ev_side, p->side));
  }
  const int transport = p->fused_count ? exchange_transport(x, p->fused_first + p->fused_count) : 0;
  if (transport) {
    // in-kernel transports, signalled per chunk (no copy streams, no pieces):
    // 1: the compress kernel releases each chunk's tag at system scope and
    //    the decode (its programmatic dependent) reads every peer's segment
    //    in the peer's own buffer once the peer's tag is there;
    // 2: the compress kernel stores each finished segment into every peer's
    //    gather buffer and releases the chunk's tags there; the decode reads
    //    the local gather buffer once the peers' tags arrived
    PieceCounter pc;
    PieceWait pw;
    if (transport == 1) {
      exchange_direct(x, k, tval, pc, pw);
    } else {
      exchange_kpush(x, k, tval, pc, pw);
      pc.done = p->d_done;
      pc.tag = ++p->tag;
      pw.done = p->d_done;
      pw.tag = pc.tag;
    }
    FGC_TRY(launch_fused_compress(p->fused, p->d_chunks, p->fused_first, p->fused_count, grad, dtype,
                                  p->desc.half_pass, p->q, message, flags, p->d_spec, s, pc));
    FGC_TRY(launch_fused_decode(p->fused, p->d_chunks, p->fused_first, p->fused_count, gathered, W, p->msg_bytes,
                                w, p->q, out, s, pw));
    exchange_trace(s, "decoded");
  } else if (p->fused_count) {
    // one compress launch; the kernel counts finished chunks per piece and the
    // copy streams push each piece the moment its count is complete
    // 4 pieces measured best at N=2 and N=4 (8: +5%, 16: +15%, 1: +20%)
    uint32_t P = 4;
    if (const char* e = getenv("FGC_EXCHANGE_PIECES")) P = (uint32_t)std::max(1, atoi(e));
    P = std::min(std::min(P, Pmax), p->fused_count);
    const uint32_t per = (p->fused_count + P - 1) / P;
    P = (p->fused_count + per - 1) / per;
    PieceCounter pc = exchange_counter(x, p->fused_first, per);
    const bool overlap = overlap_enabled();
    if (overlap) {
      pc.done = p->d_done;
      pc.tag = ++p->tag;
    }
    FGC_TRY(launch_fused_compress(p->fused, p->d_chunks, p->fused_first, p->fused_count, grad, dtype,
                                  p->desc.half_pass, p->q, message, flags, p->d_spec, s, pc));
    for (uint32_t i = 0; i < P; ++i) {
      const uint32_t c0 = p->fused_first + i * per, c1 = std::min(p->fused_first + p->fused_count, c0 + per);
      const uint64_t lo = p->seg_off[c0], hi = p->seg_off[c1];
      FGC_TRY(exchange_publish_piece(x, k, i, lo, hi - lo, exchange_piece_target(x, i, c1 - c0), tval));
    }
    // one decode launch, the compress grid's programmatic dependent: it fills
    // the SMs the compress grid's last wave leaves idle; each chunk's CTAs wait
    // for this rank's segment and for the piece from every peer
    PieceWait pw = exchange_piece_wait(x, p->fused_first, per, tval);
    if (overlap) {
      pw.done = p->d_done;
      pw.tag = pc.tag;
    }
    FGC_TRY(launch_fused_decode(p->fused, p->d_chunks, p->fused_first, p->fused_count, gathered, W, p->msg_bytes,
                                w, p->q, out, s, pw));
    exchange_trace(s, "decoded");
  }
  if (generic) FGC_CUDA(cudaStreamWaitEvent(s, ev_side, 0));
  FGC_TRY(exchange_join(x, s));
  exchange_trace(s, "end");
  *step += 1;
  (void)counter;
  return FGC_OK;
}

// Averaging step from and to HOST buffers: the PCIe transfers overlap the
// codec in pieces of consecutive chunks.  Piece i's host->device copy runs on
// a copy stream while piece i-1 compresses; piece i decodes as soon as it is
// compressed (W = 1) or its exchange landed (peer exchange), and its
// device->host copy overlaps the next pieces.  The generic (tail) chunks are
// copied in first and run their longer kernel chain on the side stream, off
// the critical path of the last piece.
static fgc_status average_host_impl(fgc_plan* p, fgc_exchange* x, const void* host_grad, int dtype,
                                    const double* weights, void* dev_grad, uint8_t* message, float* dev_out,
                                    float* host_out, uint32_t* flags, void* stream, bool* started);

extern "C" fgc_status fgc_average_host(fgc_plan* p, fgc_exchange* x, const void* host_grad, int dtype,
                                       const double* weights, void* dev_grad, uint8_t* message, float* dev_out,
                                       float* host_out, uint32_t* flags, void* stream) {
  bool started = false;
  const fgc_status st = average_host_impl(p, x, host_grad, dtype, weights, dev_grad, message, dev_out, host_out,
                                          flags, stream, &started);
  if (st != FGC_OK && started && x) exchange_poison(x);
  return st;
}

static fgc_status average_host_impl(fgc_plan* p, fgc_exchange* x, const void* host_grad, int dtype,
                                    const double* weights, void* dev_grad, uint8_t* message, float* dev_out,
                                    float* host_out, uint32_t* flags, void* stream, bool* started) {
  if (!p || !host_grad || !dev_grad || !dev_out || !host_out || !flags) {
    set_error("null argument");
    return FGC_ERR_INVALID;
  }
  FGC_TRY(check_mode(p));
  FGC_TRY(check_signal(dev_grad, dtype));
  FGC_TRY(check_out(dev_out));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int W = 1, me = 0;
  uint32_t* counter = nullptr;
  uint64_t* step = nullptr;
  uint64_t mb = p->msg_bytes;
  if (x) {
    if (!exchange_ready(x)) return exchange_not_ready(x);
    exchange_counters(x, &counter, &step, &W, &me, &mb);
    if (mb != p->msg_bytes) { set_error("exchange sized for another plan"); return FGC_ERR_INVALID; }
  } else if (!message) {
    set_error("single-rank host averaging needs a message buffer");
    return FGC_ERR_INVALID;
  }
  Weights w;
  FGC_TRY(fill_weights(weights, W, w));
  const uint32_t Pmax = exchange_max_pieces();
  const bool energy = p->desc.mode == FGC_MODE_ENERGY;
  uint32_t P = 8;
  if (const char* e = getenv("FGC_HOST_PIECES")) P = (uint32_t)std::max(1, atoi(e));
  P = (energy || !p->fused_count) ? 0 : std::min(std::min(P, Pmax), p->fused_count);
  if (!p->h2d) {
    FGC_CUDA(cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking));
    FGC_CUDA(cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking));
    FGC_CUDA(cudaEventCreateWithFlags(&p->ev_step, cudaEventDisableTiming));
  }
  while (p->ev_h.size() < P + 1) {
    cudaEvent_t a, b, c;
    FGC_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    FGC_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    FGC_CUDA(cudaEventCreateWithFlags(&c, cudaEventDisableTiming));
    p->ev_h.push_back(a);
    p->ev_c2.push_back(b);
    p->ev_d.push_back(c);
  }
  const bool overlap_steps = !getenv("FGC_HOST_SERIAL");
  while (p->ev_cin.size() < Pmax + 1) {
    cudaEvent_t a;
    FGC_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    p->ev_cin.push_back(a);
  }
  int k = 0;
  uint32_t tval = 0;
  uint8_t* gathered = message;
  if (x) {
    k = (int)(*step & 1);
    tval = (uint32_t)(*step + 1);
    FGC_TRY(fgc_exchange_message(x, k, &message, &gathered));
  }
  *started = true;
  const size_t esz = dtype == FGC_DTYPE_F64 ? 8 : 4;
  auto h2d = [&](uint64_t lo, uint64_t hi) {
    return cudaMemcpyAsync(static_cast<uint8_t*>(dev_grad) + lo * esz, static_cast<const uint8_t*>(host_grad) + lo * esz,
                           (hi - lo) * esz, cudaMemcpyHostToDevice, p->h2d);
  };
  auto d2h = [&](uint64_t lo, uint64_t hi) {
    return cudaMemcpyAsync(host_out + lo, dev_out + lo, (hi - lo) * sizeof(float), cudaMemcpyDeviceToHost, p->d2h);
  };
  // The copy-out stream follows the work already on s.  The copy-in of a
  // piece waits only until the previous call's compress has read that piece
  // of dev_grad (scratch of this call sequence), so consecutive steps
  // overlap: step e+1's host->device copies run while step e's results are
  // still copied out (the two directions of PCIe at once).  FGC_HOST_SERIAL=1
  // makes the copy-in wait for all earlier work on s instead.
  FGC_CUDA(cudaEventRecord(p->ev_step, s));
  if (!overlap_steps) FGC_CUDA(cudaStreamWaitEvent(p->h2d, p->ev_step, 0));
  FGC_CUDA(cudaStreamWaitEvent(p->d2h, p->ev_step, 0));

  // generic chunks (all of them for energy mode / plans without fused
  // chunks): elements [g_lo, n), message bytes [m_lo, end), slot P (tail slot
  // of the exchange)
  // (energy mode runs the whole message here, fused chunks included)
  const bool pieces = !energy && p->fused_count;
  const bool generic = energy || p->classes.size() > (p->fused_count ? 1u : 0u);
  const uint64_t g_lo = pieces ? p->chunks[p->fused_first + p->fused_count - 1].in_off +
                                     p->chunks[p->fused_first + p->fused_count - 1].len
                               : 0;
  const uint64_t m_lo = pieces ? p->seg_off[p->fused_first + p->fused_count] : 0;
  cudaStream_t g = P ? p->side : s;
  if (generic) {
    if (overlap_steps) FGC_CUDA(cudaStreamWaitEvent(p->h2d, p->ev_cin[Pmax], 0));
    FGC_CUDA(h2d(g_lo, p->desc.n));
    FGC_CUDA(cudaEventRecord(p->ev_h[P], p->h2d));
    FGC_CUDA(cudaStreamWaitEvent(g, p->ev_h[P], 0));
    if (energy) FGC_TRY(energy_compress(p, dev_grad, dtype, nullptr, message, nullptr, flags, g));
    else FGC_TRY(compress_range(p, dev_grad, dtype, message, flags, g, 0, 0, true));
    FGC_CUDA(cudaEventRecord(p->ev_cin[Pmax], g));
    if (x) {
      FGC_CUDA(cudaEventRecord(p->ev_c2[P], g));
      if (energy)
        FGC_TRY(exchange_publish_used(x, k, p->d_chunks, p->n_chunks, p->q.n_bits, p->ev_c2[P], tval, (int)Pmax));
      else
        FGC_TRY(exchange_publish_event(x, k, m_lo, p->msg_bytes - m_lo, p->ev_c2[P], tval, (int)Pmax));
      FGC_TRY(exchange_wait(x, g, (int)Pmax, tval));
    }
    FGC_TRY(decode_range(p, gathered, W, p->msg_bytes, w, dev_out, g, energy ? p->fused_first : 0,
                         energy ? p->fused_count : 0, true));
    FGC_CUDA(cudaEventRecord(p->ev_d[P], g));
  }
  // fused pieces: elements [chunk f[i] .. chunk f[i+1])
  std::vector<uint32_t> f(P + 1);
  // half-size first and last pieces: shorter pipeline fill (first copy-in)
  // and drain (last copy-out)
  const bool ramp = P >= 3 && p->fused_count >= 2 * P && !getenv("FGC_HOST_NO_RAMP");
  // ramp: first piece 1/2, last piece 1/tq of the middle pieces (in units of 1/tq)
  uint64_t tq = 8;                                     // measured: 2.615 ms (8) vs 2.62-2.66 (2, 4) at 25.6M
  if (const char* e = getenv("FGC_HOST_TAIL")) tq = (uint64_t)std::max(2, atoi(e));
  for (uint32_t i = 0; i <= P; ++i) {
    uint64_t u = i, un = P ? P : 1;
    if (ramp) {
      un = tq / 2 + tq * (P - 2) + 1;
      u = i == 0 ? 0 : i == P ? un : tq / 2 + tq * (i - 1);
    }
    f[i] = p->fused_first + (uint32_t)((uint64_t)p->fused_count * u / un);
  }
  auto elem_lo = [&](uint32_t i) -> uint64_t { return p->chunks[f[i]].in_off; };
  auto elem_hi = [&](uint32_t i) -> uint64_t { return i + 1 == P ? g_lo : p->chunks[f[i + 1]].in_off; };
  auto seg_hi = [&](uint32_t i) -> uint64_t { return i + 1 == P ? m_lo : p->seg_off[f[i + 1]]; };
  exchange_trace(p->h2d, "start");
  for (uint32_t i = 0; i < P; ++i) {
    if (overlap_steps) FGC_CUDA(cudaStreamWaitEvent(p->h2d, p->ev_cin[i], 0));
    FGC_CUDA(h2d(elem_lo(i), elem_hi(i)));
    FGC_CUDA(cudaEventRecord(p->ev_h[i], p->h2d));
    exchange_trace(p->h2d, "h2d");
  }
  for (uint32_t i = 0; i < P; ++i) {
    FGC_CUDA(cudaStreamWaitEvent(s, p->ev_h[i], 0));
    FGC_TRY(compress_range(p, dev_grad, dtype, message, flags, s, f[i], f[i + 1] - f[i], false));
    FGC_CUDA(cudaEventRecord(p->ev_cin[i], s));
    if (x) {
      FGC_CUDA(cudaEventRecord(p->ev_c2[i], s));
      FGC_TRY(exchange_publish_event(x, k, p->seg_off[f[i]], seg_hi(i) - p->seg_off[f[i]], p->ev_c2[i], tval,
                                     (int)i));
    } else {
      // W = 1: decode this piece right away so its copy-out overlaps the next pieces
      FGC_TRY(decode_range(p, message, 1, p->msg_bytes, w, dev_out, s, f[i], f[i + 1] - f[i], false));
      FGC_CUDA(cudaEventRecord(p->ev_d[i], s));
      exchange_trace(s, "dec");
    }
  }
  if (x) {
    for (uint32_t i = 0; i < P; ++i) {
      FGC_TRY(exchange_wait(x, s, (int)i, tval));
      FGC_TRY(decode_range(p, gathered, W, p->msg_bytes, w, dev_out, s, f[i], f[i + 1] - f[i], false));
      FGC_CUDA(cudaEventRecord(p->ev_d[i], s));
    }
  }
  // copy-out in completion order: the generic chunks finish first
  if (generic) {
    FGC_CUDA(cudaStreamWaitEvent(p->d2h, p->ev_d[P], 0));
    FGC_CUDA(d2h(g_lo, p->desc.n));
    exchange_trace(p->d2h, "d2h-tail");
  }
  for (uint32_t i = 0; i < P; ++i) {
    FGC_CUDA(cudaStreamWaitEvent(p->d2h, p->ev_d[i], 0));
    FGC_CUDA(d2h(elem_lo(i), elem_hi(i)));
    exchange_trace(p->d2h, "d2h");
  }
  FGC_CUDA(cudaEventRecord(p->ev_step, p->d2h));
  FGC_CUDA(cudaStreamWaitEvent(s, p->ev_step, 0));
  if (x) {
    FGC_TRY(exchange_join(x, s));
    *step += 1;
  }
  (void)counter;
  (void)me;
  return FGC_OK;
}

extern "C" fgc_status fgc_profile_fused_compress(fgc_plan* p, const void* grad, int dtype, uint8_t* message,
                                                 uint32_t* flags, void* stream, uint64_t* alg_bytes) {
  if (!p || !grad || !message || !flags || !alg_bytes) { set_error("null argument"); return FGC_ERR_INVALID; }
  FGC_TRY(check_mode(p));
  FGC_TRY(check_signal(grad, dtype));
  *alg_bytes = 0;
  if (!p->fused_count || p->desc.mode != FGC_MODE_COUNT) return FGC_OK;
  const uint32_t f0 = p->fused_first, f1 = f0 + p->fused_count;
  const uint64_t esz = dtype == FGC_DTYPE_F64 ? 8 : 4;
  *alg_bytes = esz * 65536ull * p->fused_count + (p->seg_off[f1] - p->seg_off[f0]);
  return launch_fused_compress(p->fused, p->d_chunks, f0, p->fused_count, grad, dtype, p->desc.half_pass, p->q,
                               message, flags, p->d_spec, static_cast<cudaStream_t>(stream));
}

extern "C" const char* fgc_last_error(void) { return g_last_error.c_str(); }
extern "C" int fgc_version(void) { return 0x000100; }
extern "C" uint64_t fgc_kernel_launches(void) { return g_launches.load(); }
