// Peer-memory exchange for the compressed average: the allgather of
// simulator.py:529-535 done by the copy engines over NVLink / NVSwitch, so it
// overlaps the codec kernels without taking SMs (NCCL's allgather kernels
// compete with the fused kernels for every SM; measured slower when
// pipelined).
//
// Every rank owns two gather buffers (double-buffered by step parity), each
// nranks * message_bytes, rank-major: rank b's message for the step lives at
// G[k] + b * message_bytes on every rank.  A rank compresses straight into its
// own slot, and after each piece (whole waves of fused chunks) its copy
// streams push that piece into the same slot of every peer's buffer
// (cudaMemcpyAsync peer-to-peer through CUDA IPC mappings) and then bump the
// rank's flag word in every peer's flag array (stream memory operation,
// ordered after the copy).  Before decoding piece i a rank waits on its own
// flag array until every peer's counter reached the piece.
//
// Reuse safety: a rank's compress of step e+1 (into buffer (e+1)&1) follows
// its decode of step e on the same stream, and a peer's push of step e+1 into
// our buffer (e+1)&1 follows the peer's decode of step e, which waited for our
// push of step e, which followed our decode of step e-1 -- the last reader of
// that buffer.  So two buffers and monotonic counters are enough.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "fgc_internal.h"

namespace {

typedef CUresult (*WriteValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

constexpr int kMaxRanks = 64;
constexpr int kMaxPieces = 32;                         // fused pieces; flag index kMaxPieces = generic chunks
constexpr int kFlagStride = kMaxPieces + 1;
constexpr int kCopyStreams = 4;                        // per publisher class (fused pieces / generic chunks)
// Per-chunk completion tags of the in-kernel transports, after the flag words
// in the same (IPC-exported) allocation: region b (nranks regions of
// 2 * kTagChunks words) holds rank b's tags.
//   direct reads:  tags_b[c] in rank b's own memory, set once b's compress
//                  kernel wrote chunk c's segment (the readers poll it remotely)
//   kernel pushes: tags_b[2c + r] in every receiver's memory, set by CTA r of
//                  b's compress cluster once it stored its half of the segment
//                  into the receiver's gather buffer (the receiver polls locally)
constexpr uint32_t kFlagWords = kMaxRanks * kFlagStride;
constexpr uint32_t kTagChunks = 1u << 14;

struct MemOps {
  WriteValueFn write = nullptr;
  WaitValueFn wait = nullptr;
  bool ok = false;
};

const MemOps& memops() {
  static MemOps m = [] {
    MemOps r;
    void* w = nullptr;
    void* v = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &v, cudaEnableDefault, &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && w && v) {
      r.write = reinterpret_cast<WriteValueFn>(w);
      r.wait = reinterpret_cast<WaitValueFn>(v);
      r.ok = true;
    }
    cudaGetLastError();
    return r;
  }();
  return m;
}

// Kernel fallbacks of the two stream memory operations.
__global__ void k_flag_write(uint32_t* addr, uint32_t value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(addr), "r"(value) : "memory");
}
__global__ void k_flag_wait(const uint32_t* flags, int nranks, int me, uint32_t target, int stride) {
  const int a = threadIdx.x;
  if (a >= nranks || a == me) return;
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + a * stride) : "memory");
    if ((int32_t)(v - target) >= 0) break;
    __nanosleep(256);
  }
}

// Variable-length push (energy mode): every chunk segment of this rank's
// message is copied to every peer only up to its used bytes -- the header,
// the bitmap and the codes the segment's own nnz says it holds (rounded to 16
// bytes, what the decode reads) -- instead of the full-capacity segment.  The
// sizes live on the device, so SMs copy (one CTA per chunk, 16-byte stores
// into the peers' IPC-mapped buffers); the last CTA to finish sets the flag
// in every peer after a system-scope fence.
struct PushPeers {
  uint8_t* dst[kMaxRanks];             // the peer's copy of this rank's slot
  uint32_t* flag[kMaxRanks];           // this rank's flag for the piece in the peer
  int n;
};

__global__ void k_push_used(const fgc::ChunkInfo* chunks, uint32_t n_chunks, const uint8_t* src, int N, PushPeers pp,
                            uint32_t value, uint32_t* done, unsigned long long* pushed) {
  const fgc::ChunkInfo ci = chunks[blockIdx.x];
  const uint8_t* seg = src + ci.seg_off;
  const uint32_t nnz = *reinterpret_cast<const uint32_t*>(seg);
  const uint64_t code_bytes = 16ull * (((uint64_t)nnz * (uint32_t)N + 127u) / 128u);
  const uint64_t cap = ci.code_off + 4ull * ((ci.code_cap + 3u) & ~3u);
  const uint64_t bytes = min((uint64_t)ci.code_off + code_bytes, cap);
  const uint4* s4 = reinterpret_cast<const uint4*>(seg);
  const uint32_t n4 = (uint32_t)(bytes / 16);
  for (int p = 0; p < pp.n; ++p) {
    uint4* d4 = reinterpret_cast<uint4*>(pp.dst[p] + ci.seg_off);
    for (uint32_t e = threadIdx.x; e < n4; e += blockDim.x) d4[e] = s4[e];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(pushed, (unsigned long long)bytes * pp.n);
    if (atomicAdd(done, 1u) == n_chunks - 1) {
      __threadfence_system();
      for (int p = 0; p < pp.n; ++p)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pp.flag[p]), "r"(value) : "memory");
      *done = 0u;                                       // ready for the next step's launch
    }
  }
}

}  // namespace

struct fgc_exchange {
  int nranks = 0, rank = 0;
  uint64_t msg_bytes = 0;
  uint8_t* gbuf = nullptr;            // 2 * nranks * msg_bytes (buffer k at k * nranks * msg_bytes)
  uint32_t* flags = nullptr;          // [kMaxRanks][kFlagStride] step counters written by the peers
  uint32_t* pcnt = nullptr;           // [kMaxPieces] completed chunks per piece (this rank's compress)
  uint32_t* push_done = nullptr;      // k_push_used: finished chunk CTAs of the running launch
  unsigned long long* pushed = nullptr;   // bytes pushed by k_push_used (diagnostics)
  uint8_t* peer_gbuf[kMaxRanks] = {};
  uint32_t* peer_flags[kMaxRanks] = {};
  // device tables (filled at open): [0, 2R) where rank b's message of buffer
  // k lives in b's memory (direct reads); [2R, 3R) rank b's tag region in b's
  // memory; [3R, 4R) rank b's tag region in this rank's memory; [4R, 6R) this
  // rank's slot of buffer k in peer p's memory (kernel pushes, peers only);
  // [6R, 7R) this rank's tag region in peer p's memory (peers only)
  void** d_tab = nullptr;
  int xmode = 0;                      // FGC_EXCHANGE_DIRECT: 0 copy-engine pushes, 1 direct reads, 2 kernel pushes
  cudaStream_t cs[2][kCopyStreams] = {};
  std::vector<cudaEvent_t> ev;        // per piece: compress done on the caller's stream
  cudaEvent_t ev_copies = nullptr;
  uint32_t counter = 0;               // pieces published so far
  uint32_t pexp[kMaxPieces] = {};     // host copy of what pcnt[i] reaches once the queued compresses finish
  uint64_t step = 0;
  bool opened = false;
  bool poisoned = false;              // a step failed mid-way: counters no longer agree with the peers
};

using fgc::set_error;

static fgc_status cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return FGC_ERR_CUDA;
}
#define XC(call)                                          \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
  } while (0)

extern "C" fgc_status fgc_exchange_create(int nranks, int rank, uint64_t message_bytes, fgc_exchange** out) {
  if (!out || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || !message_bytes) {
    set_error("bad exchange arguments");
    return FGC_ERR_INVALID;
  }
  fgc_exchange* x = new fgc_exchange();
  x->nranks = nranks;
  x->rank = rank;
  x->msg_bytes = message_bytes;
  cudaError_t e = cudaMalloc(&x->gbuf, 2ull * nranks * message_bytes);
  const size_t fwords = kFlagWords + (size_t)nranks * 2 * kTagChunks;
  if (e == cudaSuccess) e = cudaMalloc(&x->flags, sizeof(uint32_t) * fwords);
  if (e == cudaSuccess) e = cudaMemset(x->flags, 0, sizeof(uint32_t) * fwords);
  if (e == cudaSuccess) e = cudaMalloc(&x->d_tab, sizeof(void*) * 7 * kMaxRanks);
  if (const char* d = getenv("FGC_EXCHANGE_DIRECT")) x->xmode = (d[0] == '1') ? 1 : (d[0] == '2') ? 2 : 0;
  if (e == cudaSuccess) e = cudaMalloc(&x->pcnt, sizeof(uint32_t) * kMaxPieces);
  if (e == cudaSuccess) e = cudaMemset(x->pcnt, 0, sizeof(uint32_t) * kMaxPieces);
  if (e == cudaSuccess) e = cudaMalloc(&x->push_done, sizeof(uint32_t) + sizeof(unsigned long long) * 2);
  if (e == cudaSuccess) e = cudaMemset(x->push_done, 0, sizeof(uint32_t) + sizeof(unsigned long long) * 2);
  if (e == cudaSuccess) x->pushed = reinterpret_cast<unsigned long long*>(x->push_done + 2);
  if (e == cudaSuccess) e = cudaMemset(x->gbuf, 0, 2ull * nranks * message_bytes);
  for (int c = 0; c < 2; ++c)
    for (int i = 0; i < kCopyStreams && e == cudaSuccess; ++i)
      e = cudaStreamCreateWithFlags(&x->cs[c][i], cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x->ev_copies, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fgc_exchange_destroy(x);
    return cuda_fail(e, "exchange allocation");
  }
  *out = x;
  return FGC_OK;
}

extern "C" fgc_status fgc_exchange_handles(fgc_exchange* x, uint8_t handles_out[128]) {
  if (!x || !handles_out) return FGC_ERR_INVALID;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  cudaIpcMemHandle_t hg, hf;
  XC(cudaIpcGetMemHandle(&hg, x->gbuf));
  XC(cudaIpcGetMemHandle(&hf, x->flags));
  memcpy(handles_out, &hg, 64);
  memcpy(handles_out + 64, &hf, 64);
  return FGC_OK;
}

extern "C" fgc_status fgc_exchange_open(fgc_exchange* x, const uint8_t* all_handles) {
  if (!x || !all_handles) return FGC_ERR_INVALID;
  for (int a = 0; a < x->nranks; ++a) {
    if (a == x->rank) {
      x->peer_gbuf[a] = x->gbuf;
      x->peer_flags[a] = x->flags;
      continue;
    }
    cudaIpcMemHandle_t hg, hf;
    memcpy(&hg, all_handles + 128ull * a, 64);
    memcpy(&hf, all_handles + 128ull * a + 64, 64);
    void* pg = nullptr;
    void* pf = nullptr;
    XC(cudaIpcOpenMemHandle(&pg, hg, cudaIpcMemLazyEnablePeerAccess));
    XC(cudaIpcOpenMemHandle(&pf, hf, cudaIpcMemLazyEnablePeerAccess));
    x->peer_gbuf[a] = static_cast<uint8_t*>(pg);
    x->peer_flags[a] = static_cast<uint32_t*>(pf);
  }
  // tables of the in-kernel transports (rank b compresses buffer k's message
  // into its own slot b of its own buffer k)
  const int R = kMaxRanks;
  const void* tab[7 * kMaxRanks] = {};
  const uint64_t treg = 2ull * kTagChunks;
  for (int k = 0; k < 2; ++k)
    for (int b = 0; b < x->nranks; ++b)
      tab[k * R + b] = x->peer_gbuf[b] + ((uint64_t)k * x->nranks + b) * x->msg_bytes;
  for (int b = 0; b < x->nranks; ++b) {
    tab[2 * R + b] = x->peer_flags[b] + kFlagWords + b * treg;
    tab[3 * R + b] = x->flags + kFlagWords + b * treg;
  }
  int np = 0;
  for (int b = 0; b < x->nranks; ++b) {
    if (b == x->rank) continue;
    for (int k = 0; k < 2; ++k)
      tab[4 * R + k * R + np] = x->peer_gbuf[b] + ((uint64_t)k * x->nranks + x->rank) * x->msg_bytes;
    tab[6 * R + np] = x->peer_flags[b] + kFlagWords + x->rank * treg;
    ++np;
  }
  XC(cudaMemcpy(x->d_tab, tab, sizeof(tab), cudaMemcpyHostToDevice));
  x->opened = true;
  return FGC_OK;
}

extern "C" void fgc_exchange_destroy(fgc_exchange* x) {
  if (!x) return;
  cudaDeviceSynchronize();
  for (int a = 0; a < x->nranks; ++a) {
    if (a == x->rank) continue;
    if (x->peer_gbuf[a]) cudaIpcCloseMemHandle(x->peer_gbuf[a]);
    if (x->peer_flags[a]) cudaIpcCloseMemHandle(x->peer_flags[a]);
  }
  for (cudaEvent_t e : x->ev) cudaEventDestroy(e);
  if (x->ev_copies) cudaEventDestroy(x->ev_copies);
  for (int c = 0; c < 2; ++c)
    for (int i = 0; i < kCopyStreams; ++i)
      if (x->cs[c][i]) cudaStreamDestroy(x->cs[c][i]);
  cudaFree(x->gbuf);
  cudaFree(x->flags);
  cudaFree(x->pcnt);
  cudaFree(x->push_done);
  cudaFree(x->d_tab);
  delete x;
}

extern "C" fgc_status fgc_exchange_message(fgc_exchange* x, int parity, uint8_t** message, uint8_t** gathered) {
  if (!x) return FGC_ERR_INVALID;
  uint8_t* g = x->gbuf + (uint64_t)(parity & 1) * x->nranks * x->msg_bytes;
  if (gathered) *gathered = g;
  if (message) *message = g + (uint64_t)x->rank * x->msg_bytes;
  return FGC_OK;
}

namespace fgc {

// Optional timeline (FGC_EXCHANGE_TRACE=1): timing events recorded at the
// publish / wait points of the last step, read back with
// fgc_debug_exchange_trace (milliseconds relative to the first event).
static std::vector<cudaEvent_t> g_trace_ev;
static std::vector<std::string> g_trace_tag;
static bool trace_on() {
  static int on = [] { const char* e = getenv("FGC_EXCHANGE_TRACE"); return e && e[0] == '1'; }();
  return on;
}
void exchange_trace(cudaStream_t s, const char* tag) {
  if (!trace_on()) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, s);
  g_trace_ev.push_back(e);
  g_trace_tag.push_back(tag);
}

// Push bytes [lo, lo + bytes) of this rank's slot in buffer k to every peer
// on copy stream `cs`, then set flag `fi` of this rank in every peer to value.
static fgc_status push(fgc_exchange* x, cudaStream_t cs, int k, uint64_t lo, uint64_t bytes, int fi,
                       uint32_t value) {
  const uint64_t off = (uint64_t)k * x->nranks * x->msg_bytes + (uint64_t)x->rank * x->msg_bytes + lo;
  const MemOps& m = memops();
  for (int a = 0; a < x->nranks; ++a) {
    if (a == x->rank) continue;
    if (bytes) XC(cudaMemcpyAsync(x->peer_gbuf[a] + off, x->gbuf + off, bytes, cudaMemcpyDeviceToDevice, cs));
  }
  for (int a = 0; a < x->nranks; ++a) {
    if (a == x->rank) continue;
    uint32_t* dst = x->peer_flags[a] + x->rank * kFlagStride + fi;
    if (m.ok) {
      if (m.write((CUstream)cs, (CUdeviceptr)dst, value, 0) != CUDA_SUCCESS) {
        set_error("cuStreamWriteValue32 failed");
        return FGC_ERR_CUDA;
      }
    } else {
      k_flag_write<<<1, 1, 0, cs>>>(dst, value);
      FGC_LAUNCHED(1);
    }
  }
  exchange_trace(cs, fi == kMaxPieces ? "tail-copied" : "piece-copied");
  return FGC_OK;
}

// Push after `ready` (an event on the producing stream) and set flag `fi`
// (default: the generic-chunk slot).
fgc_status exchange_publish_event(fgc_exchange* x, int k, uint64_t lo, uint64_t bytes, cudaEvent_t ready,
                                  uint32_t value, int fi) {
  if (fi < 0) fi = kMaxPieces;
  cudaStream_t cs = x->cs[1][fi % kCopyStreams];
  XC(cudaStreamWaitEvent(cs, ready, 0));
  return push(x, cs, k, lo, bytes, fi, value);
}

// Variable-length publish of the whole message (energy mode) after `ready`:
// k_push_used on a copy stream, flag `fi` (default: the generic-chunk slot).
fgc_status exchange_publish_used(fgc_exchange* x, int k, const ChunkInfo* d_chunks, uint32_t n_chunks, int n_bits,
                                 cudaEvent_t ready, uint32_t value, int fi) {
  if (fi < 0) fi = kMaxPieces;
  cudaStream_t cs = x->cs[1][fi % kCopyStreams];
  XC(cudaStreamWaitEvent(cs, ready, 0));
  PushPeers pp{};
  const uint64_t off = (uint64_t)k * x->nranks * x->msg_bytes + (uint64_t)x->rank * x->msg_bytes;
  for (int a = 0; a < x->nranks; ++a) {
    if (a == x->rank) continue;
    pp.dst[pp.n] = x->peer_gbuf[a] + off;
    pp.flag[pp.n] = x->peer_flags[a] + x->rank * kFlagStride + fi;
    ++pp.n;
  }
  if (!pp.n) return FGC_OK;
  k_push_used<<<n_chunks, 256, 0, cs>>>(d_chunks, n_chunks, x->gbuf + off, n_bits, pp, value, x->push_done,
                                        x->pushed);
  FGC_LAUNCHED(1);
  exchange_trace(cs, "used-pushed");
  return FGC_OK;
}

// Fused piece i: the copy stream waits (stream memory operation) until the
// running compress kernel has counted `count_target` finished chunks of the
// piece, then pushes -- no kernel boundary between pieces.
fgc_status exchange_publish_piece(fgc_exchange* x, int k, uint32_t i, uint64_t lo, uint64_t bytes,
                                  uint32_t count_target, uint32_t value) {
  const MemOps& m = memops();
  if (!m.ok) {
    set_error("stream memory operations unavailable");
    return FGC_ERR_UNSUPPORTED;
  }
  cudaStream_t cs = x->cs[0][i % kCopyStreams];
  if (m.wait((CUstream)cs, (CUdeviceptr)(x->pcnt + i), count_target, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
    set_error("cuStreamWaitValue32 failed");
    return FGC_ERR_CUDA;
  }
  return push(x, cs, k, lo, bytes, (int)i, value);
}

// Make `s` wait until every peer's flag `fi` reached `value`.
fgc_status exchange_wait(fgc_exchange* x, cudaStream_t s, int fi, uint32_t value) {
  const MemOps& m = memops();
  if (m.ok) {
    for (int a = 0; a < x->nranks; ++a) {
      if (a == x->rank) continue;
      CUresult r = m.wait((CUstream)s, (CUdeviceptr)(x->flags + a * kFlagStride + fi), value,
                          CU_STREAM_WAIT_VALUE_GEQ);
      if (r != CUDA_SUCCESS) {
        set_error("cuStreamWaitValue32 failed");
        return FGC_ERR_CUDA;
      }
    }
  } else {
    k_flag_wait<<<1, 64, 0, s>>>(x->flags + fi, x->nranks, x->rank, value, kFlagStride);
    FGC_LAUNCHED(1);
  }
  return FGC_OK;
}

PieceCounter exchange_counter(fgc_exchange* x, uint32_t first, uint32_t per) {
  PieceCounter pc;
  pc.cnt = x->pcnt;
  pc.first = first;
  pc.per = per;
  return pc;
}

PieceWait exchange_piece_wait(fgc_exchange* x, uint32_t first, uint32_t per, uint32_t target) {
  PieceWait pw;
  pw.flags = x->flags;
  pw.stride = kFlagStride;
  pw.first = first;
  pw.per = per;
  pw.target = target;
  pw.nranks = x->nranks;
  pw.me = x->rank;
  return pw;
}

int exchange_transport(const fgc_exchange* x, uint32_t chunk_end) {
  return (x->nranks > 1 && chunk_end <= kTagChunks) ? x->xmode : 0;
}

// Direct reads: the compress kernel releases tags_me[c] in this rank's own
// memory at system scope; the decode reads message b from mtab[b] once
// rank b's tags_b[c] (remote) reached the step's tag.
void exchange_direct(fgc_exchange* x, int k, uint32_t tag, PieceCounter& pc, PieceWait& pw) {
  const int R = kMaxRanks;
  pc = PieceCounter();
  pc.done = x->flags + kFlagWords + (uint64_t)x->rank * 2 * kTagChunks;
  pc.tag = tag;
  pc.sys = 1;
  pw = PieceWait();
  pw.nranks = x->nranks;
  pw.me = x->rank;
  pw.target = tag;
  pw.done = pc.done;                  // own chunk: released by the compress grid this decode depends on
  pw.tag = tag;
  pw.mtab = reinterpret_cast<const uint8_t* const*>(x->d_tab + (k & 1) * R);
  pw.dtab = reinterpret_cast<const uint32_t* const*>(x->d_tab + 2 * R);
  pw.tstride = 1;
}

// Kernel pushes: each CTA of the compress cluster stores its half of the
// chunk's segment into every peer's gather buffer and releases tags_me[2c+r]
// there; the decode reads the local gather buffer once every peer's two tags
// of the chunk (local memory) reached the step's tag.  The caller sets the
// own-chunk done/tag pair (the decode's programmatic-dependency wait).
void exchange_kpush(fgc_exchange* x, int k, uint32_t tag, PieceCounter& pc, PieceWait& pw) {
  const int R = kMaxRanks;
  pc.pdst = reinterpret_cast<uint8_t* const*>(x->d_tab + 4 * R + (k & 1) * R);
  pc.ptag = reinterpret_cast<uint32_t* const*>(x->d_tab + 6 * R);
  pc.npeers = (uint32_t)(x->nranks - 1);
  pc.pval = tag;
  pw.nranks = x->nranks;
  pw.me = x->rank;
  pw.target = tag;
  pw.dtab = reinterpret_cast<const uint32_t* const*>(x->d_tab + 3 * R);
  pw.tstride = 2;
}

uint32_t exchange_max_pieces() { return kMaxPieces; }

// The counter value piece i reaches once a compress that adds `chunks`
// finished chunks to it completes (steps that bypass the counters -- the
// host-buffer step -- leave the targets alone).
uint32_t exchange_piece_target(fgc_exchange* x, uint32_t i, uint32_t chunks) { return x->pexp[i] += chunks; }

// Join the copy streams back into s (the caller's step is complete only when
// its pushes are).
fgc_status exchange_join(fgc_exchange* x, cudaStream_t s) {
  for (int c = 0; c < 2; ++c)
    for (int i = 0; i < kCopyStreams; ++i) {
      XC(cudaEventRecord(x->ev_copies, x->cs[c][i]));
      XC(cudaStreamWaitEvent(s, x->ev_copies, 0));
    }
  return FGC_OK;
}

fgc_status exchange_events(fgc_exchange* x, uint32_t P, std::vector<cudaEvent_t>** ev) {
  while (x->ev.size() < P + 3) {
    cudaEvent_t e;
    XC(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    x->ev.push_back(e);
  }
  *ev = &x->ev;
  return FGC_OK;
}

void exchange_counters(fgc_exchange* x, uint32_t** counter, uint64_t** step, int* nranks, int* rank,
                       uint64_t* msg_bytes) {
  *counter = &x->counter;
  *step = &x->step;
  *nranks = x->nranks;
  *rank = x->rank;
  *msg_bytes = x->msg_bytes;
}

bool exchange_ready(const fgc_exchange* x) { return x && x->opened && !x->poisoned; }
void exchange_poison(fgc_exchange* x) {
  if (x) x->poisoned = true;
}
bool exchange_poisoned(const fgc_exchange* x) { return x && x->poisoned; }

}  // namespace fgc

extern "C" int fgc_debug_exchange_trace(char* out, int cap) {
  using namespace fgc;
  std::string r;
  for (size_t i = 0; i < g_trace_ev.size(); ++i) {
    float ms = 0.f;
    cudaEventSynchronize(g_trace_ev[i]);
    cudaEventElapsedTime(&ms, g_trace_ev[0], g_trace_ev[i]);
    r += g_trace_tag[i] + " " + std::to_string(ms) + "\n";
  }
  for (cudaEvent_t e : g_trace_ev) cudaEventDestroy(e);
  g_trace_ev.clear();
  g_trace_tag.clear();
  const int n = (int)std::min<size_t>(r.size(), (size_t)cap - 1);
  memcpy(out, r.data(), n);
  out[n] = 0;
  return n;
}

extern "C" unsigned long long fgc_debug_exchange_pushed(fgc_exchange* x) {
  unsigned long long v = 0;
  if (x && x->pushed) cudaMemcpy(&v, x->pushed, sizeof(v), cudaMemcpyDeviceToHost);
  return v;
}
