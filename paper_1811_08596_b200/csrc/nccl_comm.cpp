// NCCL plumbing for the compressed average over NVLink / NVSwitch: the
// exchange the reference only simulates by value (simulator.py:529-535).
// One process per GPU; the unique id is bootstrapped by the caller (e.g. a
// torch.distributed broadcast).  Messages have a-priori fixed capacity in
// count mode, so one ncclAllGather moves every rank's message with no size
// pre-exchange.
#include <cuda_runtime.h>
#include <nccl.h>
#include <string.h>

#include <string>

#include "fgc_internal.h"

namespace {

fgc_status nccl_fail(ncclResult_t r, const char* what) {
  fgc::set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return FGC_ERR_NCCL;
}

}  // namespace

extern "C" fgc_status fgc_nccl_unique_id(uint8_t id_out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id_out, &id, 128);
  return FGC_OK;
}

extern "C" fgc_status fgc_nccl_comm_create(const uint8_t id_in[128], int nranks, int rank, void** comm_out) {
  if (!comm_out || nranks < 1 || rank < 0 || rank >= nranks) {
    fgc::set_error("bad communicator arguments");
    return FGC_ERR_INVALID;
  }
  ncclUniqueId id;
  memcpy(&id, id_in, 128);
  ncclComm_t comm;
  ncclResult_t r = ncclCommInitRank(&comm, nranks, id, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm_out = comm;
  return FGC_OK;
}

extern "C" fgc_status fgc_nccl_comm_destroy(void* comm) {
  if (!comm) return FGC_OK;
  ncclResult_t r = ncclCommDestroy(static_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return FGC_OK;
}

extern "C" fgc_status fgc_allgather(void* comm, const uint8_t* send, uint8_t* recv, uint64_t bytes, void* stream) {
  if (!comm || !send || !recv) {
    fgc::set_error("null argument");
    return FGC_ERR_INVALID;
  }
  ncclResult_t r = ncclAllGather(send, recv, bytes, ncclUint8, static_cast<ncclComm_t>(comm),
                                 static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
  return FGC_OK;
}

extern "C" fgc_status fgc_allreduce_sum_f32(void* comm, float* data, uint64_t count, void* stream) {
  if (!comm || !data) {
    fgc::set_error("null argument");
    return FGC_ERR_INVALID;
  }
  ncclResult_t r = ncclAllReduce(data, data, count, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm),
                                 static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  return FGC_OK;
}
