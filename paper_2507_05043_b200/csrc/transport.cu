// Inter-stage activation transport: NCCL 2.28 point-to-point over NVLink, plus
// the link-throttle gate that replays the reference's virtual link timing
// (transport.py:199-200, engine.py:347-372 / 546-559) in wall time.
//
// The host drains the reference's unchanged LinkQueue (transport.py:70-160);
// every Chunk it yields becomes exactly one ncclSend on the source stage's link
// stream and one ncclRecv on the destination's, covering the chunk's byte range
// [offset, offset + size) of the payload buffer -- so chunk boundaries on the
// wire are bit-identical to the virtual engine's.
#include <nccl.h>

#include "common.cuh"
#include "pl_internal.h"

namespace pl {

static int nccl_err(ncclResult_t r, const char* what) {
  return set_error(PL_ERR_PROTOCOL, "%s: %s", what, ncclGetErrorString(r));
}

__global__ void record_globaltimer_kernel(uint64_t* dst) { *dst = globaltimer_ns(); }

// One thread spins on %globaltimer: blocks the stream (and only this stream)
// until the emulated link would have delivered the bytes.
__global__ void gate_kernel(const uint64_t* t0, uint64_t offset_ns) {
  const uint64_t deadline = *t0 + offset_ns;
  while (globaltimer_ns() < deadline) {
    __nanosleep(2000);
  }
}


// Load every kernel of this file into the context now (lazy module loading would
// otherwise load it at first launch, which can wait on a spinning NCCL kernel).
template <typename K>
static int preload_one(K k, const char* name) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, k);
  return e == cudaSuccess ? PL_OK : set_cuda_error(e, name);
}

int transport_preload() {
  int rc = preload_one(record_globaltimer_kernel, "record_globaltimer_kernel");
  if (!rc) rc = preload_one(gate_kernel, "gate_kernel");
  return rc;
}

}  // namespace pl

using namespace pl;

extern "C" {

int32_t pl_nccl_version(void) {
  int v = 0;
  ncclGetVersion(&v);
  return v;
}

int32_t pl_nccl_unique_id(uint8_t* id_host, int32_t len) {
  if (!id_host || len < static_cast<int32_t>(sizeof(ncclUniqueId)))
    return set_error(PL_ERR_CONFIG, "unique id buffer must hold %d bytes", (int)sizeof(ncclUniqueId));
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_err(r, "ncclGetUniqueId");
  memcpy(id_host, &id, sizeof(id));
  return PL_OK;
}

int32_t pl_comm_init_rank(const uint8_t* id_host, int32_t nranks, int32_t rank, void** comm) {
  if (!id_host || !comm || nranks < 1 || rank < 0 || rank >= nranks)
    return set_error(PL_ERR_CONFIG, "comm_init_rank: bad arguments");
  ncclUniqueId id;
  memcpy(&id, id_host, sizeof(id));
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return nccl_err(r, "ncclCommInitRank");
  *comm = c;
  return PL_OK;
}

int32_t pl_comm_destroy(void* comm) {
  if (!comm) return PL_OK;
  ncclResult_t r = ncclCommDestroy(static_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return nccl_err(r, "ncclCommDestroy");
  return PL_OK;
}

int32_t pl_p2p_send(void* comm, const void* buf, int64_t bytes, int32_t peer, void* stream) {
  if (!comm || (!buf && bytes > 0) || bytes < 0)
    return set_error(PL_ERR_CONFIG, "p2p_send: bad arguments");
  ncclResult_t r = ncclSend(buf, static_cast<size_t>(bytes), ncclUint8, peer,
                            static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return nccl_err(r, "ncclSend");
  return PL_OK;
}

int32_t pl_p2p_recv(void* comm, void* buf, int64_t bytes, int32_t peer, void* stream) {
  if (!comm || (!buf && bytes > 0) || bytes < 0)
    return set_error(PL_ERR_CONFIG, "p2p_recv: bad arguments");
  ncclResult_t r = ncclRecv(buf, static_cast<size_t>(bytes), ncclUint8, peer,
                            static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return nccl_err(r, "ncclRecv");
  return PL_OK;
}

int32_t pl_record_globaltimer(uint64_t* dst, void* stream) {
  record_globaltimer_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(dst);
  return check_launch("record_globaltimer_kernel");
}

int32_t pl_gate_until_ns(const uint64_t* t0, uint64_t offset_ns, void* stream) {
  gate_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(t0, offset_ns);
  return check_launch("gate_kernel");
}

}  // extern "C"
