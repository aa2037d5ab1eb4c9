// comm.cpp -- NCCL for the multi-GPU path, loaded with dlopen so that the
// library builds and loads on machines without NCCL (the symbols of the
// libnccl.so.2 already mapped by PyTorch are picked up when present).
#include "comm.h"

#include <dlfcn.h>

#include <cstring>
#include <mutex>

namespace tcb {

namespace {
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return;
    }
#define LOAD(field, sym)                                   \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, sym)); \
  if (!a.field) { a.err = std::string("missing NCCL symbol ") + sym; return; }
    LOAD(GetUniqueId, "ncclGetUniqueId");
    LOAD(CommInitRank, "ncclCommInitRank");
    LOAD(CommDestroy, "ncclCommDestroy");
    LOAD(AllReduce, "ncclAllReduce");
    LOAD(AllGather, "ncclAllGather");
    LOAD(Send, "ncclSend");
    LOAD(Recv, "ncclRecv");
    LOAD(GroupStart, "ncclGroupStart");
    LOAD(GroupEnd, "ncclGroupEnd");
    LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
    a.ok = true;
  });
  return a;
}

std::string nerr(ncclResult_t r) {
  NcclApi& a = api();
  return a.GetErrorString ? a.GetErrorString(r) : "nccl error " + std::to_string((int)r);
}
}  // namespace

std::string nccl_unique_id(uint8_t out[128]) {
  NcclApi& a = api();
  if (!a.ok) return a.err;
  ncclUniqueId id;
  ncclResult_t r = a.GetUniqueId(&id);
  if (r != ncclSuccess) return nerr(r);
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out, &id, 128);
  return "";
}

std::string Comm::init(int rank_, int world_, const uint8_t id[128]) {
  NcclApi& a = api();
  if (!a.ok) return a.err;
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  ncclResult_t r = a.CommInitRank(&comm, world_, uid, rank_);
  if (r != ncclSuccess) return "ncclCommInitRank: " + nerr(r);
  rank = rank_;
  world = world_;
  return "";
}

void Comm::destroy() {
  if (comm) api().CommDestroy(comm);
  comm = nullptr;
}

std::string Comm::allreduce_sum(double* buf, size_t count, cudaStream_t s) {
  ncclResult_t r = api().AllReduce(buf, buf, count, ncclDouble, ncclSum, comm, s);
  return r == ncclSuccess ? "" : "ncclAllReduce: " + nerr(r);
}

std::string Comm::allgather(const double* send, double* recv, size_t count, cudaStream_t s) {
  ncclResult_t r = api().AllGather(send, recv, count, ncclDouble, comm, s);
  return r == ncclSuccess ? "" : "ncclAllGather: " + nerr(r);
}

std::string Comm::exchange(const std::vector<HaloMsg>& sends, const std::vector<HaloMsg>& recvs,
                           cudaStream_t s) {
  NcclApi& a = api();
  ncclResult_t r = a.GroupStart();
  if (r != ncclSuccess) return "ncclGroupStart: " + nerr(r);
  for (const HaloMsg& m : sends)
    if (m.count && (r = a.Send(m.ptr, m.count, ncclDouble, m.peer, comm, s)) != ncclSuccess) break;
  if (r == ncclSuccess)
    for (const HaloMsg& m : recvs)
      if (m.count && (r = a.Recv(m.ptr, m.count, ncclDouble, m.peer, comm, s)) != ncclSuccess) break;
  ncclResult_t r2 = a.GroupEnd();
  if (r != ncclSuccess) return "ncclSend/Recv: " + nerr(r);
  if (r2 != ncclSuccess) return "ncclGroupEnd: " + nerr(r2);
  return "";
}

}  // namespace tcb
