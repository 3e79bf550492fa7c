// Multi-GPU communicator for the time-slab decomposition.
//
// NCCL is loaded at run time with dlopen("libnccl.so.2") so the library has no
// link-time NCCL dependency; inside a PyTorch process this resolves to the
// NCCL torch already loaded.  Used for (1) grouped ncclSend/ncclRecv of the
// r_t boundary frames of the pre-multiplied iterate p with ranks +-1 and
// (2) an ncclAllReduce (fp64 sum) of the per-volume norm / Rayleigh partials
// each iteration.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

namespace sfseg {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  bool ok = false;
};

inline NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.handle) break;
    }
    if (!api.handle) return;
#define LOAD(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.handle, "nccl" #f))
    LOAD(GetUniqueId);
    LOAD(CommInitRank);
    LOAD(CommDestroy);
    LOAD(Send);
    LOAD(Recv);
    LOAD(AllReduce);
    LOAD(GroupStart);
    LOAD(GroupEnd);
#undef LOAD
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.AllReduce &&
             api.GroupStart && api.GroupEnd;
  });
  return api;
}

}  // namespace sfseg

struct sfseg_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1;
  int rank = 0;
  int device = 0;
  int32_t* flag = nullptr;  // device word of the pre-solve validation agreement (dist_agree)
  cudaStream_t cs = nullptr;  // comm stream of the overlapped time-slab schedule (SlabSched)
  cudaEvent_t ev[4] = {};     // its hand-off events
};

namespace sfseg {
// bytes of extra workspace for the two halo buffers [B][RT][H][Wp] and allreduce scratch
inline size_t comm_ws_bytes(int64_t B, int RT, int64_t H, int64_t Wp) {
  const size_t halo = (size_t)B * RT * H * Wp * sizeof(float);
  const size_t a = 256;
  return 2 * ((halo + a - 1) / a * a) + 2 * ((sizeof(double) * 2 * B + a - 1) / a * a);
}
}  // namespace sfseg
