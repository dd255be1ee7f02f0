// Data-parallel exchange of the mixed-precision step over NCCL (NVLink /
// NVSwitch), for hosts that drive the C ABI without torch.distributed.
//
// The reference keeps one replicated LossScaling state per run
// and, in data-parallel training, splits every batch across the GPUs
// (PAPER.md:282); every rank must then take the same skip / back-off decision.
// Two collectives carry that:
//   mpx_allreduce_grads  ncclAllReduce(sum) of the half (scaled) gradients —
//                        1/W is folded into the loss cotangent upstream, so a
//                        plain sum is the batch-mean gradient;
//   mpx_allreduce_flag   ncclAllReduce(min) of the u32 finite flag K2 wrote —
//                        the logical AND of every rank's all_finite
//                        (tree.py:125-131), so K3 (precision.py:156-173) and
//                        the gated K4 (optim.py:100-113) see one decision.
// libnccl.so.2 is dlopen'ed on first use (the one torch already loaded, when
// there is one, by SONAME), so the library has no link-time NCCL dependency
// and a process that never calls these never loads it.
#include "mpx_common.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
  char why[256] = {0};
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      snprintf(api.why, sizeof(api.why), "dlopen(libnccl.so.2): %s", dlerror());
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.comm_count = reinterpret_cast<decltype(api.comm_count)>(dlsym(h, "ncclCommCount"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.comm_count && api.all_reduce &&
             api.error_string;
    if (!api.ok) snprintf(api.why, sizeof(api.why), "libnccl.so.2 lacks a required symbol");
  });
  return api;
}

int nccl_fail(const char* what, ncclResult_t r) {
  return mpx::fail(MPX_ENCCL, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "?") +
                                  " (ncclResult_t " + std::to_string((int)r) + ")");
}

int need_nccl() { return nccl().ok ? 0 : mpx::fail(MPX_ENCCL, std::string("NCCL unavailable: ") + nccl().why); }

int inval(const std::string& msg) { return mpx::fail(MPX_EINVAL, msg); }

}  // namespace

extern "C" {

int mpx_comm_unique_id(uint8_t* h_id) {
  if (!h_id) return inval("mpx_comm_unique_id: null id buffer");
  if (int e = need_nccl()) return e;
  ncclUniqueId id;
  if (ncclResult_t r = nccl().get_unique_id(&id)) return nccl_fail("ncclGetUniqueId", r);
  std::memcpy(h_id, id.internal, MPX_COMM_ID_BYTES);
  return 0;
}

int mpx_comm_init(void** h_comm, int nranks, const uint8_t* h_id, int rank, int device) {
  if (!h_comm || !h_id || nranks < 1 || rank < 0 || rank >= nranks)
    return inval("mpx_comm_init: bad arguments (nranks " + std::to_string(nranks) + ", rank " + std::to_string(rank) + ")");
  if (int e = need_nccl()) return e;
  MPX_CUDA_CHECK(cudaSetDevice(device));
  ncclUniqueId id;
  std::memcpy(id.internal, h_id, MPX_COMM_ID_BYTES);
  ncclComm_t c = nullptr;
  if (ncclResult_t r = nccl().comm_init_rank(&c, nranks, id, rank)) return nccl_fail("ncclCommInitRank", r);
  *h_comm = c;
  return 0;
}

int mpx_comm_destroy(void* comm) {
  if (!comm) return 0;
  if (int e = need_nccl()) return e;
  if (ncclResult_t r = nccl().comm_destroy(static_cast<ncclComm_t>(comm))) return nccl_fail("ncclCommDestroy", r);
  return 0;
}

int mpx_comm_size(void* comm, int* h_nranks) {
  if (!comm || !h_nranks) return inval("mpx_comm_size: null argument");
  if (int e = need_nccl()) return e;
  if (ncclResult_t r = nccl().comm_count(static_cast<ncclComm_t>(comm), h_nranks)) return nccl_fail("ncclCommCount", r);
  return 0;
}

int mpx_allreduce_flag(void* comm, uint32_t* d_flag, void* stream) {
  if (!comm || !d_flag) return inval("mpx_allreduce_flag: null comm or flag");
  if (int e = need_nccl()) return e;
  if (ncclResult_t r = nccl().all_reduce(d_flag, d_flag, 1, ncclUint32, ncclMin, static_cast<ncclComm_t>(comm),
                                         static_cast<cudaStream_t>(stream)))
    return nccl_fail("ncclAllReduce(flag, min)", r);
  return 0;
}

int mpx_allreduce_grads(void* comm, void* d_grads, int64_t numel, int dtype, void* stream) {
  if (!comm || (!d_grads && numel) || numel < 0) return inval("mpx_allreduce_grads: bad arguments");
  ncclDataType_t t;
  switch (dtype) {
    case MPX_F32: t = ncclFloat32; break;
    case MPX_F16: t = ncclFloat16; break;
    case MPX_BF16: t = ncclBfloat16; break;
    default: return inval("mpx_allreduce_grads: dtype " + std::to_string(dtype));
  }
  if (numel == 0) return 0;
  if (int e = need_nccl()) return e;
  if (ncclResult_t r = nccl().all_reduce(d_grads, d_grads, static_cast<size_t>(numel), t, ncclSum,
                                         static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)))
    return nccl_fail("ncclAllReduce(grads, sum)", r);
  return 0;
}

}  // extern "C"
