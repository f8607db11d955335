// NCCL communicator for head-sharded (tensor-parallel) plans.
//
// The plan's AllReduce nodes (the only exchange of a Megatron-sharded decoder
// layer: after O-proj and after FFN-down, SURVEY.md §8 e) run as
// ncclAllReduce(sum) on the plan's stream over NVLink / NVSwitch.  NCCL is
// resolved at run time with dlopen: inside a PyTorch process the library torch
// already loaded is reused (same soname), elsewhere the system libnccl.so.2.
#include "comm.hpp"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include "vtc/errors.hpp"

namespace vtc {
namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    });
    if (!a.all_reduce || !a.comm_init_rank || !a.get_unique_id) throw NcclError("libnccl.so.2 not available");
    return a;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + (api().error_string ? api().error_string(r) : "nccl error"));
}

}  // namespace

void comm_unique_id(void* out128) {
    ncclUniqueId id;
    nck(api().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, sizeof(id));
}

Comm::Comm(const void* id128, int nranks, int rank) : nranks_(nranks), rank_(rank) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    nck(api().comm_init_rank(&comm_, nranks, id, rank), "ncclCommInitRank");
}

Comm::Comm(HostAllReduceFn fn, void* user, int nranks, int rank)
    : nranks_(nranks), rank_(rank), host_fn_(fn), host_user_(user) {
    if (!fn) throw ExecutionError("vtc_comm_init_host: null callback");
    host_cap_ = size_t(16) << 20;
    if (cudaHostAlloc(&staging_, host_cap_, cudaHostAllocDefault) != cudaSuccess)
        throw CudaError("cudaHostAlloc(allreduce staging)");
}

Comm::~Comm() {
    if (comm_ && api().comm_destroy) api().comm_destroy(comm_);
    if (staging_) cudaFreeHost(staging_);
}

void CUDART_CB Comm::host_node(void* arg) {
    auto* c = static_cast<HostCall*>(arg);
    c->status = c->fn(c->user, c->buf, c->count, c->dtype);
}

void Comm::all_reduce_sum(const void* send, void* recv, size_t count, ncclDataType_t dt, cudaStream_t s) {
    if (!host_fn_) {
        nck(api().all_reduce(send, recv, count, dt, ncclSum, comm_, s), "ncclAllReduce");
        return;
    }
    const size_t es = dt == ncclBfloat16 ? 2 : dt == ncclFloat32 ? 4 : 8;
    if (count * es > host_cap_) throw UnsupportedError("host-bridged AllReduce larger than the 16 MiB staging buffer");
    // vtc dtype codes (include/vtc.h): 0 f64, 1 f32, 2 i64, 3 bf16
    const int32_t code = dt == ncclBfloat16 ? 3 : dt == ncclFloat32 ? 1 : dt == ncclFloat64 ? 0 : 2;
    calls_.push_back(HostCall{host_fn_, host_user_, staging_, int64_t(count), code, 0});
    auto ck = [](cudaError_t e, const char* w) {
        if (e != cudaSuccess) throw CudaError(std::string(w) + ": " + cudaGetErrorString(e));
    };
    ck(cudaMemcpyAsync(staging_, send, count * es, cudaMemcpyDeviceToHost, s), "allreduce D2H");
    ck(cudaLaunchHostFunc(s, &Comm::host_node, &calls_.back()), "allreduce host node");
    ck(cudaMemcpyAsync(recv, staging_, count * es, cudaMemcpyHostToDevice, s), "allreduce H2D");
}

}  // namespace vtc
