// NCCL communicator wrapper (see comm.cpp).
#pragma once

#include <cstdint>
#include <cstring>
#include <deque>

#include <cuda_runtime.h>
#include <nccl.h>

namespace vtc {

void comm_unique_id(void* out128);

// Host-bridged sum-allreduce (include/vtc.h vtc_allreduce_fn): the buffer is
// reduced in place on the host by the caller's collective (MPI, gloo, ...).
using HostAllReduceFn = int (*)(void* user, void* buf, int64_t count, int32_t dtype);

class Comm {
public:
    Comm(const void* id128, int nranks, int rank);
    // host-bridged: every AllReduce stages through pinned host memory (D2H, the
    // callback in a stream host node, H2D) -- multi-process tests without one GPU
    // per rank, and hosts whose ranks share a device
    Comm(HostAllReduceFn fn, void* user, int nranks, int rank);
    ~Comm();
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;
    int nranks() const { return nranks_; }
    int rank() const { return rank_; }
    bool host_bridged() const { return host_fn_ != nullptr; }
    void all_reduce_sum(const void* send, void* recv, size_t count, ncclDataType_t dt, cudaStream_t s);

private:
    struct HostCall {
        HostAllReduceFn fn;
        void* user;
        void* buf;
        int64_t count;
        int32_t dtype;
        int status;
    };
    static void CUDART_CB host_node(void* arg);
    ncclComm_t comm_ = nullptr;
    int nranks_ = 1, rank_ = 0;
    HostAllReduceFn host_fn_ = nullptr;
    void* host_user_ = nullptr;
    void* staging_ = nullptr;  // pinned, host_cap_ bytes
    size_t host_cap_ = 0;
    std::deque<HostCall> calls_;  // one per recorded AllReduce (stable addresses for graph replays)
};

}  // namespace vtc
