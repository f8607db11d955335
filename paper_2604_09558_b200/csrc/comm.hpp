// NCCL communicator wrapper (see comm.cpp).
#pragma once

#include <cstring>

#include <cuda_runtime.h>
#include <nccl.h>

namespace vtc {

void comm_unique_id(void* out128);

class Comm {
public:
    Comm(const void* id128, int nranks, int rank);
    ~Comm();
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;
    int nranks() const { return nranks_; }
    int rank() const { return rank_; }
    void all_reduce_sum(const void* send, void* recv, size_t count, ncclDataType_t dt, cudaStream_t s) const;

private:
    ncclComm_t comm_ = nullptr;
    int nranks_ = 1, rank_ = 0;
};

}  // namespace vtc
