// Deterministic 256-thread row reductions shared by the row-op kernels and the
// fused GEMV prologue, so a fused RMSNorm reproduces the standalone op bit for bit.
#pragma once

#include "device.cuh"

namespace vtc {

// Thread t accumulates f(t), f(t+256), ... in order, then a warp tree, then
// the 8 warp partials in warp order.  Result broadcast to all threads.
template <typename Acc, class F>
__device__ __forceinline__ Acc block_sum_256(F f, int64_t D) {
    __shared__ Acc s_part[8];
    __shared__ Acc s_total;
    Acc s = Acc(0);
#pragma unroll 8
    for (int64_t k = threadIdx.x; k < D; k += 256) s += f(k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        Acc t = Acc(0);
#pragma unroll
        for (int w = 0; w < 8; ++w) t += s_part[w];
        s_total = t;
    }
    __syncthreads();
    Acc r = s_total;
    __syncthreads();
    return r;
}

// Same arithmetic order as block_sum_256, for 256 consumer threads that sync
// on named barrier 1 (a producer warp elsewhere in the CTA does not take part).
template <typename Acc, class F>
__device__ __forceinline__ Acc block_sum_256_bar1(F f, int64_t D) {
    __shared__ Acc s_part[8];
    __shared__ Acc s_total;
    Acc s = Acc(0);
#pragma unroll 8
    for (int64_t k = threadIdx.x; k < D; k += 256) s += f(k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = s;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (threadIdx.x == 0) {
        Acc t = Acc(0);
#pragma unroll
        for (int w = 0; w < 8; ++w) t += s_part[w];
        s_total = t;
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    Acc r = s_total;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    return r;
}

template <typename Acc, class F>
__device__ __forceinline__ Acc block_max_256(F f, int64_t D) {
    __shared__ Acc s_part[8];
    __shared__ Acc s_total;
    Acc s = -INFINITY;
#pragma unroll 8
    for (int64_t k = threadIdx.x; k < D; k += 256) s = max(s, f(k));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = max(s, __shfl_xor_sync(0xffffffffu, s, o));
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        Acc t = s_part[0];
#pragma unroll
        for (int w = 1; w < 8; ++w) t = max(t, s_part[w]);
        s_total = t;
    }
    __syncthreads();
    Acc r = s_total;
    __syncthreads();
    return r;
}

// Sum of squares of a strided bf16 row, in exactly block_sum_256's order
// (thread t: f(t), f(t+256), ... sequentially; warp tree; warps in order), but
// with the loads batched 8 deep so they are in flight together -- a rolled
// load/accumulate loop is one memory round trip per element.
template <bool BAR1>
__device__ __forceinline__ float block_sumsq_bf16_fast(const dev::bf16* __restrict__ x, int64_t stride, int64_t D) {
    __shared__ float s_part[8];
    __shared__ float s_total;
    float s = 0.f;
    for (int64_t b = threadIdx.x; b < D; b += 256 * 8) {
        float t[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t k = b + int64_t(j) * 256;
            t[j] = k < D ? __bfloat162float(x[k * stride]) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (b + int64_t(j) * 256 < D) s += t[j] * t[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = s;
    if (BAR1) asm volatile("bar.sync 1, 256;" ::: "memory");
    else __syncthreads();
    if (threadIdx.x == 0) {
        float tt = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) tt += s_part[w];
        s_total = tt;
    }
    if (BAR1) asm volatile("bar.sync 1, 256;" ::: "memory");
    else __syncthreads();
    float res = s_total;
    if (BAR1) asm volatile("bar.sync 1, 256;" ::: "memory");
    else __syncthreads();
    return res;
}

// The cross-thread part of block_sum_256 for per-thread partials already
// accumulated in its order (256 consumer threads, named barrier 1).
__device__ __forceinline__ float block_sum_regs_bar1(float s) {
    __shared__ float s_part[8];
    __shared__ float s_total;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = s;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (threadIdx.x == 0) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += s_part[w];
        s_total = t;
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    float r = s_total;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    return r;
}

// Sum of squares of row `row` of a rank-2 bf16 operand [rows, D].
__device__ __forceinline__ float block_sumsq_row_bf16(const VOperand& x, int row, int64_t D) {
    return block_sum_256<float>(
        [&](int64_t k) {
            int32_t idx[VTC_MAX_RANK] = {};
            idx[0] = row;
            idx[1] = int32_t(k);
            float v = __bfloat162float(*dev::elem_ptr<dev::bf16>(x.m, idx));
            return v * v;
        },
        D);
}

}  // namespace vtc
