// Elementwise compute (Add / Mul / SiLU / GELU) and the gather-copy kernel K0.
//
// Semantics follow run_operator (proj/src/executor.cpp:268-291 for Add/Mul/SiLU;
// SiLU evaluated in double then cast, :224-227) and, for Copy, the
// data-movement cases :292-432 expressed as out[map_out(I)] = in[map_in(I)].
// Copy is the MATERIALISING baseline kernel only: under a VTC plan no copy
// launches for eliminated operators.
//
// Each thread handles one vector of `vec` consecutive elements along the last
// axis; every operand map is evaluated once per vector, then stepped with the
// per-piece fast stride (one 16-byte access when the host proved alignment).
#include <cmath>

#include "device.cuh"

namespace vtc {
namespace {

using dev::bf16;

template <typename T, int VEC>
__device__ __forceinline__ void load_vec(const VOperand& op, int32_t (&idx)[VTC_MAX_RANK], int last, T (&v)[VEC]) {
    dev::Loc l = dev::locate(op.m, idx);
    const T* base = dev::addr<T>(op.m, l);
    if (VEC * sizeof(T) == 16 && op.vec_ok) {
        uint4 u = __ldg(reinterpret_cast<const uint4*>(base));
        const T* t = reinterpret_cast<const T*>(&u);
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] = t[j];
    } else if (op.fast_ok) {
        int64_t s = op.fast_stride[l.piece];
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] = base[j * s];
    } else {
        int32_t x0 = dev::sel(idx, last);
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            dev::set_axis(idx, last, x0 + j);
            v[j] = *dev::elem_ptr<T>(op.m, idx);
        }
        dev::set_axis(idx, last, x0);
    }
}

template <typename T, int VEC>
__device__ __forceinline__ void store_vec(const VOperand& op, int32_t (&idx)[VTC_MAX_RANK], int last, const T (&v)[VEC]) {
    dev::Loc l = dev::locate(op.m, idx);
    T* base = dev::addr<T>(op.m, l);
    if (VEC * sizeof(T) == 16 && op.vec_ok) {
        uint4 u;
        T* t = reinterpret_cast<T*>(&u);
#pragma unroll
        for (int j = 0; j < VEC; ++j) t[j] = v[j];
        *reinterpret_cast<uint4*>(base) = u;
    } else if (op.fast_ok) {
        int64_t s = op.fast_stride[l.piece];
#pragma unroll
        for (int j = 0; j < VEC; ++j) base[j * s] = v[j];
    } else {
        int32_t x0 = dev::sel(idx, last);
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            dev::set_axis(idx, last, x0 + j);
            *dev::elem_ptr<T>(op.m, idx) = v[j];
        }
        dev::set_axis(idx, last, x0);
    }
}

template <typename T>
__device__ __forceinline__ T silu_of(T x) {
    double d = (double)x;
    return (T)(d / (1.0 + exp(-d)));
}
template <>
__device__ __forceinline__ bf16 silu_of<bf16>(bf16 x) {
    float f = __bfloat162float(x);
    return __float2bfloat16_rn(f / (1.0f + expf(-f)));
}
template <>
__device__ __forceinline__ int64_t silu_of<int64_t>(int64_t x) { return x; }

template <typename T>
__device__ __forceinline__ T gelu_of(T x) {
    double d = (double)x;
    return (T)(0.5 * d * (1.0 + erf(d * 0.70710678118654752440)));
}
template <>
__device__ __forceinline__ bf16 gelu_of<bf16>(bf16 x) {
    float f = __bfloat162float(x);
    return __float2bfloat16_rn(0.5f * f * (1.0f + erff(f * 0.70710678f)));
}
template <>
__device__ __forceinline__ int64_t gelu_of<int64_t>(int64_t x) { return x; }

template <typename T>
__device__ __forceinline__ T add_of(T a, T b) { return a + b; }
template <>
__device__ __forceinline__ bf16 add_of<bf16>(bf16 a, bf16 b) {
    return __float2bfloat16_rn(__bfloat162float(a) + __bfloat162float(b));
}
template <typename T>
__device__ __forceinline__ T mul_of(T a, T b) { return a * b; }
template <>
__device__ __forceinline__ bf16 mul_of<bf16>(bf16 a, bf16 b) {
    return __float2bfloat16_rn(__bfloat162float(a) * __bfloat162float(b));
}
template <>
__device__ __forceinline__ int64_t mul_of<int64_t>(int64_t a, int64_t b) {
    return (int64_t)((uint64_t)a * (uint64_t)b);
}
template <>
__device__ __forceinline__ int64_t add_of<int64_t>(int64_t a, int64_t b) {
    return (int64_t)((uint64_t)a + (uint64_t)b);
}

template <typename T, EwOp OP, int VEC>
__global__ void __launch_bounds__(256) ew_kernel(const __grid_constant__ EwParams p) {
    const int last = p.rank - 1;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < p.nvec; v += (int64_t)gridDim.x * blockDim.x) {
        int32_t idx[VTC_MAX_RANK];
        dev::unflatten(v * VEC, p.shape, p.rank, idx);
#pragma unroll
        for (int a = 0; a < VTC_MAX_RANK; ++a) idx[a] += p.origin[a];
        T a[VEC], b[VEC], o[VEC];
        load_vec<T, VEC>(p.a, idx, last, a);
        if (OP == EwOp::Add || OP == EwOp::Mul || OP == EwOp::SiLUMul) load_vec<T, VEC>(p.b, idx, last, b);
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            if constexpr (OP == EwOp::Copy) o[j] = a[j];
            else if constexpr (OP == EwOp::Add) o[j] = add_of<T>(a[j], b[j]);
            else if constexpr (OP == EwOp::Mul) o[j] = mul_of<T>(a[j], b[j]);
            else if constexpr (OP == EwOp::SiLU) o[j] = silu_of<T>(a[j]);
            else if constexpr (OP == EwOp::GELU) o[j] = gelu_of<T>(a[j]);
            else o[j] = mul_of<T>(silu_of<T>(a[j]), b[j]);
        }
        store_vec<T, VEC>(p.out, idx, last, o);
    }
}

template <typename T, EwOp OP>
void launch_t(const EwParams& p, cudaStream_t s) {
    constexpr int V = 16 / sizeof(T);
    int64_t blocks = (p.nvec + 255) / 256;
    int grid = int(blocks < 148 * 16 ? blocks : 148 * 16);
    if (grid < 1) grid = 1;
    if (p.vec == V)
        ew_kernel<T, OP, V><<<grid, 256, 0, s>>>(p);
    else
        ew_kernel<T, OP, 1><<<grid, 256, 0, s>>>(p);
}

template <typename T>
void launch_op(const EwParams& p, cudaStream_t s) {
    switch (p.op) {
        case EwOp::Copy: launch_t<T, EwOp::Copy>(p, s); break;
        case EwOp::Add: launch_t<T, EwOp::Add>(p, s); break;
        case EwOp::Mul: launch_t<T, EwOp::Mul>(p, s); break;
        case EwOp::SiLU: launch_t<T, EwOp::SiLU>(p, s); break;
        case EwOp::GELU: launch_t<T, EwOp::GELU>(p, s); break;
        case EwOp::SiLUMul: launch_t<T, EwOp::SiLUMul>(p, s); break;
    }
}

}  // namespace

void launch_eltwise(const EwParams& p, cudaStream_t s) {
    if (p.nvec == 0) return;
    if (p.op == EwOp::Copy) {
        // copies are dtype-agnostic: dispatch on element size
        switch (p.esize) {
            case 8: launch_op<int64_t>(p, s); return;
            case 4: launch_op<float>(p, s); return;
            case 2: launch_op<bf16>(p, s); return;
        }
    }
    switch (p.dt) {
        case KDType::F64: launch_op<double>(p, s); break;
        case KDType::F32: launch_op<float>(p, s); break;
        case KDType::I64: launch_op<int64_t>(p, s); break;
        case KDType::BF16: launch_op<bf16>(p, s); break;
    }
}

}  // namespace vtc
