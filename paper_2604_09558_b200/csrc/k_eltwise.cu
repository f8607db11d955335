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
#include <cstring>

#include "device.cuh"
#include "launch.cuh"

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
    return dev::silu_bf16(x);
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
    return dev::gelu_bf16(x);
}
template <>
__device__ __forceinline__ int64_t gelu_of<int64_t>(int64_t x) { return x; }

template <typename T>
__device__ __forceinline__ T add_of(T a, T b) { return a + b; }
template <>
__device__ __forceinline__ bf16 add_of<bf16>(bf16 a, bf16 b) {
    return dev::add_bf16(a, b);
}
template <typename T>
__device__ __forceinline__ T mul_of(T a, T b) { return a * b; }
template <>
__device__ __forceinline__ bf16 mul_of<bf16>(bf16 a, bf16 b) {
    return dev::mul_bf16(a, b);
}
template <>
__device__ __forceinline__ int64_t mul_of<int64_t>(int64_t a, int64_t b) {
    return (int64_t)((uint64_t)a * (uint64_t)b);
}
template <>
__device__ __forceinline__ int64_t add_of<int64_t>(int64_t a, int64_t b) {
    return (int64_t)((uint64_t)a + (uint64_t)b);
}

template <typename T>
__device__ __forceinline__ T apply_op(EwOp op, T a, T b) {
    switch (op) {
        case EwOp::Add: return add_of<T>(a, b);
        case EwOp::Mul: return mul_of<T>(a, b);
        case EwOp::SiLU: return silu_of<T>(a);
        case EwOp::GELU: return gelu_of<T>(a);
        default: return a;
    }
}

// pp1 != nullptr: CTAs [0, blocks0) run program pp0, the rest program pp1.
// PAT 3: the program (in0 * in1) + (in2 * in3) (a RoPE tree), evaluated with
// compile-time registers; PAT 0: the general interpreter.
template <typename T, int VEC, int PAT>
__global__ void __launch_bounds__(256) ew_kernel(const EwParams* __restrict__ pp0, const EwParams* __restrict__ pp1,
                                                 int blocks0) {
    const bool second = pp1 != nullptr && int(blockIdx.x) >= blocks0;
    const EwParams* __restrict__ pp = second ? pp1 : pp0;
    const int64_t bid = second ? int64_t(blockIdx.x) - blocks0 : int64_t(blockIdx.x);
    const int64_t nblk = pp1 == nullptr ? int64_t(gridDim.x) : (second ? int64_t(gridDim.x) - blocks0 : int64_t(blocks0));
    VTC_STAGE_PARAMS(EwParams, pp);
    dev::pdl_wait(); dev::pdl_launch_dependents();
    const int last = p.rank - 1;
    const int nin = p.nin, nprog = p.nprog;
    for (int64_t v = bid * (int64_t)blockDim.x + threadIdx.x; v < p.nvec; v += nblk * blockDim.x) {
        int32_t idx[VTC_MAX_RANK];
        dev::unflatten(v * VEC, p.shape, p.rank, idx);
#pragma unroll 1
        for (int a = 0; a < p.rank; ++a) idx[a] += p.origin[a];
        // all input loads in flight at once (registers), then the program
        T in[EW_MAX_IN][VEC];
#pragma unroll
        for (int i = 0; i < EW_MAX_IN; ++i)
            if (i < nin) load_vec<T, VEC>(p.in[i], idx, last, in[i]);
        if (PAT == 3) {
            T o[VEC];
#pragma unroll
            for (int j = 0; j < VEC; ++j) o[j] = add_of<T>(mul_of<T>(in[0][j], in[1][j]), mul_of<T>(in[2][j], in[3][j]));
            store_vec<T, VEC>(p.out, idx, last, o);
            continue;
        }
        T r[EW_MAX_PROG + EW_MAX_IN][VEC];
#pragma unroll
        for (int i = 0; i < EW_MAX_IN; ++i)
#pragma unroll
            for (int j = 0; j < VEC; ++j) r[i][j] = in[i][j];
        if (nprog > 0) {
#pragma unroll 1
            for (int s = 0; s < nprog; ++s) {
                const EwInstr ins = p.prog[s];
#pragma unroll
                for (int j = 0; j < VEC; ++j) r[ins.dst][j] = apply_op<T>(ins.op, r[ins.a][j], r[ins.b][j]);
            }
        }
        store_vec<T, VEC>(p.out, idx, last, r[p.result]);
    }
}

// Flat fast path (p.flat, host-proved): every operand is a plain row-major
// bf16 buffer of the iteration box, so vector v sits at base + 8 v for all of
// them -- no index unflattening, no map evaluation, 16-byte streaming
// accesses, two vectors in flight per thread.  Programs: one op (PAT 1) or
// SiLU(in0) * in1 (PAT 2, the SwiGLU gate); rounding as the generic kernel.
template <EwOp OP, int NIN, int PAT>
__global__ void __launch_bounds__(256) ew_flat_kernel(const EwParams* __restrict__ pp) {
    VTC_STAGE_PARAMS(EwParams, pp);
    dev::pdl_wait();
    dev::pdl_launch_dependents();
    auto at = [](const VOperand& op) { return reinterpret_cast<const bf16*>(op.m.piece[0].ptr) + op.m.piece[0].base; };
    const uint4* a = reinterpret_cast<const uint4*>(at(p.in[0]));
    const uint4* b = reinterpret_cast<const uint4*>(at(p.in[NIN > 1 ? 1 : 0]));
    uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(p.out.m.piece[0].ptr) + p.out.m.piece[0].base);
    const int64_t n = p.nvec, stride = int64_t(gridDim.x) * blockDim.x;
    constexpr int U = 2;
    for (int64_t v0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v0 < n; v0 += U * stride) {
        uint4 x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + u * stride;
            if (v < n) {
                x[u] = __ldcs(a + v);
                if (NIN > 1) y[u] = __ldcs(b + v);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + u * stride;
            if (v >= n) continue;
            const bf16* xa = reinterpret_cast<const bf16*>(&x[u]);
            const bf16* yb = reinterpret_cast<const bf16*>(&y[u]);
            uint4 r;
            bf16* rr = reinterpret_cast<bf16*>(&r);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (PAT == 2) rr[j] = mul_of<bf16>(silu_of<bf16>(xa[j]), yb[j]);
                else rr[j] = apply_op<bf16>(OP, xa[j], NIN > 1 ? yb[j] : xa[j]);
            }
            __stcs(o + v, r);
        }
    }
}

void launch_flat(const EwParams& p, const EwParams* dp, cudaStream_t s) {
    const int64_t blocks = (p.nvec + 511) / 512;
    const int grid = int(blocks < 148 * 8 ? (blocks < 1 ? 1 : blocks) : 148 * 8);
    if (p.flat == 2) {
        launch_k(ew_flat_kernel<EwOp::Mul, 2, 2>, dim3(grid), dim3(256), 0, s, dp);
        return;
    }
    switch (p.prog[0].op) {
        case EwOp::Add: launch_k(ew_flat_kernel<EwOp::Add, 2, 1>, dim3(grid), dim3(256), 0, s, dp); break;
        case EwOp::Mul: launch_k(ew_flat_kernel<EwOp::Mul, 2, 1>, dim3(grid), dim3(256), 0, s, dp); break;
        case EwOp::SiLU: launch_k(ew_flat_kernel<EwOp::SiLU, 1, 1>, dim3(grid), dim3(256), 0, s, dp); break;
        default: launch_k(ew_flat_kernel<EwOp::GELU, 1, 1>, dim3(grid), dim3(256), 0, s, dp); break;
    }
}

int ew_grid(const EwParams& p) {
    int64_t blocks = (p.nvec + 255) / 256;
    int grid = int(blocks < 148 * 16 ? blocks : 148 * 16);
    return grid < 1 ? 1 : grid;
}

template <typename T>
void launch_t(const EwParams& p, const EwParams* dp, cudaStream_t s) {
    constexpr int V = 16 / sizeof(T);
    const int grid = ew_grid(p);
    const EwParams* none = nullptr;
    if (p.vec == V && p.prog_pat == 3)
        launch_k(ew_kernel<T, V, 3>, dim3(grid), dim3(256), 0, s, dp, none, grid);
    else if (p.vec == V)
        launch_k(ew_kernel<T, V, 0>, dim3(grid), dim3(256), 0, s, dp, none, grid);
    else
        launch_k(ew_kernel<T, 1, 0>, dim3(grid), dim3(256), 0, s, dp, none, grid);
}

// ---- affine operands (p.aff, host-proved): compact parameters passed by value,
// index unflattening by 32-bit multiply-shift division, one 16-byte access per
// operand per vector, the piece chosen by one compare on the last axis ----
struct EwAffArgs {
    EwAff op[EW_MAX_IN + 1];
    uint32_t shape[VTC_MAX_RANK];
    uint32_t magic[VTC_MAX_RANK];  // Granlund-Montgomery: q = (hi + ((n - hi) >> 1)) >> (l - 1), hi = umulhi(m, n)
    uint32_t shift[VTC_MAX_RANK];  // l (0: divisor 1)
    int32_t rank, nin, nprog, result;
    EwInstr prog[EW_MAX_PROG];
    int64_t nvec;
    const KHead* head;
};

__device__ __forceinline__ uint32_t fast_div(uint32_t n, uint32_t m, uint32_t l) {
    if (l == 0) return n;
    const uint32_t hi = __umulhi(m, n);
    return (hi + ((n - hi) >> 1)) >> (l - 1);
}

// a0 / a1: two independent programs (a horizontally fused pair, e.g. the Q and
// K RoPE trees) -- CTAs [0, blocks0) run a0, the rest a1 (a1.nvec == 0: single)
template <typename T, int PAT>
__global__ void __launch_bounds__(256) ew_aff_kernel(const __grid_constant__ EwAffArgs a0, const __grid_constant__ EwAffArgs a1,
                                                     int blocks0) {
    const bool second = a1.nvec > 0 && int(blockIdx.x) >= blocks0;
    const EwAffArgs& a = second ? a1 : a0;
    const int64_t bid = second ? int64_t(blockIdx.x) - blocks0 : int64_t(blockIdx.x);
    const int64_t nblk = a1.nvec == 0 ? int64_t(gridDim.x) : (second ? int64_t(gridDim.x) - blocks0 : int64_t(blocks0));
    dev::TraceScope trace_scope_(a0.head);
    constexpr int VEC = 16 / int(sizeof(T));
    dev::pdl_wait();
    dev::pdl_launch_dependents();
    const int rank = a.rank, last = rank - 1;
    // U vectors per thread per round: all their loads in flight before any use
    constexpr int U = 4;
    const int64_t stride = nblk * blockDim.x;
    auto addr_of = [&](const EwAff& op, const uint32_t (&idx)[VTC_MAX_RANK], uint32_t lastv) {
        const int k = int(lastv) >= op.split ? 1 : 0;
        int64_t off = 0;
#pragma unroll
        for (int d = 0; d < VTC_MAX_RANK; ++d)
            if (d <= last) off += op.st[k][d] * int64_t(idx[d]);
        return op.base[k] + uint64_t(off) * sizeof(T);
    };
    for (int64_t v0 = bid * blockDim.x + threadIdx.x; v0 < a.nvec; v0 += U * stride) {
        uint32_t idx[U][VTC_MAX_RANK], lastv[U];
        uint4 raw[U][EW_MAX_IN];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + u * stride;
            if (v >= a.nvec) continue;
            uint32_t f = uint32_t(v) * uint32_t(VEC);
            lastv[u] = 0;
#pragma unroll
            for (int d = VTC_MAX_RANK - 1; d >= 0; --d) {
                idx[u][d] = 0;
                if (d > last) continue;
                const uint32_t q = fast_div(f, a.magic[d], a.shift[d]);
                idx[u][d] = f - q * a.shape[d];
                if (d == last) lastv[u] = idx[u][d];
                f = q;
            }
#pragma unroll
            for (int i = 0; i < EW_MAX_IN; ++i)
                if (i < a.nin) raw[u][i] = __ldg(reinterpret_cast<const uint4*>(addr_of(a.op[1 + i], idx[u], lastv[u])));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + u * stride;
            if (v >= a.nvec) continue;
            T in[EW_MAX_IN][VEC];
#pragma unroll
            for (int i = 0; i < EW_MAX_IN; ++i) {
                const T* t = reinterpret_cast<const T*>(&raw[u][i]);
#pragma unroll
                for (int j = 0; j < VEC; ++j) in[i][j] = i < a.nin ? t[j] : T(0);
            }
            T o[VEC];
            if (PAT == 3) {
#pragma unroll
                for (int j = 0; j < VEC; ++j) o[j] = add_of<T>(mul_of<T>(in[0][j], in[1][j]), mul_of<T>(in[2][j], in[3][j]));
            } else {
                T r[EW_MAX_PROG + EW_MAX_IN][VEC];
#pragma unroll
                for (int i = 0; i < EW_MAX_IN; ++i)
#pragma unroll
                    for (int j = 0; j < VEC; ++j) r[i][j] = in[i][j];
#pragma unroll 1
                for (int s2 = 0; s2 < a.nprog; ++s2) {
                    const EwInstr ins = a.prog[s2];
#pragma unroll
                    for (int j = 0; j < VEC; ++j) r[ins.dst][j] = apply_op<T>(ins.op, r[ins.a][j], r[ins.b][j]);
                }
#pragma unroll
                for (int j = 0; j < VEC; ++j) o[j] = r[a.result][j];
            }
            uint4 w;
            T* t = reinterpret_cast<T*>(&w);
#pragma unroll
            for (int j = 0; j < VEC; ++j) t[j] = o[j];
            *reinterpret_cast<uint4*>(addr_of(a.op[0], idx[u], lastv[u])) = w;
        }
    }
}

void magic_of(uint32_t d, uint32_t& m, uint32_t& l) {
    if (d <= 1) {
        m = 0;
        l = 0;
        return;
    }
    l = 0;
    while ((uint64_t(1) << l) < d) ++l;
    m = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1);
}

EwAffArgs aff_args(const EwParams& p, const EwParams* dp) {
    EwAffArgs a;
    std::memset(&a, 0, sizeof(a));
    for (int k = 0; k <= p.nin; ++k) a.op[k] = p.affine[k];
    for (int d = 0; d < p.rank; ++d) {
        a.shape[d] = uint32_t(p.shape[d]);
        magic_of(a.shape[d], a.magic[d], a.shift[d]);
    }
    a.rank = p.rank;
    a.nin = p.nin;
    a.nprog = p.nprog;
    a.result = p.result;
    for (int i = 0; i < EW_MAX_PROG; ++i) a.prog[i] = p.prog[i];
    a.nvec = p.nvec;
    a.head = &dp->head;
    return a;
}

bool aff_usable(const EwParams& p) {
    // not for launches whose map bases move with a dynamic decode position
    // (patched on the device, KHead::ndyn)
    return p.aff && p.head.ndyn == 0 && p.nvec * (16 / p.esize) < (int64_t(1) << 31);
}

template <typename T>
void launch_aff_t(const EwParams& p, const EwParams* dp, cudaStream_t s) {
    EwAffArgs a = aff_args(p, dp), none;
    std::memset(&none, 0, sizeof(none));
    const int grid = ew_grid(p);
    if (p.prog_pat == 3) launch_k(ew_aff_kernel<T, 3>, dim3(grid), dim3(256), 0, s, a, none, grid);
    else launch_k(ew_aff_kernel<T, 0>, dim3(grid), dim3(256), 0, s, a, none, grid);
}

template <typename T>
void launch_pair_t(const EwPair& p, const EwPair* dp, cudaStream_t s) {
    constexpr int V = 16 / sizeof(T);
    const int g0 = ew_grid(p.a), g1 = ew_grid(p.b);
    if (aff_usable(p.a) && aff_usable(p.b)) {
        const EwAffArgs a0 = aff_args(p.a, &dp->a), a1 = aff_args(p.b, &dp->b);
        if (p.a.prog_pat == 3) launch_k(ew_aff_kernel<T, 3>, dim3(g0 + g1), dim3(256), 0, s, a0, a1, g0);
        else launch_k(ew_aff_kernel<T, 0>, dim3(g0 + g1), dim3(256), 0, s, a0, a1, g0);
        return;
    }
    if (p.a.vec == V && p.a.prog_pat == 3)
        launch_k(ew_kernel<T, V, 3>, dim3(g0 + g1), dim3(256), 0, s, &dp->a, &dp->b, g0);
    else if (p.a.vec == V)
        launch_k(ew_kernel<T, V, 0>, dim3(g0 + g1), dim3(256), 0, s, &dp->a, &dp->b, g0);
    else
        launch_k(ew_kernel<T, 1, 0>, dim3(g0 + g1), dim3(256), 0, s, &dp->a, &dp->b, g0);
}

}  // namespace

bool eltwise_pair_compatible(const EwParams& a, const EwParams& b) {
    return a.nvec > 0 && b.nvec > 0 && !a.copy_only && !b.copy_only && a.dt == b.dt && a.vec == b.vec &&
           a.prog_pat == b.prog_pat;
}

void launch_eltwise_pair(const EwPair& p, const EwPair* dp, cudaStream_t s) {
    switch (p.a.dt) {
        case KDType::F64: launch_pair_t<double>(p, dp, s); break;
        case KDType::F32: launch_pair_t<float>(p, dp, s); break;
        case KDType::I64: launch_pair_t<int64_t>(p, dp, s); break;
        case KDType::BF16: launch_pair_t<bf16>(p, dp, s); break;
    }
}


void launch_eltwise(const EwParams& p, const EwParams* dp, cudaStream_t s) {
    if (p.nvec == 0) return;
    if (p.flat) {
        launch_flat(p, dp, s);
        return;
    }
    if (aff_usable(p)) {  // affine compact path
        switch (p.copy_only ? (p.esize == 8 ? KDType::I64 : p.esize == 4 ? KDType::F32 : KDType::BF16) : p.dt) {
            case KDType::F64: launch_aff_t<double>(p, dp, s); return;
            case KDType::F32: launch_aff_t<float>(p, dp, s); return;
            case KDType::I64: launch_aff_t<int64_t>(p, dp, s); return;
            case KDType::BF16: launch_aff_t<bf16>(p, dp, s); return;
        }
    }
    if (p.copy_only) {
        // copies are dtype-agnostic: dispatch on element size
        switch (p.esize) {
            case 8: launch_t<int64_t>(p, dp, s); return;
            case 4: launch_t<float>(p, dp, s); return;
            case 2: launch_t<bf16>(p, dp, s); return;
        }
    }
    switch (p.dt) {
        case KDType::F64: launch_t<double>(p, dp, s); break;
        case KDType::F32: launch_t<float>(p, dp, s); break;
        case KDType::I64: launch_t<int64_t>(p, dp, s); break;
        case KDType::BF16: launch_t<bf16>(p, dp, s); break;
    }
}


// ---- host-link copies of run_host (vtc_run) --------------------------------
// Pinned host buffers are device-addressable under UVA: one small kernel reads
// the pinned input arena over the host link (or writes the outputs into pinned
// staging with posted stores) instead of a DMA memcpy node, whose fixed cost
// (~4.5 us per node on B200) exceeds the transfer of a decode step's few KB.
// Launched with PDL like every other kernel, so the next launch's static
// weight prefetch overlaps the copy-in and the copy-out overlaps the last
// kernel's tail up to its dependency wait.
namespace {
__global__ void __launch_bounds__(256) host_link_copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                            int64_t n16) {
    dev::pdl_wait();
    dev::pdl_launch_dependents();
    constexpr int U = 4;  // every load of a thread in flight before its stores
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n16; i0 += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * stride < n16) v[u] = src[i0 + u * stride];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * stride < n16) dst[i0 + u * stride] = v[u];
    }
}
}  // namespace

void launch_host_link_copy(const void* src, void* dst, int64_t bytes, cudaStream_t s) {
    const int64_t n16 = (bytes + 15) / 16;
    if (n16 == 0) return;
    const int64_t per_cta = 256 * 4;
    const unsigned grid = unsigned(std::min<int64_t>((n16 + per_cta - 1) / per_cta, 148));
    launch_k(host_link_copy_kernel, dim3(grid), dim3(256), 0, s, static_cast<const uint4*>(src), static_cast<uint4*>(dst), n16);
}

}  // namespace vtc
