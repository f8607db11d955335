// Row-wise RMSNorm / LayerNorm / Softmax over the last axis, one 256-thread
// CTA per row, reading and writing through VirtualTensor maps.
// These ops are absent from the reference (SURVEY.md §8 a'); their semantics
// are fixed here and restated in oracle/vtc_oracle.py:
//   RMSNorm   y = T((x * rsqrt(mean(x^2) + eps)) * w)
//   LayerNorm y = T(((x - mu) * rsqrt(var + eps)) * g + b)
//   Softmax   y = T(exp(x - max) / sum(exp(x - max)))
// with fp32 math for f32/bf16 and fp64 math for f64.
#include <type_traits>

#include "device.cuh"
#include "launch.cuh"
#include "rowreduce.cuh"

namespace vtc {
namespace {

using dev::bf16;

template <typename T>
struct RowIO {
    const VOperand* op;
    T* base;
    int64_t stride;
    bool fast;
    int32_t idx[VTC_MAX_RANK];
    int last;

    __device__ void init(const VOperand& o, const int32_t (&rowidx)[VTC_MAX_RANK], int last_axis) {
        op = &o;
        last = last_axis;
#pragma unroll
        for (int a = 0; a < VTC_MAX_RANK; ++a) idx[a] = rowidx[a];
        fast = o.fast_ok != 0;
        if (fast) {
            dev::set_axis(idx, last, 0);
            dev::Loc l = dev::locate(o.m, idx);
            base = dev::addr<T>(o.m, l);
            stride = o.fast_stride[l.piece];
        }
    }
    __device__ T* at(int64_t k) {
        if (fast) return base + k * stride;
        int32_t j[VTC_MAX_RANK];
#pragma unroll
        for (int a = 0; a < VTC_MAX_RANK; ++a) j[a] = idx[a];
        dev::set_axis(j, last, int32_t(k));
        return dev::elem_ptr<T>(op->m, j);
    }
};

template <typename T>
__global__ void __launch_bounds__(256) row_kernel(const RowParams* __restrict__ pp) {
    VTC_STAGE_PARAMS(RowParams, pp);
    dev::pdl_wait(); dev::pdl_launch_dependents();
    using A = std::conditional_t<std::is_same_v<T, double>, double, float>;
    const int last = p.rank - 1;
    for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
        int32_t idx[VTC_MAX_RANK];
        dev::unflatten(row * p.D, p.shape, p.rank, idx);
        RowIO<T> x, y;
        x.init(p.x, idx, last);
        y.init(p.out, idx, last);
        auto xv = [&](int64_t k) -> A { return A(dev::to_acc<T>(*x.at(k))); };
        int32_t z[VTC_MAX_RANK] = {};
        RowIO<T> w, b;
        if (p.op != RowOp::Softmax) w.init(p.w, z, 0);
        if (p.op == RowOp::LayerNorm) b.init(p.bias, z, 0);
        if (p.op == RowOp::RMSNorm) {
            A ss;
            if constexpr (std::is_same_v<T, bf16>) {
                if (x.fast) ss = block_sumsq_bf16_fast<false>(x.base, x.stride, p.D);
                else ss = block_sum_256<A>([&](int64_t k) { A v = xv(k); return v * v; }, p.D);
            } else {
                ss = block_sum_256<A>([&](int64_t k) { A v = xv(k); return v * v; }, p.D);
            }
            A r;
            if constexpr (std::is_same_v<A, double>) r = 1.0 / sqrt(ss / double(p.D) + double(p.eps));
            else r = rsqrtf(ss / float(p.D) + p.eps);
#pragma unroll 4
            for (int64_t k = threadIdx.x; k < p.D; k += 256)
                *y.at(k) = dev::from_acc<T>((xv(k) * r) * A(dev::to_acc<T>(*w.at(k))));
        } else if (p.op == RowOp::LayerNorm) {
            A mu = block_sum_256<A>([&](int64_t k) { return xv(k); }, p.D) / A(p.D);
            A var = block_sum_256<A>([&](int64_t k) { A v = xv(k) - mu; return v * v; }, p.D) / A(p.D);
            A r;
            if constexpr (std::is_same_v<A, double>) r = 1.0 / sqrt(var + double(p.eps));
            else r = rsqrtf(var + p.eps);
#pragma unroll 4
            for (int64_t k = threadIdx.x; k < p.D; k += 256)
                *y.at(k) = dev::from_acc<T>(((xv(k) - mu) * r) * A(dev::to_acc<T>(*w.at(k))) +
                                            A(dev::to_acc<T>(*b.at(k))));
        } else {
            A mx = block_max_256<A>([&](int64_t k) { return xv(k); }, p.D);
            A s = block_sum_256<A>([&](int64_t k) { return A(exp(xv(k) - mx)); }, p.D);
#pragma unroll 4
            for (int64_t k = threadIdx.x; k < p.D; k += 256) *y.at(k) = dev::from_acc<T>(A(exp(xv(k) - mx)) / s);
        }
    }
}

// Short rows (bf16, D <= 256, every operand affine along the row): one warp
// per row, the row's elements in registers (all loads in flight at once), warp
// shuffle reductions -- Swin's LayerNorm over C = 96 has 200,704 such rows.
template <int J>
__global__ void __launch_bounds__(256) row_warp_kernel(const RowParams* __restrict__ pp) {
    VTC_STAGE_PARAMS(RowParams, pp);
    dev::pdl_wait();
    dev::pdl_launch_dependents();
    const int lane = threadIdx.x % 32;
    const int D = int(p.D), last = p.rank - 1;
    const int64_t nw = int64_t(gridDim.x) * 8;
    // weights / bias once per warp
    float wv[J], bv[J];
    {
        int32_t z[VTC_MAX_RANK] = {};
        const bf16* w0 = nullptr;
        const bf16* b0 = nullptr;
        int64_t ws = 0, bs = 0;
        if (p.op != RowOp::Softmax) {
            dev::Loc l = dev::locate(p.w.m, z);
            w0 = dev::addr<bf16>(p.w.m, l);
            ws = p.w.fast_stride[l.piece];
        }
        if (p.op == RowOp::LayerNorm) {
            dev::Loc l = dev::locate(p.bias.m, z);
            b0 = dev::addr<bf16>(p.bias.m, l);
            bs = p.bias.fast_stride[l.piece];
        }
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int k = lane + 32 * j;
            wv[j] = (w0 && k < D) ? __bfloat162float(w0[int64_t(k) * ws]) : 0.f;
            bv[j] = (b0 && k < D) ? __bfloat162float(b0[int64_t(k) * bs]) : 0.f;
        }
    }
    // row r -> (x row, y row, strides): flat-linear operands (host-proved) need
    // no index arithmetic; otherwise unflatten + locate through the maps
    auto row_at = [&](int64_t row, const bf16*& xr, bf16*& yr, int64_t& xs, int64_t& ys) {
        if (p.linear) {
            xr = reinterpret_cast<const bf16*>(p.x.m.piece[0].ptr) + p.x.m.piece[0].base + row * p.D;
            yr = reinterpret_cast<bf16*>(p.out.m.piece[0].ptr) + p.out.m.piece[0].base + row * p.D;
            xs = ys = 1;
            return;
        }
        int32_t idx[VTC_MAX_RANK];
        dev::unflatten(row * p.D, p.shape, p.rank, idx);
        idx[last] = 0;
        dev::Loc lx = dev::locate(p.x.m, idx), ly = dev::locate(p.out.m, idx);
        xr = dev::addr<bf16>(p.x.m, lx);
        yr = dev::addr<bf16>(p.out.m, ly);
        xs = p.x.fast_stride[lx.piece];
        ys = p.out.fast_stride[ly.piece];
    };
    auto load_row = [&](const bf16* xr, int64_t xs, float (&v)[J]) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int k = lane + 32 * j;
            v[j] = k < D ? __bfloat162float(xr[int64_t(k) * xs]) : 0.f;
        }
    };
    // the next row's loads are issued before this row's reductions
    int64_t row = int64_t(blockIdx.x) * 8 + threadIdx.x / 32;
    const bf16* nxr = nullptr;
    bf16* nyr = nullptr;
    int64_t nxs = 0, nys = 0;
    float nv[J];
    if (row < p.rows) {
        row_at(row, nxr, nyr, nxs, nys);
        load_row(nxr, nxs, nv);
    }
    for (; row < p.rows; row += nw) {
        bf16* yr = nyr;
        const int64_t ys = nys;
        float v[J];
#pragma unroll
        for (int j = 0; j < J; ++j) v[j] = nv[j];
        if (row + nw < p.rows) {
            row_at(row + nw, nxr, nyr, nxs, nys);
            load_row(nxr, nxs, nv);
        }
        if (p.op == RowOp::Softmax) {
            float mx = -INFINITY;
#pragma unroll
            for (int j = 0; j < J; ++j)
                if (lane + 32 * j < D) mx = fmaxf(mx, v[j]);
            mx = dev::warp_max(mx);
            float sum = 0.f;
#pragma unroll
            for (int j = 0; j < J; ++j) {
                v[j] = lane + 32 * j < D ? expf(v[j] - mx) : 0.f;
                sum += v[j];
            }
            sum = dev::warp_sum(sum);
#pragma unroll
            for (int j = 0; j < J; ++j)
                if (lane + 32 * j < D) yr[int64_t(lane + 32 * j) * ys] = __float2bfloat16_rn(v[j] / sum);
            continue;
        }
        float mu = 0.f;
        if (p.op == RowOp::LayerNorm) {
            float s = 0.f;
#pragma unroll
            for (int j = 0; j < J; ++j) s += v[j];
            mu = dev::warp_sum(s) / float(D);
        }
        float s2 = 0.f;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const float c = lane + 32 * j < D ? v[j] - mu : 0.f;
            s2 += c * c;
        }
        const float r = rsqrtf(dev::warp_sum(s2) / float(D) + p.eps);
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int k = lane + 32 * j;
            if (k >= D) continue;
            const float o = p.op == RowOp::LayerNorm ? ((v[j] - mu) * r) * wv[j] + bv[j] : (v[j] * r) * wv[j];
            yr[int64_t(k) * ys] = __float2bfloat16_rn(o);
        }
    }
}

// Plain row-major bf16 rows of D = 32 U (p.linear; RMSNorm / LayerNorm):
// four lanes per row, eight rows per warp, 16-byte loads and stores (chunk
// q + 4 u of 8 elements per lane), reductions over the four lanes.
template <int U>
__global__ void __launch_bounds__(256) row_vec_kernel(const RowParams* __restrict__ pp) {
    VTC_STAGE_PARAMS(RowParams, pp);
    dev::pdl_wait();
    dev::pdl_launch_dependents();
    const int lane = threadIdx.x % 32, q = lane % 4;
    const int D = 32 * U;
    const bool ln = p.op == RowOp::LayerNorm;
    auto unpack = [](const uint4& u, float (&f)[8]) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float2 v = __bfloat1622float2(h[t]);
            f[2 * t] = v.x;
            f[2 * t + 1] = v.y;
        }
    };
    // weight / bias of the row in shared memory (fp32), read back per chunk
    __shared__ __align__(16) float sw[128], sb[128];
    {
        int32_t z[VTC_MAX_RANK] = {};
        dev::Loc lw = dev::locate(p.w.m, z);
        const bf16* w0 = dev::addr<bf16>(p.w.m, lw);
        const int64_t ws = p.w.fast_stride[lw.piece];
        const bf16* b0 = nullptr;
        int64_t bs = 0;
        if (ln) {
            dev::Loc lb = dev::locate(p.bias.m, z);
            b0 = dev::addr<bf16>(p.bias.m, lb);
            bs = p.bias.fast_stride[lb.piece];
        }
        for (int k = threadIdx.x; k < D; k += blockDim.x) {
            sw[k] = __bfloat162float(w0[int64_t(k) * ws]);
            sb[k] = ln ? __bfloat162float(b0[int64_t(k) * bs]) : 0.f;
        }
        __syncthreads();
    }
    const bf16* xb = reinterpret_cast<const bf16*>(p.x.m.piece[0].ptr) + p.x.m.piece[0].base;
    bf16* yb = reinterpret_cast<bf16*>(p.out.m.piece[0].ptr) + p.out.m.piece[0].base;
    const int64_t nrw = int64_t(gridDim.x) * 64;  // rows per grid step
    // a warp's eight rows iterate together (the row reductions shuffle across the whole warp);
    // rows past the end load the last row and store nothing
    for (int64_t row = int64_t(blockIdx.x) * 64 + threadIdx.x / 4; row - lane / 4 < p.rows; row += nrw) {
        const uint4* xr = reinterpret_cast<const uint4*>(xb + (row < p.rows ? row : p.rows - 1) * D);
        float x[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) unpack(__ldcs(xr + q + 4 * u), x[u]);
        float mu = 0.f;
        if (ln) {
            float sm = 0.f;
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int t = 0; t < 8; ++t) sm += x[u][t];
            sm += __shfl_xor_sync(0xffffffffu, sm, 1);
            sm += __shfl_xor_sync(0xffffffffu, sm, 2);
            mu = sm / float(D);
        }
        float s2 = 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const float c = x[u][t] - mu;
                s2 += c * c;
            }
        s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
        const float r = rsqrtf(s2 / float(D) + p.eps);
        if (row >= p.rows) continue;
        uint4* yr = reinterpret_cast<uint4*>(yb + row * D);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float4* w4 = reinterpret_cast<const float4*>(sw + (q + 4 * u) * 8);
            const float4* b4 = reinterpret_cast<const float4*>(sb + (q + 4 * u) * 8);
            const float4 wa = w4[0], wb = w4[1], ba = b4[0], bb = b4[1];
            const float w[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
            const float b[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
            uint4 o;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                float o0, o1;
                if (ln) {
                    o0 = ((x[u][2 * t] - mu) * r) * w[2 * t] + b[2 * t];
                    o1 = ((x[u][2 * t + 1] - mu) * r) * w[2 * t + 1] + b[2 * t + 1];
                } else {
                    o0 = (x[u][2 * t] * r) * w[2 * t];
                    o1 = (x[u][2 * t + 1] * r) * w[2 * t + 1];
                }
                h[t] = __floats2bfloat162_rn(o0, o1);
            }
            __stcs(yr + q + 4 * u, o);
        }
    }
}

// Long plain bf16 rows (p.linear, D = 2048 V, RMSNorm / LayerNorm): one CTA
// per row, each thread holds V 16-byte chunks (chunk i = tid + 256 v) in
// registers, together with the matching weight / bias chunks loaded once.
template <int V>
__global__ void __launch_bounds__(256) row_long_kernel(const RowParams* __restrict__ pp) {
    VTC_STAGE_PARAMS(RowParams, pp);
    dev::pdl_wait();
    dev::pdl_launch_dependents();
    const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
    const int D = int(p.D);
    const bool ln = p.op == RowOp::LayerNorm;
    __shared__ float s_red[2][8];
    auto unpack = [](const uint4& u, float (&f)[8]) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float2 v = __bfloat1622float2(h[t]);
            f[2 * t] = v.x;
            f[2 * t + 1] = v.y;
        }
    };
    auto block_sum = [&](float v, int slot) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s_red[slot][warp] = v;
        __syncthreads();
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += s_red[slot][w];
        return t;
    };
    // weight / bias chunks of this thread (the same columns for every row)
    uint4 wq[V], bq[V];
    {
        int32_t z[VTC_MAX_RANK] = {};
        const bf16* w0 = dev::elem_ptr<bf16>(p.w.m, z);
        const bf16* b0 = ln ? dev::elem_ptr<bf16>(p.bias.m, z) : w0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int c = tid + 256 * v;
            wq[v] = c * 8 < D ? *reinterpret_cast<const uint4*>(w0 + c * 8) : make_uint4(0, 0, 0, 0);
            bq[v] = (ln && c * 8 < D) ? *reinterpret_cast<const uint4*>(b0 + c * 8) : make_uint4(0, 0, 0, 0);
        }
    }
    const bf16* xb = reinterpret_cast<const bf16*>(p.x.m.piece[0].ptr) + p.x.m.piece[0].base;
    bf16* yb = reinterpret_cast<bf16*>(p.out.m.piece[0].ptr) + p.out.m.piece[0].base;
    int parity = 0;
    // the next row's chunks are requested before this row's reductions
    auto fetch = [&](int64_t row, uint4 (&q)[V]) {
        const uint4* xr = reinterpret_cast<const uint4*>(xb + row * D);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int c = tid + 256 * v;
            q[v] = (row < p.rows && c * 8 < D) ? __ldcs(xr + c) : make_uint4(0, 0, 0, 0);
        }
    };
    uint4 nq[V];
    fetch(blockIdx.x, nq);
    for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
        float x[V][8];
#pragma unroll
        for (int v = 0; v < V; ++v) unpack(nq[v], x[v]);
        fetch(row + gridDim.x, nq);
        float mu = 0.f;
        if (ln) {
            float sm = 0.f;
#pragma unroll
            for (int v = 0; v < V; ++v)
#pragma unroll
                for (int t = 0; t < 8; ++t) sm += x[v][t];
            mu = block_sum(sm, parity) / float(D);
            parity ^= 1;
        }
        float s2 = 0.f;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const bool ok = (tid + 256 * v) * 8 < D;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const float c = ok ? x[v][t] - mu : 0.f;
                s2 += c * c;
            }
        }
        const float r = rsqrtf(block_sum(s2, parity) / float(D) + p.eps);
        parity ^= 1;
        uint4* yr = reinterpret_cast<uint4*>(yb + row * D);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int c = tid + 256 * v;
            if (c * 8 >= D) continue;
            float w[8], b[8];
            unpack(wq[v], w);
            unpack(bq[v], b);
            uint4 o;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                float o0, o1;
                if (ln) {
                    o0 = ((x[v][2 * t] - mu) * r) * w[2 * t] + b[2 * t];
                    o1 = ((x[v][2 * t + 1] - mu) * r) * w[2 * t + 1] + b[2 * t + 1];
                } else {
                    o0 = (x[v][2 * t] * r) * w[2 * t];
                    o1 = (x[v][2 * t + 1] * r) * w[2 * t + 1];
                }
                h[t] = __floats2bfloat162_rn(o0, o1);
            }
            __stcs(yr + c, o);
        }
    }
}

}  // namespace

void launch_rowop(const RowParams& p, const RowParams* dp, cudaStream_t s) {
    if (p.rows == 0) return;
    const bool long_rows = p.dt == KDType::BF16 && p.linear && p.op != RowOp::Softmax && p.D % 8 == 0 &&
                           p.D > 128 && p.D <= 8192 && p.w.vec_ok && p.w.fast_ok &&
                           (p.op != RowOp::LayerNorm || (p.bias.vec_ok && p.bias.fast_ok)) &&
                           p.x.m.piece[0].base % 8 == 0 && p.x.m.piece[0].ptr % 16 == 0 &&
                           p.out.m.piece[0].base % 8 == 0 && p.out.m.piece[0].ptr % 16 == 0;
    if (long_rows) {
        const int grid = int(p.rows < 148 * 8 ? p.rows : 148 * 8);
        const int64_t v = (p.D / 8 + 255) / 256;
        if (v <= 1) launch_k(row_long_kernel<1>, dim3(grid), dim3(256), 0, s, dp);
        else if (v <= 2) launch_k(row_long_kernel<2>, dim3(grid), dim3(256), 0, s, dp);
        else launch_k(row_long_kernel<4>, dim3(grid), dim3(256), 0, s, dp);
        return;
    }
    const bool vec_rows = p.dt == KDType::BF16 && p.linear && p.op != RowOp::Softmax && p.D % 32 == 0 && p.D <= 128 &&
                          p.w.fast_ok && (p.op != RowOp::LayerNorm || p.bias.fast_ok) &&
                          p.x.m.piece[0].base % 8 == 0 && p.x.m.piece[0].ptr % 16 == 0 &&
                          p.out.m.piece[0].base % 8 == 0 && p.out.m.piece[0].ptr % 16 == 0;
    if (vec_rows) {
        const int64_t blocks = (p.rows + 63) / 64;
        const int grid = int(blocks < 148 * 8 ? blocks : 148 * 8);
        switch (p.D / 32) {
            case 1: launch_k(row_vec_kernel<1>, dim3(grid), dim3(256), 0, s, dp); break;
            case 2: launch_k(row_vec_kernel<2>, dim3(grid), dim3(256), 0, s, dp); break;
            case 3: launch_k(row_vec_kernel<3>, dim3(grid), dim3(256), 0, s, dp); break;
            default: launch_k(row_vec_kernel<4>, dim3(grid), dim3(256), 0, s, dp); break;
        }
        return;
    }
    const bool warp_rows = p.dt == KDType::BF16 && p.D <= 256 && p.x.fast_ok && p.out.fast_ok &&
                           (p.op == RowOp::Softmax || p.w.fast_ok) && (p.op != RowOp::LayerNorm || p.bias.fast_ok);
    if (warp_rows) {
        int64_t blocks = (p.rows + 7) / 8;
        int grid = int(blocks < 148 * 16 ? blocks : 148 * 16);
        if (p.D <= 128) launch_k(row_warp_kernel<4>, dim3(grid), dim3(256), 0, s, dp);
        else launch_k(row_warp_kernel<8>, dim3(grid), dim3(256), 0, s, dp);
        return;
    }
    int grid = int(p.rows < 148 * 8 ? p.rows : 148 * 8);
    switch (p.dt) {
        case KDType::F64: launch_k(row_kernel<double>, dim3(grid), dim3(256), 0, s, dp); break;
        case KDType::F32: launch_k(row_kernel<float>, dim3(grid), dim3(256), 0, s, dp); break;
        case KDType::BF16: launch_k(row_kernel<bf16>, dim3(grid), dim3(256), 0, s, dp); break;
        default: break;
    }
}

}  // namespace vtc
