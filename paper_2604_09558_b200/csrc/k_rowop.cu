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

}  // namespace

void launch_rowop(const RowParams& p, const RowParams* dp, cudaStream_t s) {
    if (p.rows == 0) return;
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
