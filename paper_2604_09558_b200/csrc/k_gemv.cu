// Weight-streaming GEMV / skinny GEMM for bf16 decode (M <= 16 rows).
//
// Replaces matmul_kernel (proj/src/executor.cpp:230-249) for the decode-step
// projections, where the step is bound by streaming the weight matrix B once
// from HBM.  Each CTA owns a 256-column strip of B and a K range; its 8 warps
// walk consecutive rows with 16-byte non-allocating loads, `U` rows in flight
// per warp.  A is staged into shared memory through its VirtualTensor map
// (with an optional fused SiLU*Mul or RMSNorm prologue that reproduces the
// unfused ops' bf16 roundings), C and the optional residual go through theirs.
// Split-K partials are summed in split order by the last CTA to arrive, so the
// result is deterministic and independent of the operand maps.
#include "device.cuh"
#include "launch.cuh"
#include "rowreduce.cuh"

namespace vtc {
namespace {

using dev::bf16;
constexpr int NT = 256, COLS = 256, WARPS = 8;

__device__ __forceinline__ uint4 ld_stream(const void* p, uint64_t policy) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(policy));
    return r;
}

__device__ __forceinline__ float load_bf16_at(const VOperand& op, int32_t (&idx)[VTC_MAX_RANK]) {
    return __bfloat162float(*dev::elem_ptr<bf16>(op.m, idx));
}

template <int MT, int U>
__global__ void __launch_bounds__(NT) gemv_kernel(const GemvParams* __restrict__ pp) {
    VTC_STAGE_PARAMS(GemvParams, pp);
    dev::pdl_wait(); dev::pdl_launch_dependents();
    extern __shared__ float sA[];  // [M][kchunk]
    __shared__ float red[WARPS][COLS];
    __shared__ float s_rs[16];
    __shared__ unsigned s_last;

    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int64_t n0 = int64_t(blockIdx.x) * COLS;
    const int split = blockIdx.y;
    const int64_t kb = int64_t(split) * p.kchunk;
    const int64_t ke = min(p.K, kb + p.kchunk);
    const int klen = int(ke - kb);
    const int M = int(p.M);

    // ---- prologue: A rows -> shared memory (fp32), with fused transforms ----
    // Row origins are evaluated once through the maps; elements step with the
    // per-piece stride along K (host-proved affine over whole rows).
    auto row_ptr = [&](const VOperand& op, int m, int64_t k0, int64_t& stride) -> const bf16* {
        int32_t idx[VTC_MAX_RANK] = {};
        idx[0] = m;
        idx[1] = int32_t(k0);
        dev::Loc l = dev::locate(op.m, idx);
        stride = op.fast_stride[l.piece];
        return dev::addr<bf16>(op.m, l);
    };
    auto a_at = [&](const VOperand& op, int m, int64_t k) -> float {
        if (op.fast_ok) {
            int64_t st;
            const bf16* b0 = row_ptr(op, m, 0, st);
            return __bfloat162float(b0[k * st]);
        }
        int32_t idx[VTC_MAX_RANK] = {};
        idx[0] = m;
        idx[1] = int32_t(k);
        return load_bf16_at(op, idx);
    };
    if (p.prologue == GemvPrologue::RMSNorm) {
        for (int m = 0; m < M; ++m) {
            float ss;
            if (p.a.fast_ok) {
                int64_t st;
                const bf16* b0 = row_ptr(p.a, m, 0, st);
                ss = block_sumsq_bf16_fast<false>(b0, st, p.K);
            } else {
                ss = block_sumsq_row_bf16(p.a, m, p.K);
            }
            if (tid == 0) s_rs[m] = rsqrtf(ss / float(p.K) + p.eps);
        }
        __syncthreads();
    }
    for (int m = 0; m < M; ++m) {
        int64_t sa = 0, sa2 = 0, sw = 0;
        const bf16* pa = p.a.fast_ok ? row_ptr(p.a, m, kb, sa) : nullptr;
        const bf16* pa2 = (p.prologue == GemvPrologue::SiLUMul && p.a2.fast_ok) ? row_ptr(p.a2, m, kb, sa2) : nullptr;
        const bf16* pw = nullptr;
        if (p.prologue == GemvPrologue::RMSNorm && p.normw.fast_ok) {
            int32_t widx[VTC_MAX_RANK] = {};
            widx[0] = int32_t(kb);
            dev::Loc l = dev::locate(p.normw.m, widx);
            sw = p.normw.fast_stride[l.piece];
            pw = dev::addr<bf16>(p.normw.m, l);
        }
#pragma unroll 4
        for (int e = tid; e < klen; e += NT) {
            int64_t k = kb + e;
            float v = pa ? __bfloat162float(pa[e * sa]) : a_at(p.a, m, k);
            if (p.prologue == GemvPrologue::SiLUMul) {
                float u = pa2 ? __bfloat162float(pa2[e * sa2]) : a_at(p.a2, m, k);
                float sg = __bfloat162float(__float2bfloat16_rn(dev::silu_f(v)));
                v = __bfloat162float(__float2bfloat16_rn(sg * u));
            } else if (p.prologue == GemvPrologue::RMSNorm) {
                float w;
                if (pw) {
                    w = __bfloat162float(pw[e * sw]);
                } else {
                    int32_t widx[VTC_MAX_RANK] = {};
                    widx[0] = int32_t(k);
                    w = load_bf16_at(p.normw, widx);
                }
                v = __bfloat162float(__float2bfloat16_rn(v * s_rs[m] * w));
            }
            sA[m * klen + e] = v;
        }
    }
    __syncthreads();

    // ---- stream B ----
    float acc[MT][8];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[m][j] = 0.f;
    const int64_t col = n0 + lane * 8;
    const bool col_ok = col < p.N;
    const bf16* bcol = reinterpret_cast<const bf16*>(p.b_base) + col;
    const uint64_t policy = dev::evict_first_policy();
    for (int base = 0; base < klen; base += WARPS * U) {
        uint4 w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int k = base + u * WARPS + warp;
            if (k < klen && col_ok) w[u] = ld_stream(bcol + (kb + k) * p.b_sk, policy);
            else w[u] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int k = base + u * WARPS + warp;
            if (k < klen) {
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[u]);
                float b[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float2 f = __bfloat1622float2(h[j]);
                    b[2 * j] = f.x;
                    b[2 * j + 1] = f.y;
                }
#pragma unroll
                for (int m = 0; m < MT; ++m) {
                    if (m < M) {
                        float a = sA[m * klen + k];
#pragma unroll
                        for (int j = 0; j < 8; ++j) acc[m][j] = fmaf(a, b[j], acc[m][j]);
                    }
                }
            }
        }
    }

    // ---- reduce the 8 warps, then the K splits ----
    float outv[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) {
        outv[m] = 0.f;
        if (m < M) {
#pragma unroll
            for (int j = 0; j < 8; ++j) red[warp][lane * 8 + j] = acc[m][j];
            __syncthreads();
            float v = 0.f;
#pragma unroll
            for (int w2 = 0; w2 < WARPS; ++w2) v += red[w2][tid];
            outv[m] = v;
            __syncthreads();
        }
    }
    const int64_t n = n0 + tid;
    if (p.ksplit > 1) {
        if (n < p.N)
            for (int m = 0; m < M; ++m) p.work[(int64_t(split) * M + m) * p.N + n] = outv[m];
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = (atomicAdd(&p.counters[blockIdx.x], 1u) == unsigned(p.ksplit - 1));
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        if (n < p.N)
            for (int m = 0; m < M; ++m) {
                float v = 0.f;
                for (int s2 = 0; s2 < p.ksplit; ++s2) v += __ldcg(&p.work[(int64_t(s2) * M + m) * p.N + n]);
                outv[m] = v;
            }
        if (tid == 0) p.counters[blockIdx.x] = 0u;
    }
    if (n >= p.N) return;
    // ---- epilogue: C = bf16(acc) [+ residual, rounded like an unfused Add] ----
    // strip origins evaluated once per row; columns step with the piece stride
#pragma unroll
    for (int m = 0; m < MT; ++m) {
        if (m >= M) continue;
        int32_t idx[VTC_MAX_RANK] = {};
        idx[0] = m;
        idx[1] = int32_t(n);
        bf16 c = __float2bfloat16_rn(outv[m]);
        if (p.has_res) {
            float r;
            if (p.res.fast_ok) {
                int64_t st;
                const bf16* r0 = row_ptr(p.res, m, n0, st);
                r = __bfloat162float(r0[int64_t(tid) * st]);
            } else {
                r = load_bf16_at(p.res, idx);
            }
            c = __float2bfloat16_rn(__bfloat162float(c) + r);
        }
        if (p.c.fast_ok) {
            int64_t st;
            bf16* c0 = const_cast<bf16*>(row_ptr(p.c, m, n0, st));
            c0[int64_t(tid) * st] = c;
        } else {
            *dev::elem_ptr<bf16>(p.c.m, idx) = c;
        }
    }
}

template <int MT, int U>
void launch_mt(const GemvParams& p, const GemvParams* dp, cudaStream_t s) {
    dim3 grid(unsigned((p.N + COLS - 1) / COLS), unsigned(p.ksplit));
    size_t smem = size_t(p.M) * size_t(p.kchunk) * sizeof(float);
    if (smem > 48 * 1024) allow_max_smem(gemv_kernel<MT, U>);
    launch_k(gemv_kernel<MT, U>, dim3(grid), dim3(NT), smem, s, dp);
}

}  // namespace

void launch_gemv(const GemvParams& p, const GemvParams* dp, cudaStream_t s) {
    if (p.M <= 1) launch_mt<1, 8>(p, dp, s);
    else if (p.M <= 2) launch_mt<2, 8>(p, dp, s);
    else if (p.M <= 4) launch_mt<4, 4>(p, dp, s);
    else if (p.M <= 8) launch_mt<8, 4>(p, dp, s);
    else launch_mt<16, 2>(p, dp, s);
}

}  // namespace vtc
