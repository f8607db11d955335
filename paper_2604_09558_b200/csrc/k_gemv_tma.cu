// Persistent TMA-fed weight-streaming GEMV for bf16 decode (M <= 4 rows).
//
// C[m, n] (+)= prologue(A)[m, :] . B[:, n]; B (the weight, [K, N] row-major,
// physical) is streamed exactly once from HBM.  One CTA per SM:
//   * warp 8 (producer) walks the CTA's contiguous range of (256-column strip,
//     64-row k-tile) units and issues one cp.async.bulk per weight row
//     segment (512 B) into a STAGES-deep shared-memory ring, signalling an
//     mbarrier with complete_tx -- memory-level parallelism comes from the
//     async copy engine, not from registers;
//   * warps 0-7 (consumers) first stage A through its VirtualTensor map (with
//     the fused RMSNorm / SiLU*Mul prologue, rounding like the unfused ops)
//     while the first stages are already in flight, then FMA each tile out of
//     shared memory (16-byte LDS, 8 columns per lane, 8 rows per warp).
// A strip touched by several CTAs is reduced by the last CTA to finish it, in
// CTA order (deterministic), which also applies the residual epilogue and
// stores C through its map.
#include "device.cuh"
#include "rowreduce.cuh"

namespace vtc {
namespace {

using dev::bf16;
constexpr int CONSUMERS = 8, NT = (CONSUMERS + 1) * 32, COLS = 256, KT = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct Smem {
    static constexpr size_t ring_bytes(int stages) { return size_t(stages) * KT * COLS * sizeof(bf16); }
};

template <int MT>
__global__ void __launch_bounds__(NT, 1) gemv_tma_kernel(const GemvParams* __restrict__ pp) {
    const GemvParams& p = *pp;
    extern __shared__ __align__(128) unsigned char smem[];
    const int stages = p.stages;
    bf16* ring = reinterpret_cast<bf16*>(smem);
    float* sA = reinterpret_cast<float*>(smem + Smem::ring_bytes(stages));        // [M][K]
    float* red = sA + size_t(p.M) * p.K;                                          // [CONSUMERS][COLS]
    uint64_t* full = reinterpret_cast<uint64_t*>(red + CONSUMERS * COLS);
    uint64_t* empty = full + stages;
    __shared__ float s_rs[4];
    __shared__ unsigned s_last;

    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int M = int(p.M);
    const int64_t n_strips = (p.N + COLS - 1) / COLS;
    const int64_t ktiles = (p.K + KT - 1) / KT;
    const int64_t units = n_strips * ktiles;
    const int64_t u_begin = units * blockIdx.x / gridDim.x;
    const int64_t u_end = units * (blockIdx.x + 1) / gridDim.x;

    if (tid == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CONSUMERS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == CONSUMERS) {
        // ---------------- producer ----------------
        const bf16* B = reinterpret_cast<const bf16*>(p.b_base);
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t u = u_begin; u < u_end; ++u) {
            const int64_t strip = u / ktiles, kt = u % ktiles;
            const int64_t n0 = strip * COLS, k0 = kt * KT;
            const int rows = int((int)((p.K - k0) < KT ? (p.K - k0) : KT));
            const uint32_t rowbytes = uint32_t((p.N - n0) < COLS ? (p.N - n0) : COLS) * sizeof(bf16);
            mbar_wait(&empty[stage], phase ^ 1);
            if (lane == 0) mbar_expect_tx(&full[stage], uint32_t(rows) * rowbytes);
            __syncwarp();
            bf16* dst = ring + size_t(stage) * KT * COLS;
            for (int r = lane; r < rows; r += 32)
                bulk_g2s(dst + r * COLS, B + (k0 + r) * p.b_sk + n0, rowbytes, &full[stage]);
            if (++stage == stages) {
                stage = 0;
                phase ^= 1;
            }
        }
        return;
    }

    // ---------------- consumers: A prologue (overlaps the first copies) -------
    const int ctid = tid;  // 0..255
    auto bar_consumers = [] { asm volatile("bar.sync 1, %0;" ::"n"(CONSUMERS * 32)); };
    auto row_ptr = [&](const VOperand& op, int m, int64_t& stride) -> const bf16* {
        int32_t idx[VTC_MAX_RANK] = {};
        idx[0] = m;
        dev::Loc l = dev::locate(op.m, idx);
        stride = op.fast_stride[l.piece];
        return dev::addr<bf16>(op.m, l);
    };
    auto elem = [&](const VOperand& op, int m, int64_t k) -> float {
        int32_t idx[VTC_MAX_RANK] = {};
        idx[0] = m;
        idx[1] = int32_t(k);
        return __bfloat162float(*dev::elem_ptr<bf16>(op.m, idx));
    };
    for (int m = 0; m < M; ++m) {
        int64_t sa = 0, sa2 = 0, sw = 0;
        const bf16* pa = p.a.fast_ok ? row_ptr(p.a, m, sa) : nullptr;
        const bf16* pa2 = (p.prologue == GemvPrologue::SiLUMul && p.a2.fast_ok) ? row_ptr(p.a2, m, sa2) : nullptr;
        const bf16* pw = nullptr;
        float rs = 0.f;
        if (p.prologue == GemvPrologue::RMSNorm) {
            if (p.normw.fast_ok) {
                int32_t widx[VTC_MAX_RANK] = {};
                dev::Loc l = dev::locate(p.normw.m, widx);
                sw = p.normw.fast_stride[l.piece];
                pw = dev::addr<bf16>(p.normw.m, l);
            }
            // same 256-thread reduction order as the standalone RMSNorm kernel
            float ss = block_sum_256_bar1<float>(
                [&](int64_t k) {
                    float v = pa ? __bfloat162float(pa[k * sa]) : elem(p.a, m, k);
                    return v * v;
                },
                p.K);
            if (ctid == 0) s_rs[m] = rsqrtf(ss / float(p.K) + p.eps);
            bar_consumers();
            rs = s_rs[m];
        }
        for (int64_t k = ctid; k < p.K; k += CONSUMERS * 32) {
            float v = pa ? __bfloat162float(pa[k * sa]) : elem(p.a, m, k);
            if (p.prologue == GemvPrologue::SiLUMul) {
                float u = pa2 ? __bfloat162float(pa2[k * sa2]) : elem(p.a2, m, k);
                float sg = __bfloat162float(__float2bfloat16_rn(v / (1.0f + expf(-v))));
                v = __bfloat162float(__float2bfloat16_rn(sg * u));
            } else if (p.prologue == GemvPrologue::RMSNorm) {
                float w;
                if (pw) {
                    w = __bfloat162float(pw[k * sw]);
                } else {
                    int32_t widx[VTC_MAX_RANK] = {};
                    widx[0] = int32_t(k);
                    w = __bfloat162float(*dev::elem_ptr<bf16>(p.normw.m, widx));
                }
                v = __bfloat162float(__float2bfloat16_rn(v * rs * w));
            }
            sA[size_t(m) * p.K + k] = v;
        }
    }
    bar_consumers();

    // ---------------- consumers: stream tiles ----------------
    float acc[MT][8];
    auto zero = [&] {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[m][j] = 0.f;
    };
    zero();
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t u = u_begin; u < u_end; ++u) {
        const int64_t strip = u / ktiles, kt = u % ktiles;
        const int64_t k0 = kt * KT;
        const int rows = int((int)((p.K - k0) < KT ? (p.K - k0) : KT));
        mbar_wait(&full[stage], phase);
        const bf16* tile = ring + size_t(stage) * KT * COLS;
#pragma unroll 4
        for (int r = warp; r < rows; r += CONSUMERS) {
            uint4 w = *reinterpret_cast<const uint4*>(tile + r * COLS + lane * 8);
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
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
                    float a = sA[size_t(m) * p.K + k0 + r];
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[m][j] = fmaf(a, b[j], acc[m][j]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
        }
        const bool strip_end = (kt == ktiles - 1) || (u + 1 == u_end);
        if (!strip_end) continue;

        // ---- this CTA's part of the strip is done: reduce warps -> partial slot ----
        const int64_t n0 = strip * COLS;
        const int first = p.strip_first[strip];
        const int ncontrib = p.strip_count[strip];
        const int slot = int(blockIdx.x) - first;
        float outv[MT];
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            outv[m] = 0.f;
            if (m < M) {
#pragma unroll
                for (int j = 0; j < 8; ++j) red[warp * COLS + lane * 8 + j] = acc[m][j];
                bar_consumers();
                float v = 0.f;
#pragma unroll
                for (int w2 = 0; w2 < CONSUMERS; ++w2) v += red[w2 * COLS + ctid];
                outv[m] = v;
                bar_consumers();
            }
        }
        zero();
        const int64_t n = n0 + ctid;
        bool last = true;
        if (ncontrib > 1) {
            if (n < p.N)
                for (int m = 0; m < M; ++m) p.work[((strip * p.max_contrib + slot) * M + m) * COLS + ctid] = outv[m];
            __threadfence();
            bar_consumers();
            if (ctid == 0) s_last = (atomicAdd(&p.counters[strip], 1u) == unsigned(ncontrib - 1));
            bar_consumers();
            last = s_last != 0;
            if (last) {
                __threadfence();
                if (n < p.N)
                    for (int m = 0; m < M; ++m) {
                        float v = 0.f;
                        for (int s2 = 0; s2 < ncontrib; ++s2)
                            v += __ldcg(&p.work[((strip * p.max_contrib + s2) * M + m) * COLS + ctid]);
                        outv[m] = v;
                    }
                if (ctid == 0) p.counters[strip] = 0u;
            }
        }
        if (!last || n >= p.N) continue;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            if (m >= M) continue;
            int32_t idx[VTC_MAX_RANK] = {};
            idx[0] = m;
            idx[1] = int32_t(n0);
            bf16 c = __float2bfloat16_rn(outv[m]);
            if (p.has_res) {
                float r;
                if (p.res.fast_ok) {
                    dev::Loc l = dev::locate(p.res.m, idx);
                    r = __bfloat162float(dev::addr<bf16>(p.res.m, l)[int64_t(ctid) * p.res.fast_stride[l.piece]]);
                } else {
                    idx[1] = int32_t(n);
                    r = __bfloat162float(*dev::elem_ptr<bf16>(p.res.m, idx));
                    idx[1] = int32_t(n0);
                }
                c = __float2bfloat16_rn(__bfloat162float(c) + r);
            }
            if (p.c.fast_ok) {
                dev::Loc l = dev::locate(p.c.m, idx);
                dev::addr<bf16>(p.c.m, l)[int64_t(ctid) * p.c.fast_stride[l.piece]] = c;
            } else {
                idx[1] = int32_t(n);
                *dev::elem_ptr<bf16>(p.c.m, idx) = c;
            }
        }
    }
}

template <int MT>
void launch_mt(const GemvParams& p, const GemvParams* dp, cudaStream_t s) {
    size_t smem = Smem::ring_bytes(p.stages) + size_t(p.M) * size_t(p.K) * sizeof(float) +
                  size_t(CONSUMERS) * COLS * sizeof(float) + 2 * size_t(p.stages) * sizeof(uint64_t);
    cudaFuncSetAttribute(gemv_tma_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    gemv_tma_kernel<MT><<<p.grid, NT, smem, s>>>(dp);
}

}  // namespace

size_t gemv_tma_smem(int64_t M, int64_t K, int stages) {
    return Smem::ring_bytes(stages) + size_t(M) * size_t(K) * sizeof(float) + size_t(CONSUMERS) * COLS * sizeof(float) +
           2 * size_t(stages) * sizeof(uint64_t);
}

void launch_gemv_tma(const GemvParams& p, const GemvParams* dp, cudaStream_t s) {
    if (p.M <= 1) launch_mt<1>(p, dp, s);
    else if (p.M <= 2) launch_mt<2>(p, dp, s);
    else launch_mt<4>(p, dp, s);
}

}  // namespace vtc
