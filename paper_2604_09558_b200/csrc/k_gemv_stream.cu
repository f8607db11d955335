// Persistent TMA-streamed weight GEMV for bf16 decode (M <= 4 rows).
//
// C[m, n] (+)= prologue(A)[m, :] . B[:, n] -- the decode-step projections of a
// VTC-planned decoder layer (the reference computes them with matmul_kernel,
// proj/src/executor.cpp:230-249).  The step is bound by streaming the weights
// once from HBM, so the kernel is organised around keeping HBM busy:
//
//   * one CTA per SM; the weight matrix is cut into units of one 64-row x
//     256-column tile (32 KB) and each CTA owns a contiguous range of units in
//     (strip, k-tile) order;
//   * warp 8 is the producer: one elected thread issues one 2-D TMA load
//     (cp.async.bulk.tensor) per unit into a STAGES-deep shared-memory ring,
//     completion signalled through mbarrier transaction counts;
//   * weights are static for the plan, so the producer starts streaming BEFORE
//     griddepcontrol.wait: under programmatic dependent launch the first
//     stages land while the previous kernel (attention, the previous GEMV)
//     is still draining;
//   * warps 0-7 wait for the previous kernel, stage their k-range of A through
//     its VirtualTensor map (with the fused RMSNorm / SiLU*Mul prologue,
//     rounding exactly like the unfused operators), then consume tiles with
//     16-byte LDS (8 columns per lane, 8 rows per warp per tile);
//   * a strip shared by several CTAs is reduced by the last CTA to finish it,
//     in CTA order (deterministic), which applies the residual epilogue and
//     stores C through its map.
// Up to two weight matrices that share A (sibling MatMuls such as gate/up)
// run as one launch.
#include <cuda.h>

#include <cstring>

#include "device.cuh"
#include "launch.cuh"
#include "rowreduce.cuh"

namespace vtc {
namespace {

using dev::bf16;
constexpr int CONSUMERS = 8, NT = (CONSUMERS + 1) * 32, COLS = GEMV_STREAM_COLS, KT = GEMV_STREAM_KT;
constexpr uint32_t TILE_BYTES = KT * COLS * sizeof(bf16);
static_assert(KT == 64, "a_col_to_k assumes 64-row k-tiles");

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
// Weights are read exactly once per step: stream them with an L2 evict-first
// policy so they do not push code, parameters and activations out of L2.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int32_t c0, int32_t c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 1, %0;" ::"n"(CONSUMERS * 32) : "memory"); }

template <int MT>
__global__ void __launch_bounds__(NT, 1) gemv_stream_kernel(const GemvParams* __restrict__ pp,
                                                             const __grid_constant__ GemvChainArgs ca) {
    VTC_STAGE_PARAMS(GemvParams, pp);
    extern __shared__ __align__(1024) unsigned char smem[];
    const int stages = ca.ring;
    bf16* ring = reinterpret_cast<bf16*>(smem);
    float* sA = reinterpret_cast<float*>(smem + size_t(stages) * TILE_BYTES);  // [M][a_tiles*KT] (max over stages)
    float* red = sA + ca.sA_floats;                                              // [CONSUMERS][COLS]
    uint64_t* full = reinterpret_cast<uint64_t*>(red + CONSUMERS * COLS);
    uint64_t* empty = full + stages;
    __shared__ uint64_t go;  // consumers have issued their activation loads
    __shared__ float s_rs[4];
    __shared__ unsigned s_last, s_gen;

    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;

    if (tid == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CONSUMERS);
        }
        mbar_init(&go, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    dev::pdl_launch_dependents();

    if (warp == CONSUMERS) {
        // ---------------- producer ----------------
        if (lane != 0) return;
        const uint64_t policy = dev::evict_first_policy();
        int stage = 0;
        uint32_t phase = 0;
        // one continuous ring over every chained stage: weights are static, so
        // the next stage's first tiles stream while this CTA still waits for
        // the previous stage's outputs
        for (int cs = 0; cs < ca.nst; ++cs) {
            const GemvChainStage& h = ca.st[cs];
            const CUtensorMap* tmc = reinterpret_cast<const CUtensorMap*>(ca.tmap[cs][0]);
            for (int mt = 0; mt < h.nmat; ++mt)
                asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmc[mt])) : "memory");
            const int64_t ktiles = (h.K + KT - 1) / KT;
            const int64_t strips1 = h.nmat > 1 ? (h.n1 + COLS - 1) / COLS : 0;
            const int64_t units = (int64_t(h.strips0) + strips1) * ktiles;
            const int64_t u_begin = units * blockIdx.x / gridDim.x;
            const int64_t u_end = units * (blockIdx.x + 1) / gridDim.x;
            int64_t u_pre = INT64_MAX;
            if (cs == 0) {
                if (h.b_static) {
                    // the weights do not depend on earlier launches: pull this CTA's
                    // first tiles into L2 while the previous launch is still running
                    const int64_t pf_end = u_begin + h.l2_prefetch < u_end ? u_begin + h.l2_prefetch : u_end;
                    int64_t strip = u_begin / ktiles, kt = u_begin % ktiles;
                    for (int64_t u = u_begin; u < pf_end; ++u) {
                        if (u != u_begin && ++kt == ktiles) {
                            kt = 0;
                            ++strip;
                        }
                        const int mat = strip < h.strips0 ? 0 : 1;
                        const int64_t n0 = (strip - (mat ? h.strips0 : 0)) * COLS;
                        if (u >= u_begin + h.pre_stages) tma_prefetch_2d(&tmc[mat], int32_t(n0), int32_t(kt * KT));
                    }
                } else {
                    dev::pdl_wait();
                }
                // Only PRE tiles go out before the consumers have issued their
                // activation loads: a full ring of weight requests queued ahead of
                // them would put every activation load behind ~MBs of HBM traffic.
                u_pre = u_begin + (h.pre_stages < stages ? h.pre_stages : stages);
            } else if (h.l2_prefetch > 0) {
                // chained stage: while the previous stage drains (epilogue, this
                // stage's dependency wait and prologue), pull the tiles just past
                // the ring into L2 so HBM stays busy across the boundary
                const int64_t pf_beg = u_begin + stages < u_end ? u_begin + stages : u_end;
                const int64_t pf_end = pf_beg + h.l2_prefetch < u_end ? pf_beg + h.l2_prefetch : u_end;
                for (int64_t u = pf_beg; u < pf_end; ++u) {
                    const int64_t strip = u / ktiles, kt = u % ktiles;
                    const int mat = strip < h.strips0 ? 0 : 1;
                    const int64_t n0 = (strip - (mat ? h.strips0 : 0)) * COLS;
                    tma_prefetch_2d(&tmc[mat], int32_t(n0), int32_t(kt * KT));
                }
            }
            int64_t strip = u_begin / ktiles, kt = u_begin % ktiles;
            for (int64_t u = u_begin; u < u_end; ++u) {
                if (u == u_pre) mbar_wait(&go, 0);
                if (u != u_begin && ++kt == ktiles) {
                    kt = 0;
                    ++strip;
                }
                const int mat = strip < h.strips0 ? 0 : 1;
                const int64_t n0 = (strip - (mat ? h.strips0 : 0)) * COLS;
                mbar_wait(&empty[stage], phase ^ 1);
                mbar_expect_tx(&full[stage], TILE_BYTES);
                tma_load_2d(ring + size_t(stage) * KT * COLS, &tmc[mat], int32_t(n0), int32_t(kt * KT), &full[stage], policy);
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        return;
    }

    // consumers: the ring position carries across chained stages
    int stage = 0;
    uint32_t phase = 0;
    const int ctid = tid;  // 0..255
    for (int cs = 0; cs < ca.nst; ++cs) {
    if (cs > 0) {
        // next stage: its parameter block replaces the previous one (consumers only)
        bar_consumers();
        {
            const uint4* src = reinterpret_cast<const uint4*>(pp + cs);
            uint4* dst = reinterpret_cast<uint4*>(s_params_);
            constexpr int n = int((sizeof(GemvParams) + 15) / 16);
            for (int i = ctid; i < n; i += CONSUMERS * 32) dst[i] = __ldg(src + i);
        }
        // wait until what this stage reads from earlier stages is published
        if (ctid == 0) {
            const GemvChainStage& h = ca.st[cs];
            const unsigned target = s_gen + 1u;
            auto wait_flag = [&](const unsigned* f) {
                unsigned v;
                long long spins = 0;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                    if (int(v - target) >= 0) break;
                    __nanosleep(20);
                    if (++spins > (1ll << 27)) __trap();  // a lost dependency: fail loudly, never hang
                }
            };
            for (int j = 0; j < cs; ++j) {
                if (!((h.dep_all >> j) & 1u)) continue;
                const GemvChainStage& hj = ca.st[j];
                const int ns = hj.strips0 + (hj.nmat > 1 ? int((hj.n1 + COLS - 1) / COLS) : 0);
                for (int t = 0; t < ns; ++t) wait_flag(ca.sync + 2 + int64_t(j) * ca.max_strips + t);
            }
            if (h.dep_range) {
                // k-tiles this CTA stages: (kt_first + i) mod ktiles, i < its unit count
                const GemvChainStage& hp = ca.st[cs - 1];
                const int64_t ktiles = (h.K + KT - 1) / KT;
                const int64_t strips1 = h.nmat > 1 ? (h.n1 + COLS - 1) / COLS : 0;
                const int64_t units = (int64_t(h.strips0) + strips1) * ktiles;
                const int64_t u_begin = units * blockIdx.x / gridDim.x;
                const int64_t u_end = units * (blockIdx.x + 1) / gridDim.x;
                const int64_t nk = u_end - u_begin < ktiles ? u_end - u_begin : ktiles;
                int last_strip = -1;
                for (int64_t i = 0; i < nk; ++i) {
                    const int64_t kt = (u_begin % ktiles + i) % ktiles;
                    const int ps = int(kt * KT / COLS);  // producing strip of matrix 0
                    if (ps == last_strip) continue;
                    last_strip = ps;
                    wait_flag(ca.sync + 2 + int64_t(cs - 1) * ca.max_strips + ps);
                    if (h.dep_a2) wait_flag(ca.sync + 2 + int64_t(cs - 1) * ca.max_strips + hp.strips0 + ps);
                }
            }
        }
        bar_consumers();
    }
    const int M = int(p.M);
    const int64_t ktiles = (p.K + KT - 1) / KT;
    const int64_t strips1 = p.nmat > 1 ? (p.n_mat[1] + COLS - 1) / COLS : 0;
    const int64_t units = (int64_t(p.strips0) + strips1) * ktiles;
    const int64_t u_begin = units * blockIdx.x / gridDim.x;
    const int64_t u_end = units * (blockIdx.x + 1) / gridDim.x;

    // ---------------- consumers: A prologue (overlaps the first weight tiles) ----
    if (cs == 0) {
        if (tid == 0) dev::trace_point(p.head, 4);  // parameters staged, barriers ready
        dev::pdl_wait();
        if (tid == 0) dev::trace_point(p.head, 5);  // dependency resolved
        if (ctid == 0 && ca.nst > 1) s_gen = *reinterpret_cast<volatile unsigned*>(ca.sync);
    }
    const int64_t kt_first = u_begin % ktiles;
    const int64_t a_cols = int64_t(p.a_tiles) * KT;
    // staged column e of A -> k: k-tile (kt_first + e / 64) mod ktiles, no 64-bit
    // division in the prologue loops (a division call there serialises the loads)
    const int kt_first32 = int(kt_first), ktiles32 = int(ktiles);
    auto a_col_to_k = [&](int64_t e) -> int64_t {
        const int ee = int(e);
        int kt = kt_first32 + (ee >> 6);
        if (kt >= ktiles32) kt -= ktiles32;
        return int64_t(kt) * KT + (ee & (KT - 1));
    };
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
    bool go_sent = cs > 0;  // chained stages: the producer does not wait for `go`
    auto send_go = [&] {
        if (go_sent) return;
        go_sent = true;
        bar_consumers();  // every consumer thread has issued its loads (they are in flight)
        if (ctid == 0) mbar_arrive(&go);
    };
    constexpr int XR = 16, EV = 8;  // register budgets of the fast prologue
    for (int m = 0; m < M; ++m) {
        int64_t sa = 0, sa2 = 0, sw = 0;
        const bf16 *pa = nullptr, *pa2 = nullptr, *pw = nullptr;
        if (p.rows_ok) {
            pa = static_cast<const bf16*>(p.arow[m]);
            sa = p.sa[m];
            if (p.prologue == GemvPrologue::SiLUMul) {
                pa2 = static_cast<const bf16*>(p.a2row[m]);
                sa2 = p.sa2[m];
            }
            if (p.prologue == GemvPrologue::RMSNorm) {
                pw = static_cast<const bf16*>(p.wrow);
                sw = p.sw;
            }
        } else {
        pa = p.a.fast_ok ? row_ptr(p.a, m, sa) : nullptr;
        pa2 = (p.prologue == GemvPrologue::SiLUMul && p.a2.fast_ok) ? row_ptr(p.a2, m, sa2) : nullptr;
        if (p.prologue == GemvPrologue::RMSNorm && p.normw.fast_ok) {
            int32_t widx[VTC_MAX_RANK] = {};
            dev::Loc l = dev::locate(p.normw.m, widx);
            sw = p.normw.fast_stride[l.piece];
            pw = dev::addr<bf16>(p.normw.m, l);
        }
        }
        if (ctid == 0) dev::trace_point(p.head, 7);  // operand rows located
        const bool fast = pa && (p.prologue != GemvPrologue::SiLUMul || pa2) && (p.prologue != GemvPrologue::RMSNorm || pw);
        const bool regs = fast && (p.prologue != GemvPrologue::RMSNorm || p.K <= XR * 256) && a_cols <= EV * 256;
        float rs = 0.f;
        // 16-byte path: unit-stride, 16-B aligned operands; 8 elements per load,
        // every load of the row issued (as raw bits) before any is converted
        const bool vec = fast && p.a.vec_ok && (p.prologue != GemvPrologue::SiLUMul || p.a2.vec_ok) &&
                         (p.prologue != GemvPrologue::RMSNorm || (p.normw.vec_ok && p.K <= 4 * 2048)) &&
                         a_cols <= 2 * 8 * 256 && p.K % 8 == 0;
        if (vec) {
            constexpr int XV = 4, AV = 2;
            uint4 xq[XV], aq[AV], bq[AV];
            const uint4 z4 = make_uint4(0, 0, 0, 0);
            if (p.prologue == GemvPrologue::RMSNorm) {
#pragma unroll
                for (int j = 0; j < XV; ++j) {
                    const int64_t k = (ctid + int64_t(j) * 256) * 8;
                    xq[j] = k < p.K ? *reinterpret_cast<const uint4*>(pa + k) : z4;
                }
            }
#pragma unroll
            for (int i = 0; i < AV; ++i) {
                const int64_t e = (ctid + int64_t(i) * 256) * 8;
                const int64_t k = e < a_cols ? a_col_to_k(e) : p.K;
                const bool ok = k < p.K;
                aq[i] = ok ? *reinterpret_cast<const uint4*>(pa + k) : z4;
                bq[i] = z4;
                if (p.prologue == GemvPrologue::SiLUMul && ok) bq[i] = *reinterpret_cast<const uint4*>(pa2 + k);
                if (p.prologue == GemvPrologue::RMSNorm && ok) bq[i] = *reinterpret_cast<const uint4*>(pw + k);
            }
            send_go();
            auto unpack = [](const uint4& q, float (&f)[8]) {
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    float2 v2 = __bfloat1622float2(h[t]);
                    f[2 * t] = v2.x;
                    f[2 * t + 1] = v2.y;
                }
            };
            if (p.prologue == GemvPrologue::RMSNorm) {
                float s = 0.f;
#pragma unroll
                for (int j = 0; j < XV; ++j) {
                    float f[8];
                    unpack(xq[j], f);
#pragma unroll
                    for (int t = 0; t < 8; ++t) s += f[t] * f[t];
                }
                rs = rsqrtf(block_sum_regs_bar1(s) / float(p.K) + p.eps);
                if (ctid == 0) dev::trace_point(p.head, 6);  // norm reduction done
            }
#pragma unroll
            for (int i = 0; i < AV; ++i) {
                const int64_t e = (ctid + int64_t(i) * 256) * 8;
                if (e >= a_cols) continue;
                float v[8], u[8];
                unpack(aq[i], v);
                unpack(bq[i], u);
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    if (p.prologue == GemvPrologue::SiLUMul) {
                        const float sg = __bfloat162float(__float2bfloat16_rn(dev::silu_f(v[t])));
                        v[t] = __bfloat162float(__float2bfloat16_rn(sg * u[t]));
                    } else if (p.prologue == GemvPrologue::RMSNorm) {
                        v[t] = __bfloat162float(__float2bfloat16_rn(v[t] * rs * u[t]));
                    }
                }
                float4* dst = reinterpret_cast<float4*>(sA + size_t(m) * a_cols + e);
                dst[0] = make_float4(v[0], v[1], v[2], v[3]);
                dst[1] = make_float4(v[4], v[5], v[6], v[7]);
            }
            continue;
        }
        if (regs) {
            // phase 1: issue every load of this row (registers), then let the producer go
            float xr[XR], av[EV], a2v[EV], wv[EV];
            if (p.prologue == GemvPrologue::RMSNorm) {
#pragma unroll
                for (int j = 0; j < XR; ++j) {
                    const int64_t k = ctid + int64_t(j) * 256;
                    xr[j] = k < p.K ? __bfloat162float(pa[k * sa]) : 0.f;
                }
            }
#pragma unroll
            for (int i = 0; i < EV; ++i) {
                const int64_t e = ctid + int64_t(i) * 256;
                const int64_t k = a_col_to_k(e);
                const bool ok = e < a_cols && k < p.K;
                av[i] = ok ? __bfloat162float(pa[k * sa]) : 0.f;
                if (p.prologue == GemvPrologue::SiLUMul) a2v[i] = ok ? __bfloat162float(pa2[k * sa2]) : 0.f;
                if (p.prologue == GemvPrologue::RMSNorm) wv[i] = ok ? __bfloat162float(pw[k * sw]) : 0.f;
            }
            send_go();
            // phase 2: RMSNorm statistics in block_sum_256's exact order
            if (p.prologue == GemvPrologue::RMSNorm) {
                float s = 0.f;
#pragma unroll
                for (int j = 0; j < XR; ++j)
                    if (ctid + int64_t(j) * 256 < p.K) s += xr[j] * xr[j];
                const float ss = block_sum_regs_bar1(s);
                rs = rsqrtf(ss / float(p.K) + p.eps);
                if (ctid == 0) dev::trace_point(p.head, 6);  // norm reduction done
            }
#pragma unroll
            for (int i = 0; i < EV; ++i) {
                const int64_t e = ctid + int64_t(i) * 256;
                if (e >= a_cols) continue;
                float v = av[i];
                if (p.prologue == GemvPrologue::SiLUMul) {
                    const float sg = __bfloat162float(__float2bfloat16_rn(dev::silu_f(v)));
                    v = __bfloat162float(__float2bfloat16_rn(sg * a2v[i]));
                } else if (p.prologue == GemvPrologue::RMSNorm) {
                    v = __bfloat162float(__float2bfloat16_rn(v * rs * wv[i]));
                }
                sA[size_t(m) * a_cols + e] = v;
            }
            continue;
        }
        send_go();
        if (fast) {
            // long k-ranges (e.g. gate+up: ~3K columns per CTA): batches of 8
            // elements per thread with every load of a batch in flight together
            if (p.prologue == GemvPrologue::RMSNorm) {
                const float ss = block_sumsq_bf16_fast<true>(pa, sa, p.K);
                rs = rsqrtf(ss / float(p.K) + p.eps);
            }
            for (int64_t e0 = ctid; e0 < a_cols; e0 += 8 * CONSUMERS * 32) {
                float v[8], u[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int64_t e = e0 + int64_t(j) * CONSUMERS * 32;
                    const int64_t k = a_col_to_k(e);
                    const bool ok = e < a_cols && k < p.K;
                    v[j] = ok ? __bfloat162float(pa[k * sa]) : 0.f;
                    u[j] = 0.f;
                    if (p.prologue == GemvPrologue::SiLUMul) u[j] = ok ? __bfloat162float(pa2[k * sa2]) : 0.f;
                    if (p.prologue == GemvPrologue::RMSNorm) u[j] = ok ? __bfloat162float(pw[k * sw]) : 0.f;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int64_t e = e0 + int64_t(j) * CONSUMERS * 32;
                    if (e >= a_cols) continue;
                    float x = v[j];
                    if (p.prologue == GemvPrologue::SiLUMul) {
                        const float sg = __bfloat162float(__float2bfloat16_rn(dev::silu_f(x)));
                        x = __bfloat162float(__float2bfloat16_rn(sg * u[j]));
                    } else if (p.prologue == GemvPrologue::RMSNorm) {
                        x = __bfloat162float(__float2bfloat16_rn(x * rs * u[j]));
                    }
                    sA[size_t(m) * a_cols + e] = x;
                }
            }
            continue;
        }
        if (p.prologue == GemvPrologue::RMSNorm) {
            // the same 256-thread reduction order as the standalone RMSNorm kernel
            float ss = pa ? block_sumsq_bf16_fast<true>(pa, sa, p.K)
                          : block_sum_256_bar1<float>(
                                [&](int64_t k) {
                                    float v = elem(p.a, m, k);
                                    return v * v;
                                },
                                p.K);
            if (ctid == 0) s_rs[m] = rsqrtf(ss / float(p.K) + p.eps);
            bar_consumers();
            rs = s_rs[m];
        }
        for (int64_t e = ctid; e < a_cols; e += CONSUMERS * 32) {
            const int64_t k = a_col_to_k(e);
            float v = 0.f;
            if (k < p.K) {
                v = pa ? __bfloat162float(pa[k * sa]) : elem(p.a, m, k);
                if (p.prologue == GemvPrologue::SiLUMul) {
                    float u = pa2 ? __bfloat162float(pa2[k * sa2]) : elem(p.a2, m, k);
                    float sg = __bfloat162float(__float2bfloat16_rn(dev::silu_f(v)));
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
            }
            sA[size_t(m) * a_cols + e] = v;
        }
    }
    send_go();
    bar_consumers();
    if (ctid == 0) dev::trace_point(p.head, 2);  // A prologue done

    // ---------------- consumers: stream tiles ----------------
    float acc[MT][8];
    auto zero = [&] {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[m][j] = 0.f;
    };
    zero();
    // publish a finished strip of a chained stage (its outputs are stored)
    auto strip_done = [&](int64_t strip) {
        if (ca.nst <= 1) return;
        __threadfence();
        bar_consumers();
        if (ctid == 0) atomicAdd(ca.sync + 2 + int64_t(cs) * ca.max_strips + strip, 1u);
    };
    // store a finished strip: fused trees or residual epilogue, through C's map
    // pe0 / pin0: row 0's epilogue entry and its external inputs, loaded before the
    // split-K exchange so the tail has no dependent table / input round trips
    auto finish_strip = [&](int64_t strip, const float (&outv)[MT], const EpiEntry* pe0, const float* pin0) {
        const int mat = strip < p.strips0 ? 0 : 1;
        const int64_t n0 = (strip - (mat ? p.strips0 : 0)) * COLS;
        const int64_t Nl = p.n_mat[mat];
        const int64_t n = n0 + ctid;
        if (p.has_epi) {
            // fused elementwise trees: the strip's bf16 outputs in shared memory,
            // then every element either evaluates its tree or is stored plainly
            float* sC = red;  // [M][COLS] (the warp-reduction buffer is free again)
            for (int m = 0; m < M; ++m) sC[m * COLS + ctid] = __bfloat162float(__float2bfloat16_rn(outv[m]));
            bar_consumers();
            if (n < Nl)
                for (int m = 0; m < M; ++m) {
                    const EpiEntry& e = (m == 0 && pe0) ? *pe0 : p.epi[int64_t(m) * Nl + n];
                    if (e.tree < 0) {
                        int32_t idx[VTC_MAX_RANK] = {};
                        idx[0] = m;
                        idx[1] = int32_t(n);
                        *dev::elem_ptr<bf16>(p.c.m, idx) = __float2bfloat16_rn(sC[m * COLS + ctid]);
                        continue;
                    }
                    const EpiTree& t = p.epi_tree[e.tree];
                    float r[EW_MAX_IN + EW_MAX_PROG];
#pragma unroll
                    for (int j = 0; j < EPI_MAX_IN; ++j) {
                        if (j >= t.nin) break;
                        r[j] = (e.cmask >> j) & 1u ? sC[m * COLS + int(int64_t(e.in[j]) - n0)]
                               : (m == 0 && pe0) ? pin0[j]
                                                 : __bfloat162float(*reinterpret_cast<const bf16*>(e.in[j]));
                    }
                    for (int s2 = 0; s2 < t.nprog; ++s2) {
                        const EwInstr ins = t.prog[s2];
                        const float a = r[ins.a], b = r[ins.b];
                        float v;
                        switch (ins.op) {  // bf16 rounding after every op, as the unfused kernel
                            case EwOp::Add: v = a + b; break;
                            case EwOp::Mul: v = a * b; break;
                            case EwOp::SiLU: v = dev::silu_f(a); break;
                            case EwOp::GELU: v = 0.5f * a * (1.0f + erff(a * 0.70710678f)); break;
                            default: v = a; break;
                        }
                        r[ins.dst] = __bfloat162float(__float2bfloat16_rn(v));
                    }
                    *reinterpret_cast<bf16*>(e.out + ((e.cmask & EPI_DYN_OUT) ? uint64_t(p.epi_shift) : 0ull)) =
                        __float2bfloat16_rn(r[t.result]);
                }
            bar_consumers();  // sC is the reduction buffer of the next strip
            strip_done(strip);
            return;
        }
        const VOperand& cop = mat ? p.c2 : p.c;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            if (m >= M || n >= Nl) continue;
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
            if (cop.fast_ok) {
                dev::Loc l = dev::locate(cop.m, idx);
                dev::addr<bf16>(cop.m, l)[int64_t(ctid) * cop.fast_stride[l.piece]] = c;
            } else {
                idx[1] = int32_t(n);
                *dev::elem_ptr<bf16>(cop.m, idx) = c;
            }
        }
        strip_done(strip);
    };
    int64_t strip = u_begin / ktiles, kt = u_begin % ktiles, slot = -1;
    for (int64_t u = u_begin; u < u_end; ++u) {
        if (++slot == ktiles) slot = 0;  // slot = (kt - kt_first) mod ktiles
        if (u != u_begin && ++kt == ktiles) {
            kt = 0;
            ++strip;
        }
        const float* arow = sA + slot * KT;
        mbar_wait(&full[stage], phase);
        const bf16* tile = ring + size_t(stage) * KT * COLS;
        uint4 w[KT / CONSUMERS];
#pragma unroll
        for (int i = 0; i < KT / CONSUMERS; ++i)
            w[i] = *reinterpret_cast<const uint4*>(tile + (warp + i * CONSUMERS) * COLS + lane * 8);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);  // the tile is in registers: release the slot
        if (++stage == stages) {
            stage = 0;
            phase ^= 1;
        }
#pragma unroll
        for (int i = 0; i < KT / CONSUMERS; ++i) {
            const int r = warp + i * CONSUMERS;
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w[i]);
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
                    const float a = arow[size_t(m) * a_cols + r];
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[m][j] = fmaf(a, b[j], acc[m][j]);
                }
            }
        }
        const bool strip_end = (kt == ktiles - 1) || (u + 1 == u_end);
        if (!strip_end) continue;
        if (ctid == 0 && u + 1 == u_end) dev::trace_point(p.head, 3);  // last tile consumed

        // ---- this CTA's part of the strip is done: reduce warps ----
        const int ncontrib = p.strip_count[strip];
        const int cslot = int(blockIdx.x) - p.strip_first[strip];
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
        EpiEntry pe0;
        float pin0[EPI_MAX_IN];
        bool have0 = false;
        if (p.has_epi) {
            const int mat = strip < p.strips0 ? 0 : 1;
            const int64_t n = (strip - (mat ? p.strips0 : 0)) * COLS + ctid;
            if (n < p.n_mat[mat]) {
                pe0 = p.epi[n];
                if (pe0.tree >= 0) {
                    const EpiTree& t = p.epi_tree[pe0.tree];
#pragma unroll
                    for (int j = 0; j < EPI_MAX_IN; ++j)
                        pin0[j] = (j < t.nin && !((pe0.cmask >> j) & 1u))
                                      ? __bfloat162float(*reinterpret_cast<const bf16*>(pe0.in[j]))
                                      : 0.f;
                }
                have0 = true;
            }
        }
        if (ncontrib > 1) {
            // shared strip: the last contributor to arrive sums every slot in CTA order
            for (int m = 0; m < M; ++m) p.work[((strip * p.max_contrib + cslot) * M + m) * COLS + ctid] = outv[m];
            __threadfence();
            bar_consumers();
            if (ctid == 0) s_last = (atomicAdd(&p.counters[strip], 1u) == unsigned(ncontrib - 1));
            bar_consumers();
            if (!s_last) continue;
            __threadfence();
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                float v = 0.f;
                if (m < M)
                    for (int s2 = 0; s2 < ncontrib; ++s2)
                        v += __ldcg(&p.work[((strip * p.max_contrib + s2) * M + m) * COLS + ctid]);
                outv[m] = v;
            }
            if (ctid == 0) p.counters[strip] = 0u;
        }
        finish_strip(strip, outv, have0 ? &pe0 : nullptr, pin0);
    }
    }  // chained stages
    if (ca.nst > 1) {
        // the last CTA out advances the launch generation the flags are compared against
        bar_consumers();
        if (ctid == 0) {
            __threadfence();
            if (atomicAdd(ca.sync + 1, 1u) == gridDim.x - 1) {
                ca.sync[1] = 0u;
                __threadfence();
                atomicAdd(ca.sync, 1u);
            }
        }
    }
}

template <int MT>
void launch_mt(const GemvChainArgs& ca, const GemvParams* dp, int grid, cudaStream_t s) {
    allow_max_smem(gemv_stream_kernel<MT>);
    launch_k(gemv_stream_kernel<MT>, dim3(grid), dim3(NT), gemv_chain_smem(ca.sA_floats, ca.ring), s, dp, ca);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

size_t gemv_stream_smem(int64_t M, int a_tiles, int stages) {
    size_t bytes = size_t(stages) * TILE_BYTES + size_t(M) * size_t(a_tiles) * KT * sizeof(float) +
                   size_t(CONSUMERS) * COLS * sizeof(float) + 2 * size_t(stages) * sizeof(uint64_t);
    // + the statically allocated parameter copy; 227 KB per CTA in total
    return bytes + sizeof(GemvParams) + 12 * 1024 <= 227 * 1024 ? bytes : 0;
}

bool encode_weight_tmap(void* out128, const void* base, int64_t rows, int64_t cols, int64_t ld) {
    static EncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return EncodeFn(nullptr);
        return reinterpret_cast<EncodeFn>(f);
    }();
    if (!fn || (reinterpret_cast<uintptr_t>(base) % 16) != 0 || (ld * 2) % 16 != 0) return false;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(ld) * 2};
    cuuint32_t box[2] = {COLS, KT};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(reinterpret_cast<CUtensorMap*>(out128), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

size_t gemv_chain_smem(int64_t sA_floats, int ring) {
    return size_t(ring) * TILE_BYTES + size_t(sA_floats) * sizeof(float) + size_t(CONSUMERS) * COLS * sizeof(float) +
           2 * size_t(ring) * sizeof(uint64_t);
}

void launch_gemv_chain(const GemvChainArgs& ca, const GemvParams* dp, int64_t M, int grid, cudaStream_t s) {
    if (M <= 1) launch_mt<1>(ca, dp, grid, s);
    else if (M <= 2) launch_mt<2>(ca, dp, grid, s);
    else launch_mt<4>(ca, dp, grid, s);
}

void launch_gemv_stream(const GemvParams& p, const GemvParams* dp, cudaStream_t s) {
    GemvChainArgs ca{};
    std::memcpy(ca.tmap[0], p.tmap, sizeof(p.tmap));
    GemvChainStage& h = ca.st[0];
    h.K = p.K;
    h.n0 = p.n_mat[0];
    h.n1 = p.nmat > 1 ? p.n_mat[1] : 0;
    h.nmat = p.nmat;
    h.strips0 = p.strips0;
    h.b_static = p.b_static;
    h.pre_stages = p.pre_stages;
    h.l2_prefetch = p.l2_prefetch;
    ca.nst = 1;
    ca.ring = p.stages;
    ca.sA_floats = p.M * int64_t(p.a_tiles) * KT;
    launch_gemv_chain(ca, dp, p.M, p.grid, s);
}

}  // namespace vtc
