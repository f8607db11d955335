// Persistent tcgen05 GEMM for shallow-K, narrow-N bf16 projections at large M
// (Swin-T's QKV / proj / fc1 / fc2: K, N <= 384, M = 200,704 window tokens).
//
// C[M, N] = epilogue(A[M, K] . W[K, N]) -- the reference's matmul_kernel
// (proj/src/executor.cpp:230-249) -- where the whole weight fits in shared
// memory.  Such GEMMs are HBM-bound (2-8 flop per byte) and their cost is the
// epilogue, so the kernel is built around keeping stores and loads streaming:
//
//   * one CTA per SM loops over 128-row tiles; the weight is loaded once per
//     CTA and kept in shared memory, transposed to the K-major 128-byte-swizzled
//     UMMA layout (any 8-row-aligned N slice is then a valid B descriptor);
//   * warp 0 streams A: TMA (a plain 2-D view) or 16-byte cp.async gathers
//     through host-resolved row addresses (a virtual roll + window partition),
//     into a ring of 128 x 64 k-tile slots;
//   * warp 1 issues tcgen05.mma M128 x NC x K16 into one of two TMEM
//     accumulators (a tile's N columns in `nchunks` units of NC <= 256), so the
//     next unit's MMAs overlap this unit's epilogue;
//   * warps 2-9 drain the accumulator (two warps per TMEM lane quadrant, half
//     the columns each), round to bf16 (optionally GELU), stage the unit in
//     shared memory and copy it out with coalesced 16-byte stores through the
//     output rows, adding the residual (rounded like the unfused Add).
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "device.cuh"
#include "launch.cuh"

namespace vtc {
namespace {

using dev::bf16;
constexpr int BM = 128, BK = 64, UK = 16, NPROD_NORM = 8;
constexpr int GATHER_LAG = 3;  // gathered k-tiles in flight before the oldest is published
constexpr uint32_t SLOT_BYTES = BM * BK * 2;

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
template <int NE>
__device__ __forceinline__ void bar_epi() { asm volatile("bar.sync 1, %0;" ::"n"(NE * 32) : "memory"); }

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: start >> 4, LBO (unused
// for swizzled K-major) = 16 B, SBO = 1024 B between 8-row groups, version 1.
__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t(1) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
// kind::f16 instruction descriptor: D f32, A / B bf16, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
// byte offset of element (row, k) of a [rows][64] K-major SW128 tile
__device__ __forceinline__ uint32_t sw128(int row, int k) {
    return uint32_t(row) * 128u + ((uint32_t((k >> 3) ^ (row & 7))) << 4) + uint32_t(k & 7) * 2u;
}

// NE epilogue warps; NORM: the A operand is a row normalisation (LayerNorm / RMSNorm over
// K <= 128) of host-resolved input rows, computed by NPROD_NORM producer warps
template <int NE, bool NORM>
__global__ void __launch_bounds__((2 + NE + (NORM ? NPROD_NORM - 1 : 0)) * 32, 1)
    gemm_skinny_kernel(const __grid_constant__ SkinnyParams p) {
    constexpr int NEPI = NE, NTHREADS = (2 + NE + (NORM ? NPROD_NORM - 1 : 0)) * 32;
    dev::TraceScope trace_scope_(&p.head);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int KT = p.kt, S = p.slots, NC = p.nc, NCH = p.nchunks;
    const int NP = (int(p.N) + 7) / 8 * 8;
    unsigned char* sB = smem;                                   // [KT][NP rows][128 B]
    unsigned char* sA = sB + size_t(KT) * NP * 128;             // S slots of [128][128 B]
    unsigned char* sC = sA + size_t(S) * SLOT_BYTES;            // [128][NC + 8] bf16 staging
    const int cpitch = NC + 8;                                  // elements per staged row
    __shared__ uint64_t a_full[16], a_empty[16], acc_full[2], acc_empty[2];
    __shared__ uint32_t s_tmem;
    __shared__ uint64_t s_arow[BM];  // gather: row addresses of the producer's current tile

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t mtiles = (p.M + BM - 1) / BM;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&a_full[s], NORM ? NPROD_NORM : p.a_gather ? 32 : 1);
            mbar_init(&a_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], NEPI);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // two accumulators of up to 256 fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    dev::pdl_launch_dependents();
    // the weight, transposed into K-major swizzled k-tiles: an item is a pair of weight rows
    // (k, k + 1) x 8 columns (two 16-byte loads) stored as 8 (k, k + 1) words of B rows
    // n .. n + 7. Consecutive lanes take consecutive k pairs of one column group, so each
    // 32-bit store instruction fills one 128-byte B row (no bank conflict); a thread issues
    // all loads of a batch before its stores (one memory round trip per batch).
    if (!p.b_static) dev::pdl_wait();
    {
        const int ngrp = (int(p.N) + 7) / 8, kpairs = KT * BK / 2;
        const int total = kpairs * ngrp;
        constexpr int UB = 4;
        const bf16* w = static_cast<const bf16*>(p.w);
        for (int i0 = threadIdx.x; i0 < total; i0 += UB * NTHREADS) {
            uint4 v[UB][2];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int i = i0 + u * NTHREADS;
                const int g = i / kpairs, k = 2 * (i - g * kpairs);
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    v[u][h] = (i < total && k + h < p.K) ? __ldg(reinterpret_cast<const uint4*>(w + int64_t(k + h) * p.ldw + g * 8))
                                                         : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int i = i0 + u * NTHREADS;
                if (i >= total) break;
                const int g = i / kpairs, k = 2 * (i - g * kpairs);
                const uint32_t tile = smem_u32(sB + size_t(k / BK) * NP * 128);
                const uint32_t* e0 = reinterpret_cast<const uint32_t*>(&v[u][0]);
                const uint32_t* e1 = reinterpret_cast<const uint32_t*>(&v[u][1]);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int n = g * 8 + j;
                    const uint32_t lo = (j & 1) ? (e0[j >> 1] >> 16) : (e0[j >> 1] & 0xffffu);
                    const uint32_t hi = (j & 1) ? (e1[j >> 1] & 0xffff0000u) : (e1[j >> 1] << 16);
                    if (n < NP) asm volatile("st.shared.u32 [%0], %1;" ::"r"(tile + sw128(n, k % BK)), "r"(lo | hi));
                }
            }
        }
    }
    __shared__ __align__(16) float s_nw[128], s_nb[128];  // NORM: weight / bias (fp32)
    if (NORM) {
        for (int k = threadIdx.x; k < p.K; k += NTHREADS) {
            s_nw[k] = __bfloat162float(static_cast<const bf16*>(p.norm_w)[k]);
            s_nb[k] = p.a_norm == 1 ? __bfloat162float(static_cast<const bf16*>(p.norm_b)[k]) : 0.f;
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;

    if (NORM && (warp == 0 || warp >= 2 + NEPI)) {
        // ---------------- normalising A producers ----------------
        // producer pi owns rows [16 pi, 16 pi + 16) of every tile: 4 lanes per row, lane q
        // holding 16-byte chunks q, q + 4, q + 8, ... -- the arithmetic of the row_vec
        // kernel (k_rowop.cu), so the fused and unfused normalisations round identically
        dev::pdl_wait();
        const int pi = warp == 0 ? 0 : warp - (2 + NEPI) + 1;
        const int q = lane % 4, U = int(p.K) / 32;
        const bool ln = p.a_norm == 1;
        int g = 0;
        for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
            const int64_t m0 = mt * BM;
            for (int kt = 0; kt < KT; ++kt) {
                const int s = (g + kt) % S;
                mbar_wait(&a_empty[s], (((g + kt) / S) & 1) ^ 1u);
            }
            {  // both of this lane's rows loaded before either is normalised
            uint4 raw[2][4];
#pragma unroll
            for (int pp = 0; pp < 2; ++pp) {
                const int64_t m = m0 + pi * 16 + pp * 8 + lane / 4;
                const uint4* xr = m < p.M ? reinterpret_cast<const uint4*>(p.a_rows[m]) : nullptr;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (u < U && xr) raw[pp][u] = __ldcs(xr + q + 4 * u);
            }
#pragma unroll
            for (int pp = 0; pp < 2; ++pp) {
                const int r = pi * 16 + pp * 8 + lane / 4;
                float x[4][8];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[pp][u]);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const float2 v = __bfloat1622float2(h[t]);
                        x[u][2 * t] = u < U ? v.x : 0.f;
                        x[u][2 * t + 1] = u < U ? v.y : 0.f;
                    }
                }
                float mu = 0.f;
                if (ln) {
                    float sm = 0.f;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (u < U)
#pragma unroll
                            for (int t = 0; t < 8; ++t) sm += x[u][t];
                    sm += __shfl_xor_sync(0xffffffffu, sm, 1);
                    sm += __shfl_xor_sync(0xffffffffu, sm, 2);
                    mu = sm / float(p.K);
                }
                float s2 = 0.f;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (u < U)
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            const float c = x[u][t] - mu;
                            s2 += c * c;
                        }
                s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
                s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
                const float rs = rsqrtf(s2 / float(p.K) + p.eps);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (u >= U) break;
                    const int c = q + 4 * u;  // 16-byte chunk of the row: k = 8c .. 8c + 7
                    uint4 o;
                    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int k = c * 8 + 2 * t;
                        float o0, o1;
                        if (ln) {
                            o0 = ((x[u][2 * t] - mu) * rs) * s_nw[k] + s_nb[k];
                            o1 = ((x[u][2 * t + 1] - mu) * rs) * s_nw[k + 1] + s_nb[k + 1];
                        } else {
                            o0 = (x[u][2 * t] * rs) * s_nw[k];
                            o1 = (x[u][2 * t + 1] * rs) * s_nw[k + 1];
                        }
                        h[t] = __floats2bfloat162_rn(o0, o1);
                    }
                    const int s = (g + c / 8) % S;
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(sA + size_t(s) * SLOT_BYTES) +
                                                                            sw128(r, (c % 8) * 8)),
                                 "r"(o.x), "r"(o.y), "r"(o.z), "r"(o.w)
                                 : "memory");
                }
            }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0)
                for (int kt = 0; kt < KT; ++kt) mbar_arrive(&a_full[(g + kt) % S]);
            g += KT;
        }
    } else if (warp == 0) {
        // ---------------- A producer ----------------
        if (p.b_static) dev::pdl_wait();
        int g = 0;  // global k-tile counter -> slot g % S, phase (g / S) & 1
        if (!p.a_gather) {
            if (lane == 0) {
                asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap_a)) : "memory");
                const uint64_t pol = dev::evict_first_policy();  // A is read once
                for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x)
                    for (int kt = 0; kt < KT; ++kt, ++g) {
                        const int s = g % S;
                        mbar_wait(&a_empty[s], ((g / S) & 1) ^ 1u);
                        mbar_expect_tx(&a_full[s], SLOT_BYTES);
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
                            " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(sA + size_t(s) * SLOT_BYTES)),
                            "l"(reinterpret_cast<uint64_t>(&p.tmap_a)), "r"(kt * BK), "r"(int32_t(mt * BM)),
                            "r"(smem_u32(&a_full[s])), "l"(pol)
                            : "memory");
                    }
            }
        } else {
            // gathers: 128 rows x 8 chunks of 16 B per k-tile, one lane per chunk column;
            // GATHER_LAG k-tiles stay in flight: slot g - LAG is published once its copies landed
            int oldest = 0;  // oldest k-tile not yet published
            for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
                const int64_t m0 = mt * BM;
                // the tile's 128 row addresses: one coalesced round trip, then from shared memory
                __syncwarp();
#pragma unroll
                for (int q = 0; q < BM / 32; ++q) {
                    const int64_t m = m0 + q * 32 + lane;
                    s_arow[q * 32 + lane] = m < p.M ? p.a_rows[m] : 0;
                }
                __syncwarp();
                for (int kt = 0; kt < KT; ++kt, ++g) {
                    const int s = g % S;
                    mbar_wait(&a_empty[s], ((g / S) & 1) ^ 1u);
                    const uint32_t base = smem_u32(sA + size_t(s) * SLOT_BYTES);
#pragma unroll 8
                    for (int j = 0; j < (BM * 8) / 32; ++j) {
                        const int c = lane + 32 * j, row = c >> 3, ch = c & 7;
                        const int64_t m = m0 + row, k = int64_t(kt) * BK + ch * 8;
                        const bool ok = m < p.M && k < p.K;
                        const void* src = ok ? reinterpret_cast<const void*>(s_arow[row] + uint64_t(k) * 2) : p.w;
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(base + sw128(row, ch * 8)),
                                     "l"(src), "r"(ok ? 16 : 0)
                                     : "memory");
                    }
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    if (g - oldest + 1 > GATHER_LAG) {
                        asm volatile("cp.async.wait_group %0;" ::"n"(GATHER_LAG) : "memory");
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        mbar_arrive(&a_full[oldest % S]);
                        ++oldest;
                    }
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (; oldest < g; ++oldest) mbar_arrive(&a_full[oldest % S]);
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            const uint32_t id = idesc(BM, NC);
            int g = 0, u = 0;
            for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
                const int g0 = g;
                for (int j = 0; j < NCH; ++j, ++u) {
                    const int b = u & 1;
                    mbar_wait(&acc_empty[b], ((u >> 1) & 1) ^ 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    for (int kt = 0; kt < KT; ++kt) {
                        const int gs = g0 + kt, s = gs % S;
                        if (j == 0) {
                            mbar_wait(&a_full[s], (gs / S) & 1);
                            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        }
                        const uint32_t sa = smem_u32(sA + size_t(s) * SLOT_BYTES);
                        const uint32_t sb = smem_u32(sB + size_t(kt) * NP * 128 + size_t(j) * NC * 128);
                        const int ksteps = min(BK, int(p.K) - kt * BK) / UK;
                        for (int k = 0; k < ksteps; ++k) {
                            const uint32_t acc = (kt > 0 || k > 0) ? 1u : 0u;
                            asm volatile(
                                "{\n.reg .pred q;\nsetp.ne.b32 q, %4, 0;\n"
                                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n}\n" ::"r"(tmem + uint32_t(b * 256)),
                                "l"(kdesc(sa + k * 32)), "l"(kdesc(sb + k * 32)), "r"(id), "r"(acc)
                                : "memory");
                        }
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(&acc_full[b]))
                                 : "memory");
                }
                // every chunk of this tile has been issued: its A slots free once they complete
                for (int kt = 0; kt < KT; ++kt)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(&a_empty[(g0 + kt) % S]))
                                 : "memory");
                g += KT;
            }
        }
    } else if (warp < 2 + NEPI) {
        // ---------------- epilogue: warps 2 .. NEPI + 1 ----------------
        dev::pdl_wait();
        const int et = threadIdx.x - 64;        // 0 .. NEPI * 32 - 1
        const int quad = warp & 3;              // TMEM lanes 32*quad .. +31 (hardware rule: warp id mod 4)
        const int part = (warp - 2) >> 2;       // NEPI / 4 warps per quadrant: column parts
        const int row = quad * 32 + lane;
        constexpr int PARTS = NEPI / 4;  // warps per TMEM lane quadrant
        const int hc = (NC / PARTS + 7) / 8 * 8;  // columns per part, multiple of 8
        const int c_lo = part * hc, c_hi = min(NC, c_lo + hc);
        bf16* srow = reinterpret_cast<bf16*>(sC) + size_t(row) * cpitch;
        const int cpr = NC / 8;                  // 16-byte chunks per output row
        int u = 0;
        for (int64_t mt = blockIdx.x; mt < mtiles; mt += gridDim.x) {
            const int64_t m0 = mt * BM;
            for (int j = 0; j < NCH; ++j, ++u) {
                const int b = u & 1;
                mbar_wait(&acc_full[b], (u >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t taddr = tmem + (uint32_t(quad * 32) << 16) + uint32_t(b * 256);
                for (int c = c_lo; c < c_hi; c += 8) {
                    uint32_t r[8];
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                                   "=r"(r[7])
                                 : "r"(taddr + uint32_t(c)));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    uint32_t o[4];
                    if (p.epi == 1) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) o[q] = dev::gelu2_acc(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(o[q]) : "r"(r[2 * q + 1]), "r"(r[2 * q]));
                    }
                    *reinterpret_cast<uint4*>(srow + c) = make_uint4(o[0], o[1], o[2], o[3]);
                }
                // accumulator drained: the MMA warp may refill it
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[b]);
                bar_epi<NEPI>();  // the unit is staged
                // coalesced copy-out: consecutive threads take consecutive 16-byte chunks of a row;
                // a thread's chunks (and their residual chunks) are loaded before any is stored
                const int64_t n0 = int64_t(j) * NC;
                constexpr int CH = 4;  // chunks per thread per round
                for (int i0 = et; i0 < BM * cpr; i0 += CH * NEPI * 32) {
                    uint4 v[CH], rv[CH];
                    int64_t mm[CH];
                    int cc[CH];
#pragma unroll
                    for (int q = 0; q < CH; ++q) {
                        const int i = i0 + q * NEPI * 32;
                        const int rr = i / cpr;
                        cc[q] = i - rr * cpr;
                        mm[q] = (i < BM * cpr) ? m0 + rr : p.M;
                        if (mm[q] < p.M) {
                            v[q] = *reinterpret_cast<const uint4*>(reinterpret_cast<const bf16*>(sC) + size_t(rr) * cpitch + cc[q] * 8);
                            if (p.has_res) {
                                const bf16* rp = p.r_rows ? reinterpret_cast<const bf16*>(p.r_rows[mm[q]])
                                                          : reinterpret_cast<const bf16*>(p.r_base) + mm[q] * p.r_ld;
                                rv[q] = __ldg(reinterpret_cast<const uint4*>(rp + n0 + cc[q] * 8));
                            }
                        }
                    }
#pragma unroll
                    for (int q = 0; q < CH; ++q) {
                        if (mm[q] >= p.M) continue;
                        if (p.has_res) {
                            const bf16* a = reinterpret_cast<const bf16*>(&rv[q]);
                            bf16* x = reinterpret_cast<bf16*>(&v[q]);
#pragma unroll
                            for (int e = 0; e < 8; ++e) x[e] = dev::add_bf16(a[e], x[e]);
                        }
                        bf16* cp = p.c_rows ? reinterpret_cast<bf16*>(p.c_rows[mm[q]]) : reinterpret_cast<bf16*>(p.c_base) + mm[q] * p.c_ld;
                        *reinterpret_cast<uint4*>(cp + n0 + cc[q] * 8) = v[q];
                    }
                }
                bar_epi<NEPI>();  // staging free for the next unit
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encoder() {
    static EncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return EncodeFn(nullptr);
        return reinterpret_cast<EncodeFn>(f);
    }();
    return fn;
}

}  // namespace

bool skinny_plan(SkinnyParams& p, int smem_optin) {
    if (p.K % UK || p.N % 16 || p.K > 512 || p.N > 1024) return false;
    p.kt = int((p.K + BK - 1) / BK);
    // N in units of NC <= 256 (two accumulators in 512 TMEM columns), NC a multiple of 16
    int nch = 1;
    while (nch <= 8 && (p.N % nch || (p.N / nch) % 16 || p.N / nch > 256)) ++nch;
    if (nch > 8) return false;
    p.nchunks = nch;
    p.nc = int(p.N / nch);
    const int64_t np = (p.N + 7) / 8 * 8;
    const int64_t fixed = int64_t(p.kt) * np * 128 + int64_t(BM) * (p.nc + 8) * 2 + 1024;
    // a tile's k-tiles stay resident until its last chunk: at least kt slots, two tiles' worth if they fit
    int slots = int((smem_optin - 1024 - fixed) / SLOT_BYTES);
    if (slots > 16) slots = 16;
    const int need = p.nchunks > 1 ? p.kt : 2;
    if (slots < need) return false;
    if (slots > 2 * p.kt && p.nchunks > 1) slots = std::max(2 * p.kt, std::min(slots, 4 * p.kt));
    p.slots = slots;
    p.smem = size_t(fixed + int64_t(slots) * SLOT_BYTES);
    return true;
}

bool skinny_encode_a(SkinnyParams& p, const void* a_base, int64_t lda) {
    EncodeFn fn = encoder();
    if (!fn || (reinterpret_cast<uintptr_t>(a_base) % 16) || (lda * 2) % 16) return false;
    cuuint64_t dims[2] = {cuuint64_t(p.K), cuuint64_t(p.M)};
    cuuint64_t str[1] = {cuuint64_t(lda) * 2};
    cuuint32_t box[2] = {BK, BM}, es[2] = {1, 1};
    return fn(reinterpret_cast<CUtensorMap*>(p.tmap_a), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a_base), dims,
              str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_gemm_skinny(const SkinnyParams& p, const SkinnyParams*, cudaStream_t s) {
    const int64_t mtiles = (p.M + BM - 1) / BM;
    const unsigned grid = unsigned(std::min<int64_t>(mtiles, p.sms));
    if (p.a_norm) {
        constexpr int NE = 8;
        allow_max_smem(gemm_skinny_kernel<NE, true>);
        launch_k(gemm_skinny_kernel<NE, true>, dim3(grid), dim3((2 + NE + NPROD_NORM - 1) * 32), p.smem, s, p);
    } else {
        constexpr int NE = 16;
        allow_max_smem(gemm_skinny_kernel<NE, false>);
        launch_k(gemm_skinny_kernel<NE, false>, dim3(grid), dim3((2 + NE) * 32), p.smem, s, p);
    }
}

}  // namespace vtc
