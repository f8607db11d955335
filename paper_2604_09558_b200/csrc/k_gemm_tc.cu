// bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// C[M, N] = A[M, K] . B[K, N] (+ residual), bf16 in, fp32 accumulation, the
// reference's matmul_kernel (proj/src/executor.cpp:230-249) for the projection
// GEMMs of a VTC-planned decoder at batch / prefill sizes (M > 16).
//
//   * A is read by TMA through its VirtualTensor map when the map is one
//     affine piece with unit stride along K (the map's row stride becomes the
//     TMA row pitch, its base the TMA origin -- a split / slice / reshape view
//     of the producer's buffer costs nothing); K-major, 128-byte swizzle;
//   * B (the weight, [K, N] row-major) is the MN-major UMMA operand: four
//     64-column TMA boxes per stage, 128-byte swizzle;
//   * one CTA per 128 x BN output tile (split along K when the tile grid is
//     smaller than the SM count): warp 0 = TMA producer, warp 1 = MMA issuer
//     (one thread issues tcgen05.mma M128 x N x K16 into a TMEM accumulator,
//     tcgen05.commit releases the smem stage), warps 0-3 = epilogue
//     (tcgen05.ld 32x32b -> registers -> bf16 -> the output map, with the
//     optional fused residual Add rounded like the unfused operator);
//   * K splits write fp32 partial tiles; the last CTA of a tile sums them in
//     split order (deterministic) and runs the epilogue.
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "device.cuh"
#include "launch.cuh"

namespace vtc {
namespace {

using dev::bf16;
constexpr int BM = 128, BK = 64, UK = 16, NTHREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar,
                                       uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tma_nd(void* dst, const CUtensorMap* map, const int32_t (&c)[5], int nd, uint64_t* bar,
                                       uint64_t policy) {
    const uint32_t d = smem_u32(dst), b = smem_u32(bar);
    const uint64_t m = reinterpret_cast<uint64_t>(map);
    switch (nd) {
        case 2:
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
                "{%2, %3}], [%4], %5;" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(b), "l"(policy)
                : "memory");
            break;
        case 3:
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
                "{%2, %3, %4}], [%5], %6;" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(b), "l"(policy)
                : "memory");
            break;
        case 4:
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
                "{%2, %3, %4, %5}], [%6], %7;" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(b), "l"(policy)
                : "memory");
            break;
        default:
            asm volatile(
                "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
                "{%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]),
                "r"(b), "l"(policy)
                : "memory");
            break;
    }
}
__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// UMMA shared-memory matrix descriptor: start >> 4 [0,14), LBO >> 4 [16,30),
// SBO >> 4 [32,46), version 1 [46,48), layout SWIZZLE_128B = 2 [61,64).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
// kind::f16 instruction descriptor: D f32, A/B bf16, A K-major, B MN-major.
__host__ __device__ constexpr uint32_t instr_desc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) | (uint32_t(n >> 3) << 17) |
           (uint32_t(m >> 4) << 24);
}

struct Tmaps {
    CUtensorMap a, b, b2;
};

// MT = 128-row sub-tiles per CTA (2: a 256 x BN tile whose two M=128 MMAs
// share each B stage -- half the B traffic per FLOP for prefill-sized M)
// threads per CTA: 4 warps, or 8 for the 256-row tiles (warps 4-7 join the epilogue, each
// warp draining half of its TMEM lane quadrant's columns)
template <int MT>
constexpr int tc_threads() { return MT == 2 ? 256 : NTHREADS; }

// The general case of the epilogue's 16-column emit (strided or unaligned output / residual, a
// partial last column group): out of line, so the common path stays short.
__device__ __noinline__ void emit_slow(bf16* dst, int64_t cs, const bf16* rrow, int64_t rs, int c, int ncols,
                                       const float* v, bool gelu) {
#pragma unroll 1
    for (int j = 0; j < 16; ++j) {
        if (c + j >= ncols) break;
        bf16 o;
        if (gelu) {
            o = dev::gelu_bf16(__float2bfloat16_rn(v[j]));
        } else {
            float f = __bfloat162float(__float2bfloat16_rn(v[j]));
            if (rrow) f = __bfloat162float(rrow[int64_t(c + j) * rs]) + f;
            o = __float2bfloat16_rn(f);
        }
        dst[int64_t(j) * cs] = o;
    }
}

template <int BN, int STAGES, int MT, int EPI>
__global__ void __launch_bounds__(tc_threads<MT>(), 1) gemm_tc_kernel(const GemmTcParams* __restrict__ pp,
                                                                       const __grid_constant__ Tmaps tm) {
    VTC_STAGE_PARAMS(GemmTcParams, pp);
    constexpr int NHALF = tc_threads<MT>() / NTHREADS;  // column groups per TMEM lane quadrant
    constexpr int TM = BM * MT;
    // output columns per tile: SwiGLU tiles hold gate and up halves of BN / 2 each
    constexpr int ON = EPI == GEMM_EPI_SWIGLU ? BN / 2 : BN;
    constexpr uint32_t A_SUB = BM * BK * 2, A_BYTES = A_SUB * MT, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[STAGES], empty[STAGES], done;
    __shared__ uint32_t s_tmem;
    __shared__ unsigned s_last;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tiles_n0 = int((p.N + ON - 1) / ON);
    const int tiles_n = tiles_n0 + (p.nmat > 1 ? int((p.N1 + BN - 1) / BN) : 0);
    const int tiles_m = int((p.M + TM - 1) / TM);
    const int tile = blockIdx.x;
    // grouped rasterisation: consecutive CTAs walk GROUP_M row tiles of one
    // column tile, so the CTAs in flight share a few A row blocks and B column
    // blocks through L2 (A and B are re-read by every tile of their row / column)
    constexpr int GROUP_M = 16;
    const int in_group = GROUP_M * tiles_n;
    const int first_m = (tile / in_group) * GROUP_M;
    const int gm = min(tiles_m - first_m, GROUP_M);
    const int tm_ = first_m + (tile % in_group) % gm, tn = (tile % in_group) / gm;
    const int mat = tn >= tiles_n0 ? 1 : 0;  // horizontally fused sibling (gate / up)
    const int64_t m0 = int64_t(tm_) * TM, n0 = int64_t(mat ? tn - tiles_n0 : tn) * ON;
    const int64_t Nm = mat ? p.N1 : p.N;
    const CUtensorMap* tmb = mat ? &tm.b2 : &tm.b;
    const int split = blockIdx.y;
    const int ktiles = int((p.K + BK - 1) / BK);
    const int kt0 = int(int64_t(ktiles) * split / p.splits), kt1 = int(int64_t(ktiles) * (split + 1) / p.splits);
    const int nk = kt1 - kt0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], p.a_gather ? 33 : 1);  // gather: + one arrival per loader lane
            mbar_init(&empty[s], 1);
        }
        mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {  // TMEM accumulator: 128 lanes x BN fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(BN * MT));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    dev::pdl_launch_dependents();
    const unsigned long long t_start = dev::gtime();

    if (warp == 0 && p.a_gather) {
        // ---------------- gather producer (A not TMA-readable) ----------------
        // A's rows are located once through its map (row base, unit stride
        // along K); every k-tile is then 1024 16-byte cp.asyncs written in the
        // 128-byte-swizzled layout TMA would produce.  B still comes by TMA.
        // row bases of the current K segment (re-read from the table when a k-tile
        // enters the next segment; static shared memory stays at one row table)
        __shared__ const bf16* s_arow[BM];
        const int nseg = p.a_rows ? p.a_nseg : 1;
        auto rows_of = [&](int sg) {
            for (int r = lane; r < BM; r += 32) {
                const int64_t m = m0 + r;
                const bf16* rp = nullptr;
                if (m < p.M) {
                    if (p.a_rows) {
                        rp = reinterpret_cast<const bf16*>(p.a_rows[int64_t(sg) * p.M + m]);
                    } else {
                        int32_t idx[VTC_MAX_RANK] = {};
                        idx[0] = int32_t(m);
                        rp = dev::elem_ptr<bf16>(p.a.m, idx);
                    }
                }
                s_arow[r] = rp;
            }
        };
        int seg = 0;
        while (seg + 1 < nseg && kt0 * BK >= p.a_seg_k[seg + 1]) ++seg;
        rows_of(seg);
        const uint64_t pol_b = tiles_m == 1 ? dev::evict_first_policy() : evict_last_policy();
        if (lane == 0) dev::trace_add(p.head, 5, dev::gtime() - t_start);  // sum over CTAs: rows located
        dev::pdl_wait();
        __syncwarp();
        const unsigned long long t_rows = dev::gtime();
        for (int i = 0; i < nk; ++i) {
            const int s = i % STAGES;
            const uint32_t ph = uint32_t(i / STAGES) & 1u;
            mbar_wait(&empty[s], ph ^ 1u);
            unsigned char* sa = smem + size_t(s) * STAGE_BYTES;
            unsigned char* sb = sa + A_BYTES;
            const int32_t k0 = int32_t(kt0 + i) * BK;  // all CTAs walk K in step: weight rows stream DRAM page by page
            if (seg + 1 < nseg && k0 >= p.a_seg_k[seg + 1]) {  // this k-tile starts the next K segment
                // the previous tiles' gathers still read s_arow: let them land first
                asm volatile("cp.async.wait_group 0;" ::: "memory");
                __syncwarp();
                while (seg + 1 < nseg && k0 >= p.a_seg_k[seg + 1]) ++seg;
                rows_of(seg);
                __syncwarp();
            }
            if (lane == 0) {
                mbar_expect_tx(&full[s], B_BYTES);
#pragma unroll
                for (int j = 0; j < BN / 64; ++j) {
                    if (EPI == GEMM_EPI_SWIGLU && j >= BN / 128)
                        tma_2d(sb + j * (BK * 128), &tm.b2, int32_t(n0 + 64 * (j - BN / 128)), k0, &full[s], pol_b);
                    else
                        tma_2d(sb + j * (BK * 128), tmb, int32_t(n0 + 64 * j), k0, &full[s], pol_b);
                }
            }
            const uint32_t sa_u = smem_u32(sa);
#pragma unroll 8
            for (int j = 0; j < (BM * 8) / 32; ++j) {
                const int c = lane + 32 * j;
                const int row = c >> 3, ch = c & 7;
                const bf16* rp = s_arow[row];
                const int64_t k = int64_t(k0) + ch * 8;
                const bool ok = rp != nullptr && k < p.K;
                const void* src = ok ? static_cast<const void*>(rp + k) : static_cast<const void*>(s_arow);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa_u + row * 128 + ((ch ^ (row & 7)) << 4)),
                             "l"(src), "r"(ok ? 16 : 0)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            if (i > 0) {
                // k-tile i-1 has landed (one group stays in flight: consecutive k-tiles' gathers overlap)
                asm volatile("cp.async.wait_group 1;" ::: "memory");
                // generic-proxy smem writes must be visible to the tensor core's async proxy
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[(i - 1) % STAGES])) : "memory");
            }
        }
        if (nk > 0) {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[(nk - 1) % STAGES])) : "memory");
        }
        if (lane == 0) dev::trace_add(p.head, 6, dev::gtime() - t_rows);  // sum over CTAs: gathers issued + landed
    } else if (warp == 0 && lane == 0) {
        // ---------------- TMA producer ----------------
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm.a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmb)) : "memory");
        // decode-sized M (one row tile): weights are read exactly once -> evict-first;
        // prefill: every row tile re-reads them -> keep them in L2
        const uint64_t pol_b = tiles_m == 1 ? dev::evict_first_policy() : evict_last_policy();
        const uint64_t pol_a = evict_last_policy();  // activations: re-read by every N tile
        // A's TMA coordinates: M dimensions are fixed for the CTA; K dimensions
        // advance incrementally by one 64-wide k-tile per stage (no division in the loop)
        int32_t cm[MT][5], ck[5], sub[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) {
#pragma unroll
            for (int t = 0; t < MT; ++t) {
                const uint32_t v = uint32_t(m0 + t * BM) / uint32_t(p.a_div[j]);
                cm[t][j] = int32_t(p.a_mod[j] ? v % uint32_t(p.a_mod[j]) : v);
            }
            const uint32_t kb = uint32_t(kt0) * BK, dv = uint32_t(p.a_div[j]);
            const uint32_t v = kb / dv;
            ck[j] = int32_t(p.a_mod[j] ? v % uint32_t(p.a_mod[j]) : v);
            sub[j] = int32_t(kb % dv);
        }
        dev::pdl_wait();  // A is produced by earlier kernels
        for (int i = 0; i < nk; ++i) {
            const int s = i % STAGES;
            const uint32_t ph = uint32_t(i / STAGES) & 1u;
            mbar_wait(&empty[s], ph ^ 1u);
            mbar_expect_tx(&full[s], STAGE_BYTES);
            unsigned char* sa = smem + size_t(s) * STAGE_BYTES;
            unsigned char* sb = sa + A_BYTES;
            const int32_t k0 = int32_t(kt0 + i) * BK;  // all CTAs walk K in step: weight rows stream DRAM page by page
#pragma unroll
            for (int t = 0; t < MT; ++t) {
                int32_t ca[5];
#pragma unroll
                for (int j = 0; j < 5; ++j) ca[j] = p.a_axis[j] ? ck[j] : cm[t][j];
                tma_nd(sa + t * A_SUB, &tm.a, ca, p.a_ndims, &full[s], pol_a);
            }
#pragma unroll
            for (int j = 0; j < 5; ++j) {  // advance the K coordinates by one k-tile
                if (!p.a_axis[j]) continue;
                if (p.a_div[j] == 1) {
                    ck[j] += BK;
                    if (p.a_mod[j] && ck[j] >= p.a_mod[j]) ck[j] -= int32_t(p.a_mod[j]);
                } else if ((sub[j] += BK) >= p.a_div[j]) {
                    sub[j] = 0;
                    if (++ck[j] == p.a_mod[j]) ck[j] = 0;
                }
            }
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) {
                if (EPI == GEMM_EPI_SWIGLU && j >= BN / 128)  // the up half: the same columns of B2
                    tma_2d(sb + j * (BK * 128), &tm.b2, int32_t(n0 + 64 * (j - BN / 128)), k0, &full[s], pol_b);
                else
                    tma_2d(sb + j * (BK * 128), tmb, int32_t(n0 + 64 * j), k0, &full[s], pol_b);
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer ----------------
        dev::pdl_wait();
        constexpr uint32_t idesc = instr_desc(BM, BN);
        for (int i = 0; i < nk; ++i) {
            const int s = i % STAGES;
            const uint32_t ph = uint32_t(i / STAGES) & 1u;
            mbar_wait(&full[s], ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = smem_u32(smem + size_t(s) * STAGE_BYTES);
            const uint32_t sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / UK; ++k) {
                // A: K-major SW128, +32 B per K16 step; B: MN-major SW128, +2 KB (16 rows) per step,
                // 64-column chunks BK*128 B apart (LBO), 8-row groups 1 KB apart (SBO)
                const uint64_t db = smem_desc(sb + k * 2048, BK * 128, 1024);
                const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
#pragma unroll
                for (int t = 0; t < MT; ++t) {  // sub-tile t -> TMEM columns [t*BN, (t+1)*BN)
                    const uint64_t da = smem_desc(sa + t * A_SUB + k * 32, 16, 1024);
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + uint32_t(t * BN)),
                        "l"(da), "l"(db), "r"(idesc), "r"(acc)
                        : "memory");
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&empty[s]))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&done))
                     : "memory");
    }

    // ---------------- epilogue: all 4 warps, thread = accumulator row ----------------
    dev::pdl_wait();
    __syncwarp();
    mbar_wait(&done, 0);
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned long long t_main = dev::gtime();
    if (threadIdx.x == 0) {
        dev::trace_add(p.head, 2, t_main - t_start);  // sum over CTAs: mainloop
        dev::trace_add(p.head, 4, 1);                 // CTA count
    }
    const int quad = warp & 3, half = warp >> 2;  // TMEM lane quadrant (warp id mod 4), column group
    for (int t = 0; t < MT; ++t) {
    const int row = quad * 32 + lane;  // TMEM lane == tile row (of sub-tile t)
    const int64_t m = m0 + t * BM + row;
    const uint32_t trow = tmem + (uint32_t(quad * 32) << 16) + uint32_t(t * BN);

    auto tmem_ld16 = [&](int c, float (&v)[16]) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(trow + uint32_t(c)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
    };

    bool do_epilogue = true;
    float* wtile = nullptr;
    if (p.splits > 1) {
        // fp32 partial tile -> workspace [tile][split][BN][BM] (column-major: a warp's
        // 32 rows of one column are one coalesced 128-byte store); warps whose rows
        // are all >= M skip; the last split reduces
        wtile = p.work + (int64_t(tile) * p.splits) * BM * BN;
        float* mine = wtile + int64_t(split) * BM * BN + row;
        if (m0 + warp * 32 < p.M) {
            for (int c = 0; c < BN; c += 16) {
                float v[16];
                if (nk > 0) tmem_ld16(c, v);
                else
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = 0.f;
#pragma unroll
                for (int j = 0; j < 16; ++j) mine[int64_t(c + j) * BM] = v[j];
            }
        }
        // release: the barrier orders the CTA's partial stores before thread 0's gpu-scope fence
        // and arrival (fence cumulativity), so one fence per CTA, not one per thread
        __syncthreads();
        if (p.coop_reduce) {
            // every split reduces its own slice of the tile's columns once all partials are
            // written (the host enables this only when the whole grid is co-resident, so the
            // wait cannot deadlock); the last split out resets the counters for the next replay
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(&p.counters[tile], 1u);
                unsigned v;
                long long spins = 0;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&p.counters[tile]) : "memory");
                    if (v >= unsigned(p.splits)) break;
                    __nanosleep(32);
                    if (++spins > (1ll << 26)) __trap();  // a missing split: fail loudly, never hang
                }
            }
            __syncthreads();  // thread 0's acquire, then the barrier: the CTA reads after every arrival
        } else {
            if (threadIdx.x == 0) {
                __threadfence();
                s_last = atomicAdd(&p.counters[tile], 1u) == unsigned(p.splits - 1) ? 1u : 0u;
                __threadfence();  // acquire: the other splits' partials, for the whole CTA (barrier below)
                if (s_last) p.counters[tile] = 0u;
            }
            __syncthreads();
            do_epilogue = s_last != 0;
        }
    }

    // a short SwiGLU tile without a K split (decode gate / up: 64 live rows, so only lane quadrants
    // 0-1 of TMEM hold data): warps 0-1 stage those rows' accumulators in the drained pipeline
    // buffers, then all four warps share the SiLU * Mul epilogue, columns spread over each row's threads
    const bool staged = EPI == GEMM_EPI_SWIGLU && MT == 1 && NHALF == 1 && p.splits == 1 && p.M - m0 <= 64;
    float* sacc = reinterpret_cast<float*>(smem);  // [BN][64] fp32
    if (staged) {
        if (warp < 2) {
            for (int c = 0; c < BN; c += 16) {
                float v[16];
                tmem_ld16(c, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) sacc[(c + j) * 64 + row] = v[j];
            }
        }
        __syncthreads();
    }
    if (do_epilogue) {
        // split-K reduction (partials from global, no TMEM): short tiles (decode M)
        // spread each row's columns over several threads so all 128 reduce
        int erow = row, part = 0, nparts = 1;
        if (p.splits > 1 || staged) {
            const int64_t rows_live = p.M - (m0 + int64_t(t) * BM);
            const int rp = rows_live <= 32 ? 32 : rows_live <= 64 ? 64 : 128;
            erow = int(threadIdx.x) % rp;
            part = int(threadIdx.x) / rp;
            nparts = 128 / rp;
        }
        const int64_t em = m0 + int64_t(t) * BM + erow;
        // tcgen05.ld is warp-collective: every lane loads, rows >= M only skip the stores
        const bool live = em < p.M;
        bf16* crow = nullptr;
        int64_t cs = 0;
        const bf16* rrow = nullptr;
        int64_t rs = 0;
        if (live) {
            // output row through the C map (and the residual's), stepping along N with the piece stride
            int32_t idx[VTC_MAX_RANK] = {};
            idx[0] = int32_t(em);
            idx[1] = int32_t(n0);
            if (mat) {  // the sibling's output
                crow = reinterpret_cast<bf16*>(p.c2_rows[em]) + int64_t(n0) * p.c2_rs;
                cs = p.c2_rs;
            } else if (p.c_rows) {  // host-resolved row (C's map has div/mod digits, e.g. a window reverse)
                crow = reinterpret_cast<bf16*>(p.c_rows[em]) + int64_t(n0) * p.c_rs;
                cs = p.c_rs;
            } else {
                dev::Loc lc = dev::locate(p.c.m, idx);
                crow = dev::addr<bf16>(p.c.m, lc);
                cs = p.c.fast_stride[lc.piece];
            }
            if (p.has_res) {
                dev::Loc lr = dev::locate(p.res.m, idx);
                rrow = dev::addr<bf16>(p.res.m, lr);
                rs = p.res.fast_stride[lr.piece];
            }
        }
        const int ncols = int(Nm - n0 < ON ? Nm - n0 : ON);
        // accumulator columns c..c+15 of this thread's row: TMEM, or the split-K sum
        auto get16 = [&](int c, float (&v)[16]) {
            if (p.splits > 1) {
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = 0.f;
                if (!live) return;
                // up to 4 splits' 16 columns in flight per round trip, summed in split order
                for (int s0 = 0; s0 < p.splits; s0 += 4) {
                    float tq[4][16];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float* src = wtile + int64_t(s0 + q) * BM * BN + int64_t(c) * BM + erow;
#pragma unroll
                        for (int j = 0; j < 16; ++j) tq[q][j] = s0 + q < p.splits ? __ldcg(src + int64_t(j) * BM) : 0.f;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (s0 + q < p.splits)
#pragma unroll
                            for (int j = 0; j < 16; ++j) v[j] += tq[q][j];
                }
            } else if (staged) {
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = live ? sacc[(c + j) * 64 + erow] : 0.f;
            } else {
                tmem_ld16(c, v);
            }
        };
        // 16 finished columns c..c+15 of this row: round, activation / residual, store through C's map.
        // The contiguous aligned case is a short straight line (the epilogue runs once per CTA, so
        // its code is fetched cold: i-cache misses, not math, bound it); anything else goes to a
        // shared out-of-line routine.
        auto emit = [&](int c, const float (&v)[16]) {
            bf16* dst = crow + int64_t(c) * cs;
            const bool fast = cs == 1 && c + 16 <= ncols && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 &&
                              (!rrow || (rs == 1 && (reinterpret_cast<uintptr_t>(rrow + c) & 15) == 0));
            if (!fast) {
                emit_slow(dst, cs, rrow, rs, c, ncols, v, EPI == GEMM_EPI_GELU);
                return;
            }
            uint32_t o[8];
            if (EPI == GEMM_EPI_GELU) {
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] = dev::gelu2_acc(v[2 * j], v[2 * j + 1]);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] = dev::pack_bf16x2(v[2 * j], v[2 * j + 1]);
                if (rrow) {  // bf16(bf16(acc) + residual), as the unfused Add rounds
                    uint32_t rv[8];
                    *reinterpret_cast<uint4*>(&rv[0]) = __ldg(reinterpret_cast<const uint4*>(rrow + c));
                    *reinterpret_cast<uint4*>(&rv[4]) = __ldg(reinterpret_cast<const uint4*>(rrow + c + 8));
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        o[j] = dev::pack_bf16x2(__uint_as_float(o[j] << 16) + __uint_as_float(rv[j] << 16),
                                                __uint_as_float(o[j] & 0xffff0000u) + __uint_as_float(rv[j] & 0xffff0000u));
                }
            }
            reinterpret_cast<uint4*>(dst)[0] = make_uint4(o[0], o[1], o[2], o[3]);
            reinterpret_cast<uint4*>(dst)[1] = make_uint4(o[4], o[5], o[6], o[7]);
        };
        // shallow-K variants (epilogue-bound): 64 accumulator columns per TMEM
        // round trip (4 loads, one wait), indices static so they stay in registers
        constexpr bool kBatch = MT == 1 && (EPI == GEMM_EPI_PLAIN || EPI == GEMM_EPI_GELU);
        if (EPI == GEMM_EPI_SWIGLU) {
            // columns c of the gate half and 128 + c of the up half -> SiLU(gate) * up,
            // rounded like the unfused SiLU and Mul operators
            int s_lo = 0, s_hi = ON;  // cooperative split-K: this split's slice of the columns
            if (p.coop_reduce) {
                const int gran = (ON / 16 + p.splits - 1) / p.splits;
                s_lo = min(ON, split * gran * 16);
                s_hi = min(ON, s_lo + gran * 16);
            }
            if (NHALF > 1) {  // 8 epilogue warps: this warp's half of the columns
                const int hw = (ON / NHALF + 15) / 16 * 16;
                s_lo = min(ON, half * hw);
                s_hi = min(ON, s_lo + hw);
            }
            const int cpart = ((s_hi - s_lo) / nparts + 15) / 16 * 16;
            const int c_lo = s_lo + part * cpart, c_hi = min(min(ncols, s_hi), c_lo + cpart);
            for (int c = c_lo; c < c_hi; c += 16) {
                float g[16], u[16];
                get16(c, g);
                get16(ON + c, u);
                if (!live) continue;
                bf16 o[16];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    o[j] = dev::mul_bf16(dev::silu_bf16(__float2bfloat16_rn(g[j])), __float2bfloat16_rn(u[j]));
                bf16* dst = crow + int64_t(c) * cs;
                if (cs == 1 && c + 16 <= ncols && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                    reinterpret_cast<uint4*>(dst)[0] = *reinterpret_cast<const uint4*>(&o[0]);
                    reinterpret_cast<uint4*>(dst)[1] = *reinterpret_cast<const uint4*>(&o[8]);
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (c + j < ncols) dst[int64_t(j) * cs] = o[j];
                }
            }
        } else if (kBatch && p.splits == 1) {
            for (int c0 = 0; c0 < ncols; c0 += 64) {
                uint32_t r[64];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t addr = trow + uint32_t(c0 + 16 * q < BN ? c0 + 16 * q : c0);
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                        : "=r"(r[16 * q + 0]), "=r"(r[16 * q + 1]), "=r"(r[16 * q + 2]), "=r"(r[16 * q + 3]),
                          "=r"(r[16 * q + 4]), "=r"(r[16 * q + 5]), "=r"(r[16 * q + 6]), "=r"(r[16 * q + 7]),
                          "=r"(r[16 * q + 8]), "=r"(r[16 * q + 9]), "=r"(r[16 * q + 10]), "=r"(r[16 * q + 11]),
                          "=r"(r[16 * q + 12]), "=r"(r[16 * q + 13]), "=r"(r[16 * q + 14]), "=r"(r[16 * q + 15])
                        : "r"(addr));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (!live) continue;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (c0 + 16 * q >= ncols) break;
                    float v[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[16 * q + j]);
                    emit(c0 + 16 * q, v);
                }
            }
        } else {
            int s_lo = 0, s_hi = BN;  // cooperative split-K: this split's slice of the columns
            if (p.coop_reduce) {
                const int gran = (BN / 16 + p.splits - 1) / p.splits;
                s_lo = min(BN, split * gran * 16);
                s_hi = min(BN, s_lo + gran * 16);
            }
            if (NHALF > 1) {  // 8 epilogue warps: this warp's half of the columns
                const int hw = (BN / NHALF + 15) / 16 * 16;
                s_lo = min(BN, half * hw);
                s_hi = min(BN, s_lo + hw);
            }
            const int cpart = ((s_hi - s_lo) / nparts + 15) / 16 * 16;  // this thread's columns [c_lo, c_hi)
            const int c_lo = s_lo + part * cpart, c_hi = min(min(ncols, s_hi), c_lo + cpart);
            for (int c = c_lo; c < c_hi; c += 16) {
                // trees: columns read only by the fused trees are never stored (tile-uniform test)
                if (EPI == GEMM_EPI_TREES && n0 + c >= p.skip_lo && n0 + c + 16 <= p.skip_hi) continue;
                float v[16];
                get16(c, v);
                if (!live) continue;
                emit(c, v);
            }
        }
        if (EPI == GEMM_EPI_TREES) {
            // elementwise trees over views of this tile (e.g. RoPE: x * cos + rotate_half(x) * sin):
            // head h of tree tr reads C columns of this tile only; 16 elements i0..i0+15 per step
            // split-K: the tile's (head, 16-element step) items are spread over every split's
            // threads (cooperative reduction) or the row's threads, one item each in turn, so
            // no split repeats another's work and each thread waits on few partial round trips
            const bool spread = p.splits > 1;
            const int nwork = spread ? (p.coop_reduce ? p.splits : 1) * nparts : 1;
            const int wid = spread ? (p.coop_reduce ? split : 0) * nparts + part : 0;
            int wk = 0;
            for (int tr = 0; tr < p.ntree; ++tr) {
                const GemmTree& T = p.tree[tr];
                for (int h = 0; h < T.nh; ++h) {
                    const int64_t anchor = T.c_lo + T.c_sh * h;
                    if (anchor < n0 || anchor >= n0 + ON) continue;
                    if (NHALF > 1 && (h % NHALF) != half) continue;      // 8 epilogue warps: heads over the halves
                    // external operands (the cos / sin rows) of step i0 + 16 are requested while
                    // step i0 computes: their L2 latency hides behind the TMEM loads and math
                    uint4 ext[EW_MAX_IN][2], nxt[EW_MAX_IN][2];
                    auto ext_load = [&](int i0n, uint4 (&buf)[EW_MAX_IN][2]) {
#pragma unroll
                        for (int k = 0; k < EW_MAX_IN; ++k) {
                            if (k >= T.nin) break;
                            const GemmTreeOp& op = T.op[1 + k];
                            if (op.from_c || !live || i0n >= T.hd) continue;
                            const int q = i0n >= op.split ? 1 : 0;
                            const bf16* src = reinterpret_cast<const bf16*>(op.base[q]) + op.rs[q] * em + op.sh[q] * h + i0n;
                            buf[k][0] = __ldg(reinterpret_cast<const uint4*>(src));
                            buf[k][1] = __ldg(reinterpret_cast<const uint4*>(src + 8));
                        }
                    };
                    if (!spread) ext_load(0, ext);
                    for (int i0 = 0; i0 < T.hd; i0 += 16) {
                        if (spread) {
                            if ((wk++) % nwork != wid) continue;
                            ext_load(i0, ext);
                        } else {
                            ext_load(i0 + 16, nxt);
                        }
                        bf16 in[EW_MAX_IN][16];
#pragma unroll
                        for (int k = 0; k < EW_MAX_IN; ++k) {
                            if (k < T.nin) {
                                const GemmTreeOp& op = T.op[1 + k];
                                const int q = i0 >= op.split ? 1 : 0;
                                if (op.from_c) {
                                    float v[16];
                                    get16(int(op.ccol[q] + op.sh[q] * h + i0 - n0), v);
#pragma unroll
                                    for (int j = 0; j < 16; ++j) in[k][j] = __float2bfloat16_rn(v[j]);
                                } else {
                                    *reinterpret_cast<uint4*>(&in[k][0]) = ext[k][0];
                                    *reinterpret_cast<uint4*>(&in[k][8]) = ext[k][1];
                                }
                            }
                        }
                        if (!spread)
#pragma unroll
                            for (int k = 0; k < EW_MAX_IN; ++k) {
                                ext[k][0] = nxt[k][0];
                                ext[k][1] = nxt[k][1];
                            }
                        if (!live) continue;
                        bf16 o[16];
                        if (T.pat == 3) {  // (in0 * in1) + (in2 * in3): RoPE, in registers
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                o[j] = dev::add_bf16(dev::mul_bf16(in[0][j], in[1][j]), dev::mul_bf16(in[2][j], in[3][j]));
                        } else {
                            bf16 r[EW_MAX_IN + EW_MAX_PROG][16];
#pragma unroll
                            for (int k = 0; k < EW_MAX_IN; ++k)
#pragma unroll
                                for (int j = 0; j < 16; ++j) r[k][j] = in[k][j];
#pragma unroll 1
                            for (int s2 = 0; s2 < T.nprog; ++s2) {
                                const EwInstr ins = T.prog[s2];
#pragma unroll
                                for (int j = 0; j < 16; ++j) {
                                    const bf16 a = r[ins.a][j], b = r[ins.b][j];
                                    r[ins.dst][j] = ins.op == EwOp::Add   ? dev::add_bf16(a, b)
                                                    : ins.op == EwOp::Mul  ? dev::mul_bf16(a, b)
                                                    : ins.op == EwOp::SiLU ? dev::silu_bf16(a)
                                                    : ins.op == EwOp::GELU ? dev::gelu_bf16(a)
                                                                           : a;
                                }
                            }
#pragma unroll
                            for (int j = 0; j < 16; ++j) o[j] = r[T.result][j];
                        }
                        const GemmTreeOp& out = T.op[0];
                        const int q = i0 >= out.split ? 1 : 0;
                        bf16* dst = reinterpret_cast<bf16*>(out.base[q]) + out.rs[q] * em + out.sh[q] * h + i0;
                        reinterpret_cast<uint4*>(dst)[0] = *reinterpret_cast<const uint4*>(&o[0]);
                        reinterpret_cast<uint4*>(dst)[1] = *reinterpret_cast<const uint4*>(&o[8]);
                    }
                }
            }
        }
    }
    if (p.coop_reduce && p.splits > 1) {
        // every split has read the partials: the last one out resets the tile's counters
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(&p.counters[p.ntiles_total + tile], 1u) == unsigned(p.splits - 1)) {
            p.counters[tile] = 0u;
            p.counters[p.ntiles_total + tile] = 0u;
            __threadfence();
        }
    }
    }  // sub-tiles
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) dev::trace_add(p.head, 3, dev::gtime() - t_main);  // sum over CTAs: epilogue
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN * MT));
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2) for prefill-sized M: a cluster of two CTAs on
// one TPC computes a 256 x 256 tile with M = 256 UMMAs issued by the leader
// CTA.  Each CTA loads its own 128 rows of A and its own half (128 columns) of
// B into the same shared-memory offsets, both halves' TMA transactions signal
// the leader's stage barrier, and the MMA reads the pair's operands from both
// CTAs -- half the B traffic and half the shared-memory operand reads per SM of
// a one-CTA 128 x 256 tile.  The accumulator rows of each CTA land in its own
// TMEM (128 lanes x 256 columns), so the epilogue is the one-CTA epilogue over
// 128 rows.  Three 32 KB stages per CTA: two CTAs per SM, one's epilogue
// overlapping the other's mainloop.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_2d_pair(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint32_t bar_cluster,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
        "{%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(policy)
        : "memory");
}

constexpr int PAIR_STAGES = 3;
template <int EPI>
__global__ void __launch_bounds__(NTHREADS, 1) gemm_pair_kernel(const GemmTcParams* __restrict__ pp,
                                                                 const __grid_constant__ Tmaps tm) {
    VTC_STAGE_PARAMS(GemmTcParams, pp);
    constexpr int BN = 256, HB = 128;  // tile N; B columns per CTA
    constexpr int ON = EPI == GEMM_EPI_SWIGLU ? BN / 2 : BN;
    constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = HB * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[PAIR_STAGES], empty[PAIR_STAGES], done;
    __shared__ uint32_t s_tmem;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int tiles_n = int((p.N + ON - 1) / ON);
    const int tiles_m = int((p.M + 2 * BM - 1) / (2 * BM));
    const int tile = blockIdx.x / 2;
    constexpr int GROUP_M = 16;
    const int in_group = GROUP_M * tiles_n;
    const int first_m = (tile / in_group) * GROUP_M;
    const int gm = min(tiles_m - first_m, GROUP_M);
    const int tm_ = first_m + (tile % in_group) % gm, tn = (tile % in_group) / gm;
    const int64_t m0 = int64_t(tm_) * 2 * BM + int64_t(rank) * BM, n0 = int64_t(tn) * ON;
    const int ktiles = int((p.K + BK - 1) / BK);

    if (threadIdx.x == 0) {
        for (int s = 0; s < PAIR_STAGES; ++s) {
            mbar_init(&full[s], 2);  // the leader's expect_tx arrival + the peer's arrival
            mbar_init(&empty[s], 1);
        }
        mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {  // the pair's accumulators: 128 lanes x 256 columns in each CTA
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();  // both CTAs' barriers initialised before any remote arrival
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    dev::pdl_launch_dependents();

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer (both CTAs) ----------------
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm.a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm.b)) : "memory");
        const uint64_t pol_b = evict_last_policy(), pol_a = evict_last_policy();
        int32_t cm[5], ck[5], sub[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const uint32_t v = uint32_t(m0) / uint32_t(p.a_div[j]);
            cm[j] = int32_t(p.a_mod[j] ? v % uint32_t(p.a_mod[j]) : v);
            ck[j] = 0;
            sub[j] = 0;
        }
        const uint32_t full0 = map_to_rank(smem_u32(&full[0]), 0);  // the leader's stage barriers
        dev::pdl_wait();
        for (int i = 0; i < ktiles; ++i) {
            const int s = i % PAIR_STAGES;
            const uint32_t ph = uint32_t(i / PAIR_STAGES) & 1u;
            mbar_wait(&empty[s], ph ^ 1u);
            const uint32_t fb = full0 + uint32_t(s) * 8;
            if (leader) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
            else asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(fb) : "memory");
            const uint32_t sa = smem_u32(smem + size_t(s) * STAGE_BYTES), sb = sa + A_BYTES;
            const int32_t k0 = int32_t(i) * BK;
            int32_t ca[5];
#pragma unroll
            for (int j = 0; j < 5; ++j) ca[j] = p.a_axis[j] ? ck[j] : cm[j];
            switch (p.a_ndims) {
                case 2: asm volatile(
                            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
                            " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(sa), "l"(reinterpret_cast<uint64_t>(&tm.a)), "r"(ca[0]), "r"(ca[1]),
                            "r"(fb), "l"(pol_a) : "memory"); break;
                case 3: asm volatile(
                            "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
                            " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(sa), "l"(reinterpret_cast<uint64_t>(&tm.a)), "r"(ca[0]),
                            "r"(ca[1]), "r"(ca[2]), "r"(fb), "l"(pol_a) : "memory"); break;
                default: asm volatile(
                            "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
                            " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(sa), "l"(reinterpret_cast<uint64_t>(&tm.a)), "r"(ca[0]),
                            "r"(ca[1]), "r"(ca[2]), "r"(ca[3]), "r"(fb), "l"(pol_a) : "memory"); break;
            }
#pragma unroll
            for (int j = 0; j < 5; ++j) {  // advance the K coordinates by one k-tile
                if (!p.a_axis[j]) continue;
                if (p.a_div[j] == 1) {
                    ck[j] += BK;
                    if (p.a_mod[j] && ck[j] >= p.a_mod[j]) ck[j] -= int32_t(p.a_mod[j]);
                } else if ((sub[j] += BK) >= p.a_div[j]) {
                    sub[j] = 0;
                    if (++ck[j] == p.a_mod[j]) ck[j] = 0;
                }
            }
            // this CTA's half of B: columns [rank * 128, rank * 128 + 128) of the tile (SwiGLU:
            // the leader the gate's 128, the peer the up's 128 -- the same output columns)
#pragma unroll
            for (int j = 0; j < HB / 64; ++j) {
                if (EPI == GEMM_EPI_SWIGLU)
                    tma_2d_pair(sb + j * (BK * 128), rank ? &tm.b2 : &tm.b, int32_t(n0 + 64 * j), k0, fb, pol_b);
                else
                    tma_2d_pair(sb + j * (BK * 128), &tm.b, int32_t(n0 + rank * HB + 64 * j), k0, fb, pol_b);
            }
        }
    } else if (warp == 1 && lane == 0 && leader) {
        // ---------------- MMA issuer (leader only): M = 256 over the pair ----------------
        dev::pdl_wait();
        constexpr uint32_t idesc = instr_desc(2 * BM, BN);
        for (int i = 0; i < ktiles; ++i) {
            const int s = i % PAIR_STAGES;
            const uint32_t ph = uint32_t(i / PAIR_STAGES) & 1u;
            mbar_wait(&full[s], ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = smem_u32(smem + size_t(s) * STAGE_BYTES), sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / UK; ++k) {
                const uint64_t da = smem_desc(sa + k * 32, 16, 1024);
                const uint64_t db = smem_desc(sb + k * 2048, BK * 128, 1024);
                const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc)
                    : "memory");
            }
            // frees stage s in both CTAs
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                             smem_u32(&empty[s])),
                         "h"(uint16_t(3))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         smem_u32(&done)),
                     "h"(uint16_t(3))
                     : "memory");
    }

    // ---------------- epilogue: all 4 warps of each CTA, thread = accumulator row ----------------
    dev::pdl_wait();
    __syncwarp();
    mbar_wait(&done, 0);
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = warp * 32 + lane;
    const int64_t em = m0 + row;
    const bool live = em < p.M;
    const uint32_t trow = tmem + (uint32_t(warp * 32) << 16);
    bf16* crow = nullptr;
    int64_t cs = 0;
    const bf16* rrow = nullptr;
    int64_t rs = 0;
    if (live) {
        int32_t idx[VTC_MAX_RANK] = {};
        idx[0] = int32_t(em);
        idx[1] = int32_t(n0);
        dev::Loc lc = dev::locate(p.c.m, idx);
        crow = dev::addr<bf16>(p.c.m, lc);
        cs = p.c.fast_stride[lc.piece];
        if (p.has_res) {
            dev::Loc lr = dev::locate(p.res.m, idx);
            rrow = dev::addr<bf16>(p.res.m, lr);
            rs = p.res.fast_stride[lr.piece];
        }
    }
    const int ncols = int(p.N - n0 < ON ? p.N - n0 : ON);
    auto ld16 = [&](int c, float (&v)[16]) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
              "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(trow + uint32_t(c)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
    };
    for (int c = 0; c < ON; c += 16) {
        float v[16], u[16];
        ld16(c, v);
        if (EPI == GEMM_EPI_SWIGLU) ld16(ON + c, u);
        if (!live || c >= ncols) continue;
        bf16 o[16];
        if (EPI == GEMM_EPI_SWIGLU) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                o[j] = dev::mul_bf16(dev::silu_bf16(__float2bfloat16_rn(v[j])), __float2bfloat16_rn(u[j]));
        } else {
            bf16 rv[16];
            const bool rvec = rrow && rs == 1 && c + 16 <= ncols && (reinterpret_cast<uintptr_t>(rrow + c) & 15) == 0;
            if (rvec) {
                *reinterpret_cast<uint4*>(&rv[0]) = __ldg(reinterpret_cast<const uint4*>(rrow + c));
                *reinterpret_cast<uint4*>(&rv[8]) = __ldg(reinterpret_cast<const uint4*>(rrow + c + 8));
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                float f = __bfloat162float(__float2bfloat16_rn(v[j]));
                if (rvec) f = __bfloat162float(rv[j]) + f;
                else if (rrow && c + j < ncols) f = __bfloat162float(rrow[int64_t(c + j) * rs]) + f;
                o[j] = __float2bfloat16_rn(f);
            }
        }
        bf16* dst = crow + int64_t(c) * cs;
        if (cs == 1 && c + 16 <= ncols && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            reinterpret_cast<uint4*>(dst)[0] = *reinterpret_cast<const uint4*>(&o[0]);
            reinterpret_cast<uint4*>(dst)[1] = *reinterpret_cast<const uint4*>(&o[8]);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c + j < ncols) dst[int64_t(j) * cs] = o[j];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();  // both CTAs done with the pair's TMEM before it is released
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
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

template <int BN, int STAGES, int MT>
constexpr size_t smem_bytes() {
    return size_t(STAGES) * (MT * BM * BK * 2 + BN * BK * 2) + 1024;
}

}  // namespace

bool gemm_tc_a_dims(const vtc_map& a, int64_t M, int64_t K, GemmTcParams& p, int64_t dims[5], int64_t strides[5],
                    const void** base) {
    if (a.npieces != 1 || a.rank != 2) return false;
    const vtc_piece& pc = a.piece[0];
    if (pc.ngroups != 0 || pc.ndigits < 1 || pc.ndigits > 5) return false;
    struct Dg {
        int axis;
        int64_t div, mod, coeff;
    };
    Dg dg[VTC_MAX_DIGITS];
    int n = 0;
    for (int t = 0; t < pc.ndigits; ++t) {
        const vtc_digit& d = pc.dig[t];
        if (d.coeff <= 0 || d.group >= 0 || (d.axis != 0 && d.axis != 1)) return false;
        dg[n++] = Dg{d.axis, int64_t(d.div), int64_t(d.mod), d.coeff};
    }
    std::sort(dg, dg + n, [](const Dg& x, const Dg& y) { return x.coeff < y.coeff; });
    if (dg[0].axis != 1 || dg[0].div != 1 || dg[0].coeff != 1) return false;
    bool have_m = false;
    for (int j = 0; j < n; ++j) {
        const int64_t ext_axis = dg[j].axis ? K : M;
        const int64_t tile = dg[j].axis ? BK : BM;
        const int64_t extent = dg[j].mod ? dg[j].mod : (ext_axis + dg[j].div - 1) / dg[j].div;
        if (dg[j].div == 1) {
            // the box dimension of this axis: the tile must not cross its modulus
            if (dg[j].mod && dg[j].mod % tile != 0) return false;
            if (dg[j].axis == 0) {
                if (have_m) return false;
                have_m = true;
            } else if (j != 0) {
                return false;
            }
        } else if (dg[j].div % tile != 0) {
            return false;  // constant over a tile only when the divisor is tile-aligned
        }
        if (j > 0 && (dg[j].coeff * 2) % 16 != 0) return false;
        p.a_axis[j] = dg[j].axis;
        p.a_div[j] = dg[j].div;
        p.a_mod[j] = dg[j].mod;
        dims[j] = extent;
        strides[j] = dg[j].coeff;
    }
    if (!have_m && M > 1) return false;
    for (int j = n; j < 5; ++j) {
        p.a_axis[j] = 0;
        p.a_div[j] = 1;
        p.a_mod[j] = 1;
    }
    p.a_ndims = n < 2 ? 2 : n;
    if (n < 2) {  // M == 1 without an M digit: a unit second dimension
        dims[1] = 1;
        strides[1] = K;
        p.a_axis[1] = 0;
        p.a_div[1] = 1;
        p.a_mod[1] = 1;
    }
    *base = reinterpret_cast<const char*>(pc.ptr) + pc.base * 2;
    return (reinterpret_cast<uintptr_t>(*base) % 16) == 0;
}

bool gemm_tc_encode(GemmTcParams& p, const void* a_base, const int64_t* a_dims, const int64_t* a_strides,
                    const void* b_base, int64_t b_ld) {
    EncodeFn fn = encoder();
    if (!fn) return false;
    if ((reinterpret_cast<uintptr_t>(a_base) % 16) || (reinterpret_cast<uintptr_t>(b_base) % 16)) return false;
    if ((b_ld * 2) % 16) return false;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    {
        const int nd = p.a_ndims;
        cuuint64_t dims[5], str[4];
        cuuint32_t box[5];
        for (int j = 0; j < nd; ++j) {
            dims[j] = cuuint64_t(a_dims[j]);
            if (j > 0) str[j - 1] = cuuint64_t(a_strides[j]) * 2;
            const bool boxed = p.a_div[j] == 1 && (j == 0 || p.a_axis[j] == 0);
            box[j] = boxed ? (p.a_axis[j] ? BK : BM) : 1;
        }
        if (fn(reinterpret_cast<CUtensorMap*>(p.tmap_a), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, cuuint32_t(nd), const_cast<void*>(a_base),
               dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    return gemm_tc_encode_b(p.tmap_b, b_base, p.N, p.K, b_ld);
}

bool gemm_tc_encode_b(void* out128, const void* b_base, int64_t N, int64_t K, int64_t ld) {
    EncodeFn fn = encoder();
    if (!fn || (reinterpret_cast<uintptr_t>(b_base) % 16) || (ld * 2) % 16) return false;
    cuuint32_t es[2] = {1, 1};
    cuuint64_t dims[2] = {cuuint64_t(N), cuuint64_t(K)};
    cuuint64_t str[1] = {cuuint64_t(ld) * 2};
    cuuint32_t box[2] = {64, BK};
    return fn(reinterpret_cast<CUtensorMap*>(out128), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(b_base), dims,
              str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int ST, int MT, int EPI>
void launch_variant(const GemmTcParams* dp, dim3 grid, const Tmaps& tmaps, cudaStream_t s) {
    constexpr size_t sm = smem_bytes<BN, ST, MT>();
    cudaFuncSetAttribute(gemm_tc_kernel<BN, ST, MT, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    launch_k(gemm_tc_kernel<BN, ST, MT, EPI>, grid, dim3(tc_threads<MT>()), sm, s, dp, tmaps);
}

int sm_count() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

template <int EPI>
void launch_epi(const GemmTcParams& p, const GemmTcParams* dp, const Tmaps& tmaps, cudaStream_t s) {
    const int tm = p.mt == 2 ? 2 * BM : BM;
    const int on = EPI == GEMM_EPI_SWIGLU ? p.bn / 2 : p.bn;
    const int tiles = int((p.M + tm - 1) / tm) *
                      int((p.N + on - 1) / on + (p.nmat > 1 ? (p.N1 + p.bn - 1) / p.bn : 0));
    const int64_t ktiles = (p.K + BK - 1) / BK;
    const dim3 grid(unsigned(tiles), unsigned(p.splits));
    if (p.mt == 2) {
        launch_variant<256, 3, 2, EPI>(dp, grid, tmaps, s);
    } else if (p.bn == 256 && ((ktiles <= 2 && p.splits == 1) || p.pair)) {
        // shallow K (e.g. Swin's K = 96): a 2-stage ring, two CTAs per SM, so one
        // CTA's epilogue overlaps the other's loads and MMAs
        launch_variant<256, 2, 1, EPI>(dp, grid, tmaps, s);
    } else if (p.bn == 256 || EPI == GEMM_EPI_SWIGLU) {
        launch_variant<256, 4, 1, EPI>(dp, grid, tmaps, s);
    } else if constexpr (EPI != GEMM_EPI_SWIGLU) {
        if (ktiles <= 2 && p.splits == 1) {
            launch_variant<128, 2, 1, EPI>(dp, grid, tmaps, s);  // three CTAs per SM
        } else if ((ktiles <= 6 || (p.M <= BM && tiles > sm_count())) && p.splits == 1) {
            // two CTAs per SM: shallow K, or decode-sized M with more tiles than SMs (the
            // fused gate / up weight streams then run in one wave instead of two)
            launch_variant<128, 3, 1, EPI>(dp, grid, tmaps, s);
        } else {
            launch_variant<128, 6, 1, EPI>(dp, grid, tmaps, s);
        }
    }
}

void launch_gemm_tc(const GemmTcParams& p, const GemmTcParams* dp, cudaStream_t s) {
    Tmaps tmaps;
    std::memcpy(&tmaps.a, p.tmap_a, sizeof(CUtensorMap));
    std::memcpy(&tmaps.b, p.tmap_b, sizeof(CUtensorMap));
    std::memcpy(&tmaps.b2, (p.nmat > 1 || p.epi == GEMM_EPI_SWIGLU) ? p.tmap_b2 : p.tmap_b, sizeof(CUtensorMap));
    if (p.cta_pair) {
        // clusters of two CTAs (one TPC), a 256 x 256 tile per cluster, three 32 KB stages per CTA
        const int on = p.epi == GEMM_EPI_SWIGLU ? 128 : 256;
        const int tiles = int((p.M + 255) / 256) * int((p.N + on - 1) / on);
        constexpr size_t sm = size_t(PAIR_STAGES) * (BM * BK * 2 + 128 * BK * 2) + 1024;
        if (p.epi == GEMM_EPI_SWIGLU) {
            cudaFuncSetAttribute(gemm_pair_kernel<GEMM_EPI_SWIGLU>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
            launch_k_cluster(gemm_pair_kernel<GEMM_EPI_SWIGLU>, dim3(2 * tiles), dim3(NTHREADS), sm, s, 2, dp, tmaps);
        } else {
            cudaFuncSetAttribute(gemm_pair_kernel<GEMM_EPI_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
            launch_k_cluster(gemm_pair_kernel<GEMM_EPI_PLAIN>, dim3(2 * tiles), dim3(NTHREADS), sm, s, 2, dp, tmaps);
        }
        return;
    }
    switch (p.epi) {
        case GEMM_EPI_GELU: launch_epi<GEMM_EPI_GELU>(p, dp, tmaps, s); break;
        case GEMM_EPI_SWIGLU: launch_epi<GEMM_EPI_SWIGLU>(p, dp, tmaps, s); break;
        case GEMM_EPI_TREES: launch_epi<GEMM_EPI_TREES>(p, dp, tmaps, s); break;
        default: launch_epi<GEMM_EPI_PLAIN>(p, dp, tmaps, s); break;
    }
}

}  // namespace vtc
