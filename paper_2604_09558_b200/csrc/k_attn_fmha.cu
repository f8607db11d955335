// Flash attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// bf16, head dim 128: the prefill attention of a VTC-planned decoder layer
// (BASELINE configs[4], Llama-3-8B S = 4096, GQA 32 / 8, causal).
//
// softmax(scale * Q K^T [causal]) V, with Q / K / V / O addressed through
// their VirtualTensor maps: the host proves each map affine over
// (batch, head, position, dim) (for K / V over the KV head = head / group, the
// GQA Expand's `h div G` digit) and encodes a 4-D TMA tensor per operand, so the
// QKV split, the [B,S,H,d] -> [B,H,S,d] transposes and the GQA
// Expand / Reshape stay views -- no copy kernel, no per-element map walk.
//
//   * CTA = two adjacent 128-row query tiles of one (batch, head) sharing every
//     K / V tile (half the K / V traffic per FLOP); 10 warps:
//       warps 0-3 / 4-7  softmax + epilogue of query tile 0 / 1 (thread = query
//                        row = TMEM lane),
//       warp 8           TMA producer (Q tiles once, then K / V tiles of 128 keys,
//                        2 stages each; a K stage frees when both tiles' S MMAs
//                        complete, a V stage after both PV MMAs),
//       warp 9           MMA issuer (one thread);
//   * TMEM (512 columns): S_t = Q_t K^T (fp32, 128 columns) per tile, P_t written
//     over S_t as bf16 pairs, O_t (fp32, 128 columns) per tile;
//   * per key tile: S_0, S_1 (tcgen05.mma M128 N128 K16 x 8, K-major SW128 A / B);
//     each softmax warpgroup reads its S row with tcgen05.ld, applies scale and
//     causal mask, keeps a running row max in the log2 domain and stores
//     P = exp2(S - m) back into TMEM (tcgen05.st); O_t += P_t V is a TS-MMA
//     (A from TMEM, V the MN-major B operand in smem).  While one warpgroup
//     computes its softmax the tensor core works on the other tile, and the
//     next S_t is issued right behind PV_t (tcgen05 ops run in issue order);
//   * lazy rescale: O_t and l are rescaled only when a row's max grows by more
//     than 2^8, otherwise P uses the stale max (bounded by 256);
//   * epilogue: O / l from TMEM to bf16, 16-byte stores through O's map.
// Causal query tiles stop at the diagonal key tile and are scheduled longest
// first.  Attention is absent from the reference (SURVEY.md §8 a'); CPU
// restatement: oracle/vtc_oracle.py (Attention).
#include <cuda.h>

#include <cstdlib>
#include <cstring>

#include "device.cuh"
#include "launch.cuh"
#include "lower.hpp"

namespace vtc {
namespace {

using dev::bf16;
constexpr int BQ = 128, BKV = 128, D = 128, NTHREADS = 320;
constexpr uint32_t CHUNK = 128 * 128;               // one [128 rows x 64 bf16] SW128 chunk = 16 KB
constexpr uint32_t TILE = 2 * CHUNK;                // 128 x 128 bf16
constexpr uint32_t SMEM_Q = 0, SMEM_K = 2 * TILE, SMEM_V = 4 * TILE, SMEM_BYTES = 6 * TILE;  // Q0 Q1 | K x2 | V x2
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_THRESHOLD = 8.0f;           // log2 units: rescale O only when the max grows by > 2^8

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
__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                       int32_t c3, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3, %4, %5}], [%6], %7;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// UMMA shared-memory descriptor, SWIZZLE_128B (see k_gemm_tc.cu)
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
// kind::f16 instruction descriptor: D f32, A / B bf16, A K-major, B K-major (b_mn = 0) or MN-major (1)
__host__ __device__ constexpr uint32_t idesc(int m, int n, int b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(b_mn) << 16) | (uint32_t(n >> 3) << 17) |
           (uint32_t(m >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 32 consecutive TMEM columns of this warp's 32 lanes -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

struct FmhaArgs {
    CUtensorMap q, k, v;     // 4-D {d, position, head, batch}, box {64, 128, 1, 1}, 128-byte swizzle
    bf16* o;                 // output element (b, h, s, 0) = o + b*o_sb + h*o_sh + s*o_ss
    int64_t o_sb, o_sh, o_ss;
    const KHead* head;       // timeline (VTC_TRACE)
    int32_t H, group, Sq, Sk, causal, qpairs;
    float scale_log2;
};

__global__ void __launch_bounds__(NTHREADS, 1) attn_fmha_kernel(const __grid_constant__ FmhaArgs a) {
    dev::TraceScope trace_scope_(a.head);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t q_full, k_full[2], v_full[2], k_empty[2], v_empty[2], s_full[2], p_full[2], o_done[2];
    __shared__ uint32_t s_tmem;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // CTA = query tiles 2c and 2c + 1 of one (batch, head); causal: longest first
    const int pair = a.causal ? a.qpairs - 1 - int(blockIdx.x) : int(blockIdx.x);
    const int bh = int(blockIdx.y);
    const int b = bh / a.H, h = bh - b * a.H, hkv = h / a.group;
    const int off = a.Sk - a.Sq;  // query row q sees keys t <= q + off
    auto tiles_of = [&](int t) {  // key tiles query tile t of the pair attends to
        const int q0 = (2 * pair + t) * BQ;
        const int kend = q0 >= a.Sq ? 0 : a.causal ? min(a.Sk, q0 + BQ + off) : a.Sk;
        return kend > 0 ? (kend + BKV - 1) / BKV : 0;
    };
    const int nkv0 = tiles_of(0), nkv1 = tiles_of(1);
    const int nkv = max(nkv0, nkv1);

    if (threadIdx.x == 0) {
        mbar_init(&q_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&v_full[s], 1);
            mbar_init(&k_empty[s], 1);
            mbar_init(&v_empty[s], 1);
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], 4);  // one arrival per warp of the tile's softmax warpgroup
            mbar_init(&o_done[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {  // TMEM: S / P of tile t at columns 128 t, O of tile t at 256 + 128 t
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    dev::pdl_launch_dependents();
    const uint32_t sbase = smem_u32(smem);

    if (warp == 8) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.q)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.k)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.v)) : "memory");
            const uint64_t pol = evict_last_policy();  // K / V re-read by every query tile of the head
            dev::pdl_wait();
            mbar_expect_tx(&q_full, 2 * TILE);
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const uint32_t qs = sbase + SMEM_Q + uint32_t(t) * TILE;
                tma_4d(qs, &a.q, 0, (2 * pair + t) * BQ, h, b, &q_full, pol);
                tma_4d(qs + CHUNK, &a.q, 64, (2 * pair + t) * BQ, h, b, &q_full, pol);
            }
            for (int j = 0; j < nkv; ++j) {
                const int st = j & 1;
                const uint32_t ks = sbase + SMEM_K + st * TILE, vs = sbase + SMEM_V + st * TILE;
                // K_j's stage frees when both tiles' S_{j-2} are computed, V_j's after both PV_{j-2}
                mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1u);
                mbar_expect_tx(&k_full[st], TILE);
                tma_4d(ks, &a.k, 0, j * BKV, hkv, b, &k_full[st], pol);
                tma_4d(ks + CHUNK, &a.k, 64, j * BKV, hkv, b, &k_full[st], pol);
                mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1u);
                mbar_expect_tx(&v_full[st], TILE);
                tma_4d(vs, &a.v, 0, j * BKV, hkv, b, &v_full[st], pol);
                tma_4d(vs + CHUNK, &a.v, 64, j * BKV, hkv, b, &v_full[st], pol);
            }
        }
    } else if (warp == 9) {
        if (lane == 0) {
            // ---------------- MMA issuer ----------------
            // Per key tile j: S_0 = Q_0 K^T, S_1 = Q_1 K^T, then (as each tile's P lands
            // in TMEM over its S) O_t += P_t V.  tcgen05 ops run in issue order, so S_t of
            // tile j + 1 -- issued after PV_t of tile j -- cannot overwrite P_t early.
            constexpr uint32_t id_s = idesc(BQ, BKV, 0), id_o = idesc(BQ, D, 1);
            const bool prof = a.head->trace != nullptr;
            long long w_k = 0, w_v = 0, w_p = 0;
            mbar_wait(&q_full, 0);
            auto issue_s = [&](int t, int j) {
                const uint32_t qa = sbase + SMEM_Q + uint32_t(t) * TILE, kb = sbase + SMEM_K + (j & 1) * TILE;
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const uint32_t o = (k >> 2) * CHUNK + (k & 3) * 32;  // K-major SW128: +32 B per K16, next chunk per 64
                    mma(tmem + uint32_t(t * 128), smem_desc(qa + o, 16, 1024), smem_desc(kb + o, 16, 1024), id_s,
                        k > 0 ? 1u : 0u);
                }
                commit(&s_full[t]);
            };
            auto wait_k = [&](int j) {
                const long long c0 = prof ? clock64() : 0;
                mbar_wait(&k_full[j & 1], (j >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (prof) w_k += clock64() - c0;
            };
            if (nkv > 0) {
                wait_k(0);
                if (nkv0 > 0) issue_s(0, 0);
                if (nkv1 > 0) issue_s(1, 0);
                commit(&k_empty[0]);
            }
            for (int j = 0; j < nkv; ++j) {
                const int st = j & 1;
                const long long c1 = prof ? clock64() : 0;
                mbar_wait(&v_full[st], (j >> 1) & 1);
                if (prof) w_v += clock64() - c1;
                if (j + 1 < nkv) wait_k(j + 1);
                const uint32_t vb = sbase + SMEM_V + st * TILE;
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const int nt = t ? nkv1 : nkv0;
                    if (j >= nt) continue;
                    const long long c0 = prof ? clock64() : 0;
                    mbar_wait(&p_full[t], (j & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    if (prof) w_p += clock64() - c0;
#pragma unroll
                    for (int k = 0; k < BKV / 16; ++k)  // A = P_t from TMEM (8 columns per K16), B = V MN-major
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 256u + uint32_t(t * 128)),
                            "r"(tmem + uint32_t(t * 128 + k * 8)), "l"(smem_desc(vb + uint32_t(k) * 2048u, CHUNK, 1024)),
                            "r"(id_o), "r"((j > 0 || k > 0) ? 1u : 0u)
                            : "memory");
                    commit(&o_done[t]);
                    if (j + 1 < nt) issue_s(t, j + 1);
                }
                commit(&v_empty[st]);
                if (j + 1 < nkv) commit(&k_empty[(j + 1) & 1]);
            }
            if (prof) {  // sums over CTAs, cycles: MMA thread waiting for K, P, V
                dev::trace_add(*a.head, 5, (unsigned long long)w_k);
                dev::trace_add(*a.head, 6, (unsigned long long)w_p);
                dev::trace_add(*a.head, 7, (unsigned long long)w_v);
            }
        }
    } else {
        // ---------------- softmax: warpgroup t = query tile t, thread = query row = TMEM lane ----------------
        const int t = warp >> 2, wq = warp & 3;
        const int r = wq * 32 + lane;
        const int q0 = (2 * pair + t) * BQ, q = q0 + r;
        const int lim = q + off;  // last visible key (causal)
        const int my_nkv = t ? nkv1 : nkv0;
        const uint32_t trow = tmem + (uint32_t(wq * 32) << 16);
        const uint32_t sc = uint32_t(t * 128), oc = 256u + uint32_t(t * 128);
        float m = -INFINITY, l = 0.f;
        const bool prof = a.head->trace != nullptr && threadIdx.x == 0;
        long long w_s = 0, busy = 0;
        for (int j = 0; j < my_nkv; ++j) {
            long long c0 = prof ? clock64() : 0;
            mbar_wait(&s_full[t], j & 1);
            if (prof) {
                const long long c = clock64();
                w_s += c - c0;
                c0 = c;
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint32_t sr[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(trow + sc + uint32_t(c * 32), sr[c]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int t0 = j * BKV;
            const bool masked = (a.causal && t0 + BKV - 1 > q0 + off) || t0 + BKV > a.Sk;
            if (masked) {  // diagonal / tail tiles only: invisible keys -> -inf
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int tk = t0 + c * 32 + i;
                        if (tk >= a.Sk || (a.causal && tk > lim)) sr[c][i] = __float_as_uint(-INFINITY);
                    }
            }
            // raw row max (scale > 0: max commutes with the scale); 8 independent
            // chains so the reduction is not one 128-long dependency
            float mp[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) mp[k] = -INFINITY;
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int i = 0; i < 32; ++i) mp[i & 7] = fmaxf(mp[i & 7], __uint_as_float(sr[c][i]));
            const float mr = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])), fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
            const float mx = mr * a.scale_log2;
            // lazy rescale: keep the stale max unless this tile's max exceeds it by > 2^8
            const bool grow = mx > m + RESCALE_THRESHOLD;
            const float m_use = grow ? mx : m;
            const float corr = grow ? (m == -INFINITY ? 0.f : ex2(m - mx)) : 1.f;
            // p = 2^(s * scale - m): one FFMA + one exp2 per element; -inf -> +0
            const float nm = m_use == -INFINITY ? 0.f : -m_use;
            float sp[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) sp[k] = 0.f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                    const float e0 = ex2(fmaf(__uint_as_float(sr[c][i]), a.scale_log2, nm));
                    const float e1 = ex2(fmaf(__uint_as_float(sr[c][i + 1]), a.scale_log2, nm));
                    sp[(i >> 1) & 7] += e0 + e1;
                    pk[i / 2] = pack_bf16(e0, e1);
                }
                // P_t (bf16 pairs) over the first 64 columns of S_t: keys 32c .. 32c + 31
                tmem_st16(trow + sc + uint32_t(c * 16), pk);
            }
            // (after the exponentials, so S's registers are free) S_t of this tile completing implies PV_t of the previous one completed (issue
            // order), so O_t is stable here: rescale it in place when the max grew
            if (__any_sync(0xffffffffu, grow && j > 0)) {
                const float cf = (grow && j > 0) ? corr : 1.f;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t orr[32];
                    tmem_ld32(trow + oc + uint32_t(c * 32), orr);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int i = 0; i < 32; ++i) orr[i] = __float_as_uint(__uint_as_float(orr[i]) * cf);
                    tmem_st32(trow + oc + uint32_t(c * 32), orr);
                }
            }
            const float sum = ((sp[0] + sp[1]) + (sp[2] + sp[3])) + ((sp[4] + sp[5]) + (sp[6] + sp[7]));
            l = l * corr + sum;
            m = m_use;
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[t]);
            if (prof) busy += clock64() - c0;
        }
        if (prof) {  // sums over CTAs, cycles: softmax thread 0 waiting for S and working
            dev::trace_add(*a.head, 2, (unsigned long long)w_s);
            dev::trace_add(*a.head, 4, (unsigned long long)busy);
        }
        // ---------------- epilogue: O / l -> bf16 through O's map ----------------
        if (my_nkv > 0) mbar_wait(&o_done[t], (my_nkv - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const float inv = l > 0.f ? 1.f / l : 0.f;
        bf16* orow = a.o + int64_t(b) * a.o_sb + int64_t(h) * a.o_sh + int64_t(q) * a.o_ss;
        dev::pdl_wait();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t orr[32];
            tmem_ld32(trow + oc + uint32_t(c * 32), orr);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (q < a.Sq) {
                uint32_t w[16];
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    w[i] = pack_bf16(__uint_as_float(orr[2 * i]) * inv, __uint_as_float(orr[2 * i + 1]) * inv);
                uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
                for (int i = 0; i < 4; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
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

// Element address of (b, h, s, d) of a rank-4 operand map, evaluated on the host
// from the lowered descriptor (the same formula the kernels evaluate).
bool eval_addr(const vtc_map& m, int b, int h, int s, int d, uint64_t& addr) {
    int64_t idx[VTC_MAX_RANK] = {b, h, s, d};
    int piece = -1;
    int64_t off = desc_eval(m, idx, &piece);
    if (piece < 0) return false;
    addr = m.piece[piece].ptr + uint64_t(off) * 2;
    return true;
}

// Prove the map affine over (b, h * hstep, s, d): one piece; the position and
// dim axes carry only plain (div 1, no mod below the extent, ungrouped) digits;
// the (b, h) grid is checked point by point.
bool affine4(const vtc_map& m, int B, int Hx, int hstep, int S, int Dd, uint64_t& base, int64_t (&st)[4]) {
    if (m.rank != 4 || m.npieces != 1) return false;
    const vtc_piece& pc = m.piece[0];
    if (!pc.affine) {
        for (int i = 0; i < pc.ndigits; ++i) {
            const vtc_digit& dg = pc.dig[i];
            if (dg.axis != 2 && dg.axis != 3) continue;
            const int ext = dg.axis == 2 ? S : Dd;
            if (dg.group >= 0 || dg.div != 1 || (dg.mod != 0 && int64_t(dg.mod) < ext)) return false;
        }
        for (int i = 0; i < pc.ngroups; ++i) return false;
    }
    uint64_t a0, ab = 0, ah = 0, as, ad;
    if (!eval_addr(m, 0, 0, 0, 0, a0) || !eval_addr(m, 0, 0, S > 1 ? 1 : 0, 0, as) || !eval_addr(m, 0, 0, 0, 1, ad))
        return false;
    if (B > 1 && !eval_addr(m, 1, 0, 0, 0, ab)) return false;
    if (Hx > 1 && !eval_addr(m, 0, hstep, 0, 0, ah)) return false;
    st[0] = B > 1 ? int64_t(ab - a0) / 2 : 0;
    st[1] = Hx > 1 ? int64_t(ah - a0) / 2 : 0;
    st[2] = S > 1 ? int64_t(as - a0) / 2 : 0;
    st[3] = int64_t(ad - a0) / 2;
    if (st[3] != 1) return false;
    for (int bb = 0; bb < B; ++bb)
        for (int hh = 0; hh < Hx; ++hh)
            for (int s : {0, S - 1})
                for (int d : {0, Dd - 1}) {
                    uint64_t x;
                    if (!eval_addr(m, bb, hh * hstep, s, d, x)) return false;
                    if (x != a0 + uint64_t(2 * (bb * st[0] + hh * st[1] + int64_t(s) * st[2] + d))) return false;
                }
    base = a0;
    return true;
}

bool encode4(CUtensorMap* out, uint64_t base, int S, int Hx, int B, const int64_t (&st)[4]) {
    EncodeFn fn = encoder();
    if (!fn || base % 16) return false;
    auto pitch = [](int64_t s, int64_t fallback) { return cuuint64_t(s > 0 ? s : fallback) * 2; };
    cuuint64_t dims[4] = {cuuint64_t(D), cuuint64_t(S), cuuint64_t(Hx), cuuint64_t(B)};
    cuuint64_t str[3] = {pitch(st[2], D), pitch(st[1], int64_t(D) * S), pitch(st[0], int64_t(D) * S * Hx)};
    for (auto x : str)
        if (x % 16 || x >= (cuuint64_t(1) << 40)) return false;
    cuuint32_t box[4] = {64, 128, 1, 1}, es[4] = {1, 1, 1, 1};
    return fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, reinterpret_cast<void*>(base), dims, str, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool attn_fmha_prepare(AttnParams& p, bool encode) {
    static_assert(sizeof(FmhaArgs) <= 4096, "kernel parameter space");
    static_assert(sizeof(p.fmha) >= 3 * sizeof(CUtensorMap), "AttnParams::fmha too small");
    if (p.dt != KDType::BF16 || p.D != D || p.Dv != D || p.rank != 4 || p.has_bias || p.Sq < 1 || p.Sk < 1) return false;
    if (p.H % p.group) return false;
    const int B = p.Bt, H = p.H, Hk = p.H / p.group;
    uint64_t qb, kb, vb, ob;
    int64_t qs[4], ks[4], vs[4], os[4];
    if (!affine4(p.q.m, B, H, 1, p.Sq, D, qb, qs) || !affine4(p.k.m, B, Hk, p.group, p.Sk, D, kb, ks) ||
        !affine4(p.v.m, B, Hk, p.group, p.Sk, D, vb, vs) || !affine4(p.o.m, B, H, 1, p.Sq, D, ob, os))
        return false;
    if ((os[0] * 2) % 16 || (os[1] * 2) % 16 || (os[2] * 2) % 16) return false;
    if (!encode) return true;
    if (ob % 16) return false;
    auto* t = reinterpret_cast<CUtensorMap*>(p.fmha);
    if (!encode4(&t[0], qb, p.Sq, H, B, qs) || !encode4(&t[1], kb, p.Sk, Hk, B, ks) || !encode4(&t[2], vb, p.Sk, Hk, B, vs))
        return false;
    p.fmha_o = ob;
    p.fmha_os[0] = os[0];
    p.fmha_os[1] = os[1];
    p.fmha_os[2] = os[2];
    return true;
}

void launch_attn_fmha(const AttnParams& p, const AttnParams* dp, cudaStream_t s) {
    FmhaArgs a;
    std::memset(&a, 0, sizeof(a));
    const auto* t = reinterpret_cast<const CUtensorMap*>(p.fmha);
    a.q = t[0];
    a.k = t[1];
    a.v = t[2];
    a.o = reinterpret_cast<bf16*>(p.fmha_o);
    a.o_sb = p.fmha_os[0];
    a.o_sh = p.fmha_os[1];
    a.o_ss = p.fmha_os[2];
    a.head = &dp->head;
    a.H = p.H;
    a.group = p.group;
    a.Sq = p.Sq;
    a.Sk = p.Sk;
    a.causal = p.causal;
    a.qpairs = (p.Sq + 2 * BQ - 1) / (2 * BQ);
    a.scale_log2 = p.scale * LOG2E;
    const size_t smem = SMEM_BYTES + 1024;
    const dim3 grid(unsigned(a.qpairs), unsigned(p.Bt * p.H));
    cudaFuncSetAttribute(attn_fmha_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    launch_k(attn_fmha_kernel, grid, dim3(NTHREADS), smem, s, a);
}

}  // namespace vtc
