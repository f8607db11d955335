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
//   * CTA = 128 query rows of one (batch, head); 6 warps:
//       warps 0-3  softmax + epilogue (thread = query row = TMEM lane),
//       warp 4     TMA producer (Q once, then K / V tiles of 128 keys, 2 stages each;
//                  a K stage frees when its S MMA completes, a V stage after its PV MMA),
//       warp 5     MMA issuer (one thread);
//   * S_j = Q K_j^T: tcgen05.mma M128 N128 K16 x 8 (K-major A and B, 128-byte
//     swizzle) into one of two TMEM S buffers, so S_{j+1} is computed while
//     the softmax warps work on S_j;
//   * the softmax warps read their S row with tcgen05.ld, apply scale / causal
//     mask, keep a running row max in the log2 domain and write P = exp2(S - m)
//     as bf16 into shared memory (the K-major A operand of the next MMA);
//   * O += P_j V_j: tcgen05.mma with V as the MN-major B operand, accumulated
//     in TMEM across all key tiles.  The running max is rescaled lazily: O (in
//     TMEM) and l are rescaled only when a row's max grows by more than 2^8,
//     otherwise P uses the stale max (bounded by 256, exact in fp32 / bf16);
//   * epilogue: O / l from TMEM to bf16, 16-byte stores through O's map.
// Causal query tiles stop at the diagonal key tile and are scheduled longest
// first.  Attention is absent from the reference (SURVEY.md §8 a'); CPU
// restatement: oracle/vtc_oracle.py (Attention).
#include <cuda.h>

#include <cstring>

#include "device.cuh"
#include "launch.cuh"
#include "lower.hpp"

namespace vtc {
namespace {

using dev::bf16;
constexpr int BQ = 128, BKV = 128, D = 128, NTHREADS = 192;
constexpr uint32_t CHUNK = 128 * 128;               // one [128 rows x 64 bf16] SW128 chunk = 16 KB
constexpr uint32_t TILE = 2 * CHUNK;                // 128 x 128 bf16
constexpr uint32_t SMEM_Q = 0, SMEM_K = TILE, SMEM_V = 3 * TILE, SMEM_P = 5 * TILE, SMEM_BYTES = 6 * TILE;
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
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

struct FmhaArgs {
    CUtensorMap q, k, v;     // 4-D {d, position, head, batch}, box {64, 128, 1, 1}, 128-byte swizzle
    bf16* o;                 // output element (b, h, s, 0) = o + b*o_sb + h*o_sh + s*o_ss
    int64_t o_sb, o_sh, o_ss;
    const KHead* head;       // timeline (VTC_TRACE)
    int32_t H, group, Sq, Sk, causal, qtiles;
    float scale_log2;
};

__global__ void __launch_bounds__(NTHREADS, 1) attn_fmha_kernel(const __grid_constant__ FmhaArgs a) {
    dev::TraceScope trace_scope_(a.head);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t q_full, k_full[2], v_full[2], k_empty[2], v_empty[2], s_full[2], p_full, o_done;
    __shared__ uint32_t s_tmem;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // causal: the longest query tiles (most key tiles) first
    const int qt = a.causal ? a.qtiles - 1 - int(blockIdx.x) : int(blockIdx.x);
    const int q0 = qt * BQ;
    const int bh = int(blockIdx.y);
    const int b = bh / a.H, h = bh - b * a.H, hkv = h / a.group;
    const int off = a.Sk - a.Sq;  // query row q sees keys t <= q + off
    const int kend = a.causal ? min(a.Sk, q0 + BQ + off) : a.Sk;
    const int nkv = kend > 0 ? (kend + BKV - 1) / BKV : 0;

    if (threadIdx.x == 0) {
        mbar_init(&q_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&v_full[s], 1);
            mbar_init(&k_empty[s], 1);
            mbar_init(&v_empty[s], 1);
            mbar_init(&s_full[s], 1);
        }
        mbar_init(&p_full, 4);  // one arrival per softmax warp
        mbar_init(&o_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {  // TMEM: S buffers at columns 0 / 128, O at 256
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    dev::pdl_launch_dependents();
    const uint32_t sbase = smem_u32(smem);

    if (warp == 4) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.q)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.k)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.v)) : "memory");
            const uint64_t pol = evict_last_policy();  // K / V re-read by every query tile of the head
            dev::pdl_wait();
            mbar_expect_tx(&q_full, TILE);
            tma_4d(sbase + SMEM_Q, &a.q, 0, q0, h, b, &q_full, pol);
            tma_4d(sbase + SMEM_Q + CHUNK, &a.q, 64, q0, h, b, &q_full, pol);
            for (int j = 0; j < nkv; ++j) {
                const int st = j & 1;
                const uint32_t ks = sbase + SMEM_K + st * TILE, vs = sbase + SMEM_V + st * TILE;
                // K_j's stage frees when S_{j-2} is computed, V_j's when PV_{j-2} is
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
    } else if (warp == 5) {
        if (lane == 0) {
            // ---------------- MMA issuer ----------------
            constexpr uint32_t id_s = idesc(BQ, BKV, 0), id_o = idesc(BQ, D, 1);
            mbar_wait(&q_full, 0);
            const bool prof = a.head->trace != nullptr;  // VTC_TRACE: per-CTA wait accounting (clock64)
            long long w_k = 0, w_v = 0, w_p = 0;
            auto issue_s = [&](int j) {
                const int st = j & 1;
                const long long c0 = prof ? clock64() : 0;
                mbar_wait(&k_full[st], (j >> 1) & 1);
                if (prof) w_k += clock64() - c0;
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t qa = sbase + SMEM_Q, kb = sbase + SMEM_K + st * TILE;
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const uint32_t o = (k >> 2) * CHUNK + (k & 3) * 32;  // K-major SW128: +32 B per K16, next chunk per 64
                    mma(tmem + uint32_t(st * BKV), smem_desc(qa + o, 16, 1024), smem_desc(kb + o, 16, 1024), id_s,
                        k > 0 ? 1u : 0u);
                }
                commit(&s_full[st]);
                commit(&k_empty[st]);
            };
            if (nkv > 0) issue_s(0);
            for (int j = 0; j < nkv; ++j) {
                const int st = j & 1;
                if (j + 1 < nkv) issue_s(j + 1);  // S buffer (j+1)&1 was released by softmax j-1
                const long long c0 = prof ? clock64() : 0;
                mbar_wait(&p_full, j & 1);
                if (prof) w_p += clock64() - c0;
                const long long c1 = prof ? clock64() : 0;
                mbar_wait(&v_full[st], (j >> 1) & 1);
                if (prof) w_v += clock64() - c1;
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t pa = sbase + SMEM_P, vb = sbase + SMEM_V + st * TILE;
#pragma unroll
                for (int k = 0; k < BKV / 16; ++k) {
                    // P: K-major (keys) SW128; V: MN-major, 16 keys = 2 KB per step, 64-d chunks 16 KB apart
                    const uint32_t po = (k >> 2) * CHUNK + (k & 3) * 32;
                    mma(tmem + 256u, smem_desc(pa + po, 16, 1024), smem_desc(vb + uint32_t(k) * 2048u, CHUNK, 1024), id_o,
                        (j > 0 || k > 0) ? 1u : 0u);
                }
                commit(&o_done);
                commit(&v_empty[st]);
            }
            if (prof) {  // sums over CTAs, cycles: MMA thread waiting for K, P, V
                dev::trace_add(*a.head, 5, (unsigned long long)w_k);
                dev::trace_add(*a.head, 6, (unsigned long long)w_p);
                dev::trace_add(*a.head, 7, (unsigned long long)w_v);
            }
        }
    } else {
        // ---------------- softmax (warps 0-3): thread = query row = TMEM lane ----------------
        const int r = warp * 32 + lane;
        const int q = q0 + r;
        const int lim = q + off;  // last visible key (causal)
        const uint32_t trow = tmem + (uint32_t(warp * 32) << 16);
        float m = -INFINITY, l = 0.f;
        const uint32_t prow = sbase + SMEM_P + uint32_t(r) * 128u;
        const bool prof = a.head->trace != nullptr && threadIdx.x == 0;
        long long w_s = 0, w_o = 0, busy = 0;
        for (int j = 0; j < nkv; ++j) {
            const int st = j & 1;
            long long c0 = prof ? clock64() : 0;
            mbar_wait(&s_full[st], (j >> 1) & 1);
            if (prof) {
                const long long c = clock64();
                w_s += c - c0;
                c0 = c;
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint32_t sr[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(trow + uint32_t(st * BKV + c * 32), sr[c]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int t0 = j * BKV;
            const bool masked = (a.causal && t0 + BKV - 1 > q0 + off) || t0 + BKV > a.Sk;
            if (masked) {  // diagonal / tail tiles only: invisible keys -> -inf
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int t = t0 + c * 32 + i;
                        if (t >= a.Sk || (a.causal && t > lim)) sr[c][i] = __float_as_uint(-INFINITY);
                    }
            }
            float mr = -INFINITY;  // raw row max (scale > 0: max commutes with the scale)
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int i = 0; i < 32; ++i) mr = fmaxf(mr, __uint_as_float(sr[c][i]));
            const float mx = mr * a.scale_log2;
            // lazy rescale: keep the stale max unless this tile's max exceeds it by > 2^8
            const bool grow = mx > m + RESCALE_THRESHOLD;
            const float m_use = grow ? mx : m;
            const float corr = grow ? (m == -INFINITY ? 0.f : ex2(m - mx)) : 1.f;
            // p = 2^(s * scale - m): one FFMA + one MUFU.EX2 per element; -inf -> +0
            const float nm = m_use == -INFINITY ? 0.f : -m_use;
            float sum = 0.f;
            uint32_t pk[64];
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                    const float e0 = ex2(fmaf(__uint_as_float(sr[c][i]), a.scale_log2, nm));
                    const float e1 = ex2(fmaf(__uint_as_float(sr[c][i + 1]), a.scale_log2, nm));
                    sum += e0 + e1;
                    pk[c * 16 + i / 2] = pack_bf16(e0, e1);
                }
            // PV_{j-1} complete: the P buffer is free and O is stable
            long long c1 = prof ? clock64() : 0;
            if (j > 0) mbar_wait(&o_done, (j - 1) & 1);
            if (prof) {
                const long long c = clock64();
                busy += c1 - c0;
                w_o += c - c1;
                c0 = c;
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (__any_sync(0xffffffffu, grow && j > 0)) {
                const float cf = (grow && j > 0) ? corr : 1.f;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t orr[32];
                    tmem_ld32(trow + 256u + uint32_t(c * 32), orr);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int i = 0; i < 32; ++i) orr[i] = __float_as_uint(__uint_as_float(orr[i]) * cf);
                    tmem_st32(trow + 256u + uint32_t(c * 32), orr);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            l = l * corr + sum;
            m = m_use;
            // P row -> K-major SW128 operand: 16 chunks of 8 keys; chunk c of atom c/8 at (c%8) ^ (r%8)
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const uint32_t dst = prow + (c >> 3) * CHUNK + (((c & 7) ^ (r & 7)) << 4);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(pk[4 * c]), "r"(pk[4 * c + 1]),
                             "r"(pk[4 * c + 2]), "r"(pk[4 * c + 3])
                             : "memory");
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full);
            if (prof) busy += clock64() - c0;
        }
        if (prof) {  // sums over CTAs, cycles: softmax thread 0 waiting for S, for PV, and working
            dev::trace_add(*a.head, 2, (unsigned long long)w_s);
            dev::trace_add(*a.head, 3, (unsigned long long)w_o);
            dev::trace_add(*a.head, 4, (unsigned long long)busy);
        }
        // ---------------- epilogue: O / l -> bf16 through O's map ----------------
        if (nkv > 0) mbar_wait(&o_done, (nkv - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const float inv = l > 0.f ? 1.f / l : 0.f;
        bf16* orow = a.o + int64_t(b) * a.o_sb + int64_t(h) * a.o_sh + int64_t(q) * a.o_ss;
        dev::pdl_wait();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t orr[32];
            tmem_ld32(trow + 256u + uint32_t(c * 32), orr);
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
    a.qtiles = (p.Sq + BQ - 1) / BQ;
    a.scale_log2 = p.scale * LOG2E;
    const size_t smem = SMEM_BYTES + 1024;
    cudaFuncSetAttribute(attn_fmha_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    launch_k(attn_fmha_kernel, dim3(unsigned(a.qtiles), unsigned(p.Bt * p.H)), dim3(NTHREADS), smem, s, a);
}

}  // namespace vtc
