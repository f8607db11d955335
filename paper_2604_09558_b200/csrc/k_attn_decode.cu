// Split-KV flash-decoding attention on tensor cores (bf16, head dim 128).
//
// The decode-attention fast path of the executor: softmax(scale * Q K^T) V for
// the G query heads of one GQA group (x Sq query rows, G*Sq <= 16) against one
// KV head.  In a VTC-planned decoder Q, K and V are virtual tensors -- K/V are
// the KV-cache slice -> transpose -> GQA Expand/Reshape chain composed into
// one map onto the pos-major cache, with h -> h div G -- so the kernel reads
// every K/V row exactly once for the whole group (the paper's 4x read
// reduction) and never materialises the expanded tensors.
//
//   * CTA = 4 warps; the CTA's key range (one split) is cut into 16-key
//     tiles, dealt round-robin to the warps;
//   * each warp streams its tiles through a private 3-stage cp.async ring
//     (K and V rows, 16-byte chunks, XOR-swizzled so ldmatrix is
//     conflict-free); row addresses come from the K/V maps: base + t * stride
//     when the host proved the map affine along the key axis, else one map
//     evaluation per key row;
//   * S = Q K^T and O += P V run on mma.sync m16n8k16 (bf16 in, fp32
//     accumulate), query rows in the M dimension; the online softmax works in
//     the log2 domain on the fp32 scores; P is rounded to bf16 for P V;
//   * the 4 warps' (m, l, O) are merged in shared memory in warp order; one
//     split writes O through the output map, several write fp32 partials that
//     combine_kernel (k_attention.cu) merges in split order.
// Attention itself is absent from the reference (SURVEY.md §8 a'); the CPU
// restatement is oracle/vtc_oracle.py (Attention).
#include <cfloat>

#include "device.cuh"
#include "launch.cuh"

namespace vtc {
namespace {

using dev::bf16;
constexpr int WARPS = 4, NT = WARPS * 32, TK = 16, D = 128, STAGES = 2;
constexpr int ROWB = D * 2;                     // bytes per K/V row
constexpr int TILEB = TK * ROWB;                // 4 KB per K (or V) tile
constexpr int STAGEB = 2 * TILEB;               // K + V
constexpr int WARPB = STAGES * STAGEB;          // 24 KB per warp
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid, uint64_t policy) {
    // src-size 0 zero-fills the 16 bytes (keys past the end of the range);
    // K/V rows are read once per step: L2 evict-first
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0), "l"(policy)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}
// byte offset of 16-byte chunk c of row r inside a tile (XOR swizzle on the low 3 bits)
__device__ __forceinline__ uint32_t swz(int r, int c) { return uint32_t(r * ROWB + ((c ^ (r & 7)) << 4)); }

// KVA: K/V rows affine along the key axis (host-proved p.kv_affine) -- the
// per-row map evaluation path is compiled out, which keeps the hot loop's code
// (and its instruction-cache footprint) small.
template <bool KVA>
__global__ void __launch_bounds__(NT, 2) attn_decode_kernel(const AttnParams* __restrict__ pp) {
    VTC_STAGE_PARAMS(AttnParams, pp);
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ float s_m[WARPS][16], s_l[WARPS][16];
    __shared__ const bf16* s_krow[WARPS][TK];
    __shared__ const bf16* s_vrow[WARPS][TK];
    __shared__ const bf16* s_qrow[16];
    __shared__ bf16* s_orow[16];
    __shared__ int64_t s_qstr[16], s_ostr[16];

    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int G = p.group, HG = p.H / G, Sq = p.Sq, R = G * Sq;  // R query rows (<= 16)
    const int r = p.rank, ax_h = r - 3, ax_s = r - 2, ax_d = r - 1;

    // 32-bit index arithmetic (grid dimensions fit): no 64-bit division calls
    const uint32_t qlead = blockIdx.x / uint32_t(HG);
    const int hg = int(blockIdx.x - qlead * uint32_t(HG));
    uint32_t qb = qlead;
    int32_t base_idx[VTC_MAX_RANK] = {};
    {
        uint32_t b = qb;
        for (int a = r - 4; a >= 0; --a) {
            int32_t ext = p.q.m.shape[a];
            const uint32_t nb = b / uint32_t(ext);
            base_idx[a] = int32_t(b - nb * uint32_t(ext));
            b = nb;
        }
    }
    const int h0 = hg * G;
    const int split = blockIdx.y;
    const int kbeg = split * p.chunk;
    int kend = min(p.Sk, kbeg + p.chunk);
    if (p.causal) kend = min(kend, (Sq - 1) + (p.Sk - Sq) + 1);  // last row's limit; rows masked below
    const int ntiles = kend > kbeg ? (kend - kbeg + TK - 1) / TK : 0;

    // K/V row addressing: affine along the key axis (host-proved) or per-row map evaluation
    const bf16* kb0 = nullptr;
    const bf16* vb0 = nullptr;
    if (KVA) {
        int32_t idx[VTC_MAX_RANK];
#pragma unroll
        for (int a = 0; a < VTC_MAX_RANK; ++a) idx[a] = base_idx[a];
        idx[ax_h] = h0;
        idx[ax_s] = 0;
        idx[ax_d] = 0;
        kb0 = dev::elem_ptr<bf16>(p.k.m, idx);
        vb0 = dev::elem_ptr<bf16>(p.v.m, idx);
    }
    if (tid == 0) dev::trace_point(p.head, 2);
    dev::pdl_wait();
    dev::pdl_launch_dependents();
    if (tid == 0) dev::trace_point(p.head, 3);

    const uint64_t policy = dev::evict_first_policy();
    unsigned char* wsm = smem + warp * WARPB;
    const uint32_t wsm_u = smem_u32(wsm);

    // issue the cp.asyncs of this warp's j-th tile into stage st
    auto load_tile = [&](int j, int st) {
        const int tile = warp + j * WARPS;
        const int t0 = kbeg + tile * TK;
        if (!KVA) {
            if (lane < TK) {
                int t = min(t0 + lane, kend - 1);
                int32_t idx[VTC_MAX_RANK];
#pragma unroll
                for (int a = 0; a < VTC_MAX_RANK; ++a) idx[a] = base_idx[a];
                idx[ax_h] = h0;
                idx[ax_s] = t;
                idx[ax_d] = 0;
                s_krow[warp][lane] = dev::elem_ptr<bf16>(p.k.m, idx);
                s_vrow[warp][lane] = dev::elem_ptr<bf16>(p.v.m, idx);
            }
            __syncwarp();
        }
        const uint32_t kdst = wsm_u + st * STAGEB, vdst = kdst + TILEB;
#pragma unroll
        for (int i = 0; i < (TK * ROWB / 16) / 32; ++i) {  // 8 chunks per lane per tile
            const int c = lane + i * 32;
            const int row = c >> 4, ch = c & 15;
            const int t = t0 + row;
            const bool ok = t < kend;
            const int tc = ok ? t : kbeg;
            const bf16* ks = KVA ? kb0 + int64_t(tc) * p.k_sstride : s_krow[warp][row];
            const bf16* vs = KVA ? vb0 + int64_t(tc) * p.v_sstride : s_vrow[warp][row];
            cp_async16(kdst + swz(row, ch), ks + ch * 8, ok, policy);
            cp_async16(vdst + swz(row, ch), vs + ch * 8, ok, policy);
        }
    };

    // Q first: its row loads go out ahead of the K/V prologue (which requests a
    // large share of the KV cache at once), then the K/V cp.asyncs, then Q is
    // written to shared memory and turned into fragments
    uint32_t qa[D / 16][4];
    __shared__ __align__(16) bf16 s_q[16][D];
    if (tid < R) {
        int32_t idx[VTC_MAX_RANK];
#pragma unroll
        for (int a = 0; a < VTC_MAX_RANK; ++a) idx[a] = base_idx[a];
        idx[ax_h] = h0 + tid / Sq;
        idx[ax_s] = tid % Sq;
        idx[ax_d] = 0;
        dev::Loc l = dev::locate(p.q.m, idx);
        s_qrow[tid] = dev::addr<bf16>(p.q.m, l);
        s_qstr[tid] = p.q.fast_stride[l.piece];
        dev::Loc lo = dev::locate(p.o.m, idx);
        s_orow[tid] = dev::addr<bf16>(p.o.m, lo);
        s_ostr[tid] = p.o.fast_stride[lo.piece];
    }
    __syncthreads();
    constexpr int QCH = 16 * (D / 8) / NT;  // 16-byte chunks of the 16 x D query block per thread
    uint4 qv[QCH];
#pragma unroll
    for (int i = 0; i < QCH; ++i) {
        const int c = tid + i * NT;
        const int row = c / (D / 8), ch = c % (D / 8);
        uint4 v = make_uint4(0, 0, 0, 0);
        if (row < R) {
            if (s_qstr[row] == 1 && (reinterpret_cast<uintptr_t>(s_qrow[row]) & 15) == 0) {
                v = *reinterpret_cast<const uint4*>(s_qrow[row] + ch * 8);
            } else {
                bf16 t[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) t[j] = s_qrow[row][int64_t(ch * 8 + j) * s_qstr[row]];
                v = *reinterpret_cast<const uint4*>(t);
            }
        }
        qv[i] = v;
    }

    const int my_tiles = ntiles > warp ? (ntiles - warp + WARPS - 1) / WARPS : 0;
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < my_tiles) load_tile(s, s);
        cp_async_commit();
    }
    // this CTA's share of the next projection's weights into L2, queued behind its own K / V loads
    if (p.pf_bytes > 0 && tid == 0) {
        const uint64_t nct = uint64_t(gridDim.x) * gridDim.y, cta = uint64_t(blockIdx.y) * gridDim.x + blockIdx.x;
        const uint64_t per = ((uint64_t(p.pf_bytes) + nct - 1) / nct + 15) & ~uint64_t(15);
        const uint64_t lo = cta * per, hi = min(lo + per, uint64_t(p.pf_bytes));
        for (uint64_t o = lo; o < hi; o += 32768) {
            const uint64_t left = hi - o;
            const uint32_t sz = uint32_t(left < 32768 ? left : 32768) & ~15u;
            if (sz) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.pf_base + o), "r"(sz) : "memory");
        }
    }

    {
#pragma unroll
        for (int i = 0; i < QCH; ++i) {
            const int c = tid + i * NT;
            *reinterpret_cast<uint4*>(&s_q[c / (D / 8)][(c % (D / 8)) * 8]) = qv[i];
        }
        __syncthreads();
        const int rA = lane / 4, rB = lane / 4 + 8, kc = (lane % 4) * 2;
        auto qp = [&](int row, int d) -> uint32_t { return *reinterpret_cast<const uint32_t*>(&s_q[row][d]); };
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
            const int d0 = ks * 16 + kc;
            qa[ks][0] = qp(rA, d0);
            qa[ks][1] = qp(rB, d0);
            qa[ks][2] = qp(rA, d0 + 8);
            qa[ks][3] = qp(rB, d0 + 8);
        }
    }
    if (tid == 0) dev::trace_point(p.head, 4);
    const float qscale = p.scale * LOG2E;
    const int rowA = lane / 4, rowB = lane / 4 + 8;
    // causal: query row (g, sq) may see key t iff t <= sq + Sk - Sq
    const int limA = p.causal ? (rowA % Sq) + p.Sk - Sq : INT32_MAX;
    const int limB = p.causal ? (rowB % Sq) + p.Sk - Sq : INT32_MAX;

    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;

    for (int j = 0; j < my_tiles; ++j) {
        const int st = j % STAGES;
        if (j + STAGES - 1 < my_tiles) load_tile(j + STAGES - 1, (j + STAGES - 1) % STAGES);
        cp_async_commit();
        cp_async_wait<STAGES - 1>();
        __syncwarp();
        const uint32_t kt = wsm_u + st * STAGEB, vt = kt + TILEB;
        const int t0 = kbeg + (warp + j * WARPS) * TK;

        // S[16 x 16] = Q K^T: two n8 tiles (keys 0-7, 8-15) x 8 k-steps
        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
            for (int kp = 0; kp < D / 32; ++kp) {  // two k-steps per ldmatrix.x4
                const int mi = lane / 8, rr = lane % 8;
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kt + swz(nt * 8 + rr, kp * 4 + mi), b0, b1, b2, b3);
                mma_bf16(sc[nt], qa[2 * kp], b0, b1);
                mma_bf16(sc[nt], qa[2 * kp + 1], b2, b3);
            }
        }
        // online softmax (log2 domain); thread owns rows rowA (sc[.][0..1]) and rowB (sc[.][2..3])
        float tmA = -INFINITY, tmB = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int t = t0 + nt * 8 + (lane % 4) * 2 + c;
                float a = sc[nt][c] * qscale, b = sc[nt][2 + c] * qscale;
                if (t >= kend || t > limA) a = -INFINITY;
                if (t >= kend || t > limB) b = -INFINITY;
                sc[nt][c] = a;
                sc[nt][2 + c] = b;
                tmA = fmaxf(tmA, a);
                tmB = fmaxf(tmB, b);
            }
#pragma unroll
        for (int off = 1; off < 4; off <<= 1) {
            tmA = fmaxf(tmA, __shfl_xor_sync(0xffffffffu, tmA, off));
            tmB = fmaxf(tmB, __shfl_xor_sync(0xffffffffu, tmB, off));
        }
        const float nmA = fmaxf(mA, tmA), nmB = fmaxf(mB, tmB);
        const float cA = nmA == -INFINITY ? 1.f : exp2f(mA - nmA);
        const float cB = nmB == -INFINITY ? 1.f : exp2f(mB - nmB);
        float sA = 0.f, sB = 0.f;
        uint32_t pa[4];
        float pv[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                float a = sc[nt][c] == -INFINITY ? 0.f : exp2f(sc[nt][c] - nmA);
                float b = sc[nt][2 + c] == -INFINITY ? 0.f : exp2f(sc[nt][2 + c] - nmB);
                pv[nt][c] = a;
                pv[nt][2 + c] = b;
                sA += a;
                sB += b;
            }
        lA = lA * cA + sA;  // per-thread partial row sums; reduced across the quad at the end
        lB = lB * cB + sB;
        mA = nmA;
        mB = nmB;
        pa[0] = pack_bf16(pv[0][0], pv[0][1]);
        pa[1] = pack_bf16(pv[0][2], pv[0][3]);
        pa[2] = pack_bf16(pv[1][0], pv[1][1]);
        pa[3] = pack_bf16(pv[1][2], pv[1][3]);
        // O[16 x 128] = O * corr + P V
#pragma unroll
        for (int i = 0; i < D / 8; ++i) {
            o[i][0] *= cA;
            o[i][1] *= cA;
            o[i][2] *= cB;
            o[i][3] *= cB;
        }
#pragma unroll
        for (int np = 0; np < D / 16; ++np) {  // two n8 tiles of dv per ldmatrix.x4.trans
            const int mi = lane / 8, rr = lane % 8;
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(vt + swz((mi & 1) * 8 + rr, np * 2 + (mi >> 1)), b0, b1, b2, b3);
            mma_bf16(o[2 * np], pa, b0, b1);
            mma_bf16(o[2 * np + 1], pa, b2, b3);
        }
        __syncwarp();
    }
    cp_async_wait<0>();
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
        lA += __shfl_xor_sync(0xffffffffu, lA, off);
        lB += __shfl_xor_sync(0xffffffffu, lB, off);
    }

    if (lane == 0) dev::trace_point(p.head, 5);
    // ---- merge the 4 warps (warp order) ----
    __syncthreads();  // all warps done with their rings: reuse smem for O
    float* sO = reinterpret_cast<float*>(smem);  // [WARPS][16][D]
    if (lane % 4 == 0) {
        s_m[warp][rowA] = mA;
        s_m[warp][rowB] = mB;
        s_l[warp][rowA] = lA;
        s_l[warp][rowB] = lB;
    }
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
        const int c = i * 8 + (lane % 4) * 2;
        sO[(warp * 16 + rowA) * D + c] = o[i][0];
        sO[(warp * 16 + rowA) * D + c + 1] = o[i][1];
        sO[(warp * 16 + rowB) * D + c] = o[i][2];
        sO[(warp * 16 + rowB) * D + c + 1] = o[i][3];
    }
    __syncthreads();
    for (int e = tid; e < R * D; e += NT) {
        const int row = e / D, d = e % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) M = fmaxf(M, s_m[w][row]);
        float L = 0.f, acc = 0.f;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
            const float f = s_m[w][row] == -INFINITY ? 0.f : exp2f(s_m[w][row] - M);
            L += f * s_l[w][row];
            acc += f * sO[(w * 16 + row) * D + d];
        }
        const int g = row / Sq, sq = row % Sq, h = h0 + g;
        if (p.splits == 1) {
            s_orow[row][int64_t(d) * s_ostr[row]] = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
        } else {
            const int64_t orow = (int64_t(qlead) * p.H + h) * Sq + sq;
            p.part_o[(orow * p.splits + split) * D + d] = acc;
            if (d == 0) {
                p.part_ml[(orow * p.splits + split) * 2] = M;
                p.part_ml[(orow * p.splits + split) * 2 + 1] = L;
            }
        }
    }
    if (p.splits == 1 || p.counters == nullptr) return;  // no counters: combine_fast_kernel merges
    if (tid == 0) dev::trace_point(p.head, 6);

    // ---- split-KV combine, cooperative: every split CTA of the group waits
    //      until all S partials are written (all CTAs are co-resident -- the
    //      host enables this only when the grid fits the GPU at once), then
    //      merges a 1/S slice of the group's R x D outputs in split order ----
    __shared__ unsigned s_target;
    __threadfence();
    __syncthreads();
    const int S = p.splits;
    if (tid == 0) {
        // tickets grow monotonically across executions: no reset needed
        const unsigned ticket = atomicAdd(&p.counters[blockIdx.x], 1u);
        const unsigned target = (ticket / unsigned(S) + 1u) * unsigned(S);
        unsigned seen;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(&p.counters[blockIdx.x]) : "memory");
            if (int(seen - target) < 0) __nanosleep(64);
        } while (int(seen - target) < 0);
        s_target = target;
    }
    __syncthreads();
    const int64_t orow0 = int64_t(qlead) * p.H + h0;  // (lead, h0): rows (g, sq) follow
    const int per = (R * D + S - 1) / S;
    for (int i = tid; i < per; i += NT) {
        const int e = split * per + i;
        if (e >= R * D) break;
        const int row = e / D, d = e % D;
        const int64_t base = (orow0 * Sq + row) * S;
        float L = 0.f, acc = 0.f, M = -INFINITY;
        for (int s0 = 0; s0 < S; s0 += 32) {
            float mv[32], lv[32], ov[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int s2 = s0 + j;
                mv[j] = s2 < S ? __ldcg(&p.part_ml[(base + s2) * 2]) : -INFINITY;
                lv[j] = s2 < S ? __ldcg(&p.part_ml[(base + s2) * 2 + 1]) : 0.f;
                ov[j] = s2 < S ? __ldcg(&p.part_o[(base + s2) * D + d]) : 0.f;
            }
            float Mb = -INFINITY;
#pragma unroll
            for (int j = 0; j < 32; ++j) Mb = fmaxf(Mb, mv[j]);
            const float Mn = fmaxf(M, Mb);
            const float c = M == -INFINITY ? 0.f : exp2f(M - Mn);
            L *= c;
            acc *= c;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float f = mv[j] == -INFINITY ? 0.f : exp2f(mv[j] - Mn);
                L += f * lv[j];
                acc += f * ov[j];
            }
            M = Mn;
        }
        s_orow[row][int64_t(d) * s_ostr[row]] = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
    }
}

// Split merge as a separate kernel: one CTA per (lead, h, sq) output row, all
// split partials of the row loaded at once (one memory round trip).
__global__ void __launch_bounds__(NT) combine_fast_kernel(const AttnParams* __restrict__ pp) {
    VTC_STAGE_PARAMS(AttnParams, pp);
    __shared__ bf16* s_out;
    __shared__ int64_t s_ostride;
    const int64_t row = blockIdx.x;  // (lead, h, sq)
    const int S = p.splits;
    if (threadIdx.x == 0) {
        const int r = p.rank;
        int64_t rr = row;
        int32_t idx[VTC_MAX_RANK] = {};
        idx[r - 2] = int32_t(rr % p.Sq);
        rr /= p.Sq;
        idx[r - 3] = int32_t(rr % p.H);
        rr /= p.H;
        for (int a = r - 4; a >= 0; --a) {
            idx[a] = int32_t(rr % p.o.m.shape[a]);
            rr /= p.o.m.shape[a];
        }
        dev::Loc l = dev::locate(p.o.m, idx);
        s_out = dev::addr<bf16>(p.o.m, l);
        s_ostride = p.o.fast_stride[l.piece];
    }
    dev::pdl_wait();
    dev::pdl_launch_dependents();
    __syncthreads();  // s_out / s_ostride
    // every load of the row in flight at once: (m, l) pairs and this thread's
    // column of the partial outputs (32 splits per batch)
    const int d = threadIdx.x;
    float L = 0.f, acc = 0.f, M = -INFINITY;
    for (int s0 = 0; s0 < S; s0 += 32) {
        float mv[32], lv[32], ov[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int s2 = s0 + j;
            mv[j] = s2 < S ? __ldcg(&p.part_ml[(row * S + s2) * 2]) : -INFINITY;
            lv[j] = s2 < S ? __ldcg(&p.part_ml[(row * S + s2) * 2 + 1]) : 0.f;
            ov[j] = s2 < S ? __ldcg(&p.part_o[(row * S + s2) * D + d]) : 0.f;
        }
        float Mb = -INFINITY;
#pragma unroll
        for (int j = 0; j < 32; ++j) Mb = fmaxf(Mb, mv[j]);
        const float Mn = fmaxf(M, Mb);
        const float c = M == -INFINITY ? 0.f : exp2f(M - Mn);
        L *= c;
        acc *= c;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const float f = mv[j] == -INFINITY ? 0.f : exp2f(mv[j] - Mn);
            L += f * lv[j];
            acc += f * ov[j];
        }
        M = Mn;
    }
    s_out[int64_t(d) * s_ostride] = __float2bfloat16_rn(L > 0.f ? acc / L : 0.f);
}

}  // namespace

bool attn_decode_supported(const AttnParams& p) {
    return p.dt == KDType::BF16 && p.D == D && p.Dv == D && !p.has_bias && p.group * p.Sq <= 16 && p.k.vec_ok &&
           p.v.vec_ok && p.q.fast_ok && p.o.fast_ok;
}

size_t attn_decode_smem() { return size_t(WARPS) * WARPB; }

// CTAs of attn_decode_kernel resident at once on the whole GPU (the cooperative
// split combine spins on its group's arrivals, so every CTA must be resident).
int64_t attn_decode_capacity() {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(attn_decode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(attn_decode_smem()));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, attn_decode_kernel<true>, NT, attn_decode_smem());
    return int64_t(sms) * per;
}

void launch_attn_decode(const AttnParams& p, const AttnParams* dp, cudaStream_t s) {
    int64_t qblocks = int64_t(p.Bt) * (p.H / p.group);
    dim3 grid(unsigned(qblocks), unsigned(p.splits));
    size_t smem = attn_decode_smem();
    if (p.kv_affine) {
        cudaFuncSetAttribute(attn_decode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        launch_k(attn_decode_kernel<true>, grid, dim3(NT), smem, s, dp);
    } else {
        cudaFuncSetAttribute(attn_decode_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        launch_k(attn_decode_kernel<false>, grid, dim3(NT), smem, s, dp);
    }
    if (p.splits > 1 && p.counters == nullptr)
        launch_k(combine_fast_kernel, dim3(unsigned(int64_t(p.Bt) * p.H * p.Sq)), dim3(NT), 0, s, dp);
}

}  // namespace vtc
