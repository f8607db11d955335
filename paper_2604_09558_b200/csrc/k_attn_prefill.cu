// Flash attention for long query blocks (prefill, windows), bf16, head dim 32 / 64 / 128,
// optional additive bias through its own map (Swin relative-position bias + shift mask).
//
// softmax(scale * Q K^T [causal]) V with Q, K, V and O read / written through
// their VirtualTensor maps: in a VTC-planned prefill the QKV split, the RoPE
// output, the [B,S,H,d] -> [B,H,S,d] transposes and the GQA Expand/Reshape of
// K/V are all views, so the kernel addresses the projection outputs directly
// (per query row one map evaluation, per (batch, KV head) one base + key stride).
//
//   * CTA = 4 warps x 16 query rows of one (lead, head); K/V tiles of 64 keys
//     shared by the 4 warps through a 2-stage cp.async ring (XOR-swizzled rows,
//     ldmatrix / ldmatrix.trans), zero-filled past the end;
//   * S = Q K^T and O += P V on mma.sync m16n8k16 (bf16, fp32 accumulate),
//     online softmax in the log2 domain; causal query blocks stop at the
//     diagonal key tile (masked inside it);
//   * O / l rounded to bf16 and stored through the output map.
// Attention is absent from the reference (SURVEY.md §8 a'); CPU restatement:
// oracle/vtc_oracle.py (Attention).
#include <cfloat>

#include "device.cuh"
#include "launch.cuh"

namespace vtc {
namespace {

using dev::bf16;
constexpr int WARPS = 4, NT = WARPS * 32, QR = 16 * WARPS, TK = 64, STAGES = 2;
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 32-bit global load (data the kernel never writes; no memory clobber, so loads batch)
__device__ __forceinline__ uint32_t ld_g32(const void* p) {
    uint32_t v;
    asm("ld.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
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
// byte offset of 16-byte chunk c of row r: rows of D/8 chunks, XOR-swizzled so
// the 8 rows an ldmatrix reads land in 8 distinct 16-byte bank groups
template <int D>
__device__ __forceinline__ uint32_t swz(int r, int c) {
    constexpr int ROWB = D * 2;
    if constexpr (D >= 64) return uint32_t(r * ROWB + ((c ^ (r & 7)) << 4));
    else return uint32_t(r * ROWB + ((c ^ ((r >> 1) & 3)) << 4));
}

// persistent: CTAs loop over (query block, batch x head) items, so the parameter
// block is staged once per CTA (Swin: 12,288 items of 49 queries each)
template <int D>
__global__ void __launch_bounds__(NT, D <= 32 ? 4 : 2) attn_prefill_kernel(const AttnParams* __restrict__ pp) {
    constexpr int ROWB = D * 2, TILEB = TK * ROWB, STAGEB = 2 * TILEB;
    VTC_STAGE_PARAMS(AttnParams, pp);
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ const bf16* s_qrow[QR];
    __shared__ bf16* s_orow[QR];
    __shared__ int64_t s_qstr[QR], s_ostr[QR];
    __shared__ const bf16* s_brow[QR];
    __shared__ int64_t s_bstr[QR];

    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int r = p.rank, ax_h = r - 3, ax_s = r - 2, ax_d = r - 1;
    const int Sq = p.Sq, Sk = p.Sk;
    const uint32_t nqb = uint32_t((Sq + QR - 1) / QR), nitems = nqb * uint32_t(p.Bt) * uint32_t(p.H);
    dev::pdl_wait();
    dev::pdl_launch_dependents();
    for (uint32_t item = blockIdx.x; item < nitems; item += gridDim.x) {
    const uint32_t qb = item % nqb;
    const int q0 = int(qb) * QR;
    // 32-bit index arithmetic (grid dimensions fit): no 64-bit division calls
    uint32_t bh = item / nqb;
    const uint32_t bq = bh / uint32_t(p.H);
    const int h = int(bh - bq * uint32_t(p.H));
    bh = bq;
    int32_t base_idx[VTC_MAX_RANK] = {};
    for (int a = r - 4; a >= 0; --a) {
        const uint32_t ext = uint32_t(p.q.m.shape[a]), nb = bh / ext;
        base_idx[a] = int32_t(bh - nb * ext);
        bh = nb;
    }
    // query rows: one map evaluation each
    if (tid < QR) {
        int32_t idx[VTC_MAX_RANK];
#pragma unroll
        for (int a = 0; a < VTC_MAX_RANK; ++a) idx[a] = base_idx[a];
        idx[ax_h] = h;
        idx[ax_s] = min(q0 + tid, Sq - 1);
        idx[ax_d] = 0;
        dev::Loc l = dev::locate(p.q.m, idx);
        s_qrow[tid] = dev::addr<bf16>(p.q.m, l);
        s_qstr[tid] = p.q.fast_stride[l.piece];
        dev::Loc lo = dev::locate(p.o.m, idx);
        s_orow[tid] = dev::addr<bf16>(p.o.m, lo);
        s_ostr[tid] = p.o.fast_stride[lo.piece];
        if (p.has_bias) {  // additive bias row [.., h, sq, :] (e.g. Swin relative position + shift mask)
            dev::Loc lb = dev::locate(p.bias.m, idx);
            s_brow[tid] = dev::addr<bf16>(p.bias.m, lb);
            s_bstr[tid] = p.bias.fast_stride[lb.piece];
        }
    }
    // K / V of this head: base at key 0 + key stride (host-proved affine)
    const bf16* kb0;
    const bf16* vb0;
    {
        int32_t idx[VTC_MAX_RANK];
#pragma unroll
        for (int a = 0; a < VTC_MAX_RANK; ++a) idx[a] = base_idx[a];
        idx[ax_h] = h;
        idx[ax_s] = 0;
        idx[ax_d] = 0;
        kb0 = dev::elem_ptr<bf16>(p.k.m, idx);
        vb0 = dev::elem_ptr<bf16>(p.v.m, idx);
    }
    __syncthreads();

    // causal: query row q sees keys t <= q + (Sk - Sq)
    const int kend = p.causal ? min(Sk, q0 + QR - 1 + (Sk - Sq) + 1) : Sk;
    const int ntiles = kend > 0 ? (kend + TK - 1) / TK : 0;
    const uint32_t sbase = smem_u32(smem);
    auto load_tile = [&](int j, int st) {
        const int t0 = j * TK;
        const uint32_t kd = sbase + st * STAGEB, vd = kd + TILEB;
        constexpr int CPR = D / 8;  // 16-byte chunks per row
#pragma unroll
        for (int i = 0; i < (TK * CPR) / NT; ++i) {
            const int c = tid + i * NT;
            const int row = c / CPR, ch = c % CPR;
            const int t = t0 + row;
            const bool ok = t < kend;
            const int tc = ok ? t : 0;
            cp_async16(kd + swz<D>(row, ch), kb0 + int64_t(tc) * p.k_sstride + ch * 8, ok);
            cp_async16(vd + swz<D>(row, ch), vb0 + int64_t(tc) * p.v_sstride + ch * 8, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (ntiles > 0) load_tile(0, 0);

    // Q fragments of this warp's 16 rows
    const int rA = warp * 16 + lane / 4, rB = rA + 8, kc = (lane % 4) * 2;
    uint32_t qa[D / 16][4];
    {
        auto qv = [&](int row, int d) -> float {
            return q0 + row < Sq ? __bfloat162float(s_qrow[row][int64_t(d) * s_qstr[row]]) : 0.f;
        };
        // a pair (d, d + 1) of one row: one 32-bit load when the row is contiguous and aligned
        auto qpair = [&](int row, int d) -> uint32_t {
            if (q0 + row >= Sq) return 0u;
            const bf16* rp = s_qrow[row];
            if (s_qstr[row] == 1 && (reinterpret_cast<uintptr_t>(rp + d) & 3) == 0)
                return *reinterpret_cast<const uint32_t*>(rp + d);
            return pack_bf16(qv(row, d), qv(row, d + 1));
        };
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
            const int d0 = ks * 16 + kc;
            qa[ks][0] = qpair(rA, d0);
            qa[ks][1] = qpair(rB, d0);
            qa[ks][2] = qpair(rA, d0 + 8);
            qa[ks][3] = qpair(rB, d0 + 8);
        }
    }
    const float qscale = p.scale * LOG2E;
    const int limA = p.causal ? q0 + rA + (Sk - Sq) : INT32_MAX;
    const int limB = p.causal ? q0 + rB + (Sk - Sq) : INT32_MAX;
    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;

    for (int j = 0; j < ntiles; ++j) {
        const int st = j % STAGES;
        if (j + 1 < ntiles) {
            load_tile(j + 1, (j + 1) % STAGES);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const uint32_t kt = sbase + st * STAGEB, vt = kt + TILEB;
        const int t0 = j * TK;
        // S[16 x 64]: 8 n-tiles of 8 keys
        float sc[TK / 8][4];
#pragma unroll
        for (int nt = 0; nt < TK / 8; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
        // k-step outer, key tile inner: the 8 accumulators of a k-step are
        // independent, so consecutive MMAs never wait on each other
#pragma unroll
        for (int kp = 0; kp < D / 32; ++kp) {
#pragma unroll
            for (int nt = 0; nt < TK / 8; ++nt) {
                const int mi = lane / 8, rr = lane % 8;
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kt + swz<D>(nt * 8 + rr, kp * 4 + mi), b0, b1, b2, b3);
                mma_bf16(sc[nt], qa[2 * kp], b0, b1);
                mma_bf16(sc[nt], qa[2 * kp + 1], b2, b3);
            }
        }
        float tmA = -INFINITY, tmB = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < TK / 8; ++nt)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int t = t0 + nt * 8 + (lane % 4) * 2 + c;
                float a = sc[nt][c] * qscale, b = sc[nt][2 + c] * qscale;
                if (p.has_bias && t < kend) {
                    if (q0 + rA < Sq) a += __bfloat162float(s_brow[rA][int64_t(t) * s_bstr[rA]]) * LOG2E;
                    if (q0 + rB < Sq) b += __bfloat162float(s_brow[rB][int64_t(t) * s_bstr[rB]]) * LOG2E;
                }
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
        uint32_t pa[TK / 16][4];
#pragma unroll
        for (int nt = 0; nt < TK / 8; ++nt) {
            float e[4];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                e[c] = sc[nt][c] == -INFINITY ? 0.f : exp2f(sc[nt][c] - nmA);
                e[2 + c] = sc[nt][2 + c] == -INFINITY ? 0.f : exp2f(sc[nt][2 + c] - nmB);
                sA += e[c];
                sB += e[2 + c];
            }
            // D-fragment of n-tile nt == half of the A-fragment of k-step nt/2
            const int ks = nt / 2, hi = nt % 2;
            pa[ks][hi * 2 + 0] = pack_bf16(e[0], e[1]);
            pa[ks][hi * 2 + 1] = pack_bf16(e[2], e[3]);
        }
        lA = lA * cA + sA;
        lB = lB * cB + sB;
        mA = nmA;
        mB = nmB;
#pragma unroll
        for (int i = 0; i < D / 8; ++i) {
            o[i][0] *= cA;
            o[i][1] *= cA;
            o[i][2] *= cB;
            o[i][3] *= cB;
        }
#pragma unroll
        for (int ks = 0; ks < TK / 16; ++ks)
#pragma unroll
            for (int np = 0; np < D / 16; ++np) {
                const int mi = lane / 8, rr = lane % 8;
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vt + swz<D>(ks * 16 + (mi & 1) * 8 + rr, np * 2 + (mi >> 1)), b0, b1, b2, b3);
                mma_bf16(o[2 * np], pa[ks], b0, b1);
                mma_bf16(o[2 * np + 1], pa[ks], b2, b3);
            }
        __syncthreads();  // the stage is reloaded by the next iteration's prefetch
    }
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
        lA += __shfl_xor_sync(0xffffffffu, lA, off);
        lB += __shfl_xor_sync(0xffffffffu, lB, off);
    }
    const float iA = lA > 0.f ? 1.f / lA : 0.f, iB = lB > 0.f ? 1.f / lB : 0.f;
    // pairs (d, d + 1): one 32-bit store when the output row is contiguous and aligned
    auto store_pair = [&](int row, int d, float a, float b) {
        bf16* rp = s_orow[row];
        if (s_ostr[row] == 1 && (reinterpret_cast<uintptr_t>(rp + d) & 3) == 0) {
            *reinterpret_cast<uint32_t*>(rp + d) = pack_bf16(a, b);
        } else {
            rp[int64_t(d) * s_ostr[row]] = __float2bfloat16_rn(a);
            rp[int64_t(d + 1) * s_ostr[row]] = __float2bfloat16_rn(b);
        }
    };
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
        const int d = i * 8 + (lane % 4) * 2;
        if (q0 + rA < Sq) store_pair(rA, d, o[i][0] * iA, o[i][1] * iA);
        if (q0 + rB < Sq) store_pair(rB, d, o[i][2] * iB, o[i][3] * iB);
    }
    __syncthreads();  // the row tables and K / V stages are refilled by the next item
    }  // items
}

// Short sequences (Swin windows: 49 queries x 49 keys, head dim 32): one WARP
// per (batch, head) item, all keys in one 64-key tile, so the softmax is a
// single pass; persistent warps, no CTA-wide synchronisation.  Q / K / V / O /
// bias rows are base + position * stride inside an item (host-proved), the
// bases located through the maps once per item.
constexpr int WIN_BIAS_ELEMS = 4096;  // per-warp bias staging (8 KB)
template <int D>
constexpr int window_warps() { return D <= 32 ? 12 : 8; }  // K / V tiles of every warp: 96-128 KB
template <int D>
__global__ void __launch_bounds__(window_warps<D>() * 32, 1) attn_window_kernel(const AttnParams* __restrict__ pp) {
    constexpr int WW = window_warps<D>();
    constexpr int ROWB = D * 2, TILEB = TK * ROWB;
    VTC_STAGE_PARAMS(AttnParams, pp);
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t kt = smem_u32(smem) + uint32_t(warp) * 2 * TILEB, vt = kt + TILEB;
    // the item's bias block, staged by cp.async with K / V (WIN_BIAS_ELEMS per warp)
    unsigned short* sbias = reinterpret_cast<unsigned short*>(smem + size_t(WW) * 2 * TILEB) + size_t(warp) * WIN_BIAS_ELEMS;
    const int r = p.rank, ax_h = r - 3, ax_s = r - 2, ax_d = r - 1;
    // the parameter fields the loop uses, in registers: the staged block lives in shared
    // memory, and every asm with a memory clobber (cp.async, ldmatrix) would force a reload
    const int Sq = p.Sq, Sk = p.Sk, H = p.H;
    const int64_t k_ss = p.k_sstride, v_ss = p.v_sstride, q_ss = p.q_sstride, o_ss = p.o_sstride;
    const int64_t b_ss = p.b_sstride, b_ks = p.b_kstride;
    const bool has_bias = p.has_bias != 0, causal = p.causal != 0;
    const uint64_t* __restrict__ item_base = p.item_base;
    const uint32_t nitems = uint32_t(p.Bt) * uint32_t(H);
    const float qscale = p.scale * LOG2E;
    dev::pdl_wait();
    dev::pdl_launch_dependents();
    for (uint32_t item = blockIdx.x * WW + warp; item < nitems; item += gridDim.x * WW) {
        int32_t idx[VTC_MAX_RANK] = {};
        if (!item_base) {
            uint32_t bh = item;
            const uint32_t bq = bh / uint32_t(H);
            const int h = int(bh - bq * uint32_t(H));
            bh = bq;
            for (int a = r - 4; a >= 0; --a) {
                const uint32_t ext = uint32_t(p.q.m.shape[a]), nb = bh / ext;
                idx[a] = int32_t(bh - nb * ext);
                bh = nb;
            }
            idx[ax_h] = h;
            idx[ax_s] = 0;
            idx[ax_d] = 0;
        }
        // item bases: the host-resolved table, else lanes 0..4 locate one map each
        uint64_t mine = 0;
        if (item_base) {
            if (lane < 5) mine = item_base[uint64_t(item) * 5 + lane];
        } else if (lane == 0) mine = reinterpret_cast<uint64_t>(dev::elem_ptr<bf16>(p.q.m, idx));
        else if (lane == 1) mine = reinterpret_cast<uint64_t>(dev::elem_ptr<bf16>(p.k.m, idx));
        else if (lane == 2) mine = reinterpret_cast<uint64_t>(dev::elem_ptr<bf16>(p.v.m, idx));
        else if (lane == 3) mine = reinterpret_cast<uint64_t>(dev::elem_ptr<bf16>(p.o.m, idx));
        else if (lane == 4 && p.has_bias) mine = reinterpret_cast<uint64_t>(dev::elem_ptr<bf16>(p.bias.m, idx));
        const bf16* qb = reinterpret_cast<const bf16*>(__shfl_sync(0xffffffffu, mine, 0));
        const bf16* kb = reinterpret_cast<const bf16*>(__shfl_sync(0xffffffffu, mine, 1));
        const bf16* vb = reinterpret_cast<const bf16*>(__shfl_sync(0xffffffffu, mine, 2));
        bf16* ob = reinterpret_cast<bf16*>(__shfl_sync(0xffffffffu, mine, 3));
        const bf16* bb = reinterpret_cast<const bf16*>(__shfl_sync(0xffffffffu, mine, 4));
        // K / V of the item -> this warp's tiles (zero past Sk)
        constexpr int CPR = D / 8;
#pragma unroll
        for (int i = 0; i < (TK * CPR) / 32; ++i) {
            const int c = lane + 32 * i, row = c / CPR, ch = c % CPR;
            const bool ok = row < Sk;
            const int rr = ok ? row : 0;
            cp_async16(kt + swz<D>(row, ch), kb + int64_t(rr) * k_ss + ch * 8, ok);
            cp_async16(vt + swz<D>(row, ch), vb + int64_t(rr) * v_ss + ch * 8, ok);
        }
        // the bias block (rows 0 .. Sq - 1, b_ss apart, unit key stride): the 4-byte words of the
        // span from the element-aligned-down start, plus a lone trailing element; the block then
        // sits at sbias + par. Reading a row's TK keys past its end stays inside the buffer
        // (host-checked span + TK <= WIN_BIAS_ELEMS); keys t >= Sk are masked to -inf below.
        const int par = int((reinterpret_cast<uintptr_t>(bb) >> 1) & 1);
        if (has_bias) {
            const int span = (Sq - 1) * int(b_ss) + Sk + par, nw = span / 2;
            const uint32_t sb = smem_u32(sbias);
            const char* src = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(bb) & ~uintptr_t(3));
            for (int w = lane; w < nw; w += 32)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sb + 4u * w), "l"(src + 4 * w) : "memory");
            if ((span & 1) && lane == 0) sbias[span - 1] = reinterpret_cast<const unsigned short*>(src)[span - 1];
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        const int kc = (lane % 4) * 2;
        // Q fragments of one 16-row m-tile (rows rA / rB of this thread), fetched one m-tile
        // ahead so their L2 latency overlaps the previous tile's math
        auto fetch_q = [&](int q0, uint32_t (&qa)[D / 16][4]) {
            // rows past Sq read row 0 (finite values; those rows are never stored)
            const int rA = q0 + lane / 4, rB = rA + 8;
            const int ra = rA < Sq ? rA : 0, rb = rB < Sq ? rB : 0;
            const bf16* qA = qb + int64_t(ra) * q_ss + kc;
            const bf16* qB = qb + int64_t(rb) * q_ss + kc;
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
                qa[ks][0] = ld_g32(qA + ks * 16);
                qa[ks][1] = ld_g32(qB + ks * 16);
                qa[ks][2] = ld_g32(qA + ks * 16 + 8);
                qa[ks][3] = ld_g32(qB + ks * 16 + 8);
            }
        };
        // additive bias of the m-tile's rows from the staged block
        auto fetch_b = [&](int q0, bf16 (&bA)[TK / 8][2], bf16 (&bB)[TK / 8][2]) {
            const int rA = q0 + lane / 4, rB = rA + 8;
            const int ra = rA < Sq ? rA : 0, rb = rB < Sq ? rB : 0;
            auto brow = [&](int r, bf16 (&b)[TK / 8][2]) {
                const unsigned short* rp = sbias + par + r * int(b_ss) + kc;
#pragma unroll
                for (int nt = 0; nt < TK / 8; ++nt)
#pragma unroll
                    for (int c = 0; c < 2; ++c) b[nt][c] = __ushort_as_bfloat16(has_bias ? rp[nt * 8 + c] : 0);
#pragma unroll
                for (int nt = 0; nt < TK / 8; ++nt)
                    if (nt * 8 + 8 > Sk)
#pragma unroll
                        for (int c = 0; c < 2; ++c)
                            if (nt * 8 + kc + c >= Sk) b[nt][c] = __ushort_as_bfloat16(0xff80);  // -inf
            };
            brow(ra, bA);
            brow(rb, bB);
        };
        uint32_t qcur[D / 16][4];
        bf16 bAc[TK / 8][2], bBc[TK / 8][2];
        fetch_q(0, qcur);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        fetch_b(0, bAc, bBc);
        for (int q0 = 0; q0 < Sq; q0 += 16) {
            const int rA = q0 + lane / 4, rB = rA + 8;
            uint32_t qa[D / 16][4];
            float bA[TK / 8][2], bB[TK / 8][2];
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks)
#pragma unroll
                for (int e = 0; e < 4; ++e) qa[ks][e] = qcur[ks][e];
#pragma unroll
            for (int nt = 0; nt < TK / 8; ++nt)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    bA[nt][c] = __bfloat162float(bAc[nt][c]);
                    bB[nt][c] = __bfloat162float(bBc[nt][c]);
                }
            if (q0 + 16 < Sq) {
                fetch_q(q0 + 16, qcur);
                fetch_b(q0 + 16, bAc, bBc);
            }
            float sc[TK / 8][4];
#pragma unroll
            for (int nt = 0; nt < TK / 8; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
            for (int kp = 0; kp < D / 32; ++kp) {
#pragma unroll
                for (int nt = 0; nt < TK / 8; ++nt) {
                    const int mi = lane / 8, rr = lane % 8;
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4(kt + swz<D>(nt * 8 + rr, kp * 4 + mi), b0, b1, b2, b3);
                    mma_bf16(sc[nt], qa[2 * kp], b0, b1);
                    mma_bf16(sc[nt], qa[2 * kp + 1], b2, b3);
                }
            }
            // log2-domain scores; masked keys carry a -inf bias (fetch), causal limits below
            float mA = -INFINITY, mB = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < TK / 8; ++nt)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    sc[nt][c] = fmaf(sc[nt][c], qscale, bA[nt][c] * LOG2E);
                    sc[nt][2 + c] = fmaf(sc[nt][2 + c], qscale, bB[nt][c] * LOG2E);
                }
            if (causal) {
                const int limA = rA + (Sk - Sq), limB = rB + (Sk - Sq);
#pragma unroll
                for (int nt = 0; nt < TK / 8; ++nt)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int t = nt * 8 + kc + c;
                        if (t > limA) sc[nt][c] = -INFINITY;
                        if (t > limB) sc[nt][2 + c] = -INFINITY;
                    }
            }
#pragma unroll
            for (int nt = 0; nt < TK / 8; ++nt) {
                mA = fmaxf(mA, fmaxf(sc[nt][0], sc[nt][1]));
                mB = fmaxf(mB, fmaxf(sc[nt][2], sc[nt][3]));
            }
#pragma unroll
            for (int off = 1; off < 4; off <<= 1) {
                mA = fmaxf(mA, __shfl_xor_sync(0xffffffffu, mA, off));
                mB = fmaxf(mB, __shfl_xor_sync(0xffffffffu, mB, off));
            }
            // a row whose every key is masked: exp2(-inf - 0) = 0 for all, output 0
            if (mA == -INFINITY) mA = 0.f;
            if (mB == -INFINITY) mB = 0.f;
            float lA = 0.f, lB = 0.f;
            uint32_t pa[TK / 16][4];
#pragma unroll
            for (int nt = 0; nt < TK / 8; ++nt) {
                float e[4];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    e[c] = dev::ex2_ftz(sc[nt][c] - mA);  // ex2(-inf) = +0
                    e[2 + c] = dev::ex2_ftz(sc[nt][2 + c] - mB);
                    lA += e[c];
                    lB += e[2 + c];
                }
                const int ks = nt / 2, hi = nt % 2;
                pa[ks][hi * 2 + 0] = pack_bf16(e[0], e[1]);
                pa[ks][hi * 2 + 1] = pack_bf16(e[2], e[3]);
            }
            float o[D / 8][4];
#pragma unroll
            for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
#pragma unroll
            for (int ks = 0; ks < TK / 16; ++ks)
#pragma unroll
                for (int np = 0; np < D / 16; ++np) {
                    const int mi = lane / 8, rr = lane % 8;
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4_t(vt + swz<D>(ks * 16 + (mi & 1) * 8 + rr, np * 2 + (mi >> 1)), b0, b1, b2, b3);
                    mma_bf16(o[2 * np], pa[ks], b0, b1);
                    mma_bf16(o[2 * np + 1], pa[ks], b2, b3);
                }
#pragma unroll
            for (int off = 1; off < 4; off <<= 1) {
                lA += __shfl_xor_sync(0xffffffffu, lA, off);
                lB += __shfl_xor_sync(0xffffffffu, lB, off);
            }
            const float iA = lA > 0.f ? 1.f / lA : 0.f, iB = lB > 0.f ? 1.f / lB : 0.f;
#pragma unroll
            for (int i = 0; i < D / 8; ++i) {
                const int d = i * 8 + kc;
                if (rA < Sq) *reinterpret_cast<uint32_t*>(ob + int64_t(rA) * o_ss + d) = pack_bf16(o[i][0] * iA, o[i][1] * iA);
                if (rB < Sq) *reinterpret_cast<uint32_t*>(ob + int64_t(rB) * o_ss + d) = pack_bf16(o[i][2] * iB, o[i][3] * iB);
            }
        }
        __syncwarp();  // this warp's K / V tiles are refilled by its next item
    }
}

}  // namespace

bool attn_prefill_supported(const AttnParams& p) {
    return p.dt == KDType::BF16 && p.D == p.Dv && (p.D == 32 || p.D == 64 || p.D == 128) && p.kv_affine &&
           p.k.vec_ok && p.v.vec_ok && p.q.fast_ok && p.o.fast_ok && (!p.has_bias || p.bias.fast_ok);
}

template <int D>
void launch_d(const AttnParams& p, const AttnParams* dp, cudaStream_t s) {
    const int64_t items = (p.Sq + QR - 1) / QR * int64_t(p.Bt) * p.H;
    const size_t smem = size_t(STAGES) * 2 * TK * D * 2;
    cudaFuncSetAttribute(attn_prefill_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_prefill_kernel<D>, NT, smem);
    const int64_t cap = int64_t(sms) * (per_sm > 0 ? per_sm : 1);
    launch_k(attn_prefill_kernel<D>, dim3(unsigned(items < cap ? items : cap)), dim3(NT), smem, s, dp);
}

bool attn_window_supported(const AttnParams& p) {
    return p.dt == KDType::BF16 && p.D == p.Dv && (p.D == 32 || p.D == 64) && p.Sq <= TK && p.Sk <= TK && p.kv_affine &&
           p.qo_affine && p.k.vec_ok && p.v.vec_ok &&
           (!p.has_bias || (p.bias_affine && p.b_kstride == 1 && p.b_sstride >= 0 &&
                            (p.Sq - 1) * p.b_sstride + p.Sk + 2 + TK <= WIN_BIAS_ELEMS));
}

template <int D>
void launch_w(const AttnParams& p, const AttnParams* dp, cudaStream_t s) {
    constexpr int WW = window_warps<D>();
    const size_t smem = size_t(WW) * (2 * TK * D * 2 + WIN_BIAS_ELEMS * 2);
    allow_max_smem(attn_window_kernel<D>);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t items = int64_t(p.Bt) * p.H, need = (items + WW - 1) / WW;
    launch_k(attn_window_kernel<D>, dim3(unsigned(need < sms ? need : sms)), dim3(WW * 32), smem, s, dp);
}

void launch_attn_window(const AttnParams& p, const AttnParams* dp, cudaStream_t s) {
    if (p.D == 32) launch_w<32>(p, dp, s);
    else launch_w<64>(p, dp, s);
}

void launch_attn_prefill(const AttnParams& p, const AttnParams* dp, cudaStream_t s) {
    if (p.D == 32) launch_d<32>(p, dp, s);
    else if (p.D == 64) launch_d<64>(p, dp, s);
    else launch_d<128>(p, dp, s);
}

}  // namespace vtc
