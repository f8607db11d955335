// Split-KV flash-decoding attention over VirtualTensor operands.
//
// softmax(scale * Q K^T [+ bias] [causal]) V for q:[..,H,Sq,D], k:[..,H,Sk,D],
// v:[..,H,Sk,Dv].  Attention is absent from the reference (SURVEY.md §8 a');
// in a VTC-planned decoder the K/V operands are virtual: the KV-cache slice,
// the transpose and the GQA Expand/Reshape compose into one map onto the
// cache (h -> h div G), so no expanded copy is ever materialised.  The host
// proves that the K and V maps ignore (h mod G) and hands the kernel G: one
// CTA serves G query heads and reads each K/V row once (the paper's 4x
// read reduction).
//
// CTA = 128 threads, 32-key tiles staged in shared memory (row addresses from
// one map evaluation per key row), online softmax in the log2 domain, partial
// (O, m, l) per split combined by a second kernel in split order.
#include <cfloat>

#include "device.cuh"
#include "launch.cuh"

namespace vtc {
namespace {

using dev::bf16;
constexpr int NT = 128, TK = 32, MAXD = 256, MAXG = 8;
constexpr float LOG2E = 1.4426950408889634f;

template <typename T>
__device__ __forceinline__ float ldf(const T* p) { return float(dev::to_acc<T>(*p)); }

template <typename T>
__global__ void __launch_bounds__(NT) attn_kernel(const AttnParams* __restrict__ pp) {
    VTC_STAGE_PARAMS(AttnParams, pp);
    dev::pdl_wait(); dev::pdl_launch_dependents();
    __shared__ float sQ[MAXG][MAXD];
    __shared__ float sP[MAXG][TK];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int DK = p.D + 8, DV = p.Dv + 8;  // padded rows: conflict-free 16-byte accesses
    T* sKbuf = reinterpret_cast<T*>(smem_raw);
    T* sVbuf = sKbuf + TK * DK;
    auto sK = [&](int row) { return sKbuf + row * DK; };
    auto sV = [&](int row) { return sVbuf + row * DV; };
    __shared__ const T* sKrow[TK];
    __shared__ const T* sVrow[TK];
    __shared__ int sKpiece[TK], sVpiece[TK];

    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int G = p.group, HG = p.H / G;
    const int r = p.rank;
    const int ax_h = r - 3, ax_s = r - 2, ax_d = r - 1;

    // query block -> (lead, hg, sq)
    int64_t qb = blockIdx.x;
    const int sq = int(qb % p.Sq);
    qb /= p.Sq;
    const int hg = int(qb % HG);
    qb /= HG;
    int32_t base_idx[VTC_MAX_RANK] = {};
    {
        int64_t b = qb;
        for (int a = r - 4; a >= 0; --a) {
            int32_t ext = p.q.m.shape[a];
            base_idx[a] = int32_t(b % ext);
            b /= ext;
        }
    }
    const int split = blockIdx.y;
    const int kbeg = split * p.chunk;
    int kend = min(p.Sk, kbeg + p.chunk);
    const int klimit_base = p.Sk - p.Sq;  // causal: key t allowed iff t <= sq + klimit_base
    if (p.causal) kend = min(kend, sq + klimit_base + 1);

    // stage Q (scaled into the log2 domain)
    const float qscale = p.scale * LOG2E;
    for (int e = tid; e < G * p.D; e += NT) {
        int g = e / p.D, d = e % p.D;
        int32_t idx[VTC_MAX_RANK];
#pragma unroll
        for (int a = 0; a < VTC_MAX_RANK; ++a) idx[a] = base_idx[a];
        dev::set_axis(idx, ax_h, hg * G + g);
        dev::set_axis(idx, ax_s, sq);
        dev::set_axis(idx, ax_d, d);
        sQ[g][d] = ldf<T>(dev::elem_ptr<T>(p.q.m, idx)) * qscale;
    }

    // per-thread output accumulators: heads g = warp + 4*j, dims d = lane + 32*i
    constexpr int MAXI = MAXD / 32, MAXJ = MAXG / 4;
    float o[MAXJ][MAXI];
    float m_run[MAXJ], l_run[MAXJ];
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
        m_run[j] = -INFINITY;
        l_run[j] = 0.f;
#pragma unroll
        for (int i = 0; i < MAXI; ++i) o[j][i] = 0.f;
    }
    const int h0 = hg * G;

    for (int t0 = kbeg; t0 < kend; t0 += TK) {
        const int nk = min(TK, kend - t0);
        __syncthreads();
        if (tid < TK) {
            int t = t0 + min(tid, nk - 1);
            int32_t idx[VTC_MAX_RANK];
#pragma unroll
            for (int a = 0; a < VTC_MAX_RANK; ++a) idx[a] = base_idx[a];
            dev::set_axis(idx, ax_h, h0);
            dev::set_axis(idx, ax_s, t);
            dev::set_axis(idx, ax_d, 0);
            dev::Loc lk = dev::locate(p.k.m, idx);
            sKrow[tid] = dev::addr<T>(p.k.m, lk);
            sKpiece[tid] = lk.piece;
            dev::Loc lv = dev::locate(p.v.m, idx);
            sVrow[tid] = dev::addr<T>(p.v.m, lv);
            sVpiece[tid] = lv.piece;
        }
        __syncthreads();
        // load K / V rows (16-byte chunks when the map is contiguous along d)
        {
            const int vecs = p.D / 8, vecsv = p.Dv / 8;
            for (int c = tid; c < TK * vecs; c += NT) {
                int row = c / vecs, col = (c % vecs) * 8;
                if (p.k.vec_ok && sizeof(T) == 2) {
                    *reinterpret_cast<uint4*>(sK(row) + col) = __ldg(reinterpret_cast<const uint4*>(sKrow[row] + col));
                } else {
                    int64_t s = p.k.fast_stride[sKpiece[row]];
                    for (int j = 0; j < 8; ++j) sK(row)[col + j] = sKrow[row][(col + j) * s];
                }
            }
            for (int c = tid; c < TK * vecsv; c += NT) {
                int row = c / vecsv, col = (c % vecsv) * 8;
                if (p.v.vec_ok && sizeof(T) == 2) {
                    *reinterpret_cast<uint4*>(sV(row) + col) = __ldg(reinterpret_cast<const uint4*>(sVrow[row] + col));
                } else {
                    int64_t s = p.v.fast_stride[sVpiece[row]];
                    for (int j = 0; j < 8; ++j) sV(row)[col + j] = sVrow[row][(col + j) * s];
                }
            }
        }
        __syncthreads();
        // scores: thread -> (g = tid / 32 + 4*jj, t = lane)
        #pragma unroll
        for (int jj = 0; jj < MAXJ; ++jj) {
            const int g = warp + 4 * jj;
            if (g >= G) break;
            float s = -INFINITY;
            const int t = lane;
            if (t < nk) {
                float acc = 0.f;
                for (int d = 0; d < p.D; d += 2) {
                    float2 kv;
                    if constexpr (sizeof(T) == 2) {
                        kv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sK(t) + d));
                    } else {
                        kv = make_float2(float(sK(t)[d]), float(sK(t)[d + 1]));
                    }
                    acc = fmaf(sQ[g][d], kv.x, acc);
                    acc = fmaf(sQ[g][d + 1], kv.y, acc);
                }
                s = acc;
                if (p.has_bias) {
                    int32_t idx[VTC_MAX_RANK];
#pragma unroll
                    for (int a = 0; a < VTC_MAX_RANK; ++a) idx[a] = base_idx[a];
                    dev::set_axis(idx, ax_h, h0 + g);
                    dev::set_axis(idx, ax_s, sq);
                    dev::set_axis(idx, ax_d, t0 + t);
                    s += ldf<T>(dev::elem_ptr<T>(p.bias.m, idx)) * LOG2E;
                }
            }
            // online softmax for head g (warp-uniform)
            float mt = dev::warp_max(s);
            float m_new = fmaxf(m_run[jj], mt);
            float pe = (t < nk && s != -INFINITY) ? exp2f(s - m_new) : 0.f;
            float corr = (m_run[jj] == -INFINITY) ? 0.f : exp2f(m_run[jj] - m_new);
            if (m_new == -INFINITY) corr = 1.f;
            l_run[jj] = l_run[jj] * corr + dev::warp_sum(pe);
            m_run[jj] = m_new;
#pragma unroll
            for (int i = 0; i < MAXI; ++i) o[jj][i] *= corr;
            sP[g][t] = pe;
        }
        __syncwarp();
        // P V
        #pragma unroll
        for (int jj = 0; jj < MAXJ; ++jj) {
            const int g = warp + 4 * jj;
            if (g >= G) break;
            for (int t = 0; t < nk; ++t) {
                float pt = sP[g][t];
#pragma unroll
                for (int i = 0; i < MAXI; ++i) {
                    int d = lane + 32 * i;
                    if (d < p.Dv) o[jj][i] = fmaf(pt, float(dev::to_acc<T>(sV(t)[d])), o[jj][i]);
                }
            }
        }
    }

    // write results
    #pragma unroll
        for (int jj = 0; jj < MAXJ; ++jj) {
            const int g = warp + 4 * jj;
            if (g >= G) break;
        const int h = h0 + g;
        if (p.splits == 1) {
            float inv = l_run[jj] > 0.f ? 1.f / l_run[jj] : 0.f;
#pragma unroll
            for (int i = 0; i < MAXI; ++i) {
                int d = lane + 32 * i;
                if (d >= p.Dv) continue;
                int32_t idx[VTC_MAX_RANK];
#pragma unroll
                for (int a = 0; a < VTC_MAX_RANK; ++a) idx[a] = base_idx[a];
                dev::set_axis(idx, ax_h, h);
                dev::set_axis(idx, ax_s, sq);
                dev::set_axis(idx, ax_d, d);
                *dev::elem_ptr<T>(p.o.m, idx) = dev::from_acc<T>(o[jj][i] * inv);
            }
        } else {
            int64_t row = ((int64_t(blockIdx.x) / HG / p.Sq * p.H + h) * p.Sq + sq);  // (lead, h, sq)
            float* po = p.part_o + (row * p.splits + split) * p.Dv;
#pragma unroll
            for (int i = 0; i < MAXI; ++i) {
                int d = lane + 32 * i;
                if (d < p.Dv) po[d] = o[jj][i];
            }
            if (lane == 0) {
                p.part_ml[(row * p.splits + split) * 2] = m_run[jj];
                p.part_ml[(row * p.splits + split) * 2 + 1] = l_run[jj];
            }
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(NT) combine_kernel(const AttnParams* __restrict__ pp) {
    VTC_STAGE_PARAMS(AttnParams, pp);
    dev::pdl_wait(); dev::pdl_launch_dependents();
    // one CTA per (lead, h, sq) row
    const int64_t row = blockIdx.x;
    const int r = p.rank;
    int64_t rr = row;
    const int sq = int(rr % p.Sq);
    rr /= p.Sq;
    const int h = int(rr % p.H);
    rr /= p.H;
    int32_t idx[VTC_MAX_RANK] = {};
    for (int a = r - 4; a >= 0; --a) {
        int32_t ext = p.q.m.shape[a];
        idx[a] = int32_t(rr % ext);
        rr /= ext;
    }
    dev::set_axis(idx, r - 3, h);
    dev::set_axis(idx, r - 2, sq);
    const float* ml = p.part_ml + row * p.splits * 2;
    float M = -INFINITY;
    for (int s = 0; s < p.splits; ++s) M = fmaxf(M, ml[2 * s]);
    float L = 0.f;
    for (int s = 0; s < p.splits; ++s)
        if (ml[2 * s] != -INFINITY) L += exp2f(ml[2 * s] - M) * ml[2 * s + 1];
    float inv = L > 0.f ? 1.f / L : 0.f;
    for (int d = threadIdx.x; d < p.Dv; d += NT) {
        float acc = 0.f;
        for (int s = 0; s < p.splits; ++s)
            if (ml[2 * s] != -INFINITY) acc += exp2f(ml[2 * s] - M) * p.part_o[(row * p.splits + s) * p.Dv + d];
        int32_t j[VTC_MAX_RANK];
#pragma unroll
        for (int a = 0; a < VTC_MAX_RANK; ++a) j[a] = idx[a];
        dev::set_axis(j, r - 1, d);
        *dev::elem_ptr<T>(p.o.m, j) = dev::from_acc<T>(acc * inv);
    }
}

template <typename T>
void launch_t(const AttnParams& p, const AttnParams* dp, cudaStream_t s) {
    if (p.fast == 2) {
        launch_attn_prefill(p, dp, s);
        return;
    }
    if (p.fast == 3) {
        launch_attn_fmha(p, dp, s);
        return;
    }
    if (p.fast == 4) {
        launch_attn_window(p, dp, s);
        return;
    }
    if (p.fast) {
        launch_attn_decode(p, dp, s);
    } else {
        int64_t qblocks = int64_t(p.Bt) * (p.H / p.group) * p.Sq;
        dim3 grid(unsigned(qblocks), unsigned(p.splits));
        size_t smem = size_t(TK) * size_t(p.D + 8 + p.Dv + 8) * sizeof(T);
        if (smem > 48 * 1024) allow_max_smem(attn_kernel<T>);
        launch_k(attn_kernel<T>, dim3(grid), dim3(NT), smem, s, dp);
    }
    if (p.splits > 1 && !p.fast) launch_k(combine_kernel<T>, dim3(unsigned(int64_t(p.Bt) * p.H * p.Sq)), dim3(NT), 0, s, dp);
}

}  // namespace

void launch_attention(const AttnParams& p, const AttnParams* dp, cudaStream_t s) {
    switch (p.dt) {
        case KDType::BF16: launch_t<bf16>(p, dp, s); break;
        case KDType::F32: launch_t<float>(p, dp, s); break;
        default: break;
    }
}

}  // namespace vtc
