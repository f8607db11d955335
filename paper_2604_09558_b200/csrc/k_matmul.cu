// Generic batched MatMul over virtual operands (any dtype: f64, f32, i64, bf16).
//
// Semantics: run_operator MatMul (proj/src/executor.cpp:230-249): equal batch
// dims, C[b,m,n] = sum_k A[b,m,k] * B[b,k,n]; each output accumulates k in
// ascending order inside one thread (f32/f64: FFMA; i64: wrapping; bf16 inputs:
// fp32 accumulate, RNE on store), so the arithmetic is independent of the
// operand maps and a virtual plan is bit-identical to the materialised one.
//
// Tiles of 128x128 (8x8 per thread, 256 threads), BK = 8, register-staged
// double buffering.  Operand tiles are fetched through the VirtualTensor map:
// when the host proved the map tile-affine along both tile axes, the tile
// origin is evaluated once and elements are stepped with the piece strides;
// otherwise each element is located individually (always correct).
#include <type_traits>

#include "device.cuh"
#include "launch.cuh"

namespace vtc {
namespace {

using dev::bf16;

constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8, NT = 256;

// Load a ROWS x COLS tile whose element (r, c) lives at virtual index with
// axis ax_r = row0 + r, ax_c = col0 + c (other axes from `idx`).
template <typename T, int ROWS, int COLS>
__device__ __forceinline__ void fetch_tile(const VOperand& op, int32_t (&idx)[VTC_MAX_RANK], int ax_r, int ax_c,
                                           int64_t row0, int64_t col0, int64_t nrows, int64_t ncols,
                                           const int64_t* rstride, bool r_ok, bool col_fast_first,
                                           typename dev::Acc<T>::type (&out)[ROWS * COLS / NT]) {
    using A = typename dev::Acc<T>::type;
    constexpr int PER = ROWS * COLS / NT;
    const int tid = threadIdx.x;
    bool fast = r_ok && op.fast_ok;
    const T* base = nullptr;
    int64_t sr = 0, sc = 0;
    if (fast) {
        dev::set_axis(idx, ax_r, int32_t(row0));
        dev::set_axis(idx, ax_c, int32_t(col0));
        dev::Loc l = dev::locate(op.m, idx);
        base = dev::addr<T>(op.m, l);
        sr = rstride[l.piece];
        sc = op.fast_stride[l.piece];
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        int e = tid + i * NT;
        int r, c;
        if (col_fast_first) { c = e % COLS; r = e / COLS; }
        else { r = e % ROWS; c = e / ROWS; }
        int64_t gr = row0 + r, gc = col0 + c;
        A v = A(0);
        if (gr < nrows && gc < ncols) {
            if (fast) {
                v = dev::to_acc<T>(base[r * sr + c * sc]);
            } else {
                dev::set_axis(idx, ax_r, int32_t(gr));
                dev::set_axis(idx, ax_c, int32_t(gc));
                v = dev::to_acc<T>(*dev::elem_ptr<T>(op.m, idx));
            }
        }
        out[i] = v;
    }
}

template <typename A>
__device__ __forceinline__ A mac(A acc, A a, A b, bool exact) {
    if constexpr (std::is_integral_v<A>) {
        return (A)((uint64_t)acc + (uint64_t)a * (uint64_t)b);  // wrapping, like int64 on the host
    } else if constexpr (sizeof(A) == 8) {
        return exact ? __dadd_rn(acc, __dmul_rn(a, b)) : fma(a, b, acc);
    } else {
        return exact ? __fadd_rn(acc, __fmul_rn(a, b)) : fmaf(a, b, acc);
    }
}

template <typename T, bool EXACT>
__global__ void __launch_bounds__(NT) mm_kernel(const MatmulParams* __restrict__ pp) {
    VTC_STAGE_PARAMS(MatmulParams, pp);
    dev::pdl_wait();
    using A = typename dev::Acc<T>::type;
    __shared__ A As[2][BK][BM + 4];
    __shared__ A Bs[2][BK][BN + 4];

    const int tid = threadIdx.x;
    const int tx = tid % (BN / TN), ty = tid / (BN / TN);
    const int64_t m0 = int64_t(blockIdx.y) * BM, n0 = int64_t(blockIdx.x) * BN;
    const int r = p.rank;
    const int ax_m = r - 2, ax_n = r - 1;

    // batch coordinates (leading dims) shared by A, B, C
    int32_t bidx[VTC_MAX_RANK];
    {
        int64_t b = blockIdx.z;
#pragma unroll
        for (int a = VTC_MAX_RANK - 1; a >= 0; --a) {
            if (a < r - 2) {
                bidx[a] = int32_t(b % p.shape_c[a]);
                b /= p.shape_c[a];
            } else {
                bidx[a] = 0;
            }
        }
    }
    int32_t ia[VTC_MAX_RANK], ib[VTC_MAX_RANK];
#pragma unroll
    for (int a = 0; a < VTC_MAX_RANK; ++a) ia[a] = ib[a] = bidx[a];

    // A tile: rows m (axis r-2), cols k (axis r-1): m-fastest thread order when A is M-major
    const bool a_mfast = p.a_m_ok && p.a.m.npieces == 1 && p.a_mstride[0] == 1;
    constexpr int PA = BM * BK / NT, PB = BK * BN / NT;
    A ra[PA], rb[PB];

    A acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = A(0);

    auto load = [&](int64_t k0) {
        fetch_tile<T, BM, BK>(p.a, ia, ax_m, ax_n, m0, k0, p.M, p.K, p.a_mstride, p.a_m_ok != 0, !a_mfast, ra);
        fetch_tile<T, BK, BN>(p.b, ib, ax_m, ax_n, k0, n0, p.K, p.N, p.b_kstride, p.b_k_ok != 0, true, rb);
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int i = 0; i < PA; ++i) {
            int e = tid + i * NT, rr, cc;
            if (!a_mfast) { cc = e % BK; rr = e / BK; }
            else { rr = e % BM; cc = e / BM; }
            As[buf][cc][rr] = ra[i];
        }
#pragma unroll
        for (int i = 0; i < PB; ++i) {
            int e = tid + i * NT;
            Bs[buf][e / BN][e % BN] = rb[i];
        }
    };

    int64_t ktiles = (p.K + BK - 1) / BK;
    load(0);
    stash(0);
    __syncthreads();
    for (int64_t kt = 0; kt < ktiles; ++kt) {
        int buf = int(kt & 1);
        if (kt + 1 < ktiles) load((kt + 1) * BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            A av[TM], bv[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) av[i] = As[buf][kk][ty * TM + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) bv[j] = Bs[buf][kk][tx * TN + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = mac<A>(acc[i][j], av[i], bv[j], EXACT);
        }
        if (kt + 1 < ktiles) {
            stash(buf ^ 1);
        }
        __syncthreads();
    }

    // epilogue: store through C's map (row by row, stepping along N)
    int32_t ic[VTC_MAX_RANK];
#pragma unroll
    for (int a = 0; a < VTC_MAX_RANK; ++a) ic[a] = bidx[a];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        int64_t gm = m0 + ty * TM + i;
        if (gm >= p.M) continue;
        int64_t gn0 = n0 + tx * TN;
        dev::set_axis(ic, ax_m, int32_t(gm));
        if (p.c.fast_ok && gn0 + TN <= p.N) {
            dev::set_axis(ic, ax_n, int32_t(gn0));
            dev::Loc l = dev::locate(p.c.m, ic);
            T* base = dev::addr<T>(p.c.m, l);
            int64_t s = p.c.fast_stride[l.piece];
#pragma unroll
            for (int j = 0; j < TN; ++j) base[j * s] = dev::from_acc<T>(acc[i][j]);
        } else {
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                if (gn0 + j >= p.N) continue;
                dev::set_axis(ic, ax_n, int32_t(gn0 + j));
                *dev::elem_ptr<T>(p.c.m, ic) = dev::from_acc<T>(acc[i][j]);
            }
        }
    }
}

}  // namespace

void launch_matmul(const MatmulParams& p, const MatmulParams* dp, cudaStream_t s) {
    dim3 grid(unsigned((p.N + BN - 1) / BN), unsigned((p.M + BM - 1) / BM), unsigned(p.batch));
    // exact: separate multiply and add roundings, k ascending -- bit-identical to
    // the reference's `acc += a * b` loop (executor.cpp:245) for f32 / f64.
    const bool ex = p.exact != 0;
    switch (p.dt) {
        case KDType::F64:
            if (ex) launch_k(mm_kernel<double, true>, dim3(grid), dim3(NT), 0, s, dp);
            else launch_k(mm_kernel<double, false>, dim3(grid), dim3(NT), 0, s, dp);
            break;
        case KDType::F32:
            if (ex) launch_k(mm_kernel<float, true>, dim3(grid), dim3(NT), 0, s, dp);
            else launch_k(mm_kernel<float, false>, dim3(grid), dim3(NT), 0, s, dp);
            break;
        case KDType::I64: launch_k(mm_kernel<int64_t, true>, dim3(grid), dim3(NT), 0, s, dp); break;
        case KDType::BF16: launch_k(mm_kernel<bf16, false>, dim3(grid), dim3(NT), 0, s, dp); break;
    }
}

}  // namespace vtc
