// Kernel parameter blocks and host-side launchers (sm_100a).
//
// Every operand of every kernel is a VOperand: the lowered virtual-tensor map
// plus host-derived facts about it along the kernel's fast (contiguous) axis.
// Kernels evaluate the map at row / tile / vector origins and step with the
// per-piece fast stride inside, so data-movement chains cost no kernel.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "vtc_desc.h"

namespace vtc {

enum class KDType : int32_t { F64 = 0, F32 = 1, I64 = 2, BF16 = 3 };

struct VOperand {
    vtc_map m;
    int64_t fast_stride[VTC_MAX_PIECES];  // per piece, along the kernel's fast axis
    int32_t fast_ok;   // every piece affine along the fast axis over the kernel's tile
    int32_t vec_ok;    // fast stride 1 and 16-byte aligned vector starts
    int32_t fast_axis;
    int32_t pad;
};

// ---- elementwise / copy --------------------------------------------------
enum class EwOp : int32_t { Copy = 0, Add, Mul, SiLU, GELU, SiLUMul };

struct EwParams {
    VOperand out, a, b;
    int32_t rank;
    int32_t shape[VTC_MAX_RANK];   // iteration box extents
    int32_t origin[VTC_MAX_RANK];  // iteration box origin (virtual index of element 0)
    int32_t vec;       // elements per thread-vector along the last axis
    int32_t nin;
    int64_t nvec;      // number of vectors
    EwOp op;
    KDType dt;
    int32_t esize;
};
void launch_eltwise(const EwParams& p, cudaStream_t s);

// ---- generic batched matmul (any dtype, any maps) -----------------------
struct MatmulParams {
    VOperand a, b, c;  // a:[...,M,K] fast axis K, b:[...,K,N] fast axis N, c:[...,M,N] fast axis N
    int32_t rank;
    int32_t shape_c[VTC_MAX_RANK];
    int64_t M, N, K, batch;
    int64_t a_mstride[VTC_MAX_PIECES];  // per piece strides along M (A) and K (B), when affine
    int32_t a_m_ok, b_k_ok;
    int64_t b_kstride[VTC_MAX_PIECES];
    KDType dt;
    int32_t exact;  // f32/f64: unfused multiply-add, bit-identical to the CPU reference
};
void launch_matmul(const MatmulParams& p, cudaStream_t s);

// ---- weight-streaming GEMV for bf16 decode (M <= 16) ----------------------
// C[m,n] (+)= prologue(A)[m,:] . B[:,n] ; B is a physical (single-piece affine)
// weight streamed once with 16-byte loads; A, C and the residual go through
// their VirtualTensor maps.  Split-K partials are reduced deterministically by
// the last-arriving CTA of each N tile.
enum class GemvPrologue : int32_t { None = 0, SiLUMul = 1, RMSNorm = 2 };
struct GemvParams {
    VOperand a, a2, normw, c, res;  // a:[M,K] (fast K); a2: second input of SiLUMul; normw: [K]
    const void* b_base;             // &B[0,0]
    int64_t b_sk;                   // element stride between rows k of B (columns contiguous)
    int64_t M, N, K;
    int32_t ksplit, kchunk;
    GemvPrologue prologue;
    int32_t has_res;
    float eps;
    int32_t pad;
    float* work;                    // [ksplit, M, N] partials
    unsigned int* counters;         // [ceil(N / 256)] arrival counters (self-resetting)
};
void launch_gemv(const GemvParams& p, cudaStream_t s);

// ---- row-wise normalisations / softmax -----------------------------------
enum class RowOp : int32_t { RMSNorm = 0, LayerNorm, Softmax };
struct RowParams {
    VOperand x, w, bias, out;
    int32_t rank;
    int32_t shape[VTC_MAX_RANK];
    int64_t rows, D;
    float eps;
    RowOp op;
    KDType dt;
    int32_t pad;
};
void launch_rowop(const RowParams& p, cudaStream_t s);

// ---- attention (split-KV flash decoding with GQA head grouping) ----------
struct AttnParams {
    VOperand q, k, v, o, bias;  // q:[..,H,Sq,d] k,v:[..,H,Sk,d] o:[..,H,Sq,dv]
    int32_t rank;
    int32_t has_bias;
    int32_t Bt, H, Sq, Sk, D, Dv;  // Bt = product of leading dims before H
    int32_t group;                 // heads sharing K/V addresses (GQA factor)
    int32_t splits;                // split-KV chunks
    int32_t chunk;                 // keys per split
    int32_t causal;
    float scale;
    KDType dt;
    float* part_o;                 // [Bt, H, Sq, splits, Dv]
    float* part_ml;                // [Bt, H, Sq, splits, 2]
};
void launch_attention(const AttnParams& p, cudaStream_t s);

}  // namespace vtc
