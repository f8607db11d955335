// Kernel parameter blocks and host-side launchers (sm_100a).
//
// Parameter blocks live in device memory (uploaded once when a plan is
// prepared); kernels receive one pointer.  Passing the multi-KB descriptor
// blocks as __grid_constant__ launch parameters cost ~20 us of front-end time
// per launch on B200 (measured with ncu), more than the kernels themselves.
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

// Common first member of every parameter block: optional device-side
// timeline (VTC_TRACE=1): CTA 0..n thread 0 records globaltimer at kernel entry
// (atomicMin into trace[2*id]) and exit (atomicMax into trace[2*id+1]).
//
// Dynamic-position plans (vtc_plan_set_position): the fields
// that depend on the decode position -- the base offset of a map piece that
// stores the new token's K / V row into the cache slab, a fused-epilogue
// address shift, the attention key count -- are listed as patches; after the
// block is staged into shared memory, value += coeff * (*dyn - dyn0), where
// *dyn is the plan's device-resident position for this step and dyn0 the
// position the block was lowered for.  One plan and one captured graph serve
// every step.
struct DynPatch {
    uint32_t off;    // byte offset of the field inside the staged parameter struct
    int32_t bytes;   // 4 or 8 (signed integer field)
    int64_t coeff;
};
constexpr int KHEAD_MAX_DYN = 6;
struct KHead {
    unsigned long long* trace;
    int32_t id;
    int32_t ndyn;
    const int64_t* dyn;
    int64_t dyn0;
    DynPatch patch[KHEAD_MAX_DYN];
};

// ---- elementwise / copy --------------------------------------------------
enum class EwOp : int32_t { Copy = 0, Add, Mul, SiLU, GELU };

// One step of a fused elementwise program: r[dst] = op(r[a], r[b]).
// Registers 0..nin-1 hold the inputs; every result is rounded to the tensor
// dtype, so a fused chain reproduces the unfused ops bit for bit.
struct EwInstr {
    EwOp op;
    int8_t dst, a, b, pad;
};
constexpr int EW_MAX_IN = 4, EW_MAX_PROG = 8;

// An operand whose map is one or two affine pieces split along the last axis
// (a view, a broadcast, a rotate-half): element I at
// base[k] + sum_a st[k][a] * I[a] (bytes / element size), k = I[last] >= split.
struct EwAff {
    uint64_t base[2];              // byte address of virtual index 0 of each piece's affine form
    int64_t st[2][VTC_MAX_RANK];   // element strides
    int32_t split;                 // first last-axis index of piece 1 (INT32_MAX: one piece)
    int32_t pad;
};

struct EwParams {
    KHead head;
    VOperand out;
    VOperand in[EW_MAX_IN];
    int32_t rank;
    int32_t shape[VTC_MAX_RANK];   // iteration box extents
    int32_t origin[VTC_MAX_RANK];  // iteration box origin (virtual index of element 0)
    int32_t vec;                   // elements per thread-vector along the last axis
    int32_t nin;
    int32_t nprog;
    int32_t result;                // register holding the output
    EwInstr prog[EW_MAX_PROG];
    int64_t nvec;                  // number of vectors
    KDType dt;
    int32_t esize;
    int32_t copy_only;             // pure data movement: dtype-agnostic by element size
    int32_t flat;                  // host-proved plain operands: 1 one-op program, 2 SiLU(in0) * in1
    int32_t prog_pat;              // 3: the program is (in0 * in1) + (in2 * in3) (RoPE), run without the interpreter
    int32_t aff;                   // host-proved affine operands (EwAff below): the compact-parameter kernel
    EwAff affine[EW_MAX_IN + 1];   // [0] = out, [1 + i] = in[i]
};
void launch_eltwise(const EwParams& p, const EwParams* dp, cudaStream_t s);
// Host check: the map addresses element I of an iteration box of `shape` (origin 0)
// at piece[0].ptr + piece[0].base + flat(I) (one affine piece, row-major, unit stride).
bool map_flat_linear(const vtc_map& m, int rank, const int32_t* shape);
// Two independent elementwise programs of the same element type in one launch
// (horizontal fusion of small launches, e.g. the Q and K RoPE trees).
struct EwPair {
    alignas(16) EwParams a;  // kernels stage parameter blocks with 16-byte loads
    alignas(16) EwParams b;
};
bool eltwise_pair_compatible(const EwParams& a, const EwParams& b);
void launch_eltwise_pair(const EwPair& p, const EwPair* dp, cudaStream_t s);
// 16-byte-granular copy between UVA-addressable buffers (pinned host <-> device)
void launch_host_link_copy(const void* src, void* dst, int64_t bytes, cudaStream_t s);

// ---- generic batched matmul (any dtype, any maps) -----------------------
struct MatmulParams {
    KHead head;
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
void launch_matmul(const MatmulParams& p, const MatmulParams* dp, cudaStream_t s);

// ---- weight-streaming GEMV for bf16 decode (M <= 16) ----------------------
// C[m,n] (+)= prologue(A)[m,:] . B[:,n] ; B is a physical (single-piece affine)
// weight streamed once with 16-byte loads; A, C and the residual go through
// their VirtualTensor maps.  Split-K partials are reduced deterministically by
// the last-arriving CTA of each N tile.
enum class GemvPrologue : int32_t { None = 0, SiLUMul = 1, RMSNorm = 2 };
constexpr int GEMV_MAX_MATS = 2;
// Elementwise trees fused into the GEMV epilogue (e.g. RoPE on the Q / K
// columns of the QKV projection): the tree's operands that are the GEMV output
// itself are read from the strip in shared memory (strip-local permutations
// such as the rotate-half), the others from memory; the intermediate root the
// GEMV would have written is never materialised.
constexpr int EPI_MAX_TREES = 2, EPI_MAX_IN = 4;
struct EpiTree {
    int32_t nin, nprog, result, pad;
    EwInstr prog[EW_MAX_PROG];
};
struct EpiEntry {            // one GEMV output element (m, n)
    uint64_t out;            // tree output address (bf16)
    uint64_t in[EPI_MAX_IN]; // C column (C-derived input) or element address (external input)
    int32_t tree;            // -1: plain output element, stored through the C map
    uint32_t cmask;          // bit j: input j is C-derived; EPI_DYN_OUT: out moves with the position
};
constexpr uint32_t EPI_DYN_OUT = 1u << 31;  // out += GemvParams::epi_shift (dynamic-position plans)

struct GemvParams {
    KHead head;
    VOperand a, a2, normw, c, res;  // a:[M,K] (fast K); a2: second input of SiLUMul; normw: [K]
    const void* b_base;             // &B[0,0]
    int64_t b_sk;                   // element stride between rows k of B (columns contiguous)
    int64_t M, N, K;
    int32_t ksplit, kchunk;
    GemvPrologue prologue;
    int32_t has_res;
    float eps;
    int32_t pad;
    float* work;                    // LDG variant: [ksplit, M, N] partials; stream variant: [strips, max_contrib, M, 256]
    unsigned int* counters;         // per 256-column strip arrival counters (self-resetting)
    // ---- persistent TMA-streamed variant (launch_gemv_stream) ----
    // Up to two weight matrices sharing A and the prologue (horizontally fused
    // sibling MatMuls, e.g. gate/up): strips [0, strips0) belong to matrix 0,
    // the rest to matrix 1 (output map c2).
    int32_t stream;                 // 1: use the streaming kernel
    int32_t nmat;
    int32_t stages, grid, max_contrib, a_tiles;  // a_tiles: k-tiles of A staged per CTA
    int32_t strips0, b_static;      // b_static: weights never written by the plan (prefetch before pdl_wait)
    int32_t pre_stages, l2_prefetch;  // weight tiles issued before the activation loads; tiles
                                     // prefetched into L2 while the previous launch finishes
    int64_t n_mat[GEMV_MAX_MATS];
    const int32_t* strip_first;     // first CTA touching each 256-column strip
    const int32_t* strip_count;     // number of CTAs touching it
    VOperand c2;
    // host-resolved row addressing of the prologue operands (rows_ok): the
    // element pointer of A[m, 0] / A2[m, 0] / normw[0] and the stride along K,
    // so the kernel does no map evaluation between its dependency wait and
    // its activation loads
    int32_t rows_ok, pad5;
    const void* arow[4];
    const void* a2row[4];
    const void* wrow;
    int64_t sa[4], sa2[4], sw;
    // fused epilogue trees (has_epi): table [M * N] of EpiEntry
    int32_t has_epi, epi_dyn;       // epi_dyn: bytes per position of EPI_DYN_OUT addresses
    const EpiEntry* epi;
    int64_t epi_shift;              // bytes added to the out address of EPI_DYN_OUT entries
    EpiTree epi_tree[EPI_MAX_TREES];
    alignas(64) unsigned char tmap[GEMV_MAX_MATS][128];  // CUtensorMap per weight matrix (host-encoded)
};
void launch_gemv(const GemvParams& p, const GemvParams* dp, cudaStream_t s);
void launch_gemv_stream(const GemvParams& p, const GemvParams* dp, cudaStream_t s);

// ---- chained streaming GEMVs: one persistent launch, device-side dependencies ----
// Consecutive streamed GEMVs (o_proj -> gate/up -> down) run as stages of ONE
// launch: the producer keeps streaming weights across stage boundaries (they are
// static), and each CTA starts a stage as soon as the strips of the previous
// stage it reads are published (per-strip flags), instead of at a grid boundary.
constexpr int GEMV_MAX_CHAIN = 4;
struct GemvChainStage {
    int64_t K, n0, n1;               // reduction length; columns of matrix 0 / 1
    int32_t nmat, strips0, b_static, pre_stages;
    int32_t l2_prefetch;
    int32_t dep_range;               // 1: wait only for the previous stage's strips this CTA's k-range reads
    int32_t dep_a2;                  //    ... also the matching strips of its second matrix (SiLU*Mul a2)
    uint32_t dep_all;                // bitmask of earlier stages to wait for completely
};
struct GemvChainArgs {
    alignas(64) unsigned char tmap[GEMV_MAX_CHAIN][GEMV_MAX_MATS][128];
    GemvChainStage st[GEMV_MAX_CHAIN];
    int32_t nst, ring;               // stages; weight-ring depth
    int32_t max_strips, pad;
    int64_t sA_floats;               // A staging area (max over stages)
    unsigned* sync;                  // [0] launch generation, [1] exit count, [2 + st * max_strips + strip] flags
};
// dp: nst consecutive GemvParams (one per stage, same M and grid)
void launch_gemv_chain(const GemvChainArgs& ca, const GemvParams* dp, int64_t M, int grid, cudaStream_t s);
size_t gemv_chain_smem(int64_t sA_floats, int ring);
// dynamic shared memory of the streaming kernel; 0 if the configuration does not fit
size_t gemv_stream_smem(int64_t M, int a_tiles, int stages);
constexpr int GEMV_STREAM_COLS = 256, GEMV_STREAM_KT = 64;
// Encode a 2-D TMA descriptor for a row-major bf16 [rows, cols] matrix with
// row stride `ld` elements and a {256, 64} box; returns false if unsupported.
bool encode_weight_tmap(void* out128, const void* base, int64_t rows, int64_t cols, int64_t ld);

// ---- bf16 GEMM on tcgen05 tensor cores (M > 16) ---------------------------
// C = A . B (+ residual); A [M, K] read by TMA through a single-piece affine
// map (unit stride along K), B [K, N] physical row-major; C / residual through
// their maps (affine along N per row).  K is split across `splits` CTAs per
// tile when the tile grid alone would leave SMs idle.
constexpr int GEMM_MAX_SEG = 4;
enum GemmEpi : int32_t { GEMM_EPI_PLAIN = 0, GEMM_EPI_GELU = 1, GEMM_EPI_SWIGLU = 2, GEMM_EPI_TREES = 3 };
// An elementwise tree evaluated in the tensor-core GEMM's epilogue (e.g. the
// Q / K RoPE trees over the QKV projection): the tree's index space is
// [rows = the GEMM's M, heads, hd]; operand k addresses element (m, h, i) at
//   C-derived (from_c): C column ccol[q] + sh[q] * h + i of the same row m,
//   external / output:  base[q] + (rs[q] * m + sh[q] * h + i) elements,
// with piece q = (i >= split).  Head h's C columns lie in one N tile: they
// start at anchor c_lo + c_sh * h and span less than 128 columns.
constexpr int GEMM_MAX_TREES = 2;
struct GemmTreeOp {
    uint64_t base[2];
    int64_t rs[2], sh[2], ccol[2];
    int32_t from_c, split;
};
struct GemmTree {
    int32_t nin, nprog, result, hd;
    int32_t nh, pat;  // pat 3: the program is (in0 * in1) + (in2 * in3) (RoPE), evaluated in registers
    int64_t c_lo, c_sh;
    int64_t out_dyn;  // dynamic-position plans: bytes per position the output bases move (0: static)
    EwInstr prog[EW_MAX_PROG];
    GemmTreeOp op[EW_MAX_IN + 1];  // [0] = output
};
struct GemmTcParams {
    KHead head;
    VOperand c, res;
    VOperand a;           // gather path only: A rows located through this map
    int32_t a_gather;     // 1: A by cp.async gathers (map not TMA-readable), 0: A by TMA
    int32_t mt;           // 128-row sub-tiles per CTA (1, or 2 for prefill-sized M)
    int32_t pair;         // 1: 128 x 256 tiles, two CTAs per SM (one's epilogue overlaps the other's mainloop)
    int32_t cta_pair;     // 1: cta_group::2 -- a cluster of two CTAs computes a 256 x 256 tile
    int32_t coop_reduce;  // split-K: every split reduces a column slice (grid co-resident; counters[2 * tiles])
    int32_t ntiles_total;
    int64_t M, N, K;
    int32_t bn, splits;   // N tile (128 / 256), K splits
    int32_t has_res, pad;
    float* work;          // [tiles, splits, 128, bn] fp32 partials (splits > 1)
    unsigned int* counters;
    // gather path, host-resolved rows: A's K axis in a_nseg segments [a_seg_k[s], a_seg_k[s+1])
    // (BK-aligned piece boundaries, e.g. a virtual Concat along K); a_rows[s * M + m] = address
    // of A[m, a_seg_k[s]] minus a_seg_k[s] elements.  Null: rows located on the device.
    const uint64_t* a_rows;
    // C rows resolved on the host when C's map is not affine and every row lies in one
    // piece with one stride: c_rows[m] = address of C[m, 0], c_rs = stride along N
    const uint64_t* c_rows;
    int64_t c_rs;
    int32_t a_nseg, a_pad3;
    int32_t a_seg_k[GEMM_MAX_SEG + 1];
    // A's TMA tensor: up to 5 dimensions, one per digit of A's map
    // ((idx[axis] / div) mod mod, axis 0 = M, 1 = K); coordinates of a tile at
    // (m0, k0) are computed per dimension by the producer
    int32_t a_ndims, a_pad;
    int32_t a_axis[5];
    int32_t a_pad2[3];
    int64_t a_div[5], a_mod[5];
    alignas(64) unsigned char tmap_a[128];
    alignas(64) unsigned char tmap_b[128];
    // horizontally fused sibling (gate / up reading the same A): N tiles past the
    // first matrix's use B2 (tmap_b2) and store C2 through host-resolved rows
    int32_t nmat, pad_h;
    int64_t N1;
    const uint64_t* c2_rows;
    int64_t c2_rs;
    alignas(64) unsigned char tmap_b2[128];
    // fused epilogue (GemmEpi): GELU of the rounded product; SwiGLU, where each
    // 256-column B stage holds 128 columns of B (gate) and the same 128 of B2 (up)
    // and the tile stores SiLU(gate) * up; or elementwise trees over views of C
    int32_t epi, ntree;
    int64_t skip_lo, skip_hi;  // trees: C columns [skip_lo, skip_hi) are not stored (read only by the trees)
    GemmTree tree[GEMM_MAX_TREES];
};
// Encode a B tensor map (row-major bf16 [K, N], row stride ld) into out128.
bool gemm_tc_encode_b(void* out128, const void* b_base, int64_t N, int64_t K, int64_t ld);
// Derive A's TMA dimensions from its lowered map (one piece, no groups, digits
// forming tile-aligned mixed-radix coordinates; innermost = K with unit stride).
bool gemm_tc_a_dims(const vtc_map& a, int64_t M, int64_t K, GemmTcParams& p, int64_t dims[5], int64_t strides[5],
                    const void** base);
bool gemm_tc_encode(GemmTcParams& p, const void* a_base, const int64_t* a_dims, const int64_t* a_strides,
                    const void* b_base, int64_t b_ld);
void launch_gemm_tc(const GemmTcParams& p, const GemmTcParams* dp, cudaStream_t s);

// ---- persistent shallow-K GEMM (weights resident in shared memory) --------
// C[M, N] = epi(A . W) (+ residual) for K, N <= 512 at large M (Swin's projections):
// A by TMA (tmap_a, a plain 2-D view) or 16-byte gathers from host-resolved rows
// (a_rows[m] = address of A[m, 0]); C / residual rows affine (base + m * ld) or
// host-resolved (c_rows / r_rows), unit column stride, 16-byte aligned.
struct SkinnyParams {
    KHead head;
    int64_t M, N, K;
    int32_t kt, nc, nchunks, slots;  // k-tiles, N columns per unit, units per tile, A ring slots
    int32_t epi;                     // 0: plain, 1: GELU of the rounded product
    int32_t has_res, a_gather, b_static, sms;
    int32_t a_norm;                  // 1: A = LayerNorm(rows), 2: RMSNorm(rows) -- a_rows are the norm's input rows
    float eps;
    const void* norm_w;              // [K] bf16
    const void* norm_b;              // [K] bf16 (LayerNorm)
    size_t smem;
    const void* w;  // weights [K, N] bf16, row stride ldw
    int64_t ldw;
    const uint64_t* a_rows;
    uint64_t c_base;
    int64_t c_ld;
    const uint64_t* c_rows;
    uint64_t r_base;
    int64_t r_ld;
    const uint64_t* r_rows;
    alignas(64) unsigned char tmap_a[128];
};
// Tile plan (k-tiles, N units, ring depth, shared memory); false if the weight does not fit.
bool skinny_plan(SkinnyParams& p, int smem_optin);
bool skinny_encode_a(SkinnyParams& p, const void* a_base, int64_t lda);
void launch_gemm_skinny(const SkinnyParams& p, const SkinnyParams* dp, cudaStream_t s);

// ---- row-wise normalisations / softmax -----------------------------------
enum class RowOp : int32_t { RMSNorm = 0, LayerNorm, Softmax };
struct RowParams {
    KHead head;
    VOperand x, w, bias, out;
    int32_t rank;
    int32_t shape[VTC_MAX_RANK];
    int64_t rows, D;
    float eps;
    RowOp op;
    KDType dt;
    int32_t linear;  // host-proved: x and out are flat-linear (row r at base + r * D)
};
void launch_rowop(const RowParams& p, const RowParams* dp, cudaStream_t s);

// ---- attention (split-KV flash decoding with GQA head grouping) ----------
struct AttnParams {
    KHead head;
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
    // tensor-core decode path (k_attn_decode.cu)
    int32_t fast;                  // 1: attn_decode_kernel, 2: attn_prefill_kernel
    int32_t kv_affine;             // K/V maps affine along the key axis (single piece)
    int64_t k_sstride, v_sstride;  // element stride between consecutive keys
    unsigned int* counters;        // [Bt * H / group] split arrival counters (fused combine)
    // tcgen05 flash attention (k_attn_fmha.cu, fast == 3): Q / K / V as 4-D TMA
    // tensors (CUtensorMap x 3), O as base + (batch, head, position) strides
    alignas(64) unsigned char fmha[3 * 128];
    uint64_t fmha_o;
    int64_t fmha_os[3];
    // short-sequence window attention (fast == 4): Q / O rows and the bias are
    // base + position * stride within a (batch, head) item (host-proved)
    int32_t qo_affine, bias_affine;
    int64_t q_sstride, o_sstride, b_sstride, b_kstride;
    const uint64_t* item_base;     // [Bt * H][5]: Q, K, V, O, bias addresses at position 0 (host-resolved)
    // decode: L2 prefetch of the next launch's weights while the (latency-bound)
    // attention leaves HBM idle -- [pf_base, pf_base + pf_bytes), split over the CTAs
    uint64_t pf_base;
    int64_t pf_bytes;
};
void launch_attention(const AttnParams& p, const AttnParams* dp, cudaStream_t s);
// tcgen05 / TMEM flash attention for head dim 128 (prefill): proves the Q / K / V / O
// maps affine over (batch, head, position, dim) and encodes their TMA tensors
// (encode = false: the structural check only, for dry plans).
bool attn_fmha_prepare(AttnParams& p, bool encode);
void launch_attn_fmha(const AttnParams& p, const AttnParams* dp, cudaStream_t s);
bool attn_decode_supported(const AttnParams& p);
int64_t attn_decode_capacity();
bool attn_prefill_supported(const AttnParams& p);
void launch_attn_prefill(const AttnParams& p, const AttnParams* dp, cudaStream_t s);
void launch_attn_decode(const AttnParams& p, const AttnParams* dp, cudaStream_t s);
bool attn_window_supported(const AttnParams& p);
void launch_attn_window(const AttnParams& p, const AttnParams* dp, cudaStream_t s);

}  // namespace vtc
