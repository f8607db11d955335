// GPU executor: points-to graph -> lowered descriptors -> kernel launches.
// Mirrors execute_detailed (proj/src/executor.cpp:448-498); see exec.hpp.
#include "vtc/exec.hpp"

#include <cstdlib>
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <deque>
#include <unordered_map>
#include <functional>
#include <set>

#include <cuda_runtime.h>

#include "comm.hpp"
#include "kernels.hpp"
#include "launch.cuh"
#include "lower.hpp"

namespace vtc {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// SM count of the current device (the rank's GPU, not device 0)
// A/B and test switches of the executor, read from the environment once per
// prepare (DESIGN.md §6a lists them; every default is the measured best).
struct Tuning {
    int gemv_stages = -1, gemv_pre = -1, gemv_l2pf = -1, chain_l2pf = -1, attn_ctas = -1;
    int64_t host_link_max = -1;
    bool no_ew_fast, no_ew_aff, no_tc_epi, no_tc_hfuse, no_skinny, no_skinny_norm, no_epi_fusion, debug_fusion,
        no_tc_trees, no_row_fast, gemm_pair, gemm_cta_pair, no_coop_reduce, no_fmha, no_attn_window, separate_combine, attn_l2pf, chain, trace, tree_coop,
        host_dma;
    static bool set(const char* k) { return std::getenv(k) != nullptr; }
    static bool on(const char* k) {
        const char* e = std::getenv(k);
        return e && e[0] == '1';
    }
    static Tuning from_env() {
        Tuning t;
        auto num = [](const char* k, auto& v) {
            if (const char* e = std::getenv(k)) v = std::atoll(e);
        };
        num("VTC_GEMV_STAGES", t.gemv_stages);
        num("VTC_GEMV_PRE", t.gemv_pre);
        num("VTC_GEMV_L2PF", t.gemv_l2pf);
        num("VTC_CHAIN_L2PF", t.chain_l2pf);
        num("VTC_ATTN_CTAS", t.attn_ctas);
        num("VTC_HOST_LINK_MAX", t.host_link_max);
        t.no_ew_fast = set("VTC_NO_EW_FAST");
        t.no_ew_aff = set("VTC_NO_EW_AFF");
        t.no_tc_epi = set("VTC_NO_TC_EPI");
        t.no_tc_hfuse = set("VTC_NO_TC_HFUSE");
        t.no_skinny = set("VTC_NO_SKINNY");
        t.no_skinny_norm = set("VTC_NO_SKINNY_NORM");
        t.no_epi_fusion = set("VTC_NO_EPI_FUSION");
        t.debug_fusion = set("VTC_DEBUG_FUSION");
        t.no_tc_trees = set("VTC_NO_TC_TREES");
        t.tree_coop = set("VTC_TREE_COOP");
        t.no_row_fast = set("VTC_NO_ROW_FAST");
        t.gemm_pair = on("VTC_GEMM_PAIR");
        t.gemm_cta_pair = on("VTC_GEMM_CTA_PAIR");
        t.no_coop_reduce = set("VTC_NO_COOP_REDUCE");
        t.no_fmha = set("VTC_NO_FMHA");
        t.no_attn_window = set("VTC_NO_ATTN_WINDOW");
        t.separate_combine = set("VTC_ATTN_SEPARATE_COMBINE");
        const char* pf = std::getenv("VTC_ATTN_L2PF");
        t.attn_l2pf = !(pf && pf[0] == '0');
        t.chain = on("VTC_CHAIN");
        t.trace = on("VTC_TRACE");
        t.host_dma = set("VTC_HOST_DMA");
        return t;
    }
};

int device_sms() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

KDType kdt(DType d) {
    switch (d) {
        case DType::F64: return KDType::F64;
        case DType::F32: return KDType::F32;
        case DType::I64: return KDType::I64;
        case DType::BF16: return KDType::BF16;
    }
    return KDType::F32;
}

// ---- dynamic decode position (ExecOptions::dynamic_pos) ----
// A root updated in place by a ScatterND at static row p0 (the KV caches): row
// stride rs elements, so the position's slab is elements [pos*rs, (pos+1)*rs).
struct DynRoot {
    int root = -1;
    int64_t rs = 0, es = 0;
    uint64_t ptr = 0;
    int64_t bytes = 0;
};
struct DynCtx {
    std::vector<DynRoot> roots;
    int64_t p0 = 0;
    const int64_t* dev = nullptr;  // device position (root "__pos")
    bool dry = false;
    std::string node;

    const DynRoot* find(int target) const {
        for (const auto& r : roots)
            if (r.root == target) return &r;
        return nullptr;
    }
    // element-offset range a piece addresses over its box (false: not bounded cheaply)
    static bool piece_range(const vtc_map& m, int pi, int64_t& lo, int64_t& hi) {
        const vtc_piece& pc = m.piece[pi];
        if (pc.affine) {
            lo = hi = pc.base;
            for (int a = 0; a < m.rank; ++a) {
                if (pc.hi[a] <= pc.lo[a]) return false;
                const int64_t s0 = pc.aff[a] * pc.lo[a], s1 = pc.aff[a] * (pc.hi[a] - 1);
                lo += std::min(s0, s1);
                hi += std::max(s0, s1);
            }
            return true;
        }
        int64_t vol = 1;
        for (int a = 0; a < m.rank; ++a) vol *= std::max<int64_t>(0, pc.hi[a] - pc.lo[a]);
        if (vol <= 0 || vol > (int64_t(1) << 16)) return false;
        lo = INT64_MAX;
        hi = INT64_MIN;
        int64_t idx[VTC_MAX_RANK] = {};
        for (int64_t f = 0; f < vol; ++f) {
            int64_t r = f;
            for (int a = m.rank - 1; a >= 0; --a) {
                const int64_t ext = pc.hi[a] - pc.lo[a];
                idx[a] = pc.lo[a] + r % ext;
                r /= ext;
            }
            int got = -1;
            const int64_t off = desc_eval(m, idx, &got);
            if (got != pi) continue;
            lo = std::min(lo, off);
            hi = std::max(hi, off);
        }
        return lo <= hi;
    }
    void add(KHead& h, const void* base, const void* field, int bytes, int64_t coeff) {
        if (h.ndyn >= KHEAD_MAX_DYN) throw UnsupportedError("dynamic position: too many position-dependent fields in " + node);
        const auto off = static_cast<const char*>(field) - static_cast<const char*>(base);
        h.patch[h.ndyn++] = DynPatch{uint32_t(off), int32_t(bytes), coeff};
        h.dyn = dev;
        h.dyn0 = p0;
    }
    // a piece inside the position's slab moves with the position; other pieces of a
    // dynamic root may be read (rows already in the cache) but not written
    void operand(KHead& h, const void* base, VOperand& op, bool write) {
        for (int i = 0; i < op.m.npieces; ++i) {
            const DynRoot* r = find(op.m.piece[i].target);
            if (!r) continue;
            int64_t lo = 0, hi = 0;
            const bool known = piece_range(op.m, i, lo, hi);
            if (known && lo >= p0 * r->rs && hi < (p0 + 1) * r->rs) add(h, base, &op.m.piece[i].base, 8, r->rs);
            else if (write) throw UnsupportedError("dynamic position: " + node + " writes a cache outside the position's row");
        }
    }
    bool reads(const VOperand& op) const {
        for (int i = 0; i < op.m.npieces; ++i)
            if (find(op.m.piece[i].target)) return true;
        return false;
    }
    // host-resolved addresses (row tables) cannot move with the position
    void check_ptr(const void* p, const char* what) const {
        if (dry || !p) return;
        const auto a = reinterpret_cast<uint64_t>(p);
        for (const auto& r : roots)
            if (a >= r.ptr && a < r.ptr + uint64_t(r.bytes))
                throw UnsupportedError(std::string("dynamic position: host-resolved ") + what + " of " + node + " points into a cache");
    }
};

void dyn_ops(EwParams& p, DynCtx& c) {
    c.operand(p.head, &p, p.out, true);
    for (int i = 0; i < p.nin; ++i) c.operand(p.head, &p, p.in[i], false);
}
void dyn_ops(EwPair& p, DynCtx& c) {
    dyn_ops(p.a, c);
    dyn_ops(p.b, c);
}
void dyn_ops(RowParams& p, DynCtx& c) {
    c.operand(p.head, &p, p.out, true);
    c.operand(p.head, &p, p.x, false);
    c.operand(p.head, &p, p.w, false);
    if (p.op == RowOp::LayerNorm) c.operand(p.head, &p, p.bias, false);
}
void dyn_ops(MatmulParams& p, DynCtx& c) {
    c.operand(p.head, &p, p.c, true);
    c.operand(p.head, &p, p.a, false);
    c.operand(p.head, &p, p.b, false);
}
void dyn_ops(GemvParams& p, DynCtx& c) {
    c.operand(p.head, &p, p.c, true);
    if (p.nmat > 1) c.operand(p.head, &p, p.c2, true);
    c.operand(p.head, &p, p.a, false);
    if (p.prologue == GemvPrologue::SiLUMul) c.operand(p.head, &p, p.a2, false);
    if (p.prologue == GemvPrologue::RMSNorm) c.operand(p.head, &p, p.normw, false);
    if (p.has_res) c.operand(p.head, &p, p.res, false);
    for (int m = 0; m < 4 && p.rows_ok; ++m) {
        c.check_ptr(p.arow[m], "A row");
        c.check_ptr(p.a2row[m], "A2 row");
    }
    if (p.rows_ok) c.check_ptr(p.wrow, "norm weight row");
    if (p.has_epi && p.epi_dyn) c.add(p.head, &p, &p.epi_shift, 8, p.epi_dyn);
}
void dyn_ops(GemmTcParams& p, DynCtx& c) {
    if ((p.c_rows && c.reads(p.c)) || (p.a_gather && c.reads(p.a)))
        throw UnsupportedError("dynamic position: host-resolved rows of " + c.node + " address a cache");
    c.operand(p.head, &p, p.c, true);
    if (p.has_res) c.operand(p.head, &p, p.res, false);
    // fused trees storing into the position's cache row (the roped K row): both piece bases move
    for (int k = 0; p.epi == GEMM_EPI_TREES && k < p.ntree; ++k)
        if (p.tree[k].out_dyn)
            for (int q = 0; q < 2; ++q) c.add(p.head, &p, &p.tree[k].op[0].base[q], 8, p.tree[k].out_dyn);
}
void dyn_ops(SkinnyParams& p, DynCtx& c) {
    // every address is host-resolved: none may point into a position-dependent cache
    c.check_ptr(p.w, "weights");
    c.check_ptr(reinterpret_cast<const void*>(p.c_base), "output");
    c.check_ptr(reinterpret_cast<const void*>(p.r_base), "residual");
    if (p.c_rows || p.r_rows || p.a_rows) throw UnsupportedError("dynamic position: row tables of " + c.node);
}
void dyn_ops(AttnParams& p, DynCtx& c) {
    c.operand(p.head, &p, p.o, true);
    c.operand(p.head, &p, p.q, false);
    if (p.has_bias) c.operand(p.head, &p, p.bias, false);
    const bool kr = c.reads(p.k), vr = c.reads(p.v);
    if (!kr && !vr) return;
    // keys [0, pos] of the cache: the key count follows the position
    // (every attention kernel uses Sk only as the key bound; the split-KV chunking stays
    // the one planned for p0 + 1 keys, later splits are empty)
    if (!(kr && vr) || p.Sq != 1 || p.causal || int64_t(p.Sk) != c.p0 + 1)
        throw UnsupportedError("dynamic position: attention " + c.node + " does not read the cache prefix [0, pos]");
    c.add(p.head, &p, &p.Sk, 4, 1);
}

struct Launch {
    std::string node, kernel;
    virtual ~Launch() = default;
    virtual void run(cudaStream_t s) = 0;
    virtual size_t param_bytes() const = 0;
    virtual const void* host_params() const = 0;
    virtual void set_device_params(void* d) = 0;
    virtual void set_trace(unsigned long long* t, int id) = 0;
    virtual void dyn_patch(DynCtx& c) {
        c.node = node;
        throw UnsupportedError("dynamic position: launch " + node + " (" + kernel + ") has no position patches");
    }
};

template <class P>
void set_head(P& p, unsigned long long* t, int id) {
    p.head.trace = t;
    p.head.id = id;
}
inline void set_head(EwPair& p, unsigned long long* t, int id) {
    set_head(p.a, t, id);
    set_head(p.b, t, id);
}

// Host copy of the parameter block (for dispatch decisions) + its device copy
// (what the kernel reads).
template <class P, void (*F)(const P&, const P*, cudaStream_t)>
struct LaunchT : Launch {
    P p;
    const P* dp = nullptr;
    void run(cudaStream_t s) override { F(p, dp, s); }
    size_t param_bytes() const override { return sizeof(P); }
    const void* host_params() const override { return &p; }
    void set_device_params(void* d) override { dp = static_cast<const P*>(d); }
    void set_trace(unsigned long long* t, int id) override { set_head(p, t, id); }
    void dyn_patch(DynCtx& c) override {
        c.node = node;
        dyn_ops(p, c);
    }
};

// AllReduce(sum) of a contiguous buffer over the plan's communicator; with no
// communicator (single rank) the sum over one rank is the identity.
struct AllReduceLaunch : Launch {
    const void* src = nullptr;
    void* dst = nullptr;
    size_t count = 0, bytes = 0;
    ncclDataType_t dt = ncclBfloat16;
    Comm* const* comm = nullptr;
    void run(cudaStream_t s) override {
        if (*comm) (*comm)->all_reduce_sum(src, dst, count, dt, s);
        else if (dst != src) ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s), "D2D");
    }
    size_t param_bytes() const override { return 0; }
    const void* host_params() const override { return nullptr; }
    void set_device_params(void*) override {}
    void set_trace(unsigned long long*, int) override {}
    void dyn_patch(DynCtx& c) override {
        c.node = node;
        c.check_ptr(src, "allreduce input");
        c.check_ptr(dst, "allreduce output");
    }
};

// Consecutive streamed GEMVs as the stages of one persistent launch.
struct GemvChainLaunch : Launch {
    std::vector<GemvParams> ps;
    GemvChainArgs ca{};
    const GemvParams* dp = nullptr;
    void run(cudaStream_t s) override { launch_gemv_chain(ca, dp, ps[0].M, ps[0].grid, s); }
    size_t param_bytes() const override { return ps.size() * sizeof(GemvParams); }
    const void* host_params() const override { return ps.data(); }
    void set_device_params(void* d) override { dp = static_cast<const GemvParams*>(d); }
    void set_trace(unsigned long long* t, int id) override {
        for (auto& p : ps) set_head(p, t, id);
    }
};

void launch_gemv_any(const GemvParams& p, const GemvParams* dp, cudaStream_t s) {
    if (p.stream) launch_gemv_stream(p, dp, s);
    else launch_gemv(p, dp, s);
}

// Upload a parameter block for a one-off launch; caller frees.
template <class P>
P* upload_params(const P& p) {
    P* d = nullptr;
    ck(cudaMalloc(&d, sizeof(P)), "cudaMalloc(params)");
    ck(cudaMemcpy(d, &p, sizeof(P), cudaMemcpyHostToDevice), "H2D(params)");
    return d;
}

// Host-side digest of a lowered map along the kernel's fast axis.
void finish_operand(VOperand& op, int fast_axis, int64_t tile, int64_t esize) {
    op.fast_axis = fast_axis;
    const vtc_map& d = op.m;
    bool ok = fast_axis >= 0 && fast_axis < d.rank && desc_pieces_aligned(d, fast_axis, tile);
    for (int pi = 0; pi < d.npieces && ok; ++pi) {
        int64_t s = desc_tile_stride(d.piece[pi], fast_axis, tile);
        if (s == INT64_MIN) ok = false;
        else op.fast_stride[pi] = s;
    }
    op.fast_ok = ok ? 1 : 0;
    // 16-byte vectors along the fast axis
    int64_t vec = 16 / esize;
    bool vok = ok && tile % vec == 0 && d.shape[fast_axis] % vec == 0 && desc_pieces_aligned(d, fast_axis, vec);
    for (int pi = 0; pi < d.npieces && vok; ++pi) {
        const vtc_piece& p = d.piece[pi];
        if (op.fast_stride[pi] != 1 || p.base % vec != 0 || p.ptr % 16 != 0) vok = false;
        for (int t = 0; t < p.ndigits && vok; ++t) {
            const vtc_digit& g = p.dig[t];
            bool linear_fast = g.axis == fast_axis && g.div == 1;
            if (g.group >= 0) continue;
            if (linear_fast) {
                if (g.mod && g.mod % vec != 0) vok = false;
            } else if (g.coeff % vec != 0) {
                vok = false;
            }
        }
        for (int gi = 0; gi < p.ngroups && vok; ++gi)
            if (p.grp[gi].coeff % vec != 0) vok = false;
    }
    op.vec_ok = vok ? 1 : 0;
}

}  // namespace

bool map_flat_linear(const vtc_map& m, int rank, const int32_t* shape) {
    if (m.npieces != 1 || m.rank != rank) return false;
    const vtc_piece& p = m.piece[0];
    if (!p.affine) return false;
    int64_t st = 1;
    for (int a = rank - 1; a >= 0; --a) {
        if (m.shape[a] != shape[a] || p.lo[a] > 0 || p.hi[a] < shape[a]) return false;
        if (shape[a] > 1 && p.aff[a] != st) return false;
        st *= shape[a];
    }
    return true;
}

namespace {

// K segments of a rank-2 gather operand: the distinct piece boundaries along K
// (axis 1), each a multiple of the 64-wide k-tile, at most GEMM_MAX_SEG segments,
// so every k-tile of a row lies inside one piece.
bool k_segments(const vtc_map& m, int64_t K, std::vector<int64_t>& bounds) {
    std::set<int64_t> b{0, K};
    for (int pi = 0; pi < m.npieces; ++pi) {
        for (int64_t v : {int64_t(m.piece[pi].lo[1]), int64_t(m.piece[pi].hi[1])})
            if (v > 0 && v < K) b.insert(v);
    }
    bounds.assign(b.begin(), b.end());
    if (int(bounds.size()) - 1 > GEMM_MAX_SEG) return false;
    for (int64_t v : bounds)
        if (v != K && v % 64 != 0) return false;
    return true;
}

// Heads sharing identical K/V addresses: the map ignores (h mod G).
bool ignores_mod(const vtc_map& d, int axis, int G) {
    for (int pi = 0; pi < d.npieces; ++pi) {
        const vtc_piece& p = d.piece[pi];
        if (p.lo[axis] % G != 0 || (p.hi[axis] % G != 0 && p.hi[axis] != d.shape[axis])) return false;
        for (int t = 0; t < p.ndigits; ++t) {
            const vtc_digit& g = p.dig[t];
            if (g.axis != axis) continue;
            if (g.group >= 0) return false;
            if (g.div % uint32_t(G) != 0) return false;
        }
    }
    return true;
}

}  // namespace

struct Executor::Impl {
    std::vector<std::unique_ptr<Launch>> launches;
    std::vector<void*> scratch;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t captured_on = nullptr;
    unsigned long long* trace = nullptr;  // VTC_TRACE timeline buffer (8 per launch)
    Comm* comm = nullptr;                 // tensor-parallel communicator (AllReduce nodes)

    void free_scratch() {
        for (void* p : scratch) cudaFree(p);
        scratch.clear();
    }
    // run_host graph: H2D of the input arena -> launches -> D2H of the outputs
    cudaGraphExec_t hexec = nullptr;
    std::string hkey;
    void* out_host = nullptr;  // pinned output staging
    size_t out_host_bytes = 0;
    std::vector<std::pair<std::string, int64_t>> sig_in, sig_out;  // the call hexec was built for
    std::vector<size_t> out_off;
    std::vector<int> out_kind;  // 0: staged in the graph, 1: DMA after the launch, 2: virtual (download)
    std::vector<int> in_slot;   // arena slot of a staged input, -1: DMA before the launch
    std::vector<void*> in_dev, out_dev;
    cudaStream_t fast_stream = nullptr;
    void free_graph() {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        if (hexec) cudaGraphExecDestroy(hexec);
        gexec = nullptr;
        graph = nullptr;
        hexec = nullptr;
        hkey.clear();
    }
    bool dry = false;
    DynCtx dyn;            // dynamic-position plans: cache roots, static position
    bool dyn_on = false;
    // enqueue the launch list; a dynamic-position plan's first launch is
    // stream-serialised so the step's position is written before any kernel reads it
    void launch_all(cudaStream_t s) {
        if (dyn_on) tl_serialize_next = true;
        for (auto& l : launches) l->run(s);
        tl_serialize_next = false;
    }
    void* alloc(size_t bytes, bool zero) {
        if (dry) return nullptr;
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc(scratch)");
        if (zero) ck(cudaMemset(p, 0, std::max<size_t>(bytes, 16)), "cudaMemset(scratch)");
        scratch.push_back(p);
        return p;
    }
};

Executor::Executor(const CompGraph& g, PointsToGraph ptg, ExecOptions opt)
    : g_(g), ptg_(std::move(ptg)), opt_(opt), impl_(std::make_unique<Impl>()) {
    for (const auto& id : ptg_.roots) {
        const TensorSpec& t = g_.tensor(id);
        RootBuffer rb;
        rb.id = id;
        rb.dtype = t.dtype;
        rb.shape = t.shape;
        rb.bytes = t.bytes();
        root_index_[id] = int(roots_.size());
        roots_.push_back(rb);
    }
    if (opt_.dynamic_pos) {
        RootBuffer rb;
        rb.id = "__pos";
        rb.dtype = DType::I64;
        rb.shape = {1};
        rb.bytes = 8;
        root_index_[rb.id] = int(roots_.size());
        roots_.push_back(rb);
    }
}

Executor::~Executor() {
    impl_->free_graph();
    impl_->free_scratch();
    for (auto& r : roots_)
        if (r.owned && r.ptr) cudaFree(r.ptr);
    if (arena_dev_) cudaFree(arena_dev_);
    if (arena_host_) cudaFreeHost(arena_host_);
    if (impl_->out_host) cudaFreeHost(impl_->out_host);
}

void Executor::bind_root(const std::string& id, void* dev_ptr) {
    auto it = root_index_.find(id);
    if (it == root_index_.end()) throw ExecutionError("tensor " + id + " is not a physical root of this plan");
    RootBuffer& r = roots_[size_t(it->second)];
    if (r.ptr == dev_ptr) return;
    // the launches (and any captured graph, including vtc_run's host graph) hold
    // the old address: drop them before the old buffer goes away
    invalidate();
    if (r.owned && r.ptr) cudaFree(r.ptr);
    r.ptr = dev_ptr;
    r.owned = false;
}

void Executor::invalidate() {
    impl_->free_graph();
    impl_->launches.clear();
    prepared_ = false;
}

void* Executor::root_ptr(const std::string& id) {
    auto it = root_index_.find(id);
    if (it == root_index_.end()) throw ExecutionError("tensor " + id + " is not a physical root of this plan");
    RootBuffer& r = roots_[size_t(it->second)];
    if (!r.ptr) {
        ck(cudaMalloc(&r.ptr, size_t(std::max<int64_t>(r.bytes, 16))), "cudaMalloc(root)");
        ck(cudaMemset(r.ptr, 0, size_t(std::max<int64_t>(r.bytes, 16))), "cudaMemset(root)");
        r.owned = true;
        if (prepared_) invalidate();
    }
    return r.ptr;
}

int Executor::num_kernel_launches() const {
    int n = 0;
    for (const auto& i : infos_) n += (i.kernel == "attention_splitkv") ? 2 : 1;
    return n;
}

void Executor::prepare(bool dry) {
    const Tuning tun = Tuning::from_env();
    if (!dry)
        for (auto& r : roots_) root_ptr(r.id);  // allocate every unbound root
    impl_->free_graph();
    impl_->free_scratch();
    impl_->dry = dry;
    impl_->launches.clear();
    infos_.clear();

    auto target = [&](const std::string& t) -> TargetInfo {
        auto it = root_index_.find(t);
        if (it == root_index_.end()) throw ExecutionError("map targets non-root tensor " + t);
        return TargetInfo{it->second, reinterpret_cast<uint64_t>(roots_[size_t(it->second)].ptr)};
    };
    auto operand = [&](const VMap& m, int fast_axis, int64_t tile, int64_t esize) {
        VOperand op{};
        op.m = lower_map(m, target);
        finish_operand(op, fast_axis, tile, esize);
        return op;
    };
    auto map_of = [&](const std::string& t) -> const VMap& { return ptg_.map_of(t); };
    auto targets_of = [&](const VMap& m) {
        auto v = m.targets();
        return std::set<std::string>(v.begin(), v.end());
    };
    auto lookup = [&](const std::string& t) -> const VMap* {
        if (std::find(ptg_.roots.begin(), ptg_.roots.end(), t) != ptg_.roots.end()) return nullptr;
        return &ptg_.resolved.at(t);
    };
    std::set<std::string> elim(ptg_.eliminated_ops.begin(), ptg_.eliminated_ops.end());

    // dynamic position: the caches updated in place by ScatterND at one static row p0
    impl_->dyn = DynCtx{};
    impl_->dyn_on = opt_.dynamic_pos;
    if (opt_.dynamic_pos) {
        DynCtx& dc = impl_->dyn;
        dc.dry = dry;
        bool have = false;
        for (const auto& n : g_.nodes()) {
            if (n.kind != OpKind::ScatterND) continue;
            const auto& at = std::get<ScatterNDAttrs>(n.attrs);
            const std::string& data = n.inputs[0];
            const VMap& dm = map_of(data);
            auto ts = dm.targets();
            if (at.indices.size() != 1 || at.indices[0].size() != 1 || ts.size() != 1 || !dm.is_identity_of(ts[0]) ||
                !map_of(n.outputs[0]).is_identity_of(ts[0]))
                throw UnsupportedError("dynamic position: ScatterND " + n.id +
                                       " is not a single-row in-place cache update (plan with in-place updates)");
            const int64_t p0 = at.indices[0][0];
            if (have && p0 != dc.p0) throw UnsupportedError("dynamic position: ScatterND updates at different rows");
            have = true;
            dc.p0 = p0;
            const TensorSpec& t = g_.tensor(data);
            DynRoot r;
            r.root = root_index_.at(ts[0]);
            r.rs = volume(t.shape) / t.shape[0];
            r.es = dtype_size(t.dtype);
            r.ptr = reinterpret_cast<uint64_t>(roots_[size_t(r.root)].ptr);
            r.bytes = roots_[size_t(r.root)].bytes;
            dc.roots.push_back(r);
        }
        if (!have) throw UnsupportedError("dynamic position: the graph has no ScatterND cache update");
        dc.dev = static_cast<const int64_t*>(roots_[size_t(root_index_.at("__pos"))].ptr);
        if (!dry && !pos_set_) {
            ck(cudaMemcpy(roots_[size_t(root_index_.at("__pos"))].ptr, &dc.p0, 8, cudaMemcpyHostToDevice), "H2D(pos)");
            pos_set_ = true;
        }
    }

    // algorithmic bytes of a (possibly fused) launch: tensors read from outside
    // the group (unique elements through their maps) + tensors the group emits
    auto group_bytes = [&](const std::string& names) -> int64_t {
        std::set<std::string> grp;
        size_t st = 0;
        while (st <= names.size()) {
            size_t e = names.find('+', st);
            if (e == std::string::npos) e = names.size();
            grp.insert(names.substr(st, e - st));
            st = e + 1;
        }
        std::set<std::string> produced, reads;
        int64_t bytes = 0;
        for (const auto& id : grp)
            if (const OpNode* n = g_.node(id))
                for (const auto& o : n->outputs) produced.insert(o);
        for (const auto& id : grp) {
            const OpNode* n = g_.node(id);
            if (!n) continue;
            for (const auto& in : n->inputs)
                if (!produced.count(in) && reads.insert(in).second)
                    bytes += ptg_.map_of(in).unique_elems() * dtype_size(g_.tensor(in).dtype);
            for (const auto& o : n->outputs) {
                bool internal = g_.tensor(o).kind == TensorKind::Intermediate;
                auto cs = g_.consumers(o);
                for (const OpNode* c : cs) internal = internal && grp.count(c->id);
                if (cs.empty()) internal = false;
                if (!internal) bytes += g_.tensor(o).bytes();
            }
        }
        return bytes;
    };
    auto push = [&](std::unique_ptr<Launch> l) {
        LaunchInfo li;
        li.node = l->node;
        li.kernel = l->kernel;
        li.bytes = group_bytes(l->node);
        infos_.push_back(li);
        impl_->launches.push_back(std::move(l));
    };

    // roots written by some node of the plan (weights that are not may be
    // prefetched before the kernel's dependency on earlier launches resolves)
    std::set<std::string> written_roots;
    for (const auto& n : g_.nodes())
        if (!elim.count(n.id))
            for (const auto& o : n.outputs)
                for (const auto& t : targets_of(map_of(o))) written_roots.insert(t);

    // Configure the persistent TMA-streamed GEMV: balanced contiguous ranges of
    // (256-column strip, 64-row k-tile) units, one CTA per SM.
    struct SecondMat {
        uint64_t ptr = 0;
        int64_t N = 0, ld = 0;
        std::string root;
    };
    auto stream_gemv = [&](GemvParams& p, uint64_t b_ptr, const std::string& b_root, const SecondMat* m2) -> bool {
        const int64_t COLS = GEMV_STREAM_COLS, KT = GEMV_STREAM_KT;
        const int sms = impl_->dry ? 148 : device_sms();
        int64_t strips0 = (p.N + COLS - 1) / COLS;
        int64_t strips = strips0 + (m2 ? (m2->N + COLS - 1) / COLS : 0);  // horizontal fusion: + the second matrix
        int64_t kts = (p.K + KT - 1) / KT, units = strips * kts;
        int grid = int(std::min<int64_t>(sms, units));
        std::vector<int32_t> first(size_t(strips), -1), count(size_t(strips), 0);
        int64_t maxrange = 0;
        for (int c = 0; c < grid; ++c) {
            int64_t ub = units * c / grid, ue = units * (c + 1) / grid;
            maxrange = std::max(maxrange, ue - ub);
            for (int64_t u = ub; u < ue; u = (u / kts + 1) * kts) {
                int64_t s2 = u / kts;
                if (first[size_t(s2)] < 0) first[size_t(s2)] = c;
                ++count[size_t(s2)];
            }
        }
        int a_tiles = int(std::min<int64_t>(kts, maxrange));
        int stages = 0;
        int max_st = 3;
        if (tun.gemv_stages >= 0) max_st = tun.gemv_stages;
        for (int st = max_st; st >= 2 && !stages; --st)
            if (gemv_stream_smem(p.M, a_tiles, st)) stages = st;
        if (!stages) return false;
        if (!impl_->dry && !encode_weight_tmap(p.tmap[0], reinterpret_cast<const void*>(b_ptr) , p.K, p.N, p.b_sk))
            return false;
        if (m2 && !impl_->dry && !encode_weight_tmap(p.tmap[1], reinterpret_cast<const void*>(m2->ptr), p.K, m2->N, m2->ld))
            return false;
        int maxc = *std::max_element(count.begin(), count.end());
        p.stream = 1;
        p.nmat = m2 ? 2 : 1;
        {
            // rows of the prologue operands resolved here (the kernel's row_ptr, on the host)
            auto row = [&](const VOperand& op, int64_t m, const void*& ptr, int64_t& st) {
                if (!op.fast_ok) return false;
                int64_t idx[VTC_MAX_RANK] = {};
                idx[0] = m;
                int pc = -1;
                const int64_t off = desc_eval(op.m, idx, &pc);
                if (pc < 0) return false;
                ptr = reinterpret_cast<const void*>(op.m.piece[pc].ptr + uint64_t(off) * 2);
                st = op.fast_stride[pc];
                return true;
            };
            bool ok = p.M <= 4;
            for (int64_t m = 0; ok && m < p.M; ++m) {
                ok = row(p.a, m, p.arow[m], p.sa[m]);
                if (ok && p.prologue == GemvPrologue::SiLUMul) ok = row(p.a2, m, p.a2row[m], p.sa2[m]);
            }
            if (ok && p.prologue == GemvPrologue::RMSNorm) ok = row(p.normw, 0, p.wrow, p.sw);
            p.rows_ok = ok ? 1 : 0;
        }
        p.n_mat[0] = p.N;
        if (m2) p.n_mat[1] = m2->N;
        p.strips0 = int32_t(strips0);
        p.stages = stages;
        p.grid = grid;
        p.max_contrib = maxc;
        p.a_tiles = a_tiles;
        p.b_static = (written_roots.count(b_root) || (m2 && written_roots.count(m2->root))) ? 0 : 1;
        p.pre_stages = 1;
        if (tun.gemv_pre >= 0) p.pre_stages = tun.gemv_pre;
        p.l2_prefetch = 0;
        if (tun.gemv_l2pf >= 0) p.l2_prefetch = tun.gemv_l2pf;
        p.work = static_cast<float*>(impl_->alloc(size_t(strips * maxc * p.M * COLS) * sizeof(float), false));
        p.counters = static_cast<unsigned*>(impl_->alloc(size_t(strips) * sizeof(unsigned), true));
        auto* dfirst = static_cast<int32_t*>(impl_->alloc(size_t(strips) * 4, false));
        auto* dcount = static_cast<int32_t*>(impl_->alloc(size_t(strips) * 4, false));
        if (!impl_->dry) {
            ck(cudaMemcpy(dfirst, first.data(), size_t(strips) * 4, cudaMemcpyHostToDevice), "H2D");
            ck(cudaMemcpy(dcount, count.data(), size_t(strips) * 4, cudaMemcpyHostToDevice), "H2D");
        }
        p.strip_first = dfirst;
        p.strip_count = dcount;
        return true;
    };

    // ---- elementwise / copy launches over an output shape ----
    // An EwSpec is a small program over up to EW_MAX_IN input maps.  A map with
    // more pieces than the descriptor holds is handled by one launch per piece
    // (or by bisecting the iteration box), each iterating over its own box.
    struct EwSpec {
        std::vector<const VMap*> ins;
        std::vector<EwInstr> prog;
        int result = 0;
        bool copy = false;
    };
    std::function<void(const std::string&, const EwSpec&, DType, const Index&, const VMap&, const Index&,
                       const Index&)>
        eltwise_box;
    eltwise_box = [&](const std::string& node, const EwSpec& spec, DType dt, const Index& shape, const VMap& out,
                      const Index& lo, const Index& hi) {
        auto L = std::make_unique<LaunchT<EwParams, launch_eltwise>>();
        L->node = node;
        L->kernel = spec.copy ? "gather_copy" : "eltwise";
        EwParams& p = L->p;
        std::memset(&p, 0, sizeof(p));
        int64_t es = dtype_size(dt);
        int rank = int(shape.size());
        Index ext(static_cast<size_t>(rank), 0);
        for (int i = 0; i < rank; ++i) ext[size_t(i)] = hi[size_t(i)] - lo[size_t(i)];
        int64_t vec = 16 / es;
        if (rank == 0 || ext.back() % vec != 0 || lo.back() % vec != 0) vec = 1;
        p.rank = rank;
        for (int i = 0; i < rank; ++i) {
            p.shape[i] = int32_t(ext[size_t(i)]);
            p.origin[i] = int32_t(lo[size_t(i)]);
        }
        p.vec = int32_t(vec);
        p.dt = kdt(dt);
        p.esize = int32_t(es);
        p.copy_only = spec.copy ? 1 : 0;
        p.nvec = volume(ext) / vec;
        p.nin = int32_t(spec.ins.size());
        p.nprog = int32_t(spec.prog.size());
        p.result = spec.result;
        for (size_t i = 0; i < spec.prog.size(); ++i) p.prog[i] = spec.prog[i];
        auto restrict_box = [&](const VMap& m) {
            std::vector<VPiece> ps;
            for (const auto& q : m.pieces()) {
                VPiece r = q;
                bool empty = false;
                for (int i = 0; i < rank; ++i) {
                    r.lo[size_t(i)] = std::max(q.lo[size_t(i)], lo[size_t(i)]);
                    r.hi[size_t(i)] = std::min(q.hi[size_t(i)], hi[size_t(i)]);
                    empty |= r.lo[size_t(i)] >= r.hi[size_t(i)];
                }
                if (empty) continue;
                r.off = restrict_to(q.off, r.lo, r.hi);
                ps.push_back(std::move(r));
            }
            return VMap(m.shape(), std::move(ps));
        };
        std::vector<const VMap*> maps{&out};
        for (auto* m : spec.ins) maps.push_back(m);
        for (size_t k = 0; k < maps.size(); ++k) {
            VMap rm = restrict_box(*maps[k]);
            VOperand op2{};
            try {
                op2.m = lower_map(rm, target);
            } catch (const UnsupportedError&) {
                // split the iteration box along the pieces of this map, or bisect it
                if (rm.pieces().size() > 1) {
                    for (const auto& q : rm.pieces()) eltwise_box(node, spec, dt, shape, out, q.lo, q.hi);
                    return;
                }
                int best = -1;
                int64_t bext = 1;
                for (int i = 0; i < rank; ++i)
                    if (ext[size_t(i)] > bext) {
                        bext = ext[size_t(i)];
                        best = i;
                    }
                if (best < 0) throw;
                Index h1 = hi, l2 = lo;
                h1[size_t(best)] = lo[size_t(best)] + bext / 2;
                l2[size_t(best)] = h1[size_t(best)];
                eltwise_box(node, spec, dt, shape, out, lo, h1);
                eltwise_box(node, spec, dt, shape, out, l2, hi);
                return;
            }
            finish_operand(op2, rank - 1, vec, es);
            (k == 0 ? p.out : p.in[k - 1]) = op2;
        }
        // streaming fast path: bf16, every operand a plain row-major buffer of the
        // box, and the program one op (GELU, residual adds) or SiLU(in0) * in1
        // (registers: inputs 0..nin-1, op s writes EW_MAX_IN + s; Add / Mul commute exactly)
        int pat = 0;
        const bool fast_ew = !tun.no_ew_fast;  // tests: generic interpreter everywhere
        if (fast_ew && dt == DType::BF16 && vec == 8 && !spec.copy) {
            const EwInstr* q = p.prog;
            if (p.nprog == 1 && p.result == q[0].dst && q[0].op != EwOp::Copy &&
                (p.nin == 1 ? q[0].a == 0 && (q[0].op == EwOp::SiLU || q[0].op == EwOp::GELU)
                            : p.nin == 2 && q[0].a + q[0].b == 1 && q[0].a != q[0].b &&
                                  (q[0].op == EwOp::Add || q[0].op == EwOp::Mul)))
                pat = 1;
            if (p.nprog == 2 && p.nin == 2 && q[0].op == EwOp::SiLU && q[0].a == 0 && q[1].op == EwOp::Mul &&
                p.result == q[1].dst &&
                ((q[1].a == q[0].dst && q[1].b == 1) || (q[1].b == q[0].dst && q[1].a == 1)))
                pat = 2;
        }
        // (in0 * in1) + (in2 * in3): the Q / K RoPE trees, without the register interpreter
        {
            const EwInstr* q = p.prog;
            const int r0 = EW_MAX_IN, r1 = EW_MAX_IN + 1;
            if (fast_ew && !spec.copy && p.nin == 4 && p.nprog == 3 && q[0].op == EwOp::Mul && q[0].a == 0 && q[0].b == 1 &&
                q[0].dst == r0 && q[1].op == EwOp::Mul && q[1].a == 2 && q[1].b == 3 && q[1].dst == r1 &&
                q[2].op == EwOp::Add && ((q[2].a == r0 && q[2].b == r1) || (q[2].a == r1 && q[2].b == r0)) &&
                p.result == q[2].dst)
                p.prog_pat = 3;
        }
        // affine operands (<= 2 pieces split along the last axis, vector-aligned): the
        // compact-parameter kernel, no per-element map evaluation (RoPE trees, views)
        {
            bool aff = !tun.no_ew_aff && vec * es == 16 && rank >= 1;
            for (int k = 0; k <= p.nin && aff; ++k) {
                const VOperand& op = k == 0 ? p.out : p.in[k - 1];
                const vtc_map& m = op.m;
                EwAff& A = p.affine[k];
                if (m.npieces < 1 || m.npieces > 2 || !op.vec_ok) {
                    aff = false;
                    break;
                }
                A.split = INT32_MAX;
                for (int q = 0; q < m.npieces && aff; ++q) {
                    const vtc_piece& pc = m.piece[q];
                    if (!pc.affine) aff = false;
                    for (int i = 0; i < rank - 1 && aff; ++i)
                        aff = pc.lo[i] <= p.origin[i] && pc.hi[i] >= p.origin[i] + p.shape[i];
                    if (!aff) break;
                    if (m.npieces == 2) {
                        const int lo_last = pc.lo[rank - 1] - p.origin[rank - 1];
                        if (q == 1) {
                            A.split = lo_last;
                            aff = lo_last % vec == 0 && m.piece[0].lo[rank - 1] <= p.origin[rank - 1] &&
                                  m.piece[0].hi[rank - 1] == pc.lo[rank - 1] &&
                                  pc.hi[rank - 1] >= p.origin[rank - 1] + p.shape[rank - 1];
                        }
                    }
                    // fold the iteration-box origin into the base: index I of the box = I + origin
                    int64_t off = pc.base;
                    for (int i = 0; i < rank; ++i) {
                        A.st[q][i] = pc.aff[i];
                        off += pc.aff[i] * p.origin[i];
                    }
                    A.base[q] = pc.ptr + uint64_t(off * es);
                }
            }
            p.aff = aff ? 1 : 0;
            if (aff && !spec.copy) L->kernel = "eltwise_aff";
        }
        bool flat = pat != 0;
        for (int i = 0; i < rank && flat; ++i) flat = p.origin[i] == 0;
        for (int k = 0; k <= p.nin && flat; ++k) {
            const vtc_map& m = k == 0 ? p.out.m : p.in[k - 1].m;
            flat = map_flat_linear(m, rank, p.shape) && (m.piece[0].base * es) % 16 == 0 && m.piece[0].ptr % 16 == 0;
        }
        p.flat = flat ? pat : 0;
        if (flat) L->kernel = "eltwise_flat";
        push(std::move(L));
    };
    auto eltwise = [&](const std::string& node, const EwSpec& spec, DType dt, const Index& shape, const VMap& out) {
        eltwise_box(node, spec, dt, shape, out, Index(shape.size(), 0), shape);
    };
    auto copy_spec = [](const VMap* src) {
        EwSpec sp;
        sp.ins = {src};
        sp.copy = true;
        return sp;
    };

    // A gather-copy that must not read what it writes: stage through scratch.
    auto copy_checked = [&](const std::string& node, DType dt, const Index& shape, const VMap& dst, const VMap& src) {
        auto td = targets_of(dst), ts = targets_of(src);
        bool hazard = false;
        for (const auto& t : td) hazard |= ts.count(t) > 0;
        if (!hazard) {
            eltwise(node, copy_spec(&src), dt, shape, dst);
            return;
        }
        // stage: src -> temp (identity) -> dst
        std::string tmp_id = "__stage_" + node + "_" + std::to_string(roots_.size());
        RootBuffer rb;
        rb.id = tmp_id;
        rb.dtype = dt;
        rb.shape = shape;
        rb.bytes = volume(shape) * dtype_size(dt);
        rb.ptr = impl_->alloc(size_t(rb.bytes), false);
        root_index_[tmp_id] = int(roots_.size());
        roots_.push_back(rb);
        auto tmp = std::make_shared<VMap>(VMap::identity(tmp_id, shape));
        eltwise(node, copy_spec(&src), dt, shape, *tmp);
        eltwise(node, copy_spec(tmp.get()), dt, shape, dst);
    };

    // ---- elementwise-tree fusion: a tree of Add/Mul/SiLU/GELU nodes whose
    //      internal tensors have a single consumer runs as one program ----
    auto is_ew = [](OpKind k) { return k == OpKind::Add || k == OpKind::Mul || k == OpKind::SiLU || k == OpKind::GELU; };
    auto ew_code = [](OpKind k) {
        return k == OpKind::Add ? EwOp::Add : k == OpKind::Mul ? EwOp::Mul : k == OpKind::SiLU ? EwOp::SiLU : EwOp::GELU;
    };
    // build the program for the tree rooted at `root`; members collects fused nodes
    std::function<bool(const OpNode&, EwSpec&, std::vector<std::string>&, std::vector<std::string>&, int&)> build_tree;
    build_tree = [&](const OpNode& n, EwSpec& sp, std::vector<std::string>& in_names, std::vector<std::string>& members,
                     int& reg) -> bool {
        std::vector<int> regs;
        for (const auto& t : n.inputs) {
            const OpNode* p = g_.producer(t);
            bool fuse = opt_.fuse && p && is_ew(p->kind) && g_.tensor(t).kind == TensorKind::Intermediate &&
                        g_.consumers(t).size() == 1 && g_.tensor(t).shape == g_.tensor(n.outputs[0]).shape;
            if (fuse) {
                int r = 0;
                if (!build_tree(*p, sp, in_names, members, r)) return false;
                regs.push_back(r);
            } else {
                auto it = std::find(in_names.begin(), in_names.end(), t);
                if (it != in_names.end()) {
                    regs.push_back(int(it - in_names.begin()));
                } else {
                    if (int(in_names.size()) >= EW_MAX_IN) return false;
                    in_names.push_back(t);
                    regs.push_back(int(in_names.size()) - 1);
                }
            }
        }
        if (int(sp.prog.size()) >= EW_MAX_PROG) return false;
        EwInstr ins{};
        ins.op = ew_code(n.kind);
        ins.a = int8_t(regs[0]);
        ins.b = int8_t(regs.size() > 1 ? regs[1] : regs[0]);
        ins.dst = int8_t(EW_MAX_IN + sp.prog.size());
        sp.prog.push_back(ins);
        members.push_back(n.id);
        reg = ins.dst;
        return true;
    };

    // ---- fusion pre-pass (graph structure only, so virtual and materialised
    //      plans fuse identically) ----
    struct GemvFusion {
        const OpNode* norm = nullptr;
        const OpNode* silu = nullptr;
        const OpNode* mul = nullptr;
        const OpNode* add = nullptr;
        const OpNode* view = nullptr;  // tensor-core residual: the last eliminated view between MatMul and Add
        bool perm = false;             // ... a row-permuting chain: output / residual rows host-resolved
    };
    std::map<std::string, GemvFusion> fusion;
    std::map<std::string, const OpNode*> hfuse;  // first MatMul -> its horizontally fused sibling
    std::map<std::string, const OpNode*> tc_hfuse;  // the same for the tcgen05 GEMM
    std::map<std::string, const OpNode*> tc_gelu;   // tcgen05 GEMM -> its GELU epilogue
    struct SwiGlu {
        const OpNode *gate, *up, *silu, *mul;
    };
    std::map<std::string, SwiGlu> tc_swiglu;  // launch node (earlier MatMul) -> the SwiGLU pair
    std::map<std::string, const OpNode*> skinny_norm;  // shallow-K GEMM -> the row norm its A producer computes
    std::set<std::string> hpartner;
    std::set<std::string> absorbed;
    std::map<std::string, int> topo_pos;
    for (size_t i = 0; i < g_.topo_order().size(); ++i) topo_pos[g_.nodes()[size_t(g_.topo_order()[i])].id] = int(i);
    auto only_consumer = [&](const std::string& t, const std::string& node) {
        auto cs = g_.consumers(t);
        return g_.tensor(t).kind == TensorKind::Intermediate && cs.size() == 1 && cs[0]->id == node;
    };
    // a sibling b absorbed into a's launch runs at a's topological position: a must
    // come first, everything b reads must be produced before a, and b's output must
    // be its own root (so no node between a and b writes or reads through it)
    auto absorbable_at = [&](const OpNode& a, const OpNode& b) {
        if (topo_pos.at(a.id) >= topo_pos.at(b.id)) return false;
        for (const auto& in : b.inputs) {
            const OpNode* pr = g_.producer(in);
            if (pr && topo_pos.at(pr->id) >= topo_pos.at(a.id)) return false;
            for (const auto& r : targets_of(map_of(in))) {
                const OpNode* pw = g_.producer(r);
                if (pw && topo_pos.at(pw->id) >= topo_pos.at(a.id)) return false;
            }
        }
        return map_of(b.outputs[0]).is_identity_of(b.outputs[0]);
    };
    auto gemv_eligible = [&](const OpNode& n) {
        if (n.kind != OpKind::MatMul || !opt_.use_gemv) return false;
        const TensorSpec& A = g_.tensor(n.inputs[0]);
        const TensorSpec& B = g_.tensor(n.inputs[1]);
        if (A.dtype != DType::BF16 || A.shape.size() != 2 || A.shape[0] > 16) return false;
        if (B.shape[1] % 8 != 0) return false;
        const VMap& bm = map_of(n.inputs[1]);
        if (bm.pieces().size() != 1) return false;
        const VPiece& p = bm.pieces()[0];
        auto sk = VMap::tile_stride(p, 0, B.shape[0]);
        auto sn = VMap::tile_stride(p, 1, B.shape[1]);
        if (!sk || !sn || *sn != 1) return false;
        for (const auto& tm : p.off.t)
            if (tm.a->kind != AtomKind::Axis) return false;
        if (p.off.c0 % 8 != 0 || *sk % 8 != 0) return false;
        return true;
    };
    // tcgen05 GEMM: bf16 2-D MatMul with M > 16, B physical (single affine piece, N unit
    // stride), A a single affine piece with unit stride along K (TMA-readable)
    auto affine2d = [&](const VMap& m, int64_t& ld, int64_t& c0) -> bool {
        if (m.pieces().size() != 1) return false;
        const VPiece& pc = m.pieces()[0];
        for (const auto& tm : pc.off.t)
            if (tm.a->kind != AtomKind::Axis) return false;
        auto s0 = VMap::tile_stride(pc, 0, m.shape()[0]);
        auto s1 = VMap::tile_stride(pc, 1, m.shape()[1]);
        if (!s0 || !s1 || *s1 != 1) return false;
        ld = *s0;
        c0 = pc.off.c0;
        return ld % 8 == 0 && c0 % 8 == 0;
    };
    auto tc_eligible = [&](const OpNode& n) {
        if (n.kind != OpKind::MatMul || !opt_.use_tc || gemv_eligible(n)) return false;
        const TensorSpec& A = g_.tensor(n.inputs[0]);
        const TensorSpec& B = g_.tensor(n.inputs[1]);
        if (A.dtype != DType::BF16 || A.shape.size() != 2 || A.shape[0] <= 16) return false;
        int64_t ld, c0;
        if (!affine2d(map_of(n.inputs[1]), ld, c0) || B.shape[1] % 8 != 0 || A.shape[1] % 8 != 0) return false;
        // A: TMA-readable through its map (tile-aligned mixed-radix digits)
        vtc_map am{};
        try {
            am = lower_map(map_of(n.inputs[0]), target);
        } catch (const UnsupportedError&) {
            return false;
        }
        GemmTcParams probe{};
        int64_t dims[5], strides[5];
        const void* base = nullptr;
        if (gemm_tc_a_dims(am, A.shape[0], A.shape[1], probe, dims, strides, &base)) return true;
        // gather fallback: rows located through the map, unit stride + 16-B aligned along K,
        // and every row inside one piece (a row is gathered from its base address)
        VOperand op{};
        op.m = am;
        finish_operand(op, 1, 64, 2);
        std::vector<int64_t> segs;
        return op.vec_ok != 0 && k_segments(am, A.shape[1], segs);
    };
    if (opt_.fuse) {
        for (const auto& n : g_.nodes()) {
            const bool tc = tc_eligible(n);
            if (!gemv_eligible(n) && !tc) continue;
            GemvFusion f;
            const OpNode* pa = tc ? nullptr : g_.producer(n.inputs[0]);  // TMA-fed A: no prologue fusion
            if (pa && pa->kind == OpKind::RMSNorm && g_.tensor(n.inputs[0]).kind == TensorKind::Intermediate &&
                g_.tensor(pa->inputs[0]).shape.size() == 2) {
                bool all = true;
                for (const OpNode* c : g_.consumers(n.inputs[0])) all = all && gemv_eligible(*c) && c->inputs[0] == n.inputs[0];
                if (all) f.norm = pa;
            } else if (pa && pa->kind == OpKind::Mul && only_consumer(n.inputs[0], n.id)) {
                for (int side = 0; side < 2 && !f.silu; ++side) {
                    const OpNode* ps = g_.producer(pa->inputs[size_t(side)]);
                    if (ps && ps->kind == OpKind::SiLU && only_consumer(pa->inputs[size_t(side)], pa->id) &&
                        pa->inputs[0] != pa->inputs[1]) {
                        f.silu = ps;
                        f.mul = pa;
                    }
                }
            }
            auto cs = g_.consumers(n.outputs[0]);
            if (only_consumer(n.outputs[0], cs.empty() ? "" : cs[0]->id) && cs[0]->kind == OpKind::Add &&
                cs[0]->inputs[0] != cs[0]->inputs[1]) {
                const OpNode* ad = cs[0];
                const std::string& other = ad->inputs[0] == n.outputs[0] ? ad->inputs[1] : ad->inputs[0];
                const OpNode* po = g_.producer(other);
                if (!po || topo_pos[po->id] < topo_pos[n.id]) f.add = ad;
            } else if (tc && !tun.no_tc_epi && !cs.empty()) {
                // MatMul -> virtual data-movement chain -> Add.  One Reshape keeping the last axis
                // (Swin's MLP reshape): the residual is fused through [M, N] views of the Add's
                // operands.  A longer chain that permutes whole rows (Swin's window reverse + roll
                // after proj): the persistent shallow-K GEMM stores each product row at its
                // host-resolved output row and reads the residual row there (f.perm)
                std::string t = n.outputs[0];
                const OpNode* last = nullptr;
                int len = 0;
                for (;;) {
                    auto c = g_.consumers(t);
                    if (c.empty() || !only_consumer(t, c[0]->id) || !is_data_movement(*c[0]) || !elim.count(c[0]->id) ||
                        c[0]->outputs.size() != 1)
                        break;
                    last = c[0];
                    t = c[0]->outputs[0];
                    ++len;
                }
                auto cs2 = last ? g_.consumers(t) : std::vector<const OpNode*>{};
                if (last && !cs2.empty() && only_consumer(t, cs2[0]->id) && cs2[0]->kind == OpKind::Add &&
                    cs2[0]->inputs[0] != cs2[0]->inputs[1] && g_.tensor(t).shape.back() == g_.tensor(n.outputs[0]).shape.back()) {
                    const OpNode* ad = cs2[0];
                    const std::string& other = ad->inputs[0] == t ? ad->inputs[1] : ad->inputs[0];
                    const OpNode* po = g_.producer(other);
                    const bool reshape1 = len == 1 && last->kind == OpKind::Reshape;
                    const Index& as = g_.tensor(n.inputs[0]).shape;
                    const int64_t N = g_.tensor(n.inputs[1]).shape[1];
                    const bool skinny_shape = !tun.no_skinny && as[0] >= 8192 && as[1] <= 512 && N <= 1024 && as[1] % 16 == 0 &&
                                              N % 16 == 0;
                    if ((!po || topo_pos[po->id] < topo_pos[n.id]) && (reshape1 || skinny_shape)) {
                        f.add = ad;
                        f.view = last;
                        f.perm = !reshape1;
                    }
                }
            }
            if (f.norm || f.silu || f.add) fusion[n.id] = f;
        }
        // horizontal fusion: two streamed GEMVs reading the same A with the same
        // prologue (gate / up) run as one launch over both weight matrices
        if (opt_.gemv_stream) {
            std::vector<const OpNode*> cands;
            for (const auto& n : g_.nodes())
                if (gemv_eligible(n) && g_.tensor(n.inputs[0]).shape[0] <= 4) cands.push_back(&n);
            for (size_t i = 0; i < cands.size(); ++i) {
                const OpNode* a = cands[i];
                if (hfuse.count(a->id) || hpartner.count(a->id)) continue;
                for (size_t j = i + 1; j < cands.size(); ++j) {
                    const OpNode* b = cands[j];
                    if (hfuse.count(b->id) || hpartner.count(b->id) || b->inputs[0] != a->inputs[0]) continue;
                    auto fa = fusion.find(a->id), fb = fusion.find(b->id);
                    const OpNode* na = fa != fusion.end() ? fa->second.norm : nullptr;
                    const OpNode* nb = fb != fusion.end() ? fb->second.norm : nullptr;
                    bool other = (fa != fusion.end() && (fa->second.silu || fa->second.add)) ||
                                 (fb != fusion.end() && (fb->second.silu || fb->second.add));
                    if (other || na != nb || !absorbable_at(*a, *b)) continue;
                    hfuse[a->id] = b;
                    hpartner.insert(b->id);
                    break;
                }
            }
            for (const auto& id : hpartner) absorbed.insert(id);
        }
        // activation epilogues on the tensor-core GEMM (VTC_NO_TC_EPI=1: off):
        //  * MatMul -> GELU (its only consumer): the GEMM stores GELU(round(acc));
        //  * SwiGLU: gate = A.Wg, up = A.Wu, SiLU(gate) * up, each intermediate with one
        //    consumer: one launch whose tiles hold 128 columns of both products and store
        //    only the Mul's output (gate / up are never written)
        if (!tun.no_tc_epi) {
            for (const auto& n : g_.nodes()) {
                if (!tc_eligible(n) || fusion.count(n.id) || absorbed.count(n.id)) continue;
                const std::string& o = n.outputs[0];
                auto cs = g_.consumers(o);
                if (!only_consumer(o, cs.empty() ? "" : cs[0]->id)) continue;
                const OpNode* c = cs[0];
                if (c->kind == OpKind::GELU && g_.tensor(c->outputs[0]).shape == g_.tensor(o).shape) {
                    tc_gelu[n.id] = c;
                    absorbed.insert(c->id);
                    continue;
                }
                if (c->kind != OpKind::SiLU) continue;
                const std::string& so = c->outputs[0];
                auto ms = g_.consumers(so);
                if (!only_consumer(so, ms.empty() ? "" : ms[0]->id) || ms[0]->kind != OpKind::Mul) continue;
                const OpNode* mul = ms[0];
                const std::string& other = mul->inputs[0] == so ? mul->inputs[1] : mul->inputs[0];
                if (other == so) continue;
                const OpNode* up = g_.producer(other);
                if (!up || up == &n || !tc_eligible(*up) || fusion.count(up->id) || absorbed.count(up->id) ||
                    !only_consumer(other, mul->id) || up->inputs[0] != n.inputs[0] ||
                    g_.tensor(up->inputs[1]).shape != g_.tensor(n.inputs[1]).shape ||
                    g_.tensor(mul->outputs[0]).shape != g_.tensor(o).shape ||
                    !operand(map_of(mul->outputs[0]), 1, 128, 2).fast_ok)
                    continue;
                // the launch runs at the earlier of the two MatMuls' positions; the later one's
                // inputs must be ready there
                const OpNode* first = topo_pos.at(n.id) < topo_pos.at(up->id) ? &n : up;
                const OpNode* second = first == &n ? up : &n;
                bool ready = true;
                for (const auto& in : second->inputs) {
                    const OpNode* pr = g_.producer(in);
                    if (pr && topo_pos.at(pr->id) >= topo_pos.at(first->id)) ready = false;
                    for (const auto& r : targets_of(map_of(in))) {
                        const OpNode* pw = g_.producer(r);
                        if (pw && topo_pos.at(pw->id) >= topo_pos.at(first->id)) ready = false;
                    }
                }
                if (!ready) continue;
                tc_swiglu[first->id] = SwiGlu{&n, up, c, mul};
                absorbed.insert(second->id);
                absorbed.insert(c->id);
                absorbed.insert(mul->id);
            }
        }
        // the same on the tensor cores: sibling MatMuls reading the same A with plain
        // single-piece outputs (gate / up at decode batch) run as one launch, so the
        // second does not wait for the first to complete (VTC_NO_TC_HFUSE=1: off)
        if (!tun.no_tc_hfuse) {
            std::vector<const OpNode*> cands;
            for (const auto& n : g_.nodes())
                if (tc_eligible(n) && !fusion.count(n.id) && !absorbed.count(n.id) && map_of(n.outputs[0]).pieces().size() == 1)
                    cands.push_back(&n);
            for (size_t i = 0; i < cands.size(); ++i) {
                const OpNode* a = cands[i];
                if (tc_hfuse.count(a->id) || absorbed.count(a->id)) continue;
                for (size_t j = i + 1; j < cands.size(); ++j) {
                    const OpNode* b = cands[j];
                    if (absorbed.count(b->id) || tc_hfuse.count(b->id) || b->inputs[0] != a->inputs[0] ||
                        g_.tensor(b->inputs[1]).shape[0] != g_.tensor(a->inputs[1]).shape[0])
                        continue;
                    if (!absorbable_at(*a, *b)) continue;
                    tc_hfuse[a->id] = b;
                    absorbed.insert(b->id);
                    break;
                }
            }
        }
        // a LayerNorm / RMSNorm over K <= 128 whose output only a shallow-K GEMM reads (through
        // virtual views: Swin's LN1 -> roll -> window partition -> QKV, LN2 -> reshape -> fc1) is
        // computed by that GEMM's A producers from the norm's input rows (VTC_NO_SKINNY_NORM=1: off)
        if (!tun.no_skinny && !tun.no_skinny_norm && !tun.no_tc_epi) {
            const auto gouts = g_.graph_outputs();
            const std::set<std::string> gout(gouts.begin(), gouts.end());
            for (const auto& n : g_.nodes()) {
                // not under a GELU epilogue: 8 epilogue warps leave it issue-bound (Swin fc1 178 -> 190 us)
                if (!tc_eligible(n) || absorbed.count(n.id) || tc_swiglu.count(n.id) || tc_hfuse.count(n.id) ||
                    tc_gelu.count(n.id))
                    continue;
                const Index& as = g_.tensor(n.inputs[0]).shape;
                const int64_t M = as[0], K = as[1], N = g_.tensor(n.inputs[1]).shape[1];
                if (!(M >= 8192 && K <= 128 && K % 32 == 0 && N % 16 == 0 && N <= 1024)) continue;
                const auto tg = targets_of(map_of(n.inputs[0]));
                if (tg.size() != 1) continue;
                const std::string R = *tg.begin();
                const OpNode* L = g_.producer(R);
                if (!L || (L->kind != OpKind::LayerNorm && L->kind != OpKind::RMSNorm) || gout.count(R) ||
                    g_.tensor(R).dtype != DType::BF16 || g_.tensor(R).shape.back() != K ||
                    g_.tensor(L->inputs[0]).shape.back() != K)
                    continue;
                bool only = true;  // every reader of R is n, through eliminated views
                for (const auto& [tid, m] : ptg_.resolved) {
                    const auto mt = m.targets();
                    if (std::find(mt.begin(), mt.end(), R) == mt.end()) continue;
                    if (gout.count(tid)) only = false;
                    for (const OpNode* c : g_.consumers(tid))
                        if (!(is_data_movement(*c) && elim.count(c->id)) && !(c == &n && tid == n.inputs[0])) only = false;
                }
                // the norm now runs at n's position: nothing in between may write its inputs
                std::set<std::string> lin;
                for (const auto& in : L->inputs)
                    for (const auto& r : targets_of(map_of(in))) lin.insert(r);
                for (const auto& m2 : g_.nodes()) {
                    const int pm = topo_pos.at(m2.id);
                    if (pm <= topo_pos.at(L->id) || pm >= topo_pos.at(n.id)) continue;
                    for (const auto& o : m2.outputs)
                        for (const auto& r : targets_of(map_of(o))) only = only && !lin.count(r);
                }
                if (!only) continue;
                skinny_norm[n.id] = L;
                absorbed.insert(L->id);
            }
        }
        // a norm is absorbed only if every consumer MatMul fused it
        for (auto& [id, f] : fusion) {
            if (f.norm) absorbed.insert(f.norm->id);
            if (f.silu) {
                absorbed.insert(f.silu->id);
                absorbed.insert(f.mul->id);
            }
            if (f.add) absorbed.insert(f.add->id);
        }
    }

    // elementwise trees: roots in reverse topological order; a root whose tree
    // does not fit one program runs alone and its children become roots
    struct EwTree {
        EwSpec spec;
        std::vector<std::string> in_names, members;
        int reg = 0;
    };
    std::map<std::string, EwTree> ew_trees;
    {
        std::set<std::string> in_tree;
        auto fusable_up = [&](const OpNode& n) {
            // n's output feeds a single elementwise consumer of the same shape
            const std::string& o = n.outputs[0];
            auto cs = g_.consumers(o);
            return opt_.fuse && g_.tensor(o).kind == TensorKind::Intermediate && cs.size() == 1 &&
                   is_ew(cs[0]->kind) && !absorbed.count(cs[0]->id) && g_.tensor(cs[0]->outputs[0]).shape == g_.tensor(o).shape;
        };
        std::function<void(const OpNode&)> make_root = [&](const OpNode& n) {
            EwTree t;
            if (build_tree(n, t.spec, t.in_names, t.members, t.reg)) {
                for (const auto& m : t.members) in_tree.insert(m);
                ew_trees[n.id] = std::move(t);
                return;
            }
            // fallback: n alone; each fusable child roots its own tree
            EwTree single;
            for (const auto& in : n.inputs) single.in_names.push_back(in);
            EwInstr ins{};
            ins.op = ew_code(n.kind);
            ins.a = 0;
            ins.b = int8_t(n.inputs.size() > 1 ? 1 : 0);
            ins.dst = int8_t(EW_MAX_IN);
            single.spec.prog = {ins};
            single.reg = EW_MAX_IN;
            single.members = {n.id};
            in_tree.insert(n.id);
            ew_trees[n.id] = std::move(single);
            for (const auto& in : n.inputs) {
                const OpNode* pr = g_.producer(in);
                if (pr && is_ew(pr->kind) && !absorbed.count(pr->id) && !in_tree.count(pr->id)) make_root(*pr);
            }
        };
        const auto& order = g_.topo_order();
        for (auto it = order.rbegin(); it != order.rend(); ++it) {
            const OpNode& n = g_.nodes()[size_t(*it)];
            if (!is_ew(n.kind) || absorbed.count(n.id) || in_tree.count(n.id)) continue;
            if (fusable_up(n)) continue;  // will be reached from its consumer's tree
            make_root(n);
        }
        // anything fusable_up whose consumer did not take it (should not happen) runs alone
        for (const auto& n : g_.nodes())
            if (is_ew(n.kind) && !absorbed.count(n.id) && !in_tree.count(n.id)) make_root(n);
        for (const auto& [root, t] : ew_trees)
            for (const auto& m : t.members)
                if (m != root) absorbed.insert(m);
    }

    // ---- elementwise trees folded into a streamed GEMV's epilogue: trees whose
    //      operands are strip-local views of the GEMV output (e.g. Q/K RoPE with
    //      its rotate-half) are evaluated by the GEMV's last-CTA epilogue; the
    //      intermediate roots they would have read are never written ----
    std::map<std::string, std::vector<std::string>> epi_trees;  // gemv node -> tree roots
    std::map<std::string, std::set<std::string>> epi_roots;     // gemv node -> exclusive roots
    if (opt_.fuse && opt_.gemv_stream && !tun.no_epi_fusion) {
        std::set<std::string> graph_io;
        for (const auto& t : g_.graph_inputs()) graph_io.insert(t);
        for (const auto& t : g_.graph_outputs()) graph_io.insert(t);
        std::map<std::string, std::string> tree_of_input;  // tensor -> tree root (first)
        for (const auto& [root, t] : ew_trees)
            for (const auto& in : t.in_names) tree_of_input.emplace(in, root);
        for (const auto& n : g_.nodes()) {
            if (!gemv_eligible(n) || g_.tensor(n.inputs[0]).shape[0] > 4 || hfuse.count(n.id) || hpartner.count(n.id))
                continue;
            auto fit = fusion.find(n.id);
            if (fit != fusion.end() && fit->second.add) continue;
            const std::string& C = n.outputs[0];
            if (g_.tensor(C).kind != TensorKind::Intermediate) continue;
            std::set<std::string> excl;
            for (const auto& r : targets_of(map_of(C)))
                if (!graph_io.count(r) && r != C) excl.insert(r);
            // an exclusive root is read only through views that feed ew trees, and
            // written only by this GEMV
            std::set<std::string> trees;
            for (const auto& [tid, m] : ptg_.resolved) {
                if (tid == C) continue;
                bool hits = false;
                for (const auto& r : m.targets()) hits |= excl.count(r) > 0;
                if (!hits) continue;
                auto it = tree_of_input.find(tid);
                bool consumed_by_tree = it != tree_of_input.end();
                bool other_consumer = false;
                for (const OpNode* c : g_.consumers(tid)) {
                    if (is_data_movement(*c) && elim.count(c->id)) continue;
                    bool in_tree = false;
                    for (const auto& [root, t] : ew_trees)
                        if (std::find(t.members.begin(), t.members.end(), c->id) != t.members.end()) in_tree = true;
                    if (!in_tree) other_consumer = true;
                }
                if (!consumed_by_tree && !other_consumer) continue;  // a pure intermediate view
                if (!consumed_by_tree || other_consumer) {
                    for (const auto& r : m.targets()) excl.erase(r);
                    continue;
                }
                trees.insert(it->second);
            }
            for (const auto& r : excl)
                for (const OpNode* c : g_.consumers(r))
                    if (!(is_data_movement(*c) && elim.count(c->id))) excl.erase(r);
            if (excl.empty() || trees.empty() || trees.size() > size_t(EPI_MAX_TREES)) continue;
            bool ok = true;
            for (const auto& root : trees) {
                const EwTree& t = ew_trees.at(root);
                if (t.in_names.size() > size_t(EPI_MAX_IN) || absorbed.count(root)) ok = false;
                for (const auto& in : t.in_names) {  // each operand: all C-derived or none
                    int hit = 0, miss = 0;
                    for (const auto& r : map_of(in).targets()) (excl.count(r) ? hit : miss)++;
                    if (hit && miss) ok = false;
                }
            }
            if (!ok) continue;
            epi_trees[n.id] = std::vector<std::string>(trees.begin(), trees.end());
            epi_roots[n.id] = excl;
            for (const auto& root : trees)
                for (const auto& m : ew_trees.at(root).members) absorbed.insert(m);
        }
    }

    // ---- elementwise trees folded into a tensor-core GEMM's epilogue: trees whose
    //      operands are views of the GEMM output C (same row, columns of one N tile
    //      per head: e.g. the prefill Q / K RoPE trees over the QKV projection) or
    //      row-linear external tensors (the cos / sin tables).  The columns of C that
    //      only these trees read are not stored (VTC_NO_TC_EPI=1: off) ----
    struct TcTrees {
        std::vector<GemmTree> trees;
        std::vector<std::string> roots;
        int64_t skip_lo = 0, skip_hi = 0;
    };
    std::map<std::string, TcTrees> tc_trees;
    const bool dbg_fuse = tun.debug_fusion;
    // (VTC_NO_TC_TREES=1: off.)  With one CTA per SM the per-row epilogue's table loads
    // serialised (QKV + trees 2.53 ms vs 1.64 + 0.67 ms at C5); with two 128-row CTAs per SM
    // the co-resident CTA's mainloop hides them (1.98 ms vs 1.48 + 0.65 ms)
    if (opt_.fuse && !tun.no_tc_trees && !tun.no_tc_epi) {
        const auto gouts = g_.graph_outputs();
        const std::set<std::string> graph_out(gouts.begin(), gouts.end());
        for (const auto& n : g_.nodes()) {
            if (!tc_eligible(n) || absorbed.count(n.id) || fusion.count(n.id) || tc_gelu.count(n.id) ||
                tc_swiglu.count(n.id) || tc_hfuse.count(n.id))
                continue;
            const std::string& C = n.outputs[0];
            if (g_.tensor(C).kind != TensorKind::Intermediate) continue;
            const int64_t M = g_.tensor(C).shape[0], N = g_.tensor(C).shape[1];
            // decode batch (one 128-row tile, K splits over the weight stream): the trees in the
            // split-K epilogue measured slower than the separate eltwise launch (C3 QKV 58.7 us
            // last-split, 41.1 us cooperative, vs 25.0 + 7.7 us); VTC_TREE_COOP=1 fuses them anyway
            if (M <= 128 && !tun.tree_coop) continue;
            int64_t ldc = 0, cc0 = 0;
            std::string R;
            // C's roots the trees may read by column: root index -> (row stride, column-0 offset)
            std::map<int, std::pair<int64_t, int64_t>> croots;
            std::set<std::string> cnames;
            if (affine2d(map_of(C), ldc, cc0)) {
                R = map_of(C).pieces()[0].target;
            } else {
                // C split over roots (decode QKV: Q and K columns into two intermediates, V straight
                // into the cache row): the trees read the row-affine pieces on intermediate roots
                for (const VPiece& pc : map_of(C).pieces()) {
                    bool axes = pc.lo[0] == 0 && pc.hi[0] == M && g_.tensor(pc.target).kind == TensorKind::Intermediate;
                    for (const auto& tm : pc.off.t) axes = axes && tm.a->kind == AtomKind::Axis;
                    if (!axes) continue;
                    auto s0 = VMap::tile_stride(pc, 0, M), s1 = VMap::tile_stride(pc, 1, pc.hi[1] - pc.lo[1]);
                    if (!s0 || !s1 || *s1 != 1 || *s0 % 8 || pc.off.c0 % 8) continue;
                    const int ti = target(pc.target).index;
                    if (croots.count(ti)) {  // one root in two pieces: not resolved here
                        R.clear();
                        break;
                    }
                    croots[ti] = {*s0, pc.off.c0};
                    cnames.insert(pc.target);
                    if (R.empty()) R = pc.target;
                }
                if (R.empty()) {
                    if (dbg_fuse) fprintf(stderr, "[vtc fuse] %s: output map has no row-affine intermediate piece\n", n.id.c_str());
                    continue;
                }
            }
            const int Ridx = target(R).index;
            if (croots.empty()) {
                croots[Ridx] = {ldc, cc0};
                cnames.insert(R);
            }
            const int pos_n = topo_pos.at(n.id);
            TcTrees tt;
            std::vector<std::string> roots_fused;
            std::vector<char> mark(size_t(N), 0);  // C columns read by the fused trees
            for (const auto& [root, t] : ew_trees) {
                if (absorbed.count(root) || int(tt.trees.size()) == GEMM_MAX_TREES) continue;
                bool hits = false;
                for (const auto& in : t.in_names)
                    for (const auto& r : targets_of(map_of(in))) hits |= cnames.count(r) > 0;
                if (!hits) continue;
                const OpNode* rn = g_.node(root);
                const std::string& O = rn->outputs[0];
                const Index& shp = g_.tensor(O).shape;
                const int r = int(shp.size());
                if (r < 3 || g_.tensor(O).dtype != DType::BF16 || graph_out.count(O)) continue;
                int64_t rows = 1;
                for (int d = 0; d + 2 < r; ++d) rows *= shp[size_t(d)];
                const int64_t nh = shp[size_t(r - 2)], hd = shp[size_t(r - 1)];
                if (rows != M || hd % 16 != 0 || hd > 256) continue;
                // the tree now runs at n's position: its external inputs must be ready there,
                // and nothing between n and the tree may touch its output's roots
                bool ok = true;
                for (const auto& in : t.in_names) {
                    bool fromc = false;
                    for (const auto& r2 : targets_of(map_of(in))) fromc |= cnames.count(r2) > 0;
                    if (fromc) continue;
                    const OpNode* pr = g_.producer(in);  // an eliminated view runs nothing: its roots count
                    if (pr && !(is_data_movement(*pr) && elim.count(pr->id)) && topo_pos.at(pr->id) >= pos_n) ok = false;
                    for (const auto& r2 : targets_of(map_of(in))) {
                        const OpNode* pw = g_.producer(r2);
                        if (pw && topo_pos.at(pw->id) >= pos_n) ok = false;
                    }
                }
                const auto oroots = targets_of(map_of(O));
                for (const auto& m2 : g_.nodes()) {
                    const int pm = topo_pos.at(m2.id);
                    if (pm <= pos_n || pm >= topo_pos.at(root)) continue;
                    if (std::find(t.members.begin(), t.members.end(), m2.id) != t.members.end()) continue;
                    for (const auto* lst : {&m2.inputs, &m2.outputs})
                        for (const auto& tn : *lst)
                            for (const auto& r2 : targets_of(map_of(tn))) ok = ok && !oroots.count(r2);
                }
                if (!ok) {
                    if (dbg_fuse) fprintf(stderr, "[vtc fuse] %s: tree %s not movable to the GEMM\n", n.id.c_str(), root.c_str());
                    continue;
                }
                // operands as row-linear pieces: element (m, h, i) at base + rs*m + sh*h + i
                GemmTree T{};
                T.nin = int32_t(t.in_names.size());
                T.nprog = int32_t(t.spec.prog.size());
                T.result = t.reg;
                T.hd = int32_t(hd);
                T.nh = int32_t(nh);
                for (size_t k = 0; k < t.spec.prog.size(); ++k) T.prog[k] = t.spec.prog[k];
                {
                    const EwInstr* q = T.prog;
                    const int r0 = EW_MAX_IN, r1 = EW_MAX_IN + 1;
                    if (T.nin == 4 && T.nprog == 3 && q[0].op == EwOp::Mul && q[0].a == 0 && q[0].b == 1 && q[0].dst == r0 &&
                        q[1].op == EwOp::Mul && q[1].a == 2 && q[1].b == 3 && q[1].dst == r1 && q[2].op == EwOp::Add &&
                        ((q[2].a == r0 && q[2].b == r1) || (q[2].a == r1 && q[2].b == r0)) && T.result == q[2].dst)
                        T.pat = 3;
                }
                int64_t csh = INT64_MIN, clo = INT64_MAX, chi = INT64_MIN;
                auto lower_op = [&](const std::string& name, GemmTreeOp& op, bool is_out) -> bool {
                    vtc_map lm;
                    try {
                        lm = lower_map(map_of(name), target);
                    } catch (const UnsupportedError&) {
                        return false;
                    }
                    if (lm.npieces < 1 || lm.npieces > 2) return false;
                    op.split = lm.npieces == 2 ? lm.piece[1].lo[r - 1] : int32_t(hd);
                    int fromc = -1;
                    for (int q = 0; q < lm.npieces; ++q) {
                        const vtc_piece& pc = lm.piece[q];
                        if (!pc.affine) return false;
                        for (int d = 0; d + 1 < r; ++d)
                            if (pc.lo[d] > 0 || pc.hi[d] < shp[size_t(d)]) return false;
                        if (lm.npieces == 2) {
                            if (q == 0 && (pc.lo[r - 1] > 0 || pc.hi[r - 1] != lm.piece[1].lo[r - 1])) return false;
                            if (q == 1 && (pc.hi[r - 1] < hd || pc.lo[r - 1] % 16 != 0)) return false;
                        } else if (pc.lo[r - 1] > 0 || pc.hi[r - 1] < hd) {
                            return false;
                        }
                        if (pc.aff[r - 1] != 1) return false;
                        if (shp[size_t(r - 3)] == 1 && rows > 1) return false;  // the row stride is not the innermost's
                        const int64_t rs = pc.aff[r - 3];
                        int64_t want = rs;
                        for (int d = r - 3; d >= 0; --d) {
                            if (shp[size_t(d)] > 1 && pc.aff[d] != want) return false;  // unit axes: any stride
                            want *= shp[size_t(d)];
                        }
                        const auto cr = croots.find(pc.target);
                        const bool c_side = cr != croots.end();
                        if (fromc >= 0 && fromc != int(c_side)) return false;
                        fromc = int(c_side);
                        op.rs[q] = rs;
                        op.sh[q] = pc.aff[r - 2];
                        if (c_side) {
                            if (is_out || rs != cr->second.first) return false;
                            op.ccol[q] = pc.base - cr->second.second;
                            const int64_t lo_i = q == 0 ? 0 : op.split, hi_i = q == 0 && lm.npieces == 2 ? op.split : hd;
                            if (csh != INT64_MIN && csh != op.sh[q]) return false;
                            csh = op.sh[q];
                            clo = std::min(clo, op.ccol[q] + lo_i);
                            chi = std::max(chi, op.ccol[q] + hi_i - 1);
                        } else {
                            if (pc.target == Ridx) return false;
                            if ((pc.base * 2) % 16 || rs % 8 || op.sh[q] % 8) return false;
                            op.base[q] = pc.ptr + uint64_t(pc.base * 2);
                            // dynamic position: only the output may address a cache, inside the
                            // position's row (its bases are patched per step); inputs stay static
                            if (const DynRoot* dr = impl_->dyn_on ? impl_->dyn.find(pc.target) : nullptr) {
                                int64_t lo = 0, hi = 0;
                                const int64_t row = dr->rs * dr->es;
                                if (!is_out || !DynCtx::piece_range(lm, q, lo, hi) || lo < impl_->dyn.p0 * dr->rs ||
                                    hi >= (impl_->dyn.p0 + 1) * dr->rs || (T.out_dyn && T.out_dyn != row))
                                    return false;
                                T.out_dyn = row;
                            }
                        }
                    }
                    if (lm.npieces == 1) {
                        op.rs[1] = op.rs[0];
                        op.sh[1] = op.sh[0];
                        op.ccol[1] = op.ccol[0];
                        op.base[1] = op.base[0];
                    }
                    op.from_c = fromc;
                    return true;
                };
                ok = lower_op(O, T.op[0], true);
                for (size_t k = 0; k < t.in_names.size() && ok; ++k) {
                    ok = lower_op(t.in_names[k], T.op[1 + k], false);
                    if (!ok && dbg_fuse) fprintf(stderr, "[vtc fuse] %s: tree %s operand %s not row-linear\n", n.id.c_str(), root.c_str(), t.in_names[k].c_str());
                }
                if (!ok || csh == INT64_MIN) {
                    if (dbg_fuse) fprintf(stderr, "[vtc fuse] %s: tree %s output / C operands not row-linear\n", n.id.c_str(), root.c_str());
                    continue;
                }
                for (int64_t h = 0; h < nh && ok; ++h) {
                    const int64_t a = clo + csh * h, b = chi + csh * h;
                    ok = a >= 0 && b < N && a / 128 == b / 128;
                }
                if (!ok) {
                    if (dbg_fuse) fprintf(stderr, "[vtc fuse] %s: tree %s head columns cross a 128-column tile\n", n.id.c_str(), root.c_str());
                    continue;
                }
                T.c_lo = clo;
                T.c_sh = csh;
                for (int k = 0; k < T.nin; ++k) {
                    const GemmTreeOp& op = T.op[1 + k];
                    if (!op.from_c) continue;
                    for (int64_t h = 0; h < nh; ++h)
                        for (int64_t i = 0; i < hd; ++i) {
                            const int q = i >= op.split ? 1 : 0;
                            mark[size_t(op.ccol[q] + op.sh[q] * h + i)] = 1;
                        }
                }
                tt.trees.push_back(T);
                roots_fused.push_back(root);
            }
            if (tt.trees.empty()) continue;
            // columns read only by the trees: the longest marked run, 16-aligned inward;
            // dropped if any other reader of C's root may read inside it
            int64_t best_lo = 0, best_hi = 0;
            for (int64_t c = 0; c < N;) {
                if (!mark[size_t(c)]) {
                    ++c;
                    continue;
                }
                int64_t e = c;
                while (e < N && mark[size_t(e)]) ++e;
                if (e - c > best_hi - best_lo) {
                    best_lo = c;
                    best_hi = e;
                }
                c = e;
            }
            best_lo = (best_lo + 15) / 16 * 16;
            best_hi = best_hi / 16 * 16;
            std::set<std::string> members;
            for (const auto& root : roots_fused)
                for (const auto& m2 : ew_trees.at(root).members) members.insert(m2);
            bool clean = best_hi > best_lo && croots.size() == 1 && !graph_out.count(R) && ldc == N && cc0 == 0;
            for (const auto& [tid, m] : ptg_.resolved) {
                if (!clean) break;
                const auto mt = m.targets();
                if (std::find(mt.begin(), mt.end(), R) == mt.end() || tid == C) continue;
                bool read = graph_out.count(tid) > 0;
                for (const OpNode* c : g_.consumers(tid))
                    if (!(is_data_movement(*c) && elim.count(c->id)) && !members.count(c->id)) read = true;
                if (!read) continue;
                vtc_map lm;
                try {
                    lm = lower_map(m, target);
                } catch (const UnsupportedError&) {
                    clean = false;
                    break;
                }
                for (int q = 0; q < lm.npieces && clean; ++q) {
                    const vtc_piece& pc = lm.piece[q];
                    if (pc.target != Ridx) continue;
                    if (!pc.affine) {
                        clean = false;
                        break;
                    }
                    int64_t lo = pc.base, hi = pc.base;
                    for (int d = 0; d < lm.rank; ++d) {
                        const int64_t st = pc.aff[d];
                        if (st % ldc == 0) continue;
                        const int64_t x0 = st * pc.lo[d], x1 = st * (pc.hi[d] - 1);
                        lo += std::min(x0, x1);
                        hi += std::max(x0, x1);
                    }
                    if (lo < 0 || lo / ldc != hi / ldc) {
                        clean = false;
                        break;
                    }
                    const int64_t clo2 = lo % ldc, chi2 = hi % ldc;
                    if (chi2 >= best_lo && clo2 < best_hi) clean = false;
                }
            }
            if (clean) {
                tt.skip_lo = best_lo;
                tt.skip_hi = best_hi;
            }
            for (const auto& root : roots_fused) absorbed.insert(ew_trees.at(root).members.begin(), ew_trees.at(root).members.end());
            tt.roots = roots_fused;
            tc_trees[n.id] = std::move(tt);
        }
    }

    for (int ni : g_.topo_order()) {
        const OpNode& n = g_.nodes()[size_t(ni)];
        if (absorbed.count(n.id)) continue;
        const TensorSpec& o0 = g_.tensor(n.outputs[0]);
        DType dt = g_.tensor(n.inputs[0]).dtype;
        int64_t es = dtype_size(dt);

        if (is_data_movement(n)) {
            if (elim.count(n.id)) continue;  // eliminated: no kernel
            for (const auto& o : n.outputs) {
                VMap src = gather_map(n, o, g_).compose(lookup);
                const VMap& dst = map_of(o);
                const Index& shp = g_.tensor(o).shape;
                // Only what moves is copied (the estimate's `moved`, proj/src/cost_model.cpp:150-165):
                // pieces whose source already is where the output lives (a ScatterND whose output
                // aliases its data in place, rule (i)) need no copy.
                std::vector<const VPiece*> moving;
                for (const auto& q : src.pieces()) {
                    int64_t vol = 1;
                    for (size_t a = 0; a < q.lo.size(); ++a) vol *= q.hi[a] - q.lo[a];
                    if (VMap(src.shape(), {q}).agree_volume(dst) != vol) moving.push_back(&q);
                }
                if (moving.size() == src.pieces().size()) {
                    copy_checked(n.id, dt, shp, dst, src);
                    continue;
                }
                for (const VPiece* q : moving) {
                    auto part = std::make_shared<VMap>(src.shape(), std::vector<VPiece>{*q});
                    bool hazard = false;
                    for (const auto& t : targets_of(dst)) hazard |= targets_of(*part).count(t) > 0;
                    if (hazard) throw UnsupportedError("in-place copy of " + n.id + " reads what it writes");
                    const size_t before = infos_.size();
                    eltwise_box(n.id, copy_spec(part.get()), dt, shp, dst, q->lo, q->hi);
                    int64_t vol = 1;
                    for (size_t a = 0; a < q->lo.size(); ++a) vol *= q->hi[a] - q->lo[a];
                    for (size_t i = before; i < infos_.size(); ++i)  // the moved region, read + written
                        infos_[i].bytes = 2 * vol * es / int64_t(infos_.size() - before);
                }
            }
            continue;
        }

        // hazard: a compute node writing a root it also reads (other than identical elementwise maps)
        for (const auto& o : n.outputs)
            for (const auto& in : n.inputs) {
                auto to = targets_of(map_of(o)), ti = targets_of(map_of(in));
                bool clash = false;
                for (const auto& t : to) clash |= ti.count(t) > 0;
                bool same_elementwise = (n.kind == OpKind::Add || n.kind == OpKind::Mul || n.kind == OpKind::SiLU ||
                                         n.kind == OpKind::GELU) && map_of(o).equivalent(map_of(in));
                if (clash && !same_elementwise && !map_of(o).images_disjoint(map_of(in)))
                    throw UnsupportedError("node " + n.id + " writes a root it reads (" + o + " / " + in + ")");
            }

        switch (n.kind) {
            case OpKind::Add:
            case OpKind::Mul:
            case OpKind::SiLU:
            case OpKind::GELU: {
                EwTree& t = ew_trees.at(n.id);
                EwSpec sp = t.spec;
                for (const auto& name : t.in_names) sp.ins.push_back(&map_of(name));
                sp.result = t.reg;
                std::string label;
                for (const auto& m : t.members) label += (label.empty() ? "" : "+") + m;
                eltwise(label, sp, dt, o0.shape, map_of(n.outputs[0]));
                break;
            }
            case OpKind::AllReduce: {
                // NCCL on contiguous views of roots (the tensor-parallel partial sums)
                auto contiguous = [&](const VMap& m) -> const char* {
                    if (m.pieces().size() != 1) return nullptr;
                    const VPiece& pc = m.pieces()[0];
                    for (const auto& tm : pc.off.t)
                        if (tm.a->kind != AtomKind::Axis) return nullptr;
                    int64_t want = 1;
                    for (int a = int(m.rank()) - 1; a >= 0; --a) {
                        auto st = VMap::tile_stride(pc, a, m.shape()[size_t(a)]);
                        if (!st || (m.shape()[size_t(a)] > 1 && *st != want)) return nullptr;
                        want *= m.shape()[size_t(a)];
                    }
                    return reinterpret_cast<const char*>(target(pc.target).ptr) + pc.off.c0 * es;
                };
                const char* src = contiguous(map_of(n.inputs[0]));
                const char* dst = contiguous(map_of(n.outputs[0]));
                if ((!src || !dst) && !impl_->dry)
                    throw UnsupportedError("AllReduce " + n.id + " needs contiguous input / output views");
                auto L = std::make_unique<AllReduceLaunch>();
                L->node = n.id;
                L->kernel = "allreduce_nccl";
                L->src = src;
                L->dst = const_cast<char*>(dst);
                L->count = size_t(volume(o0.shape));
                L->bytes = L->count * size_t(es);
                L->dt = dt == DType::BF16 ? ncclBfloat16 : dt == DType::F32 ? ncclFloat32 : dt == DType::F64 ? ncclFloat64 : ncclInt64;
                L->comm = &impl_->comm;
                push(std::move(L));
                break;
            }
            case OpKind::RMSNorm:
            case OpKind::LayerNorm:
            case OpKind::Softmax: {
                if (dt == DType::I64) throw UnsupportedError(std::string(to_string(n.kind)) + " on i64");
                auto L = std::make_unique<LaunchT<RowParams, launch_rowop>>();
                L->node = n.id;
                L->kernel = "rowop";
                RowParams& p = L->p;
                std::memset(&p, 0, sizeof(p));
                const Index& sh = o0.shape;
                int rank = int(sh.size());
                p.rank = rank;
                for (int i = 0; i < rank; ++i) p.shape[i] = int32_t(sh[size_t(i)]);
                p.D = sh.back();
                p.rows = volume(sh) / p.D;
                p.dt = kdt(dt);
                p.op = n.kind == OpKind::RMSNorm ? RowOp::RMSNorm : n.kind == OpKind::LayerNorm ? RowOp::LayerNorm : RowOp::Softmax;
                if (const auto* na = std::get_if<NormAttrs>(&n.attrs)) p.eps = float(na->eps);
                p.x = operand(map_of(n.inputs[0]), rank - 1, p.D, es);
                p.out = operand(map_of(n.outputs[0]), rank - 1, p.D, es);
                if (n.kind != OpKind::Softmax) p.w = operand(map_of(n.inputs[1]), 0, p.D, es);
                if (n.kind == OpKind::LayerNorm) p.bias = operand(map_of(n.inputs[2]), 0, p.D, es);
                p.linear = map_flat_linear(p.x.m, rank, p.shape) && map_flat_linear(p.out.m, rank, p.shape) ? 1 : 0;
                if (tun.no_row_fast) p.linear = 0;  // tests: map-evaluating row kernels
                push(std::move(L));
                break;
            }
            case OpKind::MatMul: {
                const TensorSpec& A = g_.tensor(n.inputs[0]);
                const TensorSpec& B = g_.tensor(n.inputs[1]);
                int rank = int(A.shape.size());
                int64_t M = A.shape[size_t(rank - 2)], K = A.shape[size_t(rank - 1)], N = B.shape[size_t(rank - 1)];
                if (gemv_eligible(n)) {
                    auto L = std::make_unique<LaunchT<GemvParams, launch_gemv_any>>();
                    L->node = n.id;
                    L->kernel = "gemv_bf16";
                    GemvParams& p = L->p;
                    std::memset(&p, 0, sizeof(p));
                    p.M = M;
                    p.N = N;
                    p.K = K;
                    GemvFusion f;
                    auto fit = fusion.find(n.id);
                    if (fit != fusion.end()) f = fit->second;
                    if (f.norm) {
                        p.prologue = GemvPrologue::RMSNorm;
                        p.a = operand(map_of(f.norm->inputs[0]), 1, K, es);
                        p.normw = operand(map_of(f.norm->inputs[1]), 0, K, es);
                        p.eps = float(std::get<NormAttrs>(f.norm->attrs).eps);
                        L->node = f.norm->id + "+" + n.id;
                    } else if (f.silu) {
                        p.prologue = GemvPrologue::SiLUMul;
                        const std::string& sg = f.silu->outputs[0];
                        const std::string& other = f.mul->inputs[0] == sg ? f.mul->inputs[1] : f.mul->inputs[0];
                        p.a = operand(map_of(f.silu->inputs[0]), 1, K, es);
                        p.a2 = operand(map_of(other), 1, K, es);
                        L->node = f.silu->id + "+" + f.mul->id + "+" + n.id;
                    } else {
                        p.a = operand(map_of(n.inputs[0]), 1, K, es);
                    }
                    if (f.add) {
                        const std::string& other =
                            f.add->inputs[0] == n.outputs[0] ? f.add->inputs[1] : f.add->inputs[0];
                        p.has_res = 1;
                        p.res = operand(map_of(other), 1, 256, es);
                        p.c = operand(map_of(f.add->outputs[0]), 1, 256, es);
                        L->node += "+" + f.add->id;
                    } else {
                        p.c = operand(map_of(n.outputs[0]), 1, 256, es);
                    }
                    const VMap& bm = map_of(n.inputs[1]);
                    const VPiece& bp = bm.pieces()[0];
                    TargetInfo bt = target(bp.target);
                    p.b_base = reinterpret_cast<const char*>(bt.ptr) + bp.off.c0 * es;
                    p.b_sk = *VMap::tile_stride(bp, 0, K);
                    // persistent TMA-streamed variant: one CTA per SM, balanced (strip, k-tile) ranges
                    SecondMat m2;
                    const SecondMat* m2p = nullptr;
                    auto hf = hfuse.find(n.id);
                    if (hf != hfuse.end()) {
                        const OpNode& n2 = *hf->second;
                        const VPiece& bp2 = map_of(n2.inputs[1]).pieces()[0];
                        TargetInfo bt2 = target(bp2.target);
                        m2.ptr = reinterpret_cast<uint64_t>(reinterpret_cast<const char*>(bt2.ptr) + bp2.off.c0 * es);
                        m2.N = g_.tensor(n2.inputs[1]).shape[1];
                        m2.ld = *VMap::tile_stride(bp2, 0, K);
                        m2.root = bp2.target;
                        m2p = &m2;
                        p.c2 = operand(map_of(n2.outputs[0]), 1, 256, es);
                        L->node += "+" + n2.id;
                    }
                    auto ef = epi_trees.find(n.id);
                    if (ef != epi_trees.end()) {
                        // the fused-epilogue table: one entry per output element (m, col)
                        const std::string& C = n.outputs[0];
                        const VMap& cm = map_of(C);
                        const std::set<std::string>& excl = epi_roots.at(n.id);
                        std::map<std::pair<std::string, int64_t>, int64_t> inv;  // (root, offset) -> m * N + col
                        for (int64_t m = 0; m < M; ++m)
                            for (int64_t c = 0; c < N; ++c) {
                                auto te = cm.eval(Index{m, c});
                                if (excl.count(te.first)) inv[te] = m * N + c;
                            }
                        std::vector<EpiEntry> tab(size_t(M * N));
                        for (auto& x : tab) {
                            std::memset(&x, 0, sizeof(x));
                            x.tree = -1;
                        }
                        auto addr_of = [&](const std::pair<std::string, int64_t>& te) -> uint64_t {
                            return target(te.first).ptr + uint64_t(te.second * es);
                        };
                        for (size_t ti = 0; ti < ef->second.size(); ++ti) {
                            const std::string& root = ef->second[ti];
                            const EwTree& t = ew_trees.at(root);
                            const OpNode* rn = g_.node(root);
                            const VMap& om = map_of(rn->outputs[0]);
                            EpiTree& et = p.epi_tree[ti];
                            et.nin = int32_t(t.in_names.size());
                            et.nprog = int32_t(t.spec.prog.size());
                            et.result = t.reg;
                            for (size_t k2 = 0; k2 < t.spec.prog.size(); ++k2) et.prog[k2] = t.spec.prog[k2];
                            const Index& shp = g_.tensor(rn->outputs[0]).shape;
                            Index idx(shp.size(), 0);
                            for (int64_t f = 0; f < volume(shp); ++f) {
                                int64_t r = f;
                                for (int a = int(shp.size()) - 1; a >= 0; --a) {
                                    idx[size_t(a)] = r % shp[size_t(a)];
                                    r /= shp[size_t(a)];
                                }
                                EpiEntry ent{};
                                ent.tree = int32_t(ti);
                                const auto oe = om.eval(idx);
                                ent.out = addr_of(oe);
                                if (impl_->dyn_on) {
                                    const DynCtx& dc = impl_->dyn;
                                    const DynRoot* r = dc.find(root_index_.at(oe.first));
                                    if (r && oe.second >= dc.p0 * r->rs && oe.second < (dc.p0 + 1) * r->rs) {
                                        ent.cmask |= EPI_DYN_OUT;
                                        if (p.epi_dyn && p.epi_dyn != r->rs * r->es)
                                            throw UnsupportedError("dynamic position: caches with different row sizes in one epilogue");
                                        p.epi_dyn = int32_t(r->rs * r->es);
                                    } else if (r) {
                                        throw UnsupportedError("dynamic position: fused epilogue writes a cache outside the row");
                                    }
                                }
                                int64_t anchor = -1;
                                for (size_t j = 0; j < t.in_names.size(); ++j) {
                                    auto te = map_of(t.in_names[j]).eval(idx);
                                    if (excl.count(te.first)) {
                                        auto it = inv.find(te);
                                        if (it == inv.end()) throw UnsupportedError("fused epilogue: operand outside the GEMV output");
                                        if (anchor < 0) anchor = it->second;
                                        if (it->second / N != anchor / N ||
                                            (it->second % N) / GEMV_STREAM_COLS != (anchor % N) / GEMV_STREAM_COLS)
                                            throw UnsupportedError("fused epilogue: operand crosses a 256-column strip");
                                        ent.in[j] = uint64_t(it->second % N);
                                        ent.cmask |= 1u << j;
                                    } else {
                                        ent.in[j] = addr_of(te);
                                        if (impl_->dyn_on && impl_->dyn.find(root_index_.at(te.first)))
                                            throw UnsupportedError("dynamic position: fused epilogue reads a cache");
                                    }
                                }
                                if (anchor < 0 || tab[size_t(anchor)].tree >= 0)
                                    throw UnsupportedError("fused epilogue: tree element without a unique anchor");
                                tab[size_t(anchor)] = ent;
                            }
                            for (const auto& m : t.members) L->node += "+" + m;
                        }
                        auto* dtab = static_cast<EpiEntry*>(impl_->alloc(tab.size() * sizeof(EpiEntry), false));
                        if (!impl_->dry)
                            ck(cudaMemcpy(dtab, tab.data(), tab.size() * sizeof(EpiEntry), cudaMemcpyHostToDevice), "H2D(epi)");
                        p.has_epi = 1;
                        p.epi = dtab;
                    }
                    if (M <= 4 && opt_.gemv_stream && stream_gemv(p, reinterpret_cast<uint64_t>(p.b_base), bp.target, m2p)) {
                        L->kernel = "gemv_stream_bf16";
                        push(std::move(L));
                        break;
                    }
                    if (p.has_epi) throw UnsupportedError("fused GEMV epilogue " + L->node + " needs the streaming kernel");
                    if (m2p) throw UnsupportedError("horizontally fused GEMV " + L->node + " needs the streaming kernel");
                    // grid: 256-column strips x K splits, ~3 CTAs per SM
                    int64_t ntiles = (N + 255) / 256;
                    int64_t want = (148 * 3 + ntiles - 1) / ntiles;
                    int64_t maxsplit = std::max<int64_t>(1, K / 64);
                    int64_t ks = std::min(want, maxsplit);
                    int64_t kchunk = ((K + ks - 1) / ks + 63) / 64 * 64;
                    int64_t smem_cap = 48 * 1024 / (4 * std::max<int64_t>(M, 1));
                    if (kchunk > smem_cap) kchunk = smem_cap / 64 * 64;
                    ks = (K + kchunk - 1) / kchunk;
                    p.ksplit = int32_t(ks);
                    p.kchunk = int32_t(kchunk);
                    if (ks > 1) {
                        p.work = static_cast<float*>(impl_->alloc(size_t(ks * M * N) * sizeof(float), false));
                        p.counters = static_cast<unsigned*>(impl_->alloc(size_t(ntiles) * sizeof(unsigned), true));
                    }
                    push(std::move(L));
                    break;
                }
                if (tc_eligible(n)) {
                    auto T = std::make_unique<LaunchT<GemmTcParams, launch_gemm_tc>>();
                    T->node = n.id;
                    T->kernel = "gemm_tc_bf16";
                    GemmTcParams& p = T->p;
                    std::memset(&p, 0, sizeof(p));
                    p.M = M;
                    p.N = N;
                    p.K = K;
                    GemvFusion f;
                    auto fit = fusion.find(n.id);
                    if (fit != fusion.end()) f = fit->second;
                    auto gl = tc_gelu.find(n.id);
                    auto sw = tc_swiglu.find(n.id);
                    const std::string& cout = f.add ? f.add->outputs[0]
                                              : gl != tc_gelu.end() ? gl->second->outputs[0]
                                              : sw != tc_swiglu.end() ? sw->second.mul->outputs[0]
                                                                      : n.outputs[0];
                    // the residual Add's operands as [M, N] (a Reshape between MatMul and Add)
                    std::deque<VMap> views;
                    auto mn = [&](const std::string& t) -> const VMap& {
                        if (!f.view || g_.tensor(t).shape == Index{M, N}) return map_of(t);
                        const VMap v = VMap::affine(Index{M, N}, Index{N, 1}, 0, t);
                        views.push_back(v.compose([&](const std::string& x) -> const VMap* {
                            return map_of(x).is_identity_of(x) ? nullptr : &map_of(x);
                        }));
                        return views.back();
                    };
                    const std::string& f_in = f.view ? f.view->outputs[0] : n.outputs[0];  // the Add's MatMul-side input
                    // shallow K, narrow N, many rows (Swin's projections): the persistent kernel with
                    // the weight resident in shared memory (VTC_NO_SKINNY=1: off)
                    if (sw == tc_swiglu.end() && !tc_trees.count(n.id) && !tc_hfuse.count(n.id) && M >= 8192 && K <= 512 &&
                        N <= 1024 && K % 16 == 0 && N % 16 == 0 && !tun.no_skinny) {
                        auto S = std::make_unique<LaunchT<SkinnyParams, launch_gemm_skinny>>();
                        SkinnyParams& q = S->p;
                        std::memset(&q, 0, sizeof(q));
                        q.M = M;
                        q.N = N;
                        q.K = K;
                        q.epi = gl != tc_gelu.end() ? 1 : 0;
                        q.sms = impl_->dry ? 148 : device_sms();
                        int optin = 232448;
                        if (!impl_->dry) {
                            int dev = 0;
                            cudaGetDevice(&dev);
                            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
                        }
                        bool sk = skinny_plan(q, optin - 2048);
                        // weights: one affine piece, rows 16-byte aligned
                        int64_t ldw = 0, cw = 0;
                        sk = sk && affine2d(map_of(n.inputs[1]), ldw, cw);
                        if (sk) {
                            const VMap& wm = map_of(n.inputs[1]);
                            q.w = reinterpret_cast<const char*>(target(wm.pieces()[0].target).ptr) + cw * es;
                            q.ldw = ldw;
                            const OpNode* wp = g_.producer(wm.pieces()[0].target);
                            q.b_static = wp == nullptr && g_.producer(n.inputs[1]) == nullptr;
                            sk = (reinterpret_cast<uintptr_t>(q.w) % 16) == 0 && ldw % 8 == 0;
                        }
                        // rows of a 2-D operand: affine (base, ld) or resolved per row on the host
                        auto rows_of = [&](const VMap& m, int64_t cols, uint64_t& base, int64_t& ld,
                                           const uint64_t*& table, const char* what) -> bool {
                            int64_t l = 0, c0 = 0;
                            if (affine2d(m, l, c0)) {
                                base = target(m.pieces()[0].target).ptr + uint64_t(c0 * es);
                                ld = l;
                                return base % 16 == 0 && l % 8 == 0;
                            }
                            VOperand op = operand(m, 1, cols, es);
                            if (!op.vec_ok) return false;
                            for (int pi = 0; pi < op.m.npieces; ++pi)
                                if (op.m.piece[pi].lo[1] > 0 || op.m.piece[pi].hi[1] < m.shape()[1]) return false;
                            if (impl_->dry) return true;
                            const int64_t rows = m.shape()[0];
                            std::vector<uint64_t> tab(static_cast<size_t>(rows));
                            int64_t idx[VTC_MAX_RANK] = {};
                            for (int64_t r2 = 0; r2 < rows; ++r2) {
                                idx[0] = r2;
                                int pc = -1;
                                const int64_t off = desc_eval(op.m, idx, &pc);
                                if (pc < 0) return false;
                                tab[size_t(r2)] = op.m.piece[pc].ptr + uint64_t(off) * es;
                                if (tab[size_t(r2)] % 16) return false;
                            }
                            auto* d = static_cast<uint64_t*>(impl_->alloc(tab.size() * 8, false));
                            ck(cudaMemcpy(d, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice), what);
                            table = d;
                            return true;
                        };
                        if (sk && f.perm) {
                            // residual behind a row-permuting view chain: product row m goes to the Add's
                            // output row r with pu[r, :] = C[m, :], and reads the residual row r there
                            const std::string& other = f.add->inputs[0] == f_in ? f.add->inputs[1] : f.add->inputs[0];
                            q.has_res = 1;
                            if (!impl_->dry) {
                                const int64_t R = volume(g_.tensor(cout).shape) / N;
                                auto rowview = [&](const std::string& t) {
                                    return lower_map(VMap::affine(Index{R, N}, Index{N, 1}, 0, t)
                                                         .compose([&](const std::string& x) -> const VMap* {
                                                             return map_of(x).is_identity_of(x) ? nullptr : &map_of(x);
                                                         }),
                                                     target);
                                };
                                const vtc_map pv = rowview(f_in), yv = rowview(cout), xv = rowview(other);
                                // product row m and view row r meet where both land in the same root
                                // element (either side may be the virtual one)
                                const vtc_map cv = lower_map(map_of(n.outputs[0]), target);
                                std::vector<uint64_t> ct(static_cast<size_t>(M), 0), rt(static_cast<size_t>(M), 0);
                                auto row_key = [&](const vtc_map& mp, int64_t row, uint64_t& key) {
                                    int64_t ix[VTC_MAX_RANK] = {};
                                    ix[0] = row;
                                    int pa = -1, pb = -1;
                                    const int64_t a = desc_eval(mp, ix, &pa);
                                    ix[1] = N - 1;
                                    const int64_t b = desc_eval(mp, ix, &pb);
                                    if (pa < 0 || pb != pa || b != a + N - 1 || a < 0 || a >= (int64_t(1) << 47)) return false;
                                    key = (uint64_t(mp.piece[pa].target) << 48) | uint64_t(a);
                                    return true;
                                };
                                std::unordered_map<uint64_t, int64_t> view_row;
                                view_row.reserve(size_t(R) * 2);
                                for (int64_t r = 0; r < R && sk; ++r) {
                                    uint64_t key = 0;
                                    sk = row_key(pv, r, key) && view_row.emplace(key, r).second;
                                }
                                std::vector<char> used(static_cast<size_t>(R), 0);
                                int64_t idx[VTC_MAX_RANK] = {};
                                for (int64_t m = 0; m < M && sk; ++m) {
                                    uint64_t key = 0;
                                    sk = row_key(cv, m, key);
                                    auto it = sk ? view_row.find(key) : view_row.end();
                                    sk = sk && it != view_row.end() && !used[size_t(it->second)];
                                    if (!sk) break;
                                    const int64_t r = it->second;
                                    used[size_t(r)] = 1;
                                    idx[0] = r;
                                    idx[1] = 0;
                                    int py = -1, px = -1;
                                    const int64_t oy = desc_eval(yv, idx, &py), ox = desc_eval(xv, idx, &px);
                                    sk = py >= 0 && px >= 0;
                                    if (!sk) break;
                                    ct[size_t(m)] = yv.piece[py].ptr + uint64_t(oy) * es;
                                    rt[size_t(m)] = xv.piece[px].ptr + uint64_t(ox) * es;
                                    sk = ct[size_t(m)] % 16 == 0 && rt[size_t(m)] % 16 == 0;
                                }
                                for (int64_t m = 0; m < M && sk; ++m) sk = ct[size_t(m)] != 0;  // a permutation
                                if (sk) {
                                    auto* dc = static_cast<uint64_t*>(impl_->alloc(size_t(M) * 8, false));
                                    auto* dr = static_cast<uint64_t*>(impl_->alloc(size_t(M) * 8, false));
                                    ck(cudaMemcpy(dc, ct.data(), size_t(M) * 8, cudaMemcpyHostToDevice), "H2D(skinny perm rows)");
                                    ck(cudaMemcpy(dr, rt.data(), size_t(M) * 8, cudaMemcpyHostToDevice), "H2D(skinny perm rows)");
                                    q.c_rows = dc;
                                    q.r_rows = dr;
                                }
                            }
                        } else {
                            sk = sk && rows_of(mn(cout), N, q.c_base, q.c_ld, q.c_rows, "H2D(skinny c_rows)");
                            if (sk && f.add) {
                                const std::string& other = f.add->inputs[0] == f_in ? f.add->inputs[1] : f.add->inputs[0];
                                q.has_res = 1;
                                sk = rows_of(mn(other), N, q.r_base, q.r_ld, q.r_rows, "H2D(skinny r_rows)");
                            }
                        }
                        auto sn = skinny_norm.find(n.id);
                        if (sk && sn != skinny_norm.end()) {
                            // A = norm(x rows): the producers read x's row behind each A row
                            const OpNode& L = *sn->second;
                            q.a_norm = L.kind == OpKind::LayerNorm ? 1 : 2;
                            q.eps = float(std::get<NormAttrs>(L.attrs).eps);
                            q.a_gather = 1;
                            bool vec_ok = true;
                            auto vec_ptr = [&](const std::string& t) -> const void* {
                                const VMap& m = map_of(t);
                                auto st = m.pieces().size() == 1 ? VMap::tile_stride(m.pieces()[0], 0, K) : std::nullopt;
                                if (!st || *st != 1) {
                                    vec_ok = false;
                                    return nullptr;
                                }
                                return reinterpret_cast<const char*>(target(m.pieces()[0].target).ptr) + m.pieces()[0].off.c0 * es;
                            };
                            q.norm_w = vec_ptr(L.inputs[1]);
                            q.norm_b = L.kind == OpKind::LayerNorm ? vec_ptr(L.inputs[2]) : nullptr;
                            sk = vec_ok;
                            if (sk && !impl_->dry) {
                                const std::string& R = L.outputs[0];
                                const int64_t xrows = volume(g_.tensor(L.inputs[0]).shape) / K;
                                const VMap xv = VMap::affine(Index{xrows, K}, Index{K, 1}, 0, L.inputs[0])
                                                    .compose([&](const std::string& x) -> const VMap* {
                                                        return map_of(x).is_identity_of(x) ? nullptr : &map_of(x);
                                                    });
                                const vtc_map xl = lower_map(xv, target);
                                const vtc_map al = lower_map(map_of(n.inputs[0]), target);
                                const int rid = target(R).index;
                                std::vector<uint64_t> tab(static_cast<size_t>(M));
                                int64_t idx[VTC_MAX_RANK] = {};
                                for (int64_t m = 0; m < M && sk; ++m) {
                                    idx[0] = m;
                                    idx[1] = 0;
                                    int pc = -1;
                                    const int64_t off = desc_eval(al, idx, &pc);
                                    sk = pc >= 0 && al.piece[pc].target == rid && off % K == 0;
                                    if (!sk) break;
                                    idx[0] = off / K;
                                    const int64_t xo = desc_eval(xl, idx, &pc);
                                    sk = pc >= 0;
                                    if (sk) tab[size_t(m)] = xl.piece[pc].ptr + uint64_t(xo) * es;
                                    sk = sk && tab[size_t(m)] % 16 == 0;
                                }
                                if (sk) {
                                    auto* d = static_cast<uint64_t*>(impl_->alloc(tab.size() * 8, false));
                                    ck(cudaMemcpy(d, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice), "H2D(skinny norm rows)");
                                    q.a_rows = d;
                                }
                            }
                            if (!sk) throw UnsupportedError("gemm_skinny: fused " + L.id + " rows not resolvable for " + n.id);
                            S->node = L.id + "+" + T->node;
                        } else if (sk) {
                            const VMap& am = map_of(n.inputs[0]);
                            int64_t lda = 0, ca = 0;
                            if (affine2d(am, lda, ca)) {
                                const char* ab = reinterpret_cast<const char*>(target(am.pieces()[0].target).ptr) + ca * es;
                                sk = impl_->dry || skinny_encode_a(q, ab, lda);
                            } else {
                                uint64_t abase = 0;
                                int64_t ald = 0;
                                const uint64_t* at = nullptr;
                                q.a_gather = 1;
                                // A rows: the K axis contiguous inside one piece per row
                                VOperand op = operand(am, 1, 64, es);
                                std::vector<int64_t> segs;
                                sk = op.vec_ok && k_segments(op.m, K, segs) && segs.size() == 2;
                                sk = sk && rows_of(am, K, abase, ald, at, "H2D(skinny a_rows)") && (impl_->dry || at != nullptr);
                                sk = sk && q.slots >= q.kt + 3;  // the gather keeps 3 k-tiles in flight
                                q.a_rows = at;
                            }
                        }
                        if (!sk && (sn != skinny_norm.end() || f.perm))
                            throw UnsupportedError("gemm_skinny: " + n.id + " with a fused norm / permuted residual is not launchable");
                        if (sk) {
                            S->node = (sn != skinny_norm.end() ? sn->second->id + "+" : std::string()) + T->node +
                                      (f.add ? "+" + f.add->id : "") + (gl != tc_gelu.end() ? "+" + gl->second->id : "");
                            S->kernel = "gemm_skinny_bf16";
                            push(std::move(S));
                            break;
                        }
                    }
                    bool ok = true;
                    if (sw != tc_swiglu.end()) {
                        // 256-column B stages: 128 columns of W_gate then the same 128 of W_up
                        p.epi = GEMM_EPI_SWIGLU;
                        p.bn = 256;
                        p.c = operand(map_of(cout), 1, 128, es);
                        ok = p.c.fast_ok != 0;
                    } else {
                        if (gl != tc_gelu.end()) p.epi = GEMM_EPI_GELU;
                        // small M: 128-column tiles so the K split (and its reduction) stays shallow
                        // (256-column tiles with deeper splits measured slower at C3: 675 vs 563 us)
                        p.bn = M <= 128 ? 128 : 256;
                        p.c = operand(mn(cout), 1, p.bn, es);
                        if (!p.c.fast_ok || N % 256 != 0) {
                            p.bn = 128;
                            p.c = operand(mn(cout), 1, p.bn, es);
                        }
                        ok = p.c.fast_ok != 0;
                    }
                    if (f.add) {
                        const std::string& other = f.add->inputs[0] == f_in ? f.add->inputs[1] : f.add->inputs[0];
                        p.has_res = 1;
                        p.res = operand(mn(other), 1, p.bn, es);
                        ok = ok && p.res.fast_ok;
                        T->node += "+" + f.add->id;
                    }
                    // B: the weights (SwiGLU: the gate's; the up weights follow as B2)
                    const OpNode& nbw = sw != tc_swiglu.end() ? *sw->second.gate : n;
                    int64_t ldb, cb;
                    affine2d(map_of(nbw.inputs[1]), ldb, cb);
                    const VMap& bmm = map_of(nbw.inputs[1]);
                    const char* bbase = reinterpret_cast<const char*>(target(bmm.pieces()[0].target).ptr) + cb * es;
                    int64_t adims[5], astr[5];
                    const void* abase = nullptr;
                    const vtc_map alow = lower_map(map_of(n.inputs[0]), target);
                    if (ok && !gemm_tc_a_dims(alow, M, K, p, adims, astr, &abase)) {
                        // A through 16-byte cp.async gathers (row bases from its map)
                        p.a = operand(map_of(n.inputs[0]), 1, 64, es);
                        std::vector<int64_t> segs;
                        ok = p.a.vec_ok != 0 && k_segments(p.a.m, K, segs);
                        p.a_gather = 1;
                        p.a_ndims = 2;  // the (unused) A tensor map: a dummy over B
                        adims[0] = K;
                        adims[1] = 1;
                        astr[1] = K;
                        abase = bbase;
                        for (int j = 0; j < 5; ++j) {
                            p.a_axis[j] = j == 0 ? 1 : 0;
                            p.a_div[j] = 1;
                            p.a_mod[j] = 0;
                        }
                        if (ok) T->kernel = "gemm_tc_bf16_gather";
                        if (ok && p.bn == 128 && N > 128 && p.epi != GEMM_EPI_SWIGLU) {
                            // gathered A is re-gathered for every N tile: 256-wide tiles (a
                            // partial last one) halve that (Swin QKV N = 288: 218 -> 180 us)
                            VOperand c256 = operand(mn(cout), 1, 256, es);
                            VOperand r256{};
                            bool rok = true;
                            if (f.add) {
                                const std::string& other = f.add->inputs[0] == f_in ? f.add->inputs[1] : f.add->inputs[0];
                                r256 = operand(mn(other), 1, 256, es);
                                rok = r256.fast_ok != 0;
                            }
                            if (c256.fast_ok && rok) {
                                p.bn = 256;
                                p.c = c256;
                                if (f.add) p.res = r256;
                            }
                        }
                        if (ok && !impl_->dry) {
                            // A's row addresses resolved once per plan (the map is static): a
                            // per-CTA device locate through a multi-piece div/mod map costs
                            // more than the gathers themselves (Swin: 7.8 of 11.5 us)
                            const int nseg = int(segs.size()) - 1;
                            std::vector<uint64_t> rows(static_cast<size_t>(M * nseg));
                            int64_t idx[VTC_MAX_RANK] = {};
                            for (int sg = 0; sg < nseg && ok; ++sg) {
                                idx[1] = segs[size_t(sg)];
                                for (int64_t m = 0; m < M && ok; ++m) {
                                    idx[0] = m;
                                    int pc = -1;
                                    const int64_t off = desc_eval(p.a.m, idx, &pc);
                                    ok = pc >= 0;
                                    // rp + k addresses A[m, k] for every k of the segment
                                    if (ok) rows[size_t(sg * M + m)] = p.a.m.piece[pc].ptr + uint64_t(off - idx[1]) * 2;
                                }
                            }
                            p.a_nseg = nseg;
                            for (int sg = 0; sg <= nseg; ++sg) p.a_seg_k[sg] = int32_t(segs[size_t(sg)]);
                            if (ok) {
                                auto* d = static_cast<uint64_t*>(impl_->alloc(rows.size() * 8, false));
                                ck(cudaMemcpy(d, rows.data(), rows.size() * 8, cudaMemcpyHostToDevice), "H2D(a_rows)");
                                p.a_rows = d;
                            }
                        }
                    }
                    if (ok && !impl_->dry) ok = gemm_tc_encode(p, abase, adims, astr, bbase, ldb);
                    if (ok && !impl_->dry) {
                        // C through a non-affine map (Swin's window reverse + roll): resolve its
                        // rows here once instead of a div/mod locate per row in every epilogue
                        bool affine = true, one = true;
                        for (int pi = 0; pi < p.c.m.npieces; ++pi) {
                            affine &= p.c.m.piece[pi].affine != 0;
                            one &= p.c.m.piece[pi].lo[1] <= 0 && p.c.m.piece[pi].hi[1] >= N &&
                                   p.c.fast_stride[pi] == p.c.fast_stride[0];
                        }
                        if (!affine && one) {
                            std::vector<uint64_t> rows(static_cast<size_t>(M));
                            int64_t idx[VTC_MAX_RANK] = {};
                            bool good = true;
                            for (int64_t m = 0; m < M && good; ++m) {
                                idx[0] = m;
                                int pc = -1;
                                const int64_t off = desc_eval(p.c.m, idx, &pc);
                                good = pc >= 0;
                                if (good) rows[size_t(m)] = p.c.m.piece[pc].ptr + uint64_t(off) * 2;
                            }
                            if (good) {
                                auto* d = static_cast<uint64_t*>(impl_->alloc(rows.size() * 8, false));
                                ck(cudaMemcpy(d, rows.data(), rows.size() * 8, cudaMemcpyHostToDevice), "H2D(c_rows)");
                                p.c_rows = d;
                                p.c_rs = p.c.fast_stride[0];
                            }
                        }
                    }
                    if (sw != tc_swiglu.end()) {
                        const OpNode& nu = *sw->second.up;
                        int64_t ldb2, cb2;
                        if (!affine2d(map_of(nu.inputs[1]), ldb2, cb2)) throw UnsupportedError("SwiGLU B2 of " + nu.id);
                        const VMap& bm2 = map_of(nu.inputs[1]);
                        const char* b2 = reinterpret_cast<const char*>(target(bm2.pieces()[0].target).ptr) + cb2 * es;
                        if (ok && !impl_->dry && !gemm_tc_encode_b(p.tmap_b2, b2, N, K, ldb2))
                            throw UnsupportedError("SwiGLU B2 tensor map of " + nu.id);
                        T->node = sw->second.gate->id + "+" + nu.id + "+" + sw->second.silu->id + "+" + sw->second.mul->id;
                    }
                    if (gl != tc_gelu.end()) T->node += "+" + gl->second->id;
                    auto tr = tc_trees.find(n.id);
                    if (tr != tc_trees.end()) {
                        p.epi = GEMM_EPI_TREES;
                        p.ntree = int32_t(tr->second.trees.size());
                        for (int k = 0; k < p.ntree; ++k) p.tree[k] = tr->second.trees[size_t(k)];
                        p.skip_lo = tr->second.skip_lo;
                        p.skip_hi = tr->second.skip_hi;
                        for (const auto& root : tr->second.roots) {
                            std::string label;
                            for (const auto& m2 : ew_trees.at(root).members) label += (label.empty() ? "" : "+") + m2;
                            T->node += "|" + label;
                        }
                    }
                    auto th = tc_hfuse.find(n.id);
                    if (th != tc_hfuse.end()) {
                        // the absorbed sibling: its weights as B2, its output rows resolved here
                        const OpNode& nb = *th->second;
                        if (!ok || f.add) throw UnsupportedError("horizontally fused GEMM " + n.id + " not launchable");
                        int64_t ldb2, cb2;
                        if (!affine2d(map_of(nb.inputs[1]), ldb2, cb2)) throw UnsupportedError("fused GEMM B2 of " + nb.id);
                        const VMap& bm2 = map_of(nb.inputs[1]);
                        const char* b2 = reinterpret_cast<const char*>(target(bm2.pieces()[0].target).ptr) + cb2 * es;
                        VOperand c2 = operand(map_of(nb.outputs[0]), 1, p.bn, es);
                        if (!c2.fast_ok || c2.m.npieces != 1) throw UnsupportedError("fused GEMM C2 of " + nb.id);
                        p.nmat = 2;
                        p.N1 = g_.tensor(nb.inputs[1]).shape[1];
                        p.c2_rs = c2.fast_stride[0];
                        if (!impl_->dry) {
                            if (!gemm_tc_encode_b(p.tmap_b2, b2, p.N1, K, ldb2))
                                throw UnsupportedError("fused GEMM B2 tensor map of " + nb.id);
                            std::vector<uint64_t> rows(static_cast<size_t>(M));
                            int64_t idx[VTC_MAX_RANK] = {};
                            for (int64_t m = 0; m < M; ++m) {
                                idx[0] = m;
                                int pc = -1;
                                const int64_t off = desc_eval(c2.m, idx, &pc);
                                rows[size_t(m)] = c2.m.piece[0].ptr + uint64_t(off) * 2;
                            }
                            auto* d = static_cast<uint64_t*>(impl_->alloc(rows.size() * 8, false));
                            ck(cudaMemcpy(d, rows.data(), rows.size() * 8, cudaMemcpyHostToDevice), "H2D(c2_rows)");
                            p.c2_rows = d;
                        }
                        T->node += "+" + nb.id;
                    }
                    if (ok) {
                        // prefill-sized M: 256-row tiles (two M=128 MMAs per B stage)
                        p.mt = (!p.a_gather && p.bn == 256 && M >= 4096) ? 2 : 1;
                        // opt-in (VTC_GEMM_PAIR=1): 128 x 256 tiles, two CTAs per SM, so one CTA's epilogue
                        // overlaps the other's mainloop.  It won while the 256-row tiles drained TMEM with 4
                        // warps (C5 QKV 1585 -> 1519 us); with 8 epilogue warps the 256-row tiles are faster
                        // again (QKV 2053 vs 2115 us, O-proj 1060 vs 1118 us on one box)
                        if (p.mt == 2 && K <= 4096 && (p.epi == GEMM_EPI_PLAIN || p.epi == GEMM_EPI_TREES) && tun.gemm_pair) {
                            p.mt = 1;
                            p.pair = 1;
                        }
                        const int64_t on = p.epi == GEMM_EPI_SWIGLU ? p.bn / 2 : p.bn;  // output columns per tile
                        const int64_t ntl = (N + on - 1) / on + (p.nmat > 1 ? (p.N1 + p.bn - 1) / p.bn : 0);
                        int64_t tiles = (M + 128 * p.mt - 1) / (128 * p.mt) * ntl;
                        int64_t ktiles = (K + 63) / 64;
                        const int sms = impl_->dry ? 148 : device_sms();
                        if (p.mt == 2 && tiles < sms) {  // not enough 256-row tiles: back to 128 rows
                            p.mt = 1;
                            tiles = (M + 127) / 128 * ntl;
                        }
                        // K splits as for the first matrix alone: a fused sibling launch sums in
                        // the same order as two separate launches would (bit-identical results)
                        int64_t tiles0 = tiles / ntl * ((N + on - 1) / on);
                        int64_t splits = tiles0 >= sms ? 1 : std::min<int64_t>(ktiles, std::max<int64_t>(1, sms / tiles0));
                        if (splits > 1 && p.mt == 2) {
                            // the split-K workspace and counters are per 128-row tile: a K split
                            // (a narrow first matrix) runs 128-row tiles
                            p.mt = 1;
                            tiles = (M + 127) / 128 * ntl;
                            tiles0 = tiles / ntl * ((N + on - 1) / on);
                            splits = tiles0 >= sms ? 1 : std::min<int64_t>(ktiles, std::max<int64_t>(1, sms / tiles0));
                        }
                        // (two CTAs per SM with twice the K splits measured slower at C3: 604 vs 546 us --
                        // the decode GEMMs are bound by the split-K epilogue, not the weight stream)
                        // prefill: CTA pairs (cta_group::2, M = 256 UMMAs over two SMs) -- VTC_GEMM_CTA_PAIR=1
                        if (tun.gemm_cta_pair && splits == 1 && p.bn == 256 && M >= 4096 && !p.a_gather && p.a_ndims <= 4 &&
                            p.nmat <= 1 && (p.epi == GEMM_EPI_PLAIN || p.epi == GEMM_EPI_SWIGLU)) {
                            p.cta_pair = 1;
                            p.pair = 0;
                            p.mt = 1;
                        }
                        p.splits = int32_t(splits);
                        if (splits > 1) {
                            p.work = static_cast<float*>(impl_->alloc(size_t(tiles * splits * 128 * p.bn) * 4, false));
                            p.counters = static_cast<unsigned*>(impl_->alloc(size_t(tiles) * 2 * 4, true));
                            p.ntiles_total = int32_t(tiles);
                            // the split-K reduction spread over every split (one CTA per SM, so the
                            // grid is co-resident when it fits the SMs): VTC_NO_COOP_REDUCE=1 off
                            p.coop_reduce = (tiles * splits <= sms && p.mt == 1 && (p.epi != GEMM_EPI_TREES || tun.tree_coop) &&
                                             !tun.no_coop_reduce)
                                                ? 1
                                                : 0;
                        }
                        push(std::move(T));
                        break;
                    }
                    if (f.add || p.epi != GEMM_EPI_PLAIN)
                        throw UnsupportedError("gemm_tc: fused epilogue without a tensor-core launch for " + n.id);
                }
                auto L = std::make_unique<LaunchT<MatmulParams, launch_matmul>>();
                L->node = n.id;
                L->kernel = "matmul_tiled";
                MatmulParams& p = L->p;
                std::memset(&p, 0, sizeof(p));
                p.rank = rank;
                for (int i = 0; i < rank; ++i) p.shape_c[i] = int32_t(o0.shape[size_t(i)]);
                p.M = M;
                p.N = N;
                p.K = K;
                p.batch = volume(o0.shape) / (M * N);
                p.dt = kdt(dt);
                p.exact = opt_.exact_fp ? 1 : 0;
                p.a = operand(map_of(n.inputs[0]), rank - 1, 8, es);
                p.b = operand(map_of(n.inputs[1]), rank - 1, 128, es);
                p.c = operand(map_of(n.outputs[0]), rank - 1, 8, es);
                // strides along M for A (tile 128) and along K for B (tile 8)
                {
                    const vtc_map& d = p.a.m;
                    bool ok = desc_pieces_aligned(d, rank - 2, 128);
                    for (int pi = 0; pi < d.npieces && ok; ++pi) {
                        int64_t s = desc_tile_stride(d.piece[pi], rank - 2, 128);
                        if (s == INT64_MIN) ok = false;
                        else p.a_mstride[pi] = s;
                    }
                    p.a_m_ok = ok;
                    const vtc_map& e = p.b.m;
                    ok = desc_pieces_aligned(e, rank - 2, 8);
                    for (int pi = 0; pi < e.npieces && ok; ++pi) {
                        int64_t s = desc_tile_stride(e.piece[pi], rank - 2, 8);
                        if (s == INT64_MIN) ok = false;
                        else p.b_kstride[pi] = s;
                    }
                    p.b_k_ok = ok;
                }
                push(std::move(L));
                break;
            }
            case OpKind::Attention: {
                if (dt != DType::BF16 && dt != DType::F32) throw UnsupportedError("Attention supports bf16/f32");
                const auto& at = std::get<AttentionAttrs>(n.attrs);
                const Index& qs = g_.tensor(n.inputs[0]).shape;
                const Index& ks = g_.tensor(n.inputs[1]).shape;
                const Index& vs = g_.tensor(n.inputs[2]).shape;
                int rank = int(qs.size());
                if (rank < 3 || rank > VTC_MAX_RANK) throw UnsupportedError("Attention needs rank >= 3");
                auto L = std::make_unique<LaunchT<AttnParams, launch_attention>>();
                L->node = n.id;
                AttnParams& p = L->p;
                std::memset(&p, 0, sizeof(p));
                p.rank = rank;
                p.H = int32_t(qs[size_t(rank - 3)]);
                p.Sq = int32_t(qs[size_t(rank - 2)]);
                p.D = int32_t(qs[size_t(rank - 1)]);
                p.Sk = int32_t(ks[size_t(rank - 2)]);
                p.Dv = int32_t(vs[size_t(rank - 1)]);
                if (p.D % 8 || p.Dv % 8 || p.D > 256 || p.Dv > 256) throw UnsupportedError("Attention head dims must be multiples of 8 and <= 256");
                p.Bt = int32_t(volume(Index(qs.begin(), qs.end() - 3)));
                p.scale = float(at.scale);
                p.causal = at.causal ? 1 : 0;
                p.dt = kdt(dt);
                p.q = operand(map_of(n.inputs[0]), rank - 1, p.D, es);
                p.k = operand(map_of(n.inputs[1]), rank - 1, p.D, es);
                p.v = operand(map_of(n.inputs[2]), rank - 1, p.Dv, es);
                p.o = operand(map_of(n.outputs[0]), rank - 1, p.Dv, es);
                if (n.inputs.size() == 4) {
                    p.has_bias = 1;
                    p.bias = operand(map_of(n.inputs[3]), rank - 1, 1, es);
                }
                int G = 1;
                for (int cand : {8, 4, 2})
                    if (p.H % cand == 0 && ignores_mod(p.k.m, rank - 3, cand) && ignores_mod(p.v.m, rank - 3, cand)) {
                        G = cand;
                        break;
                    }
                p.group = G;
                // tensor-core decode path: K/V rows addressed as base + t * stride when
                // the maps are single-piece affine along the key axis
                p.fast = attn_decode_supported(p) ? 1 : 0;
                if (p.k.m.npieces == 1 && p.v.m.npieces == 1) {
                    int64_t ks_ = desc_tile_stride(p.k.m.piece[0], rank - 2, p.Sk);
                    int64_t vs_ = desc_tile_stride(p.v.m.piece[0], rank - 2, p.Sk);
                    if (ks_ != INT64_MIN && vs_ != INT64_MIN) {
                        p.kv_affine = 1;
                        p.k_sstride = ks_;
                        p.v_sstride = vs_;
                    }
                }
                // long query blocks (prefill), head dim 128: tcgen05 / TMEM flash attention
                // with TMA-loaded Q / K / V (maps proved affine on the host)
                if (!p.fast && p.Sq >= 64 && !tun.no_fmha && attn_fmha_prepare(p, !impl_->dry)) {
                    p.fast = 3;
                    p.splits = 1;
                    p.chunk = p.Sk;
                    L->kernel = "attn_fmha_tc";
                    push(std::move(L));
                    break;
                }
                // short sequences (Swin windows): one warp per (batch, head) item
                if (!p.fast && p.Sq <= 64 && p.Sk <= 64 && p.q.m.npieces == 1 && p.o.m.npieces == 1 &&
                    !tun.no_attn_window) {
                    const int64_t qs_ = desc_tile_stride(p.q.m.piece[0], rank - 2, p.Sq);
                    const int64_t os_ = desc_tile_stride(p.o.m.piece[0], rank - 2, p.Sq);
                    const int64_t qd_ = desc_tile_stride(p.q.m.piece[0], rank - 1, p.D);
                    const int64_t od_ = desc_tile_stride(p.o.m.piece[0], rank - 1, p.Dv);
                    // 32-bit accesses of (d, d + 1) pairs: every element offset of an even d is even
                    auto even = [](const vtc_map& m) {
                        for (int pi = 0; pi < m.npieces; ++pi) {
                            const vtc_piece& pc = m.piece[pi];
                            if (pc.base % 2 || pc.ngroups || pc.ptr % 4) return false;
                            for (int t = 0; t < pc.ndigits; ++t)
                                if (pc.dig[t].coeff % 2 && pc.dig[t].axis != m.rank - 1) return false;
                            if (pc.affine)
                                for (int a = 0; a + 1 < m.rank; ++a)
                                    if (pc.aff[a] % 2) return false;
                        }
                        return true;
                    };
                    p.qo_affine = qs_ != INT64_MIN && os_ != INT64_MIN && qd_ == 1 && od_ == 1 && even(p.q.m) && even(p.o.m);
                    p.q_sstride = qs_;
                    p.o_sstride = os_;
                    if (p.has_bias && p.bias.m.npieces == 1) {
                        p.b_sstride = desc_tile_stride(p.bias.m.piece[0], rank - 2, p.Sq);
                        p.b_kstride = desc_tile_stride(p.bias.m.piece[0], rank - 1, p.Sk);
                        p.bias_affine = p.b_sstride != INT64_MIN && p.b_kstride != INT64_MIN;
                    }
                    if (attn_window_supported(p) && !impl_->dyn_on) {  // a dynamic key count may outgrow the tile
                        p.fast = 4;
                        p.splits = 1;
                        p.chunk = p.Sk;
                        if (!impl_->dry) {
                            // per-item bases resolved once (Swin's maps carry (i + 3) mod 56 / t div 7 digits:
                            // five device locates per item cost more than the item's math)
                            const int64_t items = int64_t(p.Bt) * p.H;
                            std::vector<uint64_t> tab(static_cast<size_t>(items * 5), 0);
                            int64_t idx[VTC_MAX_RANK] = {};
                            const vtc_map* ms[5] = {&p.q.m, &p.k.m, &p.v.m, &p.o.m, &p.bias.m};
                            bool good = true;
                            for (int64_t it = 0; it < items && good; ++it) {
                                int64_t bh = it;
                                idx[rank - 3] = bh % p.H;
                                bh /= p.H;
                                for (int a = rank - 4; a >= 0; --a) {
                                    idx[a] = bh % qs[size_t(a)];
                                    bh /= qs[size_t(a)];
                                }
                                idx[rank - 2] = 0;
                                idx[rank - 1] = 0;
                                for (int k2 = 0; k2 < (p.has_bias ? 5 : 4) && good; ++k2) {
                                    int pc = -1;
                                    const int64_t off = desc_eval(*ms[k2], idx, &pc);
                                    good = pc >= 0;
                                    if (good) tab[size_t(it * 5 + k2)] = ms[k2]->piece[pc].ptr + uint64_t(off) * es;
                                }
                            }
                            if (good) {
                                auto* d = static_cast<uint64_t*>(impl_->alloc(tab.size() * 8, false));
                                ck(cudaMemcpy(d, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice), "H2D(attn item bases)");
                                p.item_base = d;
                            }
                        }
                        L->kernel = "attn_window_tc";
                        push(std::move(L));
                        break;
                    }
                }
                // other long query blocks: flash attention on mma.sync, no K split
                if (!p.fast && attn_prefill_supported(p)) {
                    p.fast = 2;
                    p.splits = 1;
                    p.chunk = p.Sk;
                    L->kernel = "attn_prefill_tc";
                    push(std::move(L));
                    break;
                }
                int64_t qblocks = int64_t(p.Bt) * (p.H / G) * (p.fast ? 1 : p.Sq);
                int splits = opt_.attn_splits;
                const int kgran = p.fast ? 64 : 32;  // keys per split granule (4 warps x 16 on the fast path)
                if (splits <= 0) {
                    // fast path: one wave (2 CTAs per SM) when the KV is short, ~4 waves when long
                    const int64_t wave = int64_t(impl_->dry ? 148 : device_sms()) * 2;  // 2 CTAs per SM
                    const bool longkv = int64_t(p.Sk) * qblocks >= wave * 512;
                    int64_t target = p.fast ? (longkv ? wave * 4 : wave) : wave;
                    const bool ev = tun.attn_ctas > 0;
                    if (ev) target = tun.attn_ctas;
                    splits = int((target + qblocks - 1) / qblocks);
                    const int smax = (p.Sk + kgran - 1) / kgran;
                    splits = std::max(1, std::min(splits, smax));
                    if (p.fast && longkv && !ev) {
                        // several waves: the split count whose last wave is fullest (C3: 3 splits =
                        // 5.19 waves -> 4 splits = 6.92 waves, attention 396 -> 379 us)
                        int best = splits;
                        double best_fill = 0.0;
                        for (int sc = std::max(1, splits - 1); sc <= std::min(smax, 2 * splits); ++sc) {
                            const double w = double(qblocks) * sc / double(wave);
                            const double fill = w / std::ceil(w);
                            if (fill > best_fill + 0.02) {
                                best_fill = fill;
                                best = sc;
                            }
                        }
                        splits = best;
                    }
                }
                int chunk = (p.Sk + splits - 1) / splits;
                chunk = (chunk + kgran - 1) / kgran * kgran;
                splits = (p.Sk + chunk - 1) / chunk;
                p.splits = splits;
                p.chunk = chunk;
                L->kernel = p.fast ? (splits > 1 ? "attn_decode_tc_splitkv" : "attn_decode_tc") : (splits > 1 ? "attention_splitkv" : "attention");
                // cooperative in-kernel split combine when every CTA fits on the GPU at once
                if (splits > 1 && p.fast == 1 && !impl_->dry && !tun.separate_combine &&
                    qblocks * splits <= attn_decode_capacity())
                    p.counters = static_cast<unsigned*>(impl_->alloc(size_t(qblocks) * sizeof(unsigned), true));
                if (splits > 1) {
                    int64_t rows = int64_t(p.Bt) * p.H * p.Sq;
                    p.part_o = static_cast<float*>(impl_->alloc(size_t(rows * splits * p.Dv) * sizeof(float), false));
                    p.part_ml = static_cast<float*>(impl_->alloc(size_t(rows * splits * 2) * sizeof(float), false));
                }
                push(std::move(L));
                break;
            }
            default:
                throw UnsupportedError(std::string("no kernel for operator ") + to_string(n.kind));
        }
    }
    // horizontal fusion of adjacent independent elementwise launches (e.g. the Q
    // and K RoPE trees): one launch, CTAs split between the two programs
    if (opt_.fuse) {
        using EwL = LaunchT<EwParams, launch_eltwise>;
        auto roots_of = [](const vtc_map& m, std::set<int>& out) {
            for (int i = 0; i < m.npieces; ++i) out.insert(m.piece[i].target);
        };
        std::vector<std::unique_ptr<Launch>> merged;
        std::vector<LaunchInfo> minfos;
        for (size_t i = 0; i < impl_->launches.size(); ++i) {
            auto* a = dynamic_cast<EwL*>(impl_->launches[i].get());
            auto* b = i + 1 < impl_->launches.size() ? dynamic_cast<EwL*>(impl_->launches[i + 1].get()) : nullptr;
            if (a && b && eltwise_pair_compatible(a->p, b->p)) {
                std::set<int> wa, rb, wb, ra;
                roots_of(a->p.out.m, wa);
                roots_of(b->p.out.m, wb);
                for (int k = 0; k < b->p.nin; ++k) roots_of(b->p.in[k].m, rb);
                for (int k = 0; k < a->p.nin; ++k) roots_of(a->p.in[k].m, ra);
                bool dep = false;
                for (int t : wa) dep |= rb.count(t) > 0 || wb.count(t) > 0;
                for (int t : wb) dep |= ra.count(t) > 0;
                if (!dep) {
                    auto P = std::make_unique<LaunchT<EwPair, launch_eltwise_pair>>();
                    P->node = a->node + "|" + b->node;
                    P->kernel = a->p.aff && b->p.aff ? "eltwise_aff" : "eltwise";
                    P->p.a = a->p;
                    P->p.b = b->p;
                    LaunchInfo li = infos_[i];
                    li.node = P->node;
                    li.bytes += infos_[i + 1].bytes;
                    merged.push_back(std::move(P));
                    minfos.push_back(li);
                    ++i;
                    continue;
                }
            }
            merged.push_back(std::move(impl_->launches[i]));
            minfos.push_back(infos_[i]);
        }
        impl_->launches = std::move(merged);
        infos_ = std::move(minfos);
    }
    // decode attention -> streamed GEMV: the attention CTAs prefetch the GEMV's weights
    // into L2 (HBM is idle while the split-KV attention is latency-bound; W_o is 32 MB
    // at Llama-3-8B).  VTC_ATTN_L2PF=0: off
    {
        const bool on = tun.attn_l2pf;
        using AL = LaunchT<AttnParams, launch_attention>;
        using GL = LaunchT<GemvParams, launch_gemv_any>;
        for (size_t i = 0; on && i + 1 < impl_->launches.size(); ++i) {
            auto* a = dynamic_cast<AL*>(impl_->launches[i].get());
            auto* b = dynamic_cast<GL*>(impl_->launches[i + 1].get());
            if (!a || !b || a->p.fast != 1 || !b->p.stream || !b->p.b_static || b->p.b_sk != b->p.N) continue;
            const int64_t bytes = b->p.K * b->p.N * 2;
            if (bytes <= 0 || bytes > (int64_t(64) << 20) || reinterpret_cast<uintptr_t>(b->p.b_base) % 16) continue;
            a->p.pf_base = reinterpret_cast<uint64_t>(b->p.b_base);
            a->p.pf_bytes = bytes;
        }
    }
    // chain consecutive streamed GEMVs (o_proj -> gate/up -> down) into one
    // persistent launch with per-strip dependencies.  Opt-in (VTC_CHAIN=1):
    // on C2 it measured equal to separate launches (113.6 vs 113.6 us) because
    // every strip of a split-K stage completes at the stage's end, so the next
    // stage cannot start early; kept for multi-layer chains.
    if (opt_.fuse && tun.chain) {
        using GL = LaunchT<GemvParams, launch_gemv_any>;
        auto roots_of = [](const VOperand& op, std::set<int>& out) {
            for (int i = 0; i < op.m.npieces; ++i) out.insert(op.m.piece[i].target);
        };
        auto reads_of = [&](const GemvParams& p) {
            std::set<int> r;
            roots_of(p.a, r);
            if (p.prologue == GemvPrologue::SiLUMul) roots_of(p.a2, r);
            if (p.prologue == GemvPrologue::RMSNorm) roots_of(p.normw, r);
            if (p.has_res) roots_of(p.res, r);
            return r;
        };
        auto writes_of = [&](const GemvParams& p) {
            std::set<int> w;
            roots_of(p.c, w);
            if (p.nmat > 1) roots_of(p.c2, w);
            return w;
        };
        auto chainable = [](const GemvParams& p) { return p.stream == 1 && p.has_epi == 0 && p.b_static == 1; };
        auto same_map = [](const VOperand& x, const VOperand& y) { return std::memcmp(&x.m, &y.m, sizeof(vtc_map)) == 0; };
        std::vector<std::unique_ptr<Launch>> merged;
        std::vector<LaunchInfo> minfos;
        size_t i = 0;
        while (i < impl_->launches.size()) {
            auto* a = dynamic_cast<GL*>(impl_->launches[i].get());
            if (!a || !chainable(a->p)) {
                merged.push_back(std::move(impl_->launches[i]));
                minfos.push_back(infos_[i]);
                ++i;
                continue;
            }
            std::vector<GemvParams> run{a->p};
            std::vector<GemvChainStage> hs(1);
            std::set<int> rd = reads_of(a->p), wr = writes_of(a->p);
            std::vector<std::set<int>> wr_st{writes_of(a->p)};
            int64_t sA = a->p.M * int64_t(a->p.a_tiles) * GEMV_STREAM_KT;
            size_t j = i + 1;
            for (; j < impl_->launches.size() && run.size() < size_t(GEMV_MAX_CHAIN); ++j) {
                auto* b = dynamic_cast<GL*>(impl_->launches[j].get());
                if (!b || !chainable(b->p) || b->p.M != a->p.M || b->p.grid != a->p.grid) break;
                const GemvParams& q = b->p;
                std::set<int> rq = reads_of(q), wq = writes_of(q);
                bool hazard = false;  // WAR / WAW against earlier stages
                for (int t : wq) hazard |= rd.count(t) > 0 || wr.count(t) > 0;
                if (hazard) break;
                int64_t sAq = std::max<int64_t>(sA, q.M * int64_t(q.a_tiles) * GEMV_STREAM_KT);
                if (gemv_chain_smem(sAq, 2) + sizeof(GemvParams) + 12 * 1024 > 227 * 1024) break;
                GemvChainStage h{};
                const GemvParams& pv = run.back();
                const size_t k = run.size();
                for (size_t t = 0; t < k; ++t) {
                    bool touches = false;
                    for (int r : rq) touches |= wr_st[t].count(r) > 0;
                    if (touches) h.dep_all |= 1u << t;
                }
                // A exactly the previous stage's output columns: wait per strip
                if ((h.dep_all >> (k - 1)) & 1u) {
                    std::set<int> rest;
                    if (q.prologue == GemvPrologue::RMSNorm) roots_of(q.normw, rest);
                    if (q.has_res) roots_of(q.res, rest);
                    bool other = false;
                    for (int r : rest) other |= wr_st[k - 1].count(r) > 0;
                    const bool a_ok = same_map(q.a, pv.c);
                    const bool a2_ok = q.prologue != GemvPrologue::SiLUMul || (pv.nmat > 1 && same_map(q.a2, pv.c2));
                    if (!other && a_ok && a2_ok && q.prologue != GemvPrologue::RMSNorm) {
                        h.dep_all &= ~(1u << (k - 1));
                        h.dep_range = 1;
                        h.dep_a2 = q.prologue == GemvPrologue::SiLUMul ? 1 : 0;
                    }
                }
                run.push_back(q);
                hs.push_back(h);
                rd.insert(rq.begin(), rq.end());
                wr.insert(wq.begin(), wq.end());
                wr_st.push_back(wq);
                sA = sAq;
            }
            if (run.size() < 2) {
                merged.push_back(std::move(impl_->launches[i]));
                minfos.push_back(infos_[i]);
                ++i;
                continue;
            }
            auto C = std::make_unique<GemvChainLaunch>();
            C->kernel = a->kernel;
            LaunchInfo li = infos_[i];
            int max_strips = 0;
            for (size_t t = 0; t < run.size(); ++t) {
                const GemvParams& p = run[t];
                GemvChainStage& h = hs[t];
                h.K = p.K;
                h.n0 = p.n_mat[0];
                h.n1 = p.nmat > 1 ? p.n_mat[1] : 0;
                h.nmat = p.nmat;
                h.strips0 = p.strips0;
                h.b_static = p.b_static;
                h.pre_stages = p.pre_stages;
                h.l2_prefetch = p.l2_prefetch;
                if (t) {
                    h.l2_prefetch = 0;  // measured: any boundary prefetch slowed C2 (133 us at 4 tiles)
                    if (tun.chain_l2pf >= 0) h.l2_prefetch = tun.chain_l2pf;
                }
                C->ca.st[t] = h;
                std::memcpy(C->ca.tmap[t], p.tmap, sizeof(p.tmap));
                const int ns = p.strips0 + (p.nmat > 1 ? int((p.n_mat[1] + GEMV_STREAM_COLS - 1) / GEMV_STREAM_COLS) : 0);
                max_strips = std::max(max_strips, ns);
                if (t) {
                    li.node += "|" + infos_[i + t].node;
                    li.bytes += infos_[i + t].bytes;
                }
            }
            C->node = li.node;
            C->ps = run;
            C->ca.nst = int32_t(run.size());
            C->ca.ring = gemv_chain_smem(sA, 3) + sizeof(GemvParams) + 12 * 1024 <= 227 * 1024 ? 3 : 2;
            C->ca.max_strips = max_strips;
            C->ca.sA_floats = sA;
            C->ca.sync = static_cast<unsigned*>(impl_->alloc(size_t(2 + run.size() * max_strips) * 4, true));
            merged.push_back(std::move(C));
            minfos.push_back(li);
            i = j;
        }
        impl_->launches = std::move(merged);
        infos_ = std::move(minfos);
    }
    // dynamic position: register the position-dependent fields of every launch
    if (impl_->dyn_on)
        for (auto& l : impl_->launches) l->dyn_patch(impl_->dyn);
    // optional device timeline (VTC_TRACE=1): [entry, exit] globaltimer per launch
    impl_->trace = nullptr;
    if (!dry && Tuning::on("VTC_TRACE")) {
        impl_->trace = static_cast<unsigned long long*>(impl_->alloc(impl_->launches.size() * 64, false));
        for (size_t i = 0; i < impl_->launches.size(); ++i) impl_->launches[i]->set_trace(impl_->trace, int(i));
        reset_trace();
    }
    // all parameter blocks in one device allocation, uploaded once
    if (!dry) {
        size_t total = 0;
        std::vector<size_t> offs;
        for (auto& l : impl_->launches) {
            offs.push_back(total);
            total += (l->param_bytes() + 255) / 256 * 256;
        }
        if (total) {
            auto* base = static_cast<char*>(impl_->alloc(total, false));
            std::vector<char> host(total);
            for (size_t i = 0; i < impl_->launches.size(); ++i) {
                if (impl_->launches[i]->param_bytes() == 0) continue;
                std::memcpy(host.data() + offs[i], impl_->launches[i]->host_params(), impl_->launches[i]->param_bytes());
                impl_->launches[i]->set_device_params(base + offs[i]);
            }
            ck(cudaMemcpy(base, host.data(), total, cudaMemcpyHostToDevice), "H2D(params)");
        }
    }
    prepared_ = !dry;
}

void Executor::run(void* stream) {
    if (!prepared_) prepare();
    auto s = static_cast<cudaStream_t>(stream);
    impl_->launch_all(s);
    ck(cudaGetLastError(), "kernel launch");
}

void Executor::run_graph(void* stream) {
    if (!prepared_) prepare();
    auto s = static_cast<cudaStream_t>(stream);
    if (!impl_->gexec) {
        cudaStream_t cap;
        ck(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
        impl_->launch_all(cap);
        cudaError_t e = cudaStreamEndCapture(cap, &impl_->graph);
        cudaStreamDestroy(cap);
        ck(e, "cudaStreamEndCapture");
        ck(cudaGraphInstantiate(&impl_->gexec, impl_->graph, 0), "cudaGraphInstantiate");
    }
    ck(cudaGraphLaunch(impl_->gexec, s), "cudaGraphLaunch");
}

void Executor::set_comm(Comm* c) {
    impl_->comm = c;
    impl_->free_graph();  // a captured graph holds the previous collective
}

void Executor::reset_trace() {
    if (!impl_->trace) return;
    std::vector<unsigned long long> init(impl_->launches.size() * 8, 0ull);
    for (size_t i = 0; i < impl_->launches.size(); ++i) init[8 * i] = ~0ull;
    ck(cudaMemcpy(impl_->trace, init.data(), init.size() * 8, cudaMemcpyHostToDevice), "H2D(trace)");
}

int Executor::read_trace(unsigned long long* out, int n) {
    if (!impl_->trace) return 0;
    int L = int(impl_->launches.size());
    std::vector<unsigned long long> buf(size_t(L) * 8);
    ck(cudaDeviceSynchronize(), "sync");
    ck(cudaMemcpy(buf.data(), impl_->trace, buf.size() * 8, cudaMemcpyDeviceToHost), "D2H(trace)");
    for (int i = 0; i < 8 * L && i < n; ++i) out[i] = buf[size_t(i)];
    reset_trace();
    return L;
}

void Executor::run_timed(void* stream, float* ms, int n) {
    // Launches with an event between each, captured into a CUDA graph so the
    // per-launch intervals contain no host launch gaps.
    if (!prepared_) prepare();
    auto s = static_cast<cudaStream_t>(stream);
    size_t L = impl_->launches.size();
    std::vector<cudaEvent_t> ev(L + 1);
    for (auto& e : ev) ck(cudaEventCreate(&e), "cudaEventCreate");
    cudaStream_t cap;
    ck(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    ck(cudaEventRecordWithFlags(ev[0], cap, cudaEventRecordExternal), "cudaEventRecord");
    for (size_t i = 0; i < L; ++i) {
        if (i == 0 && impl_->dyn_on) tl_serialize_next = true;
        impl_->launches[i]->run(cap);
        ck(cudaEventRecordWithFlags(ev[i + 1], cap, cudaEventRecordExternal), "cudaEventRecord");
    }
    cudaGraph_t graph;
    cudaError_t e = cudaStreamEndCapture(cap, &graph);
    cudaStreamDestroy(cap);
    ck(e, "cudaStreamEndCapture");
    cudaGraphExec_t gexec;
    ck(cudaGraphInstantiate(&gexec, graph, 0), "cudaGraphInstantiate");
    ck(cudaGraphLaunch(gexec, s), "cudaGraphLaunch");
    ck(cudaStreamSynchronize(s), "sync");
    for (size_t i = 0; i < L && int(i) < n; ++i) ck(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]), "elapsed");
    cudaGraphExecDestroy(gexec);
    cudaGraphDestroy(graph);
    for (auto& x : ev) cudaEventDestroy(x);
}

void Executor::set_position(int64_t pos, void* stream) {
    if (!opt_.dynamic_pos) throw ExecutionError("set_position: plan was not created with a dynamic position");
    if (!prepared_) prepare();
    if (pos < 0 || pos > impl_->dyn.p0)
        throw OutOfBoundsError("set_position: " + std::to_string(pos) + " outside [0, " + std::to_string(impl_->dyn.p0) + "]");
    upload("__pos", &pos, 8, stream);
    ck(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "sync");  // pageable source
}

int64_t Executor::max_position() const { return opt_.dynamic_pos ? impl_->dyn.p0 : -1; }

void Executor::upload(const std::string& id, const void* host, int64_t bytes, void* stream) {
    auto it = root_index_.find(id);
    if (it == root_index_.end()) throw ExecutionError("upload target " + id + " is not a physical root");
    RootBuffer& r = roots_[size_t(it->second)];
    if (bytes != r.bytes) throw ShapeMismatchError("upload of " + id + ": byte count mismatch");
    if (id == "__pos") pos_set_ = true;
    void* d = root_ptr(id);
    ck(cudaMemcpyAsync(d, host, size_t(bytes), cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)), "H2D");
}

void Executor::run_host(const std::vector<HostIn>& ins, const std::vector<HostOut>& outs, void* stream) {
    // Small transfers (a decode step's activations) go through pinned staging and
    // host-link copy kernels captured in the host graph -- a DMA node costs more
    // than moving a few KB.  Large ones (prefill activations) are DMA'd straight
    // between the caller's buffer and the root around the graph launch.
    int64_t kLinkMax = 64 << 10;  // measured: link copies win at 8 KB (C2), DMA at 512 KB (C3)
    if (const int64_t e = Tuning::from_env().host_link_max; e >= 0) kLinkMax = e;  // tests: force either path
    auto s = static_cast<cudaStream_t>(stream);
    Impl& I = *impl_;
    bool same = prepared_ && I.hexec && ins.size() == I.sig_in.size() && outs.size() == I.sig_out.size() && I.fast_stream == s;
    for (size_t i = 0; same && i < ins.size(); ++i) same = ins[i].bytes == I.sig_in[i].second && ins[i].id == I.sig_in[i].first;
    for (size_t i = 0; same && i < outs.size(); ++i)
        same = outs[i].bytes == I.sig_out[i].second && outs[i].id == I.sig_out[i].first;
    if (!same) {
        I.sig_in.clear();
        I.sig_out.clear();
        if (I.hexec) cudaGraphExecDestroy(I.hexec);
        I.hexec = nullptr;
        // inputs: validate, pick the staged (small) ones, (re)build their arena
        std::string key;
        std::vector<int> small;
        for (size_t i = 0; i < ins.size(); ++i) {
            auto it = root_index_.find(ins[i].id);
            if (it == root_index_.end()) throw ExecutionError("input " + ins[i].id + " is not a physical root");
            if (ins[i].bytes != roots_[size_t(it->second)].bytes)
                throw ShapeMismatchError("input " + ins[i].id + ": byte count mismatch");
            if (ins[i].bytes <= kLinkMax) {
                small.push_back(int(i));
                key += ins[i].id;
                key += '\n';
            }
        }
        bool ok = key == arena_key_ && (arena_dev_ || small.empty());
        for (size_t j = 0; ok && j < small.size(); ++j)
            ok = root_ptr(ins[size_t(small[j])].id) == static_cast<char*>(arena_dev_) + arena_off_[j];
        if (!ok) {
            if (arena_dev_) {
                // roots staged by an earlier call but not named in this one keep their
                // contents: move them out of the old arena before it is freed
                std::set<std::string> now;
                for (int i : small) now.insert(ins[size_t(i)].id);
                char* lo = static_cast<char*>(arena_dev_);
                for (auto& r : roots_) {
                    char* rp = static_cast<char*>(r.ptr);
                    if (r.owned || !rp || rp < lo || rp >= lo + arena_bytes_ || now.count(r.id)) continue;
                    void* own = nullptr;
                    ck(cudaMalloc(&own, size_t(std::max<int64_t>(r.bytes, 16))), "cudaMalloc(root)");
                    ck(cudaMemcpy(own, rp, size_t(r.bytes), cudaMemcpyDeviceToDevice), "D2D(arena root)");
                    bind_root(r.id, own);
                    r.owned = true;
                }
                ck(cudaFree(arena_dev_), "cudaFree(arena)");
            }
            if (arena_host_) ck(cudaFreeHost(arena_host_), "cudaFreeHost(arena)");
            arena_dev_ = arena_host_ = nullptr;
            arena_off_.clear();
            int64_t total = 0;
            for (int i : small) {
                arena_off_.push_back(total);
                total += (std::max<int64_t>(ins[size_t(i)].bytes, 16) + 255) / 256 * 256;
            }
            arena_bytes_ = total;
            if (total) {
                ck(cudaMalloc(&arena_dev_, size_t(total)), "cudaMalloc(arena)");
                ck(cudaHostAlloc(&arena_host_, size_t(total), cudaHostAllocMapped | cudaHostAllocPortable),
                   "cudaHostAlloc(arena)");
                for (size_t j = 0; j < small.size(); ++j)
                    bind_root(ins[size_t(small[j])].id, static_cast<char*>(arena_dev_) + arena_off_[j]);
            }
            arena_key_ = key;
        }
        I.in_slot.assign(ins.size(), -1);
        for (size_t j = 0; j < small.size(); ++j) I.in_slot[size_t(small[j])] = int(j);
        // outputs: small physical -> staged in the graph; large physical -> DMA; virtual -> download
        I.out_off.assign(outs.size(), SIZE_MAX);
        I.out_kind.assign(outs.size(), 2);
        size_t out_total = 0;
        for (size_t i = 0; i < outs.size(); ++i) {
            const HostOut& o = outs[i];
            if (o.bytes != g_.tensor(o.id).bytes()) throw ShapeMismatchError("output " + o.id + ": byte count mismatch");
            if (root_index_.count(o.id) && ptg_.map_of(o.id).is_identity_of(o.id)) {
                const bool link = o.bytes <= kLinkMax && o.bytes % 16 == 0;
                I.out_kind[i] = link ? 0 : 1;
                if (link) {
                    I.out_off[i] = out_total;
                    out_total += (size_t(o.bytes) + 255) / 256 * 256;
                }
            }
        }
        if (!prepared_) prepare();
        if (out_total > I.out_host_bytes) {
            if (I.out_host) ck(cudaFreeHost(I.out_host), "cudaFreeHost(out)");
            I.out_host = nullptr;
            ck(cudaHostAlloc(&I.out_host, out_total, cudaHostAllocMapped | cudaHostAllocPortable), "cudaHostAlloc(out)");
            I.out_host_bytes = out_total;
        }
        std::vector<void*> out_dev(outs.size(), nullptr);
        for (size_t i = 0; i < outs.size(); ++i)
            if (I.out_kind[i] != 2) out_dev[i] = root_ptr(outs[i].id);
        void *arena_host_dev = nullptr, *out_host_dev = nullptr;  // device views of the pinned buffers
        if (arena_host_) ck(cudaHostGetDevicePointer(&arena_host_dev, arena_host_, 0), "cudaHostGetDevicePointer");
        if (I.out_host) ck(cudaHostGetDevicePointer(&out_host_dev, I.out_host, 0), "cudaHostGetDevicePointer");
        const bool dma = Tuning::set("VTC_HOST_DMA");  // A/B: DMA nodes for the small copies too
        cudaStream_t cap;
        cudaGraph_t hg = nullptr;
        ck(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
        if (arena_bytes_) {
            if (!dma) launch_host_link_copy(arena_host_dev, arena_dev_, arena_bytes_, cap);
            else cudaMemcpyAsync(arena_dev_, arena_host_, size_t(arena_bytes_), cudaMemcpyHostToDevice, cap);
        }
        I.launch_all(cap);
        for (size_t i = 0; i < outs.size(); ++i) {
            if (I.out_kind[i] != 0) continue;
            if (!dma)
                launch_host_link_copy(out_dev[i], static_cast<char*>(out_host_dev) + I.out_off[i], outs[i].bytes, cap);
            else
                cudaMemcpyAsync(static_cast<char*>(I.out_host) + I.out_off[i], out_dev[i], size_t(outs[i].bytes),
                                cudaMemcpyDeviceToHost, cap);
        }
        cudaError_t e = cudaStreamEndCapture(cap, &hg);
        cudaStreamDestroy(cap);
        ck(e, "cudaStreamEndCapture(host graph)");
        e = cudaGraphInstantiate(&I.hexec, hg, 0);
        cudaGraphDestroy(hg);
        ck(e, "cudaGraphInstantiate(host graph)");
        I.out_dev = out_dev;
        I.in_dev.assign(ins.size(), nullptr);
        for (size_t i = 0; i < ins.size(); ++i)
            if (I.in_slot[i] < 0) I.in_dev[i] = root_ptr(ins[i].id);
        for (const auto& in : ins) I.sig_in.emplace_back(in.id, in.bytes);
        for (const auto& o : outs) I.sig_out.emplace_back(o.id, o.bytes);
        I.fast_stream = s;
    }
    for (size_t i = 0; i < ins.size(); ++i) {
        if (!ins[i].bytes) continue;
        if (I.in_slot[i] >= 0)
            std::memcpy(static_cast<char*>(arena_host_) + arena_off_[size_t(I.in_slot[i])], ins[i].ptr, size_t(ins[i].bytes));
        else
            ck(cudaMemcpyAsync(I.in_dev[i], ins[i].ptr, size_t(ins[i].bytes), cudaMemcpyHostToDevice, s), "H2D");
    }
    ck(cudaGraphLaunch(I.hexec, s), "cudaGraphLaunch(host graph)");
    for (size_t i = 0; i < outs.size(); ++i) {
        if (I.out_kind[i] == 1)
            ck(cudaMemcpyAsync(outs[i].ptr, I.out_dev[i], size_t(outs[i].bytes), cudaMemcpyDeviceToHost, s), "D2H");
        else if (I.out_kind[i] == 2)
            download(outs[i].id, outs[i].ptr, outs[i].bytes, stream);  // virtual: materialised through its map
    }
    ck(cudaStreamSynchronize(s), "sync");
    for (size_t i = 0; i < outs.size(); ++i)
        if (I.out_kind[i] == 0)
            std::memcpy(outs[i].ptr, static_cast<char*>(I.out_host) + I.out_off[i], size_t(outs[i].bytes));
}

void Executor::download(const std::string& id, void* host, int64_t bytes, void* stream) {
    const TensorSpec& t = g_.tensor(id);
    if (bytes != t.bytes()) throw ShapeMismatchError("download of " + id + ": byte count mismatch");
    auto s = static_cast<cudaStream_t>(stream);
    const VMap& m = ptg_.map_of(id);
    auto it = root_index_.find(id);
    if (it != root_index_.end() && m.is_identity_of(id)) {
        ck(cudaMemcpyAsync(host, root_ptr(id), size_t(bytes), cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaStreamSynchronize(s), "sync");
        return;
    }
    if (!prepared_) prepare();
    // materialise through the map into a temporary buffer
    void* tmp = nullptr;
    ck(cudaMalloc(&tmp, size_t(std::max<int64_t>(bytes, 16))), "cudaMalloc(download)");
    std::string tmp_id = "__download__";
    auto target = [&](const std::string& tt) -> TargetInfo {
        if (tt == tmp_id) return TargetInfo{-1, reinterpret_cast<uint64_t>(tmp)};
        auto jt = root_index_.find(tt);
        if (jt == root_index_.end()) throw ExecutionError("map targets non-root tensor " + tt);
        return TargetInfo{jt->second, reinterpret_cast<uint64_t>(roots_[size_t(jt->second)].ptr)};
    };
    EwParams p;
    std::memset(&p, 0, sizeof(p));
    int rank = int(t.shape.size());
    int64_t es = dtype_size(t.dtype);
    p.rank = rank;
    for (int i = 0; i < rank; ++i) p.shape[i] = int32_t(t.shape[size_t(i)]);
    p.vec = 1;
    p.copy_only = 1;
    p.dt = kdt(t.dtype);
    p.esize = int32_t(es);
    p.nvec = t.elems();
    p.nin = 1;
    p.out.m = lower_map(VMap::identity(tmp_id, t.shape), target);
    finish_operand(p.out, rank - 1, 1, es);
    p.in[0].m = lower_map(m, target);
    finish_operand(p.in[0], rank - 1, 1, es);
    EwParams* dp = upload_params(p);
    launch_eltwise(p, dp, s);
    cudaError_t e = cudaMemcpyAsync(host, tmp, size_t(bytes), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(tmp);
    cudaFree(dp);
    ck(e, "download");
}

}  // namespace vtc
