// GPU executor for VTC-planned graphs.
//
// Same shape as the reference interpreter's execute_detailed
// (proj/src/executor.cpp:448-498): only physical roots own device buffers,
// nodes run in the graph's deterministic topological order, eliminated
// data-movement operators launch nothing, and every operand is read / written
// through its resolved map onto the roots -- inside the consumer kernel.
// The all-physical points-to graph gives the materialising baseline executor
// on the same kernels (each data-movement op becomes one gather-copy launch).
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "vtc/graph.hpp"
#include "vtc/plan.hpp"

namespace vtc {

struct ExecOptions {
    bool exact_fp = true;     // generic f32/f64 MatMul: unfused mul+add (bit-exact vs CPU reference)
    bool use_gemv = true;     // bf16 decode projections on the weight-streaming kernel
    bool use_tc = true;       // bf16 MatMul with M > 16 on the tcgen05 GEMM
    bool gemv_stream = true;  // persistent TMA-streamed GEMV for M <= 4 (else the LDG split-K GEMV)
    bool fuse = true;         // RMSNorm->MatMul, SiLU*Mul->MatMul, MatMul->Add(residual) fusion
    int attn_splits = 0;      // 0: automatic
    // Dynamic decode position: the plan is lowered once at the
    // static index p0 of its in-place ScatterND cache updates (write row p0, attend
    // over keys [0, p0]); each step's position pos <= p0 is read on the device from
    // the root "__pos" (int64[1]: vtc_run input or set_position), so the same
    // captured graph writes row pos and attends over pos + 1 keys.
    bool dynamic_pos = false;
};

struct RootBuffer {
    std::string id;
    DType dtype = DType::F32;
    Index shape;
    int64_t bytes = 0;
    void* ptr = nullptr;
    bool owned = false;
};

struct LaunchInfo {
    std::string node;    // graph node id (or "node+node" for a fused group)
    std::string kernel;  // kernel family
    int64_t bytes = 0;   // algorithmic bytes: unique elements read through the maps + elements written
};

class Executor {
public:
    Executor(const CompGraph& g, PointsToGraph ptg, ExecOptions opt = {});
    ~Executor();
    Executor(const Executor&) = delete;
    Executor& operator=(const Executor&) = delete;

    const CompGraph& graph() const { return g_; }
    const PointsToGraph& ptg() const { return ptg_; }

    void bind_root(const std::string& id, void* dev_ptr);
    void* root_ptr(const std::string& id);
    const std::vector<RootBuffer>& roots() const { return roots_; }

    // Lower descriptors against the current root pointers and build the launch list.
    // dry: plan the launches without touching the device (no allocation; null pointers).
    void prepare(bool dry = false);
    // Enqueue every launch on `stream` (asynchronous).
    void run(void* stream);
    // Capture the launch list into a CUDA graph once, then replay it.
    void run_graph(void* stream);
    // Enqueue every launch with a CUDA event on each side; per-launch device
    // milliseconds are written to ms[0..n) after the stream drains.
    void run_timed(void* stream, float* ms, int n);
    // VTC_TRACE=1 timeline: out[2i], out[2i+1] = globaltimer (ns) at entry / exit
    // of launch i over the runs since the last read; returns the launch count.
    int read_trace(unsigned long long* out, int n);
    // Communicator for the plan's AllReduce nodes (nullptr: single rank).
    void set_comm(class Comm* c);
    void reset_trace();

    void upload(const std::string& id, const void* host, int64_t bytes, void* stream);
    // Dynamic-position plans: the next steps write cache row `pos` and attend over
    // pos + 1 keys (0 <= pos <= the plan's static position); stream-ordered.
    void set_position(int64_t pos, void* stream);
    int64_t max_position() const;
    // Materialise any tensor (virtual or physical) into host memory.
    void download(const std::string& id, void* host, int64_t bytes, void* stream);

    // One call per step from host buffers (the reference's execute(g, ptg, inputs),
    // proj/include/vtelim/executor.hpp:77): the inputs' roots live in one device
    // arena filled by a single H2D copy from a pinned staging buffer, then the
    // CUDA-graph replay, then one D2H per output and a stream synchronisation.
    struct HostIn {
        std::string id;
        const void* ptr;
        int64_t bytes;
    };
    struct HostOut {
        std::string id;
        void* ptr;
        int64_t bytes;
    };
    void run_host(const std::vector<HostIn>& ins, const std::vector<HostOut>& outs, void* stream);

    const std::vector<LaunchInfo>& launches() const { return infos_; }
    int num_kernel_launches() const;

private:
    // drop the launch list and every captured graph (a root address changed)
    void invalidate();
    struct Impl;
    const CompGraph& g_;
    PointsToGraph ptg_;
    ExecOptions opt_;
    std::vector<RootBuffer> roots_;
    std::map<std::string, int> root_index_;
    std::vector<LaunchInfo> infos_;
    std::unique_ptr<Impl> impl_;
    bool prepared_ = false;
    bool pos_set_ = false;  // dynamic position written by the caller (else p0 at prepare)
    // run_host staging: device arena holding the per-step input roots + pinned mirror
    std::string arena_key_;
    void* arena_dev_ = nullptr;
    void* arena_host_ = nullptr;
    int64_t arena_bytes_ = 0;
    std::vector<int64_t> arena_off_;
};

}  // namespace vtc
