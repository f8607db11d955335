/* vtc -- C ABI of the B200-native executor for VTC-planned graphs.
 *
 * This is the drop-in boundary: plain pointers, sizes and status codes, no
 * C++ or torch types.  Each entry point replaces one reference interface
 * (paths relative to /root/reference):
 *
 *   vtc_graph_parse       <- vtelim::parse_graph          proj/include/vtelim/graph_ir.hpp:108 (src/graph_ir.cpp:455-485)
 *   vtc_graph_serialize   <- vtelim::serialize_graph      proj/include/vtelim/graph_ir.hpp:109
 *   vtc_graph_vtog        <- vtelim::build_vtog           proj/include/vtelim/vtog.hpp:42
 *   vtc_plan_create       <- vtelim::validate_ptg / all_physical_ptg (+ the planner's selection)
 *                                                         proj/include/vtelim/vtog.hpp:58, cost_model.hpp:61
 *   vtc_plan_info         <- PointsToGraph {roots, eliminated_ops} + vtelim::estimate
 *                                                         proj/include/vtelim/vtog.hpp:45-53, cost_model.hpp:59
 *   vtc_plan_upload / vtc_execute / vtc_plan_download
 *                         <- vtelim::execute / execute_detailed / ExecutionResult::materialize
 *                                                         proj/include/vtelim/executor.hpp:77-83, 71
 *   vtc_graph_estimate    <- vtelim::estimate(g, ptg, MachineParams) + breakdown
 *                                                         proj/include/vtelim/cost_model.hpp:59, 74-80
 *   vtc_graph_enumerate   <- vtelim::enumerate_ptgs       proj/include/vtelim/vtog.hpp:62
 *   vtc_graph_greedy      <- greedy_build (Alg. 2) over saving_oracle / executor_timed_oracle
 *                            (proj/include/vtelim/cost_model.hpp:64-73; the
 *                            reference snapshot lacks src/greedy.cpp, proj/CMakeLists.txt:21)
 *   vtc_map_eval          <- vtelim::IndexMap::eval       proj/include/vtelim/mapping.hpp:70
 *   vtc_launch_gather_copy<- vtelim::load_virtual + store_virtual (one copy through two maps)
 *                                                         proj/include/vtelim/executor.hpp:59-62
 *
 * Errors: C++ exceptions never cross this boundary.  Every int-returning call
 * returns VTC_OK or the status code of the reference error class
 * (proj/include/vtelim/errors.hpp:14-38); vtc_last_error() gives the message.
 * Threading: one plan per host thread; plans are independent.
 */
#ifndef VTC_H
#define VTC_H

#include <stdint.h>

#include "vtc_desc.h"

#ifdef __cplusplus
extern "C" {
#endif

enum vtc_status {
    VTC_OK = 0,
    VTC_ERR_GENERIC = 1,
    VTC_ERR_SCHEMA = 2,
    VTC_ERR_CYCLE = 3,
    VTC_ERR_SHAPE = 4,
    VTC_ERR_UNKNOWN_OPERATOR = 5,
    VTC_ERR_OUT_OF_BOUNDS = 6,
    VTC_ERR_MISSING_BASE_MAP = 7,
    VTC_ERR_COMPOSE_LIMIT = 8,
    VTC_ERR_CONFLICT = 9,
    VTC_ERR_INCOMPLETE_SELECTION = 10,
    VTC_ERR_CYCLE_DETECTED = 11,
    VTC_ERR_WRITE_ALIASING = 12,
    VTC_ERR_SPACE_TOO_LARGE = 13,
    VTC_ERR_MISSING_INPUT = 14,
    VTC_ERR_SHAPE_MISMATCH = 15,
    VTC_ERR_EXECUTION = 16,
    VTC_ERR_EQUIVALENCE = 17,
    VTC_ERR_INVALID_VTOG = 18,
    VTC_ERR_BUDGET = 19,
    VTC_ERR_CUDA = 20,
    VTC_ERR_NCCL = 21,
    VTC_ERR_UNSUPPORTED = 22
};

enum vtc_plan_mode {
    VTC_PLAN_MATERIALIZE = 0,     /* all-physical points-to graph: materialising baseline */
    VTC_PLAN_SELECTED = 1,        /* caller-selected VTOG edges (validate_ptg) */
    VTC_PLAN_MAX_ELIMINATION = 2, /* built-in strategy: eliminate every eliminable DM op */
    VTC_PLAN_INPLACE_UPDATES = 3, /* strong materialising comparator: ScatterND in place (rule i,
                                     proj/src/vt_rules.cpp:346-349), every other DM op copied */
    VTC_PLAN_GREEDY = 4           /* Alg. 2 global greedy over the B200-calibrated analytic oracle
                                     (MachineParams fitted by scripts/calibrate.py) */
};

enum vtc_plan_flags {
    VTC_FLAG_FAST_FP = 1u << 0,  /* generic f32/f64 MatMul with FMA instead of the bit-exact mul+add */
    VTC_FLAG_NO_GEMV = 1u << 1,  /* disable the weight-streaming decode kernel */
    VTC_FLAG_NO_FUSE = 1u << 2,  /* disable RMSNorm/SiLU*Mul/residual and elementwise-tree fusion */
    VTC_FLAG_GEMV_LDG = 1u << 3, /* decode GEMV on the LDG split-K kernel instead of the persistent TMA-streamed one */
    VTC_FLAG_NO_TC = 1u << 4,    /* bf16 MatMul with M > 16 on the generic tiled kernel instead of tcgen05 */
    VTC_FLAG_DYNAMIC_POS = 1u << 5 /* decode position read on the device each step (vtc_plan_set_position or
                                      the vtc_run input "__pos", int64[1]); the graph's ScatterND row is the
                                      largest position.  Replaces the reference's static index
                                      (proj/src/vt_rules.cpp:63-109) for multi-step decode. */
};

typedef struct vtc_graph vtc_graph;
typedef struct vtc_plan vtc_plan;
typedef struct vtc_comm vtc_comm;

const char* vtc_last_error(void);
const char* vtc_version(void);

int vtc_graph_parse(const char* json_text, vtc_graph** out);
void vtc_graph_free(vtc_graph* g);
/* Returned strings stay valid until the next call on the same thread. */
int vtc_graph_serialize(vtc_graph* g, const char** json_out);
int vtc_graph_vtog(vtc_graph* g, const char** json_out);

/* Planner (host only, no GPU unless the device oracle is chosen).
 * params_json: MachineParams {"bandwidth","coalesce_unit","kernel_launch_overhead",
 * "noncoalesced_penalty","partial_penalty"} (cost_model.hpp:18-28); NULL or "" = the
 * reference defaults, "b200" = the calibrated B200 parameters.
 * vtc_graph_estimate: selected == NULL && n_selected < 0 -> the all-physical plan.
 *   JSON: total_time, kernels[{node, data_movement, time, reads/writes[{tensor, bytes, factor}]}],
 *   breakdown {data_movement_time, compute_time, ...}.
 * vtc_graph_enumerate: {"ptgs": [{selected, roots, eliminated_ops}]} in the reference's order.
 * vtc_graph_greedy: config {"oracle": "analytic"|"device", "params": <params>|"b200",
 *   "trials": n, "executable": bool} -> {selected, roots, eliminated_ops, total_saving,
 *   final_saving, iterations, oracle_calls, decisions[{iteration, node, edges, saving}]}. */
int vtc_graph_estimate(vtc_graph* g, const int32_t* selected, int32_t n_selected, const char* params_json,
                       const char** json_out);
int vtc_graph_enumerate(vtc_graph* g, int64_t limit, const char** json_out);
int vtc_graph_greedy(vtc_graph* g, const char* config_json, const char** json_out);

int vtc_plan_create(vtc_graph* g, int mode, const int32_t* selected, int32_t n_selected, uint32_t flags,
                    vtc_plan** out);
void vtc_plan_free(vtc_plan* p);
/* JSON: roots, eliminated_ops, selected, resolved map text, launches, bytes
 * (all-physical vs this plan, per reference estimate), data_movement_kernels.
 * dry != 0 plans the launch list without touching the GPU. */
int vtc_plan_info(vtc_plan* p, int dry, const char** json_out);

int vtc_plan_bind_root(vtc_plan* p, const char* tensor, void* dev_ptr);
int vtc_plan_root_ptr(vtc_plan* p, const char* tensor, void** dev_ptr);
int vtc_plan_upload(vtc_plan* p, const char* tensor, const void* host, int64_t bytes, void* stream);
int vtc_plan_download(vtc_plan* p, const char* tensor, void* host, int64_t bytes, void* stream);
/* One step from host buffers -- the drop-in for the reference's
 * execute(g, ptg, inputs) (proj/include/vtelim/executor.hpp:77-83): every
 * input lands in its root with ONE H2D copy (the inputs' roots share a device
 * arena staged through pinned memory), the plan runs as a CUDA-graph replay,
 * each output (physical or virtual) is copied back, and the stream is
 * synchronised before returning.  Inputs not named keep their device contents. */
int vtc_run(vtc_plan* p, int32_t n_in, const char* const* in_ids, const void* const* in_host, const int64_t* in_bytes,
            int32_t n_out, const char* const* out_ids, void* const* out_host, const int64_t* out_bytes, void* stream);
int vtc_plan_prepare(vtc_plan* p);
/* Dynamic-position plans: the following executions write the cache row `pos`
 * and attend over keys [0, pos] (0 <= pos <= the ScatterND row the graph was
 * built with); stream-ordered, no re-planning, the captured graph is reused. */
int vtc_plan_set_position(vtc_plan* p, int64_t pos, void* stream);
int vtc_execute(vtc_plan* p, void* stream);        /* async launches on `stream` (cudaStream_t) */
int vtc_execute_graph(vtc_plan* p, void* stream);  /* CUDA-graph replay of the same launches */
int vtc_plan_num_launches(vtc_plan* p);
/* Same launches with a CUDA event between each; ms[i] = device time of launch
 * record i (vtc_plan_info "launches" order).  For measurement only. */
int vtc_execute_timed(vtc_plan* p, void* stream, float* ms, int32_t n);
/* Device timeline of the launches when the plan was prepared with VTC_TRACE=1
 * in the environment: out[8i] / out[8i+1] = first CTA entry / last CTA exit
 * (globaltimer ns) of launch i, out[8i+2..8i+7] = kernel-specific checkpoints
 * (latest CTA; 0 if unused), accumulated over executions since the last call
 * (which resets it).  Returns the number of launches, 0 when tracing is
 * off.  For measurement only. */
int vtc_plan_trace(vtc_plan* p, uint64_t* out, int32_t n);

/* Host evaluation (no GPU) of a tensor's resolved map over its whole index
 * space in row-major order: targets[i] = index into the sorted target list
 * (vtc_plan_map_json "targets"), offsets[i] = element offset.  lowered != 0
 * evaluates the device descriptor instead of the symbolic map. */
int vtc_map_eval(vtc_plan* p, const char* tensor, int lowered, int32_t* targets, int64_t* offsets, int64_t cap);
int vtc_plan_map_json(vtc_plan* p, const char* tensor, const char** json_out);
/* Analyses of a tensor's resolved map (IndexMap::contiguity / injective / unique_elems /
 * is_total, proj/include/vtelim/mapping.hpp:43-51, 100-125):
 * {injective, unique_elems, is_total, min_contiguous_dim, contiguous_run_elems, class, type}. */
int vtc_plan_map_analyze(vtc_plan* p, const char* tensor, int64_t elem_size, int64_t coalesce_unit,
                         const char** json_out);

/* Tensor-parallel plans (SURVEY.md §8 e): one NCCL communicator per process /
 * GPU.  Rank 0 creates the 128-byte unique id, the host side distributes it
 * (any channel), every rank calls vtc_comm_init on its current CUDA device.
 * The plan's AllReduce nodes then run ncclAllReduce(sum) on the plan's stream;
 * without a communicator an AllReduce is the single-rank identity.  NCCL is
 * resolved at run time (libnccl.so.2). */
int vtc_comm_unique_id(void* out, int32_t bytes);
int vtc_comm_init(const void* unique_id, int32_t bytes, int32_t nranks, int32_t rank, vtc_comm** out);
void vtc_comm_free(vtc_comm* c);
int vtc_plan_set_comm(vtc_plan* p, vtc_comm* c);
/* Host-bridged communicator: every AllReduce of the plan copies its buffer to
 * pinned host memory, calls fn(user, buf, count, dtype) from a stream host node
 * (dtype: 0 f64, 1 f32, 2 i64, 3 bf16; fn sums buf over the ranks in place with
 * the caller's own collective -- MPI, gloo, ... -- and returns 0), and copies it
 * back.  For ranks that share a GPU (multi-process tests) or have no NCCL; fn
 * must not call CUDA.  Same role as vtc_comm_init (SURVEY.md §8 e). */
typedef int (*vtc_allreduce_fn)(void* user, void* buf, int64_t count, int32_t dtype);
int vtc_comm_init_host(vtc_allreduce_fn fn, void* user, int32_t nranks, int32_t rank, vtc_comm** out);

/* Low-level kernel entry: dst[map_dst(I)] = src[map_src(I)] over dst->shape. */
int vtc_launch_gather_copy(const vtc_map* dst, const vtc_map* src, int32_t elem_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VTC_H */
