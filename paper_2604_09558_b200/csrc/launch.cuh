// Host-side kernel launch with programmatic dependent launch (PDL).
//
// Every vtc kernel stages its parameter block, then calls dev::pdl_wait()
// before touching data written by earlier kernels, and
// dev::pdl_launch_dependents() once its own CTAs are resident.  Launching
// with programmaticStreamSerialization lets the next kernel of the plan be
// scheduled while the current one drains, so launch latency and parameter
// staging overlap the previous kernel's tail (also inside CUDA graphs).
// VTC_NO_PDL=1 in the environment launches with plain stream order (A/B).
#pragma once

#include <cstdlib>
#include <mutex>
#include <set>

#include <cuda_runtime.h>

namespace vtc {

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("VTC_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

// Opt a kernel into the largest dynamic shared memory it can use, once.
// (Setting the attribute per launch to that launch's size is wrong under CUDA
// graphs: the attribute is read at replay, after a later capture may have
// lowered it for a launch with a smaller footprint.)
template <typename... KArgs>
inline void allow_max_smem(void (*kern)(KArgs...)) {
    // once per kernel function (a function-local static would be shared by every
    // kernel with the same signature)
    static std::mutex mu;
    static std::set<const void*> done;
    std::lock_guard<std::mutex> lock(mu);
    if (!done.insert(reinterpret_cast<const void*>(kern)).second) return;
    cudaFuncAttributes a{};
    cudaFuncGetAttributes(&a, kern);
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - int(a.sharedSizeBytes));
}

// Set by the executor before a dynamic-position plan's first launch: that
// launch is stream-serialised (no PDL), so every kernel of the step starts after
// the position write that precedes the plan has completed.  Consumed by the
// next launch_k on this thread.
inline thread_local bool tl_serialize_next = false;

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pdl_enabled() && !tl_serialize_next) ? 1 : 0;
    tl_serialize_next = false;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// The same with a thread-block cluster of `cx` CTAs along x (CTA pairs for cta_group::2).
template <typename... KArgs, typename... Args>
inline void launch_k_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, unsigned cx,
                             Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cx;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pdl_enabled() && !tl_serialize_next) ? 2 : 1;
    tl_serialize_next = false;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace vtc
