// condgraph.cuh -- "run the head; run the body only if a device flag says so" as ONE CUDA graph:
// the head's kernels, a 1-thread kernel that sets a conditional handle from the flag, and a
// conditional IF node whose body holds the fallback kernels.  The body's kernels are not launched
// at all when the flag is 0 -- no empty grids -- and nothing waits on the host.  One instantiated
// graph per argument set (pointers, sizes, device), cached and replayed on later calls; the
// caller's stream order is kept (cudaGraphLaunch on it).
#pragma once

#include <cstring>
#include <mutex>
#include <vector>

#include "csrk_internal.cuh"

namespace csrk {

struct CondKey {
    uint64_t w[16];
    int n;
    bool operator==(const CondKey &o) const { return n == o.n && !memcmp(w, o.w, sizeof(uint64_t) * n); }
};

inline CondKey cond_key(std::initializer_list<uint64_t> v)
{
    CondKey k{};
    for (uint64_t x : v) if (k.n < 16) k.w[k.n++] = x;
    return k;
}

// cond = (*flag != 0), evaluated on the device when the graph runs
__global__ void k_set_cond(cudaGraphConditionalHandle h, const int *flag);

cudaStream_t cond_capture_stream(int which);   // private non-blocking streams for capture (per device)

// Looks up / builds the graph for `key` (tag: the calling op) and launches it on s.  head(cs) and
// body(cs) enqueue on the capture stream they are given and return a csrk status.
template <typename Head, typename Body>
int cond_graph_run(int tag, const CondKey &key, cudaStream_t s, const int *flag, Head head, Body body)
{
    struct Entry {
        int tag, dev;
        CondKey key;
        cudaGraphExec_t exec;
        uint64_t head_kernels;   // kernels of the head (+ the condition setter), counted per replay
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    int dev = 0;
    CSRK_CUDA(cudaGetDevice(&dev));
    cudaGraphExec_t exec = nullptr;
    uint64_t nk = 0;
    {
        std::lock_guard<std::mutex> g(mu);
        for (auto &e : cache)
            if (e.tag == tag && e.dev == dev && e.key == key) {
                exec = e.exec;
                nk = e.head_kernels;
            }
    }
    if (exec) {
        g_launches.fetch_add(nk, std::memory_order_relaxed);
    } else {
        cudaStream_t cs = cond_capture_stream(0), cb = cond_capture_stream(1);
        if (!cs || !cb) return CSRK_ERR_CUDA;
        cudaGraph_t graph = nullptr, body_g = nullptr;
        int st = CSRK_OK;
        const uint64_t l0 = g_launches.load(std::memory_order_relaxed);
        CSRK_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        st = head(cs);
        cudaGraph_t cap = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t ndeps = 0;
        cudaStreamCaptureStatus cst;
        cudaGraphConditionalHandle h = 0;
        cudaGraphNode_t cnode = nullptr;
        if (st == CSRK_OK && cudaStreamGetCaptureInfo_v3(cs, &cst, nullptr, &cap, nullptr, nullptr, nullptr) != cudaSuccess)
            st = CSRK_ERR_CUDA;
        if (st == CSRK_OK && cudaGraphConditionalHandleCreate(&h, cap, 0, cudaGraphCondAssignDefault) != cudaSuccess)
            st = CSRK_ERR_CUDA;
        if (st == CSRK_OK) {
            k_set_cond<<<1, 1, 0, cs>>>(h, flag);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            if (cudaGetLastError() != cudaSuccess) st = CSRK_ERR_CUDA;
        }
        const uint64_t head_kernels = g_launches.load(std::memory_order_relaxed) - l0;
        if (st == CSRK_OK &&
            cudaStreamGetCaptureInfo_v3(cs, &cst, nullptr, &cap, &deps, nullptr, &ndeps) != cudaSuccess)
            st = CSRK_ERR_CUDA;
        if (st == CSRK_OK) {
            cudaGraphNodeParams p{};
            p.type = cudaGraphNodeTypeConditional;
            p.conditional.handle = h;
            p.conditional.type = cudaGraphCondTypeIf;
            p.conditional.size = 1;
            if (cudaGraphAddNode(&cnode, cap, deps, ndeps, &p) != cudaSuccess) st = CSRK_ERR_CUDA;
            else body_g = p.conditional.phGraph_out[0];
        }
        if (st == CSRK_OK && cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies) !=
                                 cudaSuccess)
            st = CSRK_ERR_CUDA;
        const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
        if (st == CSRK_OK && ce != cudaSuccess) st = CSRK_ERR_CUDA;
        if (st == CSRK_OK) {
            // the body: captured into the conditional node's graph on a second stream
            if (cudaStreamBeginCaptureToGraph(cb, body_g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
                cudaSuccess) {
                st = CSRK_ERR_CUDA;
            } else {
                st = body(cb);
                cudaGraph_t tmp = nullptr;
                if (cudaStreamEndCapture(cb, &tmp) != cudaSuccess && st == CSRK_OK) st = CSRK_ERR_CUDA;
            }
        }
        if (st == CSRK_OK && cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) st = CSRK_ERR_CUDA;
        if (graph) cudaGraphDestroy(graph);
        if (st != CSRK_OK) {
            (void)cudaGetLastError();
            return st;
        }
        std::lock_guard<std::mutex> g(mu);
        if (cache.size() >= 16) {
            cudaGraphExecDestroy(cache.front().exec);
            cache.erase(cache.begin());
        }
        cache.push_back(Entry{tag, dev, key, exec, head_kernels});
    }
    CSRK_CUDA(cudaGraphLaunch(exec, s));
    return CSRK_OK;
}

}  // namespace csrk
