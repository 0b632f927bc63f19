// Host-side helpers shared by the libgsicp translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

namespace gsicp {

// kernels launched by the calling thread (diagnostic counter behind gsicp_kernel_launch_count)
void note_launch(int n = 1);
// thread-local error detail behind gsicp_last_error
void set_error(const char *fmt, ...);

// diagnostic kernel timer (gsicp_debug_kernel_timer): when enabled on the calling thread, the
// hot kernels record a start / stop CUDA event pair around their launch (graph-capture safe)
enum KTimerId { KT_KNN_SEARCH = 0, KT_ALIGN = 1, KT_SEED = 2, KT_BP = 3, KT_COVS = 4, KT_WIDE = 5, KT_TAIL = 6, KT_COUNT = 7 };
void ktimer_mark(int id, bool stop, cudaStream_t s);

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller workspace; with base == nullptr it only measures.
struct Carver {
    char *base;
    size_t off = 0;
    explicit Carver(void *b) : base(static_cast<char *>(b)) {}
    template <typename T>
    T *take(size_t count) {
        off = align_up(off);
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
    size_t bytes() const { return align_up(off); }
};

inline int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

inline unsigned blocks_for(long long n, int threads) { return (unsigned)((n + threads - 1) / threads); }

// Programmatic dependent launch (sm_90+): the kernel may be launched while its stream
// predecessor is still running and waits for it in-kernel (pdl_wait() at its top, before any
// dependent read), which hides the launch latency between consecutive kernels of the frame
// (CUDA-graph edges included).  GSICP_PDL=0 turns it off (A/B).
inline bool &pdl_suspended() {  // set while capturing into a conditional-node body
    static thread_local bool off = false;
    return off;
}
inline bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("GSICP_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1 && !pdl_suspended();
}

// Launch priorities: the frame's critical path (A1 -> A2-A4 -> A6-A9) runs high, the work
// overlapped on side streams (iteration-0 seeds, the fallback hash) low, so that it fills idle
// SM slots instead of slowing the critical kernels.  Honoured in graphs instantiated with
// cudaGraphInstantiateFlagUseNodePriority (gsicp_graph_instantiate).  GSICP_PRIO=0: off.
inline int launch_priority(bool high) {
    static int lo = 1, hi = 1, on = -1;
    if (on < 0) {
        const char *e = getenv("GSICP_PRIO");
        on = (e && e[0] == '0') ? 0 : 1;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) on = 0;
    }
    if (!on) return 0;
    return high ? hi : lo;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    at[1].id = cudaLaunchAttributePriority;
    at[1].val.priority = launch_priority(true);
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// a launch at low priority (work overlapped with the critical path on a side stream)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_low(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    static int flip = -1;  // GSICP_SIDE_HIGH=1: side work at high priority too (A/B)
    if (flip < 0) {
        const char *e = getenv("GSICP_SIDE_HIGH");
        flip = (e && e[0] == '1') ? 1 : 0;
    }
    at[0].val.priority = launch_priority(flip == 1);
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace gsicp

#define GSICP_LAUNCH_CHECK(what)                                                    \
    do {                                                                            \
        cudaError_t e_ = cudaGetLastError();                                        \
        if (e_ != cudaSuccess) {                                                    \
            ::gsicp::set_error("%s: %s", what, cudaGetErrorString(e_));             \
            return e_;                                                              \
        }                                                                           \
    } while (0)
