// Host-side helpers shared by the libgsicp translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

#include <mutex>
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

// A value per CUDA device, computed once per device on first use (thread-safe: std::call_once)
// and immutable afterwards — device properties and kernel occupancies, which may differ between
// the devices one process drives.  This is the library's only process-wide state besides
// thread-local diagnostics (gsicp.h, "State").
template <typename T>
struct PerDevice {
    static constexpr int kMaxDevices = 64;
    std::once_flag once[kMaxDevices];
    T value[kMaxDevices];
    template <typename F>
    const T &get(F &&compute) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
        std::call_once(once[dev], [&] { value[dev] = compute(dev); });
        return value[dev];
    }
};

inline int num_sms() {
    static PerDevice<int> cache;
    return cache.get([](int dev) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return sms > 0 ? sms : 148;
    });
}

inline unsigned blocks_for(long long n, int threads) { return (unsigned)((n + threads - 1) / threads); }

// Programmatic dependent launch (sm_90+): the kernel may be launched while its stream
// predecessor is still running and waits for it in-kernel (pdl_wait() at its top, before any
// dependent read), which hides the launch latency between consecutive kernels of the frame
// (CUDA-graph edges included).  Off only while a conditional-node body is being captured.
inline bool &pdl_suspended() {  // set while capturing into a conditional-node body
    static thread_local bool off = false;
    return off;
}
inline bool pdl_enabled() { return !pdl_suspended(); }

// Launch priorities: the frame's critical path (A1 -> A2-A4 -> A6-A9) runs high, the work
// overlapped on side streams (iteration-0 seeds, the fallback hash) low, so that it fills idle
// SM slots instead of slowing the critical kernels.  Honoured in graphs instantiated with
// cudaGraphInstantiateFlagUseNodePriority (gsicp_graph_instantiate).
inline int launch_priority(bool high) {
    static PerDevice<int2> cache;  // (least, greatest) stream priority of the device
    const int2 r = cache.get([](int) {
        int lo = 0, hi = 0;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) lo = hi = 0;
        return make_int2(lo, hi);
    });
    return high ? r.y : r.x;
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
    at[0].val.priority = launch_priority(false);
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
