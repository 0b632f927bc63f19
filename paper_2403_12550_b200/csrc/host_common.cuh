// Host-side helpers shared by the libgsicp translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace gsicp {

// kernels launched by the calling thread (diagnostic counter behind gsicp_kernel_launch_count)
void note_launch(int n = 1);
// thread-local error detail behind gsicp_last_error
void set_error(const char *fmt, ...);

// diagnostic kernel timer (gsicp_debug_kernel_timer): when enabled on the calling thread, the
// hot kernels record a start / stop CUDA event pair around their launch (graph-capture safe)
enum KTimerId { KT_KNN_SEARCH = 0, KT_ALIGN = 1, KT_SEED = 2, KT_COUNT = 3 };
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

}  // namespace gsicp

#define GSICP_LAUNCH_CHECK(what)                                                    \
    do {                                                                            \
        cudaError_t e_ = cudaGetLastError();                                        \
        if (e_ != cudaSuccess) {                                                    \
            ::gsicp::set_error("%s: %s", what, cudaGetErrorString(e_));             \
            return e_;                                                              \
        }                                                                           \
    } while (0)
