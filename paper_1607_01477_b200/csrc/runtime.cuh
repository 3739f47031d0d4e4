// runtime.cuh -- library-wide runtime state shared by the translation units of libmstrsm:
// the current stream, launch counter, error string, live profiling (CUDA events on the
// launching stream) and the launcher prototypes of the kernels compiled in separate units.
#pragma once
#include <utility>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <vector>

#include "common.cuh"
#include "diag_kernel.cuh"
#include "gemm_kernel.cuh"

namespace mstrsm {
namespace rt {

// Library state is per calling thread and per device: every API call runs
// ensure_init(), which binds the thread-local pointers below to the calling thread's context on
// the current device.  Two host threads (or one thread driving two GPUs) therefore never share a
// stream, event, side stream or status flag.  Only the NCCL communicator of the multi-GPU entry
// points is process-wide (one communicator per process, one process per GPU).
extern thread_local cudaStream_t g_stream;   // the calling thread's library stream (mstrsm_set_stream)
// > 0: launches of the update GEMM and the diagonal kernel use at most this many CTAs (one per
// SM), leaving the other SMs to a kernel running concurrently on another stream (look-ahead)
extern thread_local int g_cta_cap;
extern std::atomic<int64_t> g_launches;
extern thread_local int *g_flag;             // non-finite input seen (this thread, this device)
extern thread_local char g_errmsg[512];
extern thread_local int g_num_sms;
extern thread_local int g_dev;               // the device ensure_init() bound
extern bool g_debug_sync;
extern int g_diag_force_fb;
extern int g_pdl;            // MSTRSM_PDL: programmatic dependent launch of the diag / GEMM kernels

// Streams and events of the calling thread on the current device: the look-ahead's side stream
// and events, the host-buffer entries' copy streams.  Created on first use.
struct DevRes {
    cudaStream_t side = nullptr, h2d = nullptr, d2h = nullptr, comm = nullptr;
    cudaEvent_t ev_d = nullptr, ev_rest = nullptr;
};
DevRes *dev_res();
#ifdef MSTRSM_PHASE_TIMES
long long *phase_next(int kind = 0);   // the next launch's row block of the phase-time buffer (0 diag, 1 GEMM)
#endif           // nullptr (and the error recorded) if creation fails
// True the first time it is asked for the current device (per-device one-shot setup such as
// cudaFuncSetAttribute; bit d of mask = device d done).
inline bool first_on_device(std::atomic<uint64_t> &mask) {
    const uint64_t bit = uint64_t(1) << (g_dev & 63);
    return (mask.fetch_or(bit) & bit) == 0;
}

// Launch with the programmatic-stream-serialization attribute when g_pdl >= lvl (1: the diagonal
// and update-GEMM kernels, 2: also the solve's finalize and the Lanczos kernels): the grid may be
// scheduled while the preceding kernel in the stream drains; the kernel calls pdl_wait() before
// touching global memory, which returns once that kernel has completed and its writes are visible.
template <typename... KArgs, typename... Args>
cudaError_t launch_k_lvl(int lvl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                         Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl >= lvl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    return launch_k_lvl(1, kern, grid, block, smem, st, std::forward<Args>(args)...);
}


int set_cuda_error(cudaError_t e, const char *where);
cudaError_t last_cuda_error();   // the error recorded by the last set_cuda_error on this thread
int ensure_init();

#define CK(call)                                                       \
    do {                                                               \
        cudaError_t e_ = (call);                                       \
        if (e_ != cudaSuccess) return ::mstrsm::rt::set_cuda_error(e_, #call); \
    } while (0)
#define CK_LAUNCH(name)                                                \
    do {                                                               \
        ::mstrsm::rt::g_launches.fetch_add(1, std::memory_order_relaxed); \
        cudaError_t e_ = cudaGetLastError();                           \
        if (e_ != cudaSuccess) return ::mstrsm::rt::set_cuda_error(e_, name); \
    } while (0)

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// live kernel profiling
enum { PK_GEMM = 0, PK_DIAG = 1, PK_OTHER = 2, PK_N = 3 };
struct ProfRec { int kind; cudaEvent_t e0, e1; double flops; };
extern thread_local bool g_prof;
extern thread_local std::vector<ProfRec> g_prof_recs;
extern thread_local std::vector<cudaEvent_t> g_ev_pool;
cudaEvent_t ev_get();
struct ProfScope {
    ProfRec r{};
    bool on;
    ProfScope(int kind, double flops) : on(g_prof) {
        if (!on) return;
        r.kind = kind; r.flops = flops; r.e0 = ev_get(); r.e1 = ev_get();
        cudaEventRecord(r.e0, g_stream);
    }
    ~ProfScope() {
        if (!on) return;
        cudaEventRecord(r.e1, g_stream);
        g_prof_recs.push_back(r);
    }
};

template <typename K>
int occupancy(K kern, int threads, size_t smem) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem) != cudaSuccess) nb = 1;
    return nb > 1 ? nb : 1;
}

// launchers compiled in their own translation units (diag_*.cu, gemm_launch.cu)
template <typename T, bool SAFE, int OP> int launch_diag(const DiagArgs<T> &a, int nb);
template <typename T, bool SAFE> int launch_diag_gen(const DiagArgs<T> &a, int nb);
template <typename T, bool OPC> int launch_gemm(const GemmArgs<T> &g);
bool gemm_presum_enabled();   // complex 3M with precomputed operand sums (gemm_ws3p.cuh)
int gemm_variant();   // 0 = warp-specialised (complex: 3 real products), 1 = classic, 2 = ws 4 products

}  // namespace rt
}  // namespace mstrsm
