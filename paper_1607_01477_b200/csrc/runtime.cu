// runtime.cu -- definitions of the library-wide runtime state (see runtime.cuh).
#include <stdio.h>
#include <stdlib.h>

#include <mutex>

#include "runtime.cuh"

namespace mstrsm {
namespace rt {

thread_local cudaStream_t g_stream = nullptr;
thread_local int g_cta_cap = 0;
std::atomic<int64_t> g_launches{0};
thread_local int *g_flag = nullptr;
thread_local char g_errmsg[512] = "no error";
thread_local int g_num_sms = 0;
thread_local int g_dev = -1;
bool g_debug_sync = getenv("MSTRSM_DEBUG_SYNC") != nullptr;   // synchronise + log after each diag launch
int g_diag_force_fb = getenv("MSTRSM_DIAG_FORCE_FALLBACK") != nullptr;   // testing: synchronous diag path
int g_pdl = [] { const char *e = getenv("MSTRSM_PDL"); return (e && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 2; }();
thread_local bool g_prof = false;
thread_local std::vector<ProfRec> g_prof_recs;
thread_local std::vector<cudaEvent_t> g_ev_pool;

static thread_local cudaError_t g_last_err = cudaSuccess;
int set_cuda_error(cudaError_t e, const char *where) {
    snprintf(g_errmsg, sizeof(g_errmsg), "CUDA error in %s: %s", where, cudaGetErrorString(e));
    g_last_err = e;
    return 1;
}
cudaError_t last_cuda_error() { return g_last_err; }

// Per (thread, device) context.  Devices beyond kMaxDev are refused.
namespace {
constexpr int kMaxDev = 64;
struct Ctx {
    bool init = false;
    int sms = 0;
    int *flag = nullptr;
    DevRes res;
};
thread_local Ctx t_ctx[kMaxDev];
std::atomic<uint64_t> g_pool_done{0};
}  // namespace

int ensure_init() {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDev) return set_cuda_error(cudaErrorInvalidDevice, "ensure_init (device index)");
    Ctx &c = t_ctx[dev];
    g_dev = dev;
    if (!c.init) {
        CK(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev));
        if (first_on_device(g_pool_done)) {
            // keep stream-ordered allocations cached between calls (workspace, host-entry staging)
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        }
        CK(cudaMalloc(&c.flag, sizeof(int)));
        CK(cudaMemset(c.flag, 0, sizeof(int)));
        c.init = true;
    }
    g_flag = c.flag;
    g_num_sms = c.sms;
    return 0;
}

DevRes *dev_res() {
    if (g_dev < 0 && ensure_init()) return nullptr;
    DevRes &r = t_ctx[g_dev].res;
    if (!r.side) {
        cudaError_t e = cudaStreamCreateWithFlags(&r.side, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r.h2d, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r.d2h, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r.comm, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.ev_d, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.ev_rest, cudaEventDisableTiming);
        if (e != cudaSuccess) {
            set_cuda_error(e, "dev_res (stream / event creation)");
            r = DevRes{};
            return nullptr;
        }
    }
    return &r;
}

cudaEvent_t ev_get() {
    if (!g_ev_pool.empty()) { cudaEvent_t e = g_ev_pool.back(); g_ev_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

}  // namespace rt
}  // namespace mstrsm

#ifdef MSTRSM_PHASE_TIMES
// Phase-time buffers of the experiment build (0: diagonal kernels, 1: update GEMM): 512 launches x
// 256 CTAs x 16 slots each (rings).
namespace mstrsm {
namespace rt {
static long long *g_pt[2] = {nullptr, nullptr};
static int g_pt_next[2] = {0, 0};
static const size_t kPtBytes = size_t(512) * 256 * 16 * 8;
long long *phase_next(int kind) {
    if (!g_pt[kind]) {
        if (cudaMalloc(&g_pt[kind], kPtBytes) != cudaSuccess) return nullptr;
        cudaMemset(g_pt[kind], 0, kPtBytes);
    }
    long long *p = g_pt[kind] + size_t(g_pt_next[kind] % 512) * 256 * 16;
    g_pt_next[kind]++;
    return p;
}
}  // namespace rt
}  // namespace mstrsm
extern "C" int mstrsm_phase_read2(int kind, long long *host, int64_t n_launches, int reset) {
    using namespace mstrsm::rt;
    cudaDeviceSynchronize();
    if (g_pt[kind] && n_launches > 0)
        cudaMemcpy(host, g_pt[kind], size_t(n_launches < 512 ? n_launches : 512) * 256 * 16 * 8, cudaMemcpyDeviceToHost);
    const int used = g_pt_next[kind];
    if (reset) {
        g_pt_next[kind] = 0;
        if (g_pt[kind]) cudaMemset(g_pt[kind], 0, kPtBytes);
    }
    return used;
}
extern "C" int mstrsm_phase_read(long long *host, int64_t n_launches, int reset) {
    return mstrsm_phase_read2(0, host, n_launches, reset);
}
#endif
