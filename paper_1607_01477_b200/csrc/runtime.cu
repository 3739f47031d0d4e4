// runtime.cu -- definitions of the library-wide runtime state (see runtime.cuh).
#include <stdio.h>
#include <stdlib.h>

#include <mutex>

#include "runtime.cuh"

namespace mstrsm {
namespace rt {

cudaStream_t g_stream = nullptr;
int g_cta_cap = 0;
std::atomic<int64_t> g_launches{0};
int *g_flag = nullptr;                 // device: non-finite input seen
char g_errmsg[512] = "no error";
int g_num_sms = 0;
bool g_debug_sync = getenv("MSTRSM_DEBUG_SYNC") != nullptr;   // synchronise + log after each diag launch
int g_diag_force_fb = getenv("MSTRSM_DIAG_FORCE_FALLBACK") != nullptr;   // testing: synchronous diag path
int g_pdl = [] { const char *e = getenv("MSTRSM_PDL"); return (e && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 2; }();
static std::mutex g_mu;
bool g_prof = false;
std::vector<ProfRec> g_prof_recs;
std::vector<cudaEvent_t> g_ev_pool;

static thread_local cudaError_t g_last_err = cudaSuccess;
int set_cuda_error(cudaError_t e, const char *where) {
    snprintf(g_errmsg, sizeof(g_errmsg), "CUDA error in %s: %s", where, cudaGetErrorString(e));
    g_last_err = e;
    return 1;
}
cudaError_t last_cuda_error() { return g_last_err; }

int ensure_init() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_flag) return 0;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
    // keep stream-ordered allocations cached between calls (workspace, host-entry staging)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    CK(cudaMalloc(&g_flag, sizeof(int)));
    CK(cudaMemset(g_flag, 0, sizeof(int)));
    return 0;
}

cudaEvent_t ev_get() {
    if (!g_ev_pool.empty()) { cudaEvent_t e = g_ev_pool.back(); g_ev_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

}  // namespace rt
}  // namespace mstrsm
