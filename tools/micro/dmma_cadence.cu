// Microbenchmark (not part of the library): DMMA.8x8x4 throughput per SM for the consumer
// structures of the update GEMM -- warps per SM sub-partition x accumulators per warp, operands
// fixed in registers or re-loaded from shared memory every 36 DMMAs (as the 3M consumer loop).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_cadence dmma_cadence.cu && ./dmma_cadence
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// NA x NB fragments -> NA*NB accumulators; LDS=1: a, b re-read from shared memory every step
template <int NA, int NB, bool LDS>
__global__ void kern(double *out, int iters) {
    __shared__ double sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 1e-3 * (i % 7);
    __syncthreads();
    double a[NA], b[NB], c[NA][NB][2];
#pragma unroll
    for (int i = 0; i < NA; i++) a[i] = 1e-3 * (threadIdx.x + i);
#pragma unroll
    for (int j = 0; j < NB; j++) b[j] = 1.0 - 1e-3 * j;
#pragma unroll
    for (int i = 0; i < NA; i++)
#pragma unroll
        for (int j = 0; j < NB; j++) c[i][j][0] = c[i][j][1] = 0.0;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; it++) {
        if (LDS) {
            const int o = ((it & 7) * 64 + lane * 2) & 2047;
#pragma unroll
            for (int i = 0; i < NA; i++) a[i] = sm[(o + i * 97) & 2047];
#pragma unroll
            for (int j = 0; j < NB; j++) b[j] = sm[(o + 1000 + j * 61) & 2047];
        }
#pragma unroll
        for (int i = 0; i < NA; i++)
#pragma unroll
            for (int j = 0; j < NB; j++) dmma(c[i][j][0], c[i][j][1], a[i], b[j]);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NA; i++)
#pragma unroll
        for (int j = 0; j < NB; j++) s += c[i][j][0] + c[i][j][1];
    if (s == 1234.5) out[0] = s;
}

// software-pipelined: the next step's operands are loaded before this step's DMMAs
template <int NA, int NB>
__global__ void kern_pipe(double *out, int iters) {
    __shared__ double sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 1e-3 * (i % 7);
    __syncthreads();
    double a[NA], b[NB], an[NA], bn[NB], c[NA][NB][2];
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < NA; i++) a[i] = sm[(lane * 2 + i * 97) & 2047];
#pragma unroll
    for (int j = 0; j < NB; j++) b[j] = sm[(lane * 2 + 1000 + j * 61) & 2047];
#pragma unroll
    for (int i = 0; i < NA; i++)
#pragma unroll
        for (int j = 0; j < NB; j++) c[i][j][0] = c[i][j][1] = 0.0;
    for (int it = 0; it < iters; it++) {
        const int o = (((it + 1) & 7) * 64 + lane * 2) & 2047;
#pragma unroll
        for (int i = 0; i < NA; i++) an[i] = sm[(o + i * 97) & 2047];
#pragma unroll
        for (int j = 0; j < NB; j++) bn[j] = sm[(o + 1000 + j * 61) & 2047];
#pragma unroll
        for (int i = 0; i < NA; i++)
#pragma unroll
            for (int j = 0; j < NB; j++) dmma(c[i][j][0], c[i][j][1], a[i], b[j]);
#pragma unroll
        for (int i = 0; i < NA; i++) a[i] = an[i];
#pragma unroll
        for (int j = 0; j < NB; j++) b[j] = bn[j];
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NA; i++)
#pragma unroll
        for (int j = 0; j < NB; j++) s += c[i][j][0] + c[i][j][1];
    if (s == 1234.5) out[0] = s;
}

template <int NA, int NB>
void run_pipe(const char *name, int warps_per_sm, int sms) {
    double *out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int iters = 20000;
    float best = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
        cudaEventRecord(e0);
        kern_pipe<NA, NB><<<sms, warps_per_sm * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float t;
        cudaEventElapsedTime(&t, e0, e1);
        if (rep > 0 && t < best) best = t;
    }
    const double flops = double(sms) * warps_per_sm * iters * NA * NB * 512.0;
    printf("{\"case\": \"%s\", \"warps_per_smsp\": %d, \"acc\": %d, \"lds\": 1, \"pipelined\": 1, \"tflops\": %.2f}\n",
           name, warps_per_sm / 4, NA * NB, flops / (best * 1e-3) / 1e12);
    cudaFree(out);
}

template <int NA, int NB, bool LDS>
void run(const char *name, int warps_per_sm, int sms) {
    double *out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int iters = 20000;
    float best = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
        cudaEventRecord(e0);
        kern<NA, NB, LDS><<<sms, warps_per_sm * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float t;
        cudaEventElapsedTime(&t, e0, e1);
        if (rep > 0 && t < best) best = t;
    }
    const double flops = double(sms) * warps_per_sm * iters * NA * NB * 512.0;
    printf("{\"case\": \"%s\", \"warps_per_smsp\": %d, \"acc\": %d, \"lds\": %d, \"tflops\": %.2f}\n", name,
           warps_per_sm / 4, NA * NB, int(LDS), flops / (best * 1e-3) / 1e12);
    cudaFree(out);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<3, 12, false>("36acc fixed", 4, sms);
    run<3, 12, false>("36acc fixed", 8, sms);
    run<3, 12, true>("36acc lds", 4, sms);
    run<3, 12, true>("36acc lds", 8, sms);
    run<3, 12, true>("36acc lds", 12, sms);
    run<2, 12, true>("24acc lds", 12, sms);
    run_pipe<3, 12>("36acc lds pipelined", 4, sms);
    run_pipe<3, 12>("36acc lds pipelined", 8, sms);
    run<2, 4, false>("8acc fixed", 16, sms);
    return 0;
}
