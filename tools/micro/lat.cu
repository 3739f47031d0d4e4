// Dependent-chain latencies on sm_100a (one warp): DADD, DMUL, DFMA, SHFL.IDX (64-bit as 2 x 32),
// IADD, and a DMUL + DADD pair; cycles per op from clock64 around 1024 chained ops.
#include <cstdio>
__global__ void lat(double *out, long long *cyc, double a, double b, int it) {
    double x = a, y = b;
    long long t0, t1;
    int lane = threadIdx.x & 31;
#define CHAIN(name, k, body)                                \
    t0 = clock64();                                         \
    for (int i = 0; i < it; i++) { body; }                  \
    t1 = clock64();                                         \
    if (threadIdx.x == 0) cyc[k] = t1 - t0;
    CHAIN("dadd", 0, x = __dadd_rn(x, y));
    CHAIN("dmul", 1, x = __dmul_rn(x, y));
    CHAIN("dfma", 2, x = __fma_rn(x, y, a));
    CHAIN("shfl", 3, x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31));
    int v = int(a);
    CHAIN("iadd", 4, v = v * 3 + lane);
    CHAIN("dmul+dadd", 5, x = __dadd_rn(__dmul_rn(x, y), a));
    CHAIN("dsetp+sel", 6, x = (x >= a) ? __dadd_rn(x, y) : __dmul_rn(x, y));
    CHAIN("bexp-roundtrip", 7, { int e = (__double2hiint(x) >> 20) & 0x7ff; x = __hiloint2double(__double2hiint(x) + (e & 1), __double2loint(x)); });
    out[threadIdx.x] = x + v;
}
int main() {
    double *o; long long *c, h[8];
    cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 8 * 8);
    const int it = 4096;
    lat<<<1, 32>>>(o, c, 1.0000001, 0.9999999, it);
    lat<<<1, 32>>>(o, c, 1.0000001, 0.9999999, it);
    cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    const char *n[8] = {"dadd", "dmul", "dfma", "shfl(f64)", "imad", "dmul+dadd", "dsetp+sel+dop", "bexp int roundtrip"};
    for (int k = 0; k < 8; k++) printf("%-22s %.1f cycles/op\n", n[k], double(h[k]) / it);
    return 0;
}
