// Microbenchmark: fp64 FMA and DADD throughput / latency per SM (perf experiment only).
#include <cstdio>
template <int CHAINS>
__global__ void k(double* out, int iters, double a) {
    double x[CHAINS];
    for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) x[i] = fma(x[i], a, 1e-9);
    double s = 0;
    for (int i = 0; i < CHAINS; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}
template <int CHAINS>
void run(int threads, int ctas_per_sm) {
    double* out; cudaMalloc(&out, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 4096;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k<CHAINS><<<sms * ctas_per_sm, threads>>>(out, iters, 0.999999);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = double(sms) * ctas_per_sm * threads * iters * CHAINS;
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("chains %d threads %4d ctas/SM %d: %.2f DFMA/clk/SM  (%.2f T DFMA/s at max clk); per-thread cyc/op %.1f\n",
           CHAINS, threads, ctas_per_sm, ops / cyc / sms, ops / (ms * 1e-3) / 1e12, cyc / (double(iters) * CHAINS));
}
int main() {
    run<1>(32, 1);
    run<4>(32, 1);
    run<8>(256, 1);
    run<8>(512, 2);
    run<4>(1024, 2);
    return 0;
}
