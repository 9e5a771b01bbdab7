// Microbenchmark (perf experiment only): dependent-chain latency of DADD, fp64 exp and __ddiv_rn
// on one warp, and of the same ops with 4 / 8 independent chains per thread -- the cost model of
// K2's sequential fp64 row denominators (row_select_kernel).
#include <cstdio>
#include <stdint.h>

template <int OP, int CH>
__global__ void k(double* out, long long* cyc, int n, double seed) {
    double a[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = seed + threadIdx.x * 1e-3 + c;
    const double b = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (OP == 0) a[c] = __dadd_rn(a[c], b);
            else if (OP == 1) a[c] = exp(a[c] * 1e-9);
            else a[c] = __ddiv_rn(b, a[c]);
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += a[c];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int OP, int CH>
void run(const char* name) {
    double* out; long long* cyc; cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
    const int n = 1000;
    k<OP, CH><<<1, 32>>>(out, cyc, n, 1.5);
    k<OP, CH><<<1, 32>>>(out, cyc, n, 1.5);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-8s chains/thread=%d: %.1f cycles per op per chain-step (%.1f per op)\n", name, CH, double(h) / n,
           double(h) / n / CH);
    cudaFree(out); cudaFree(cyc);
}

int main() {
    run<0, 1>("dadd"); run<0, 4>("dadd"); run<0, 8>("dadd");
    run<1, 1>("exp64"); run<1, 4>("exp64");
    run<2, 1>("ddiv"); run<2, 4>("ddiv");
    return 0;
}
