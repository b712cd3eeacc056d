// FP64 pipe probe for the roofline of the on-chip-bound stages (K1, observer pass, FFT, far projection):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_probe.cu -o /tmp/fp64_probe && /tmp/fp64_probe
// (a) dependent DFMA latency in cycles (one warp, one chain);
// (b) DFMA throughput (TFLOP/s, FMA = 2 flops) against warps per SM and independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_fma(double* out, int iters, double a, double b, long long* cyc) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (cyc && threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CH>
static void run(int warps_per_sm, int sms, double* d, long long* dc) {
    const int iters = 20000;
    const int threads = std::min(1024, warps_per_sm * 32), blocks_per_sm = (warps_per_sm * 32 + threads - 1) / threads;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fma<CH><<<sms * blocks_per_sm, threads>>>(d, 100, 1.0000001, 1e-9, nullptr);
    cudaEventRecord(e0);
    k_fma<CH><<<sms * blocks_per_sm, threads>>>(d, iters, 1.0000001, 1e-9, dc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c = 0;
    cudaMemcpy(&c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    const double flops = 2.0 * CH * iters * (double)sms * blocks_per_sm * threads;
    printf("warps/SM %2d chains %d: %.2f TFLOP/s, %.2f cycles per DFMA per warp (%.1f cycles per loop pass)\n", warps_per_sm, CH,
           flops / (ms * 1e-3) / 1e12, (double)c / iters / CH, (double)c / iters);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    long long* dc;
    cudaMalloc(&d, sizeof(double) * sms * 2048 * 2);
    cudaMalloc(&dc, sizeof(long long));
    printf("SMs %d\n", sms);
    k_fma<1><<<1, 32>>>(d, 20000, 1.0000001, 1e-9, dc);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("dependent DFMA latency: %.2f cycles (one warp, one chain)\n", (double)c / 20000);
    for (int w : {4, 8, 12, 16, 32, 64}) {
        run<1>(w, sms, d, dc);
        run<2>(w, sms, d, dc);
        run<4>(w, sms, d, dc);
        run<8>(w, sms, d, dc);
    }
    return 0;
}
