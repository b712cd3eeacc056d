// stream_probe.cu -- microbenchmark for the correction-matvec access pattern
// (DESIGN.md "K4"): pure streaming of the 20 B/pair (int32 index + complex128
// coefficient) stream vs the same stream with the q gathers of a CSR matvec.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/stream_probe.cu -o stream_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void k_stream(const int* __restrict__ src, const double2* __restrict__ coef, long long n, double* out) {
    double acc = 0;
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += stride) {
        double2 c = __ldcs(coef + p);
        acc += c.x + c.y + __ldcs(src + p);
    }
    if (acc == 12345.0) *out = acc;
}

template <int U>
__global__ void k_stream_u(const int* __restrict__ src, const double2* __restrict__ coef, long long n, double* out) {
    double acc = 0;
    long long stride = (long long)gridDim.x * blockDim.x * U;
    for (long long b = (blockIdx.x * (long long)blockDim.x) * U + threadIdx.x; b < n; b += stride) {
        double2 c[U];
        int s[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            long long p = b + k * blockDim.x;
            c[k] = p < n ? __ldcs(coef + p) : make_double2(0, 0);
            s[k] = p < n ? __ldcs(src + p) : 0;
        }
#pragma unroll
        for (int k = 0; k < U; ++k) acc += c[k].x + c[k].y + s[k];
    }
    if (acc == 12345.0) *out = acc;
}

// gathers q[src] (q small, L2 resident) -- the matvec's access pattern without rows
template <int U>
__global__ void k_gather_u(const int* __restrict__ src, const double2* __restrict__ coef, const double2* __restrict__ q,
                           long long n, double* out) {
    double ar = 0, ai = 0;
    long long stride = (long long)gridDim.x * blockDim.x * U;
    for (long long b = (blockIdx.x * (long long)blockDim.x) * U + threadIdx.x; b < n; b += stride) {
        double2 c[U];
        int s[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            long long p = b + k * blockDim.x;
            c[k] = p < n ? __ldcs(coef + p) : make_double2(0, 0);
            s[k] = p < n ? __ldcs(src + p) : 0;
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            double2 v = q[s[k]];
            ar += c[k].x * v.x - c[k].y * v.y;
            ai += c[k].x * v.y + c[k].y * v.x;
        }
    }
    if (ar == 12345.0) *out = ar + ai;
}

int main(int argc, char** argv) {
    long long n = argc > 1 ? atoll(argv[1]) : 14514148LL;
    int nq = argc > 2 ? atoi(argv[2]) : 65536;
    int* src;
    double2 *coef, *q;
    double* out;
    cudaMalloc(&src, n * 4);
    cudaMalloc(&coef, n * 16);
    cudaMalloc(&q, nq * 16);
    cudaMalloc(&out, 8);
    std::vector<int> hs(n);
    // locality like the real matrix: rows of ~221 sources near the row index
    for (long long p = 0; p < n; ++p) hs[p] = (int)(((p / 221) + (p * 7919) % 512) % nq);
    cudaMemcpy(src, hs.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemset(coef, 0, n * 16);
    cudaMemset(q, 0, nq * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double bytes = n * 20.0;
    auto run = [&](const char* name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 20;
        printf("%-28s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
    int sms = 148;
    for (int bpsm : {4, 8, 16}) {
        char nm[64];
        snprintf(nm, 64, "stream u1 %d blk/SM", bpsm);
        run(nm, [&] { k_stream<<<sms * bpsm, 256>>>(src, coef, n, out); });
        snprintf(nm, 64, "stream u4 %d blk/SM", bpsm);
        run(nm, [&] { k_stream_u<4><<<sms * bpsm, 256>>>(src, coef, n, out); });
        snprintf(nm, 64, "gather u4 %d blk/SM", bpsm);
        run(nm, [&] { k_gather_u<4><<<sms * bpsm, 256>>>(src, coef, q, n, out); });
        snprintf(nm, 64, "gather u8 %d blk/SM", bpsm);
        run(nm, [&] { k_gather_u<8><<<sms * bpsm, 256>>>(src, coef, q, n, out); });
    }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
