// direct_kernels.cu -- brute-force periodic superposition on the device
// (SURVEY.md 8f rank 4): the reference's accuracy oracle
//   eval_direct          u_m = sum_n G_p(r_m - r_n) q_n          oracle.py:92-97
//   eval_direct_farzone  same with G_p - G_near(i_d)              oracle.py:100-111
//   eval_free_space      sum_n exp(-j k0 r)/(4 pi r) q_n          oracle.py:114-123
// with one converged series per (observer, source) pair (series.cuh).
//
// The reference walks the observers in chunks of 64 (oracle.py:20, :67-87):
// a chunk holding any pair that violates the separation rule
// (_pair_failures, oracle.py:35-59) is skipped -- its potentials stay 0 and
// only its separation failures are reported -- otherwise every pair is
// evaluated and its non-converged pairs are reported.  The 3D lattice lead
// sums a z-image range taken over the whole chunk (pgf.py:394-397), so each
// pair carries its chunk's z extrema.  Pass 1 flags separation per pair and
// counts it per chunk; pass 2 evaluates the pairs of the clean chunks into a
// (chunk rows x N) buffer of G q; pass 3 sums each observer's row in a fixed
// order (warp per observer) -- deterministic, no atomics on values.
#include "series.cuh"

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

#define DIRECT_CHUNK 64   // oracle.py:20 _OBS_CHUNK

// numpy.remainder (npy_divmod): fmod with the sign of the divisor
__device__ __forceinline__ double np_remainder(double a, double b) {
    double mod = fmod(a, b);
    if (mod != 0.0) {
        if ((b < 0.0) != (mod < 0.0)) mod += b;
    } else {
        mod = copysign(0.0, b);
    }
    return mod;
}

// _pair_failures' separation rule (oracle.py:35-51)
__device__ __forceinline__ bool separation_bad(const DirectArgs& a, double dy, double dz) {
    if (a.dim == 1) return hypot(dy, dz) <= a.floor_t;
    if (!a.npsp) return false;
    const double ly = a.L[1], lz = a.L[2];
    const double ry = fabs(np_remainder(dy + ly / 2.0, ly) - ly / 2.0);
    const double rz = a.dim == 2 ? fabs(dz) : fabs(np_remainder(dz + lz / 2.0, lz) - lz / 2.0);
    return hypot(ry, rz) <= a.floor_t;
}

// pass 1: separation flags (1) per pair and per chunk
__global__ void k_direct_separation(DirectArgs a) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= a.mc * a.N) return;
    const int64_t i = a.m0 + t / a.N, j = t % a.N;
    const double dy = a.obs[3 * i + 1] - a.src[3 * j + 1], dz = a.obs[3 * i + 2] - a.src[3 * j + 2];
    const bool bad = !a.free_space && separation_bad(a, dy, dz);
    a.flags[t] = bad ? 1 : 0;
    if (bad) atomicAdd(&a.chunk_sep[i / DIRECT_CHUNK], 1);
}

// pass 2: G(r_m - r_n) q_n for the pairs of clean chunks; flag 2 = not converged
__global__ void __launch_bounds__(128) k_direct_pairs(DirectArgs a, FarSeriesParams fp, ImageSet im, GLTable gl,
                                                      DevStatus* st) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= a.mc * a.N) return;
    const int64_t i = a.m0 + t / a.N, j = t % a.N;
    const int64_t c = i / DIRECT_CHUNK;
    if (a.chunk_sep[c]) {
        a.vals[t] = mk(0.0);
        return;
    }
    const double x = a.obs[3 * i] - a.src[3 * j], y = a.obs[3 * i + 1] - a.src[3 * j + 1],
                 z = a.obs[3 * i + 2] - a.src[3 * j + 2];
    cplx g;
    if (a.free_space) {
        const double r = sqrt(x * x + y * y + z * z);
        if (r == 0.0) {
            set_status(st, FFTPIM_DOMAIN, 60, i, j);   // ZeroDivisionError, oracle.py:120-121
            a.vals[t] = mk(0.0);
            return;
        }
        // exp(-j k0 r) / (4 pi r)
        g = cexp_mj(cplx{fp.k0_re, fp.k0_im} * r) / (4.0 * M_PI * r);
        a.flags[t] = 0;
    } else {
        const Drive d = fp.npsp ? lattice_series(fp, gl, x, y, z, a.zr[2 * c], a.zr[2 * c + 1], st, t)
                                : spectral_series(fp, gl, x, y, z, st, t);
        g = d.total;
        if (a.far_only) {
            bool bad = false;
            g = g - image_sum(im, x, y, z, im.sep_tol, false, &bad);   // pgf.py:141-147 (no drop)
            if (bad) set_status(st, FFTPIM_DOMAIN, 61, i, j);
        }
        a.flags[t] = d.done ? 0 : 2;
        atomicMax(&a.chunk_terms[c], (long long)d.terms);
    }
    a.vals[t] = g * a.q[j];
}

// pass 3: warp per observer, lane-strided partial sums then a fixed xor tree
__global__ void k_direct_reduce(DirectArgs a, cplx* __restrict__ u) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= a.mc) return;
    const int64_t i = a.m0 + w;
    cplx s = mk(0.0);
    if (!a.chunk_sep[i / DIRECT_CHUNK]) {
        const cplx* row = a.vals + w * a.N;
        for (int64_t j = lane; j < a.N; j += 32) s = s + row[j];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s.re += __shfl_xor_sync(0xffffffffu, s.re, o);
        s.im += __shfl_xor_sync(0xffffffffu, s.im, o);
    }
    if (lane == 0) u[i] = s;
}

void launch_direct(const DirectArgs& a, const FarSeriesParams& fp, const ImageSet& im, const GLTable& gl,
                   cplx* u, DevStatus* st, cudaStream_t s) {
    const int64_t n = a.mc * a.N;
    if (n == 0) return;
    k_direct_separation<<<nblk(n, 256), 256, 0, s>>>(a);
    k_direct_pairs<<<nblk(n, 128), 128, 0, s>>>(a, fp, im, gl, st);
    k_direct_reduce<<<nblk(a.mc * 32, 256), 256, 0, s>>>(a, u);
    fftpim_count_launch(3);
}
