// sweep_kernels.cu -- batched excitation sweep.
//
// E excitations whose Floquet shifts differ only along one periodic axis a
// share the geometry, the stencils, the K1 operator and the correction-pair
// list.  Each pair's coefficient (nearzone.py:405-457) is linear in the image
// phases exp(-j i_a k_a L_a) and the code phase exp(-j c_a k_a L_a), so the plan
// stores 2 i_d + 1 components B_j (image index i_a = j - i_d, every other phase
// folded in) and
//     coef_e = sum_j exp(-j (c_a + j - i_d) k_e L_a) B_j.
// The batched K4 below streams the components once for all E excitations: a
// warp per observer, lanes own excitations, per-component accumulators
// S_j = sum_pairs B_j omega_e^(c_a) q_e[src] (the code phase is pre-applied to
// three copies of the charges), and at the row end
// corr_e = sum_j omega_e^(j - i_d) S_j.  Fixed order, no atomics.
#include <cstdlib>

#include "geom.cuh"
#include "kernels.h"

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// pair_src <- sorted source | (code along the sweep axis + 1) << 30
__global__ void k_sweep_pack_src(int* pair_src, const unsigned char* __restrict__ codeid, SweepCodeAxis ca,
                                 int64_t P) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    pair_src[p] = pair_src[p] | ((ca.c[codeid[p]] + 1) << 30);
}

void launch_sweep_pack_src(int* pair_src, const unsigned char* codeid, const signed char* code_axis, int64_t P,
                           cudaStream_t s) {
    if (P == 0) return;
    SweepCodeAxis ca;
    for (int c = 0; c < 27; ++c) ca.c[c] = code_axis[c];
    k_sweep_pack_src<<<nblk(P, 256), 256, 0, s>>>(pair_src, codeid, ca, P);
    fftpim_count_launch();
}

// Code-phased charges: qt3[c + 1][i][e] = omega_e^c q[e][perm[i]], c = -1, 0, 1
// (sorted order, excitation fastest), omega_e^m = exp(-j m k_e L_a).  The code
// phase of a pair then rides on the charge row it reads, so the batched K4
// keeps one accumulator per component and never branches on the code.
__global__ void k_sweep_permute(const cplx* __restrict__ q, const int* __restrict__ perm, int64_t N, int E,
                                const cplx* __restrict__ omega, int NS, int h, cplx* __restrict__ qt3) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N * E) return;
    const int64_t i = t / E;
    const int e = (int)(t - i * E);
    const cplx v = q[(int64_t)e * N + perm[i]];
    qt3[t] = omega[e * NS + h] * v;           // m = -1
    qt3[N * E + t] = v;                       // m = 0
    qt3[2 * N * E + t] = omega[e * NS + h + 2] * v;   // m = +1
}

void launch_sweep_permute(const cplx* q, const int* perm, int64_t N, int E, const cplx* omega, int NS, int h,
                          cplx* qt3, cudaStream_t s) {
    if (N == 0) return;
    k_sweep_permute<<<nblk(N * E, 256), 256, 0, s>>>(q, perm, N, E, omega, NS, h, qt3);
    fftpim_count_launch();
}

// Warp per sorted observer; lane l owns excitations l and l + 32 (E <= 64).
// Pairs are taken 32 at a time: lane k stages pair k's packed source and
// components in shared memory (coalesced loads), then the warp walks the 32
// pairs reading them as broadcasts, SWEEP_U pairs' charge rows in flight at a
// time.  S_j += B_j qt3[c][src]; at the row end corr_e = sum_j omega_e^(j - h) S_j.
#ifndef SWEEP_U   // pairs whose q rows are in flight together
#define SWEEP_U 2
#endif
#ifndef SWEEP_MINB
#define SWEEP_MINB 3
#endif
template <int NC, bool TWO, bool FULL, bool TAIL>
__device__ __forceinline__ void sweep_pairs(const int* sv, const cplx (*sb)[32], int cnt, const cplx* __restrict__ qt3,
                                            int64_t NE, int E, int e0, int e1, bool ok0, bool ok1, double* s0r,
                                            double* s0i, double* s1r, double* s1i) {
    const int kend = TAIL ? cnt : 32;
    for (int k0 = 0; k0 < kend; k0 += SWEEP_U) {
        cplx q0[SWEEP_U], q1[SWEEP_U];
#pragma unroll
        for (int u = 0; u < SWEEP_U; ++u) {
            const bool in = !TAIL || k0 + u < cnt;
            const int v = in ? sv[k0 + u] : 0;
            const cplx* qrow = qt3 + (int64_t)((unsigned)v >> 30) * NE + (int64_t)(v & 0x3fffffff) * E;
            q0[u] = (in && (FULL || ok0)) ? qrow[e0] : mk(0.0);
            if (TWO) q1[u] = (in && (FULL || ok1)) ? qrow[e1] : mk(0.0);
        }
#pragma unroll
        for (int u = 0; u < SWEEP_U; ++u) {
            const int k = TAIL ? min(k0 + u, 31) : k0 + u;   // tail: padded pairs carry q = 0
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                const cplx b = sb[j][k];
                s0r[j] = fma(b.re, q0[u].re, s0r[j]);
                s0r[j] = fma(-b.im, q0[u].im, s0r[j]);
                s0i[j] = fma(b.re, q0[u].im, s0i[j]);
                s0i[j] = fma(b.im, q0[u].re, s0i[j]);
                if (TWO) {
                    s1r[j] = fma(b.re, q1[u].re, s1r[j]);
                    s1r[j] = fma(-b.im, q1[u].im, s1r[j]);
                    s1i[j] = fma(b.re, q1[u].im, s1i[j]);
                    s1i[j] = fma(b.im, q1[u].re, s1i[j]);
                }
            }
        }
    }
}

template <int NC, bool TWO, bool FULL>
__global__ void __launch_bounds__(256, SWEEP_MINB)
    k_corr_sweep(const int64_t* __restrict__ ptr, const int* __restrict__ psrc, const cplx* __restrict__ comp,
                 int64_t P, const cplx* __restrict__ qt3, int64_t N, int E, const cplx* __restrict__ omega,
                 cplx* __restrict__ corr, int64_t M) {
    constexpr int h = NC / 2, NS = NC + 2;
    __shared__ cplx s_b[8][NC][32];
    __shared__ int s_v[8][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (i >= M) return;
    const int e0 = lane, e1 = lane + 32;
    const bool ok0 = e0 < E, ok1 = TWO && e1 < E;
    const int64_t NE = N * E;
    double s0r[NC], s0i[NC], s1r[NC], s1i[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) s0r[k] = s0i[k] = s1r[k] = s1i[k] = 0.0;
    const int64_t p0 = ptr[i], p1 = ptr[i + 1];
    for (int64_t b = p0; b < p1; b += 32) {
        const int cnt = (int)min((int64_t)32, p1 - b);
        __syncwarp();
        if (lane < cnt) {
            s_v[wid][lane] = psrc[b + lane];
#pragma unroll
            for (int j = 0; j < NC; ++j) s_b[wid][j][lane] = comp[(int64_t)j * P + b + lane];
        } else {
            s_v[wid][lane] = 0;
#pragma unroll
            for (int j = 0; j < NC; ++j) s_b[wid][j][lane] = mk(0.0);
        }
        __syncwarp();
        if (cnt == 32)
            sweep_pairs<NC, TWO, FULL, false>(s_v[wid], s_b[wid], cnt, qt3, NE, E, e0, e1, ok0, ok1, s0r, s0i, s1r, s1i);
        else
            sweep_pairs<NC, TWO, FULL, true>(s_v[wid], s_b[wid], cnt, qt3, NE, E, e0, e1, ok0, ok1, s0r, s0i, s1r, s1i);
    }
    // corr_e = sum_j omega_e^(j - h) S_j   (table index m + h + 1)
    if (FULL || ok0) {
        double r = 0.0, im = 0.0;
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            const cplx w = omega[(int64_t)e0 * NS + k + 1];
            r += w.re * s0r[k] - w.im * s0i[k];
            im += w.re * s0i[k] + w.im * s0r[k];
        }
        corr[i * E + e0] = cplx{r, im};
    }
    if (TWO && (FULL || ok1)) {
        double r = 0.0, im = 0.0;
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            const cplx w = omega[(int64_t)e1 * NS + k + 1];
            r += w.re * s1r[k] - w.im * s1i[k];
            im += w.re * s1i[k] + w.im * s1r[k];
        }
        corr[i * E + e1] = cplx{r, im};
    }
}

void launch_corr_sweep(const int64_t* ptr, const int* pair_src, const cplx* comp, int ncomp, int64_t P,
                       const cplx* qt3, int64_t N, int E, const cplx* omega, cplx* corr, int64_t M, cudaStream_t s) {
    if (M == 0) return;
    const int blocks = nblk(M * 32, 256);
#define KS(NC)                                                                                                   \
    if (E == 64)                                                                                                 \
        k_corr_sweep<NC, true, true><<<blocks, 256, 0, s>>>(ptr, pair_src, comp, P, qt3, N, E, omega, corr, M); \
    else if (E > 32)                                                                                             \
        k_corr_sweep<NC, true, false><<<blocks, 256, 0, s>>>(ptr, pair_src, comp, P, qt3, N, E, omega, corr, M); \
    else if (E == 32)                                                                                            \
        k_corr_sweep<NC, false, true><<<blocks, 256, 0, s>>>(ptr, pair_src, comp, P, qt3, N, E, omega, corr, M); \
    else                                                                                                         \
        k_corr_sweep<NC, false, false><<<blocks, 256, 0, s>>>(ptr, pair_src, comp, P, qt3, N, E, omega, corr, M);
    if (ncomp == 1) {
        KS(1)
    } else if (ncomp == 3) {
        KS(3)
    } else {
        KS(5)
    }
#undef KS
    fftpim_count_launch();
}

// multi-RHS batches on one plan: qt[i][e] = q[e][perm[i]] (no phases)
__global__ void k_batch_permute(const cplx* __restrict__ q, const int* __restrict__ perm, int64_t N, int E,
                                cplx* __restrict__ qt) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N * E) return;
    const int64_t i = t / E;
    const int e = (int)(t - i * E);
    qt[t] = q[(int64_t)e * N + perm[i]];
}

void launch_batch_permute(const cplx* q, const int* perm, int64_t N, int E, cplx* qt, cudaStream_t s) {
    if (N == 0) return;
    k_batch_permute<<<nblk(N * E, 256), 256, 0, s>>>(q, perm, N, E, qt);
    fftpim_count_launch();
}

// u[e][obs_perm[i]] += corr[i][e]: the batched K4 sums into the potentials the
// per-excitation observer passes wrote (thread per (observer, excitation),
// excitation fastest: coalesced corr reads)
__global__ void k_sweep_add_corr(cplx* __restrict__ u, const cplx* __restrict__ corr, const int* __restrict__ perm,
                                 int64_t M, int E) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= M * E) return;
    const int64_t i = t / E;
    const int e = (int)(t - i * E);
    cplx* d = u + (int64_t)e * M + perm[i];
    *d = *d + corr[t];
}

void launch_sweep_add_corr(cplx* u, const cplx* corr, const int* obs_perm, int64_t M, int E, cudaStream_t s) {
    if (M == 0) return;
    k_sweep_add_corr<<<nblk(M * E, 256), 256, 0, s>>>(u, corr, obs_perm, M, E);
    fftpim_count_launch();
}
