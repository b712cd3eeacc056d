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
// warp per observer, lanes own excitations, per-power accumulators
// S_m = sum_pairs B_j q_e[src] (m = c_a + j - i_d), and at the row end
// corr_e = sum_m omega_e^m S_m.  Fixed order, no atomics.
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

// qt[i][e] = q[e][perm[i]]  (sorted order, excitation fastest)
__global__ void k_sweep_permute(const cplx* __restrict__ q, const int* __restrict__ perm, int64_t N, int E,
                                cplx* __restrict__ qt) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= N * E) return;
    const int64_t i = t / E;
    const int e = (int)(t - i * E);
    qt[t] = q[(int64_t)e * N + perm[i]];
}

void launch_sweep_permute(const cplx* q, const int* perm, int64_t N, int E, cplx* qt, cudaStream_t s) {
    if (N == 0) return;
    k_sweep_permute<<<nblk(N * E, 256), 256, 0, s>>>(q, perm, N, E, qt);
    fftpim_count_launch();
}

// warp per sorted observer; lane l owns excitations l and l + 32 (E <= 64).
// Pairs are taken 32 at a time: lane k stages pair k's packed source and
// components in shared memory (coalesced loads), then the warp walks the 32
// pairs reading them as broadcasts, four pairs' q rows in flight at a time.
#ifndef SWEEP_U   // pairs whose q rows are in flight together
#define SWEEP_U 2
#endif
template <int NC, bool TWO, bool HALVES>
__global__ void __launch_bounds__(256) k_corr_sweep(const int64_t* __restrict__ ptr, const int* __restrict__ psrc,
                                                    const cplx* __restrict__ comp, int64_t P,
                                                    const cplx* __restrict__ qt, int E,
                                                    const cplx* __restrict__ omega, cplx* __restrict__ corr,
                                                    int64_t M) {
    constexpr int NS = NC + 2;   // powers m = -(h+1) .. h+1, h = NC / 2
    __shared__ cplx s_b[8][NC][32];
    __shared__ int s_v[8][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t i = HALVES ? gw >> 1 : gw;
    if (i >= M) return;
    const int e0 = HALVES ? lane + 32 * (int)(gw & 1) : lane, e1 = lane + 32;
    const bool ok0 = e0 < E, ok1 = TWO && e1 < E;
    double s0r[NS], s0i[NS], s1r[NS], s1i[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) s0r[k] = s0i[k] = s1r[k] = s1i[k] = 0.0;
    const int64_t p0 = ptr[i], p1 = ptr[i + 1];
    for (int64_t b = p0; b < p1; b += 32) {
        const int cnt = (int)min((int64_t)32, p1 - b);
        __syncwarp();
        if (lane < cnt) {
            s_v[wid][lane] = psrc[b + lane];
#pragma unroll
            for (int j = 0; j < NC; ++j) s_b[wid][j][lane] = comp[(int64_t)j * P + b + lane];
        }
        __syncwarp();
        for (int k0 = 0; k0 < cnt; k0 += SWEEP_U) {
            int v[SWEEP_U];
            cplx q0[SWEEP_U], q1[SWEEP_U];
#pragma unroll
            for (int u = 0; u < SWEEP_U; ++u) {
                const bool in = k0 + u < cnt;
                v[u] = in ? s_v[wid][k0 + u] : 0;
                const cplx* qrow = qt + (int64_t)(v[u] & 0x3fffffff) * E;
                q0[u] = (in && ok0) ? qrow[e0] : mk(0.0);
                q1[u] = (in && ok1) ? qrow[e1] : mk(0.0);
            }
#pragma unroll
            for (int u = 0; u < SWEEP_U; ++u) {
                if (k0 + u >= cnt) break;
                const int ca = (v[u] >> 30) & 3;   // code along the axis + 1 (warp-uniform)
                cplx bj[NC];
#pragma unroll
                for (int j = 0; j < NC; ++j) bj[j] = s_b[wid][j][k0 + u];
                // S[ca + j] += B_j q
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (ca != c) continue;
#pragma unroll
                    for (int j = 0; j < NC; ++j) {
                        s0r[c + j] += bj[j].re * q0[u].re - bj[j].im * q0[u].im;
                        s0i[c + j] += bj[j].re * q0[u].im + bj[j].im * q0[u].re;
                        if (TWO) {
                            s1r[c + j] += bj[j].re * q1[u].re - bj[j].im * q1[u].im;
                            s1i[c + j] += bj[j].re * q1[u].im + bj[j].im * q1[u].re;
                        }
                    }
                }
            }
        }
    }
    // corr_e = sum_m omega_e^m S_m
    if (ok0) {
        double r = 0.0, im = 0.0;
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const cplx w = omega[(int64_t)e0 * NS + k];
            r += w.re * s0r[k] - w.im * s0i[k];
            im += w.re * s0i[k] + w.im * s0r[k];
        }
        corr[i * E + e0] = cplx{r, im};
    }
    if (ok1) {
        double r = 0.0, im = 0.0;
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const cplx w = omega[(int64_t)e1 * NS + k];
            r += w.re * s1r[k] - w.im * s1i[k];
            im += w.re * s1i[k] + w.im * s1r[k];
        }
        corr[i * E + e1] = cplx{r, im};
    }
}

void launch_corr_sweep(const int64_t* ptr, const int* pair_src, const cplx* comp, int ncomp, int64_t P,
                       const cplx* qt, int E, const cplx* omega, cplx* corr, int64_t M, cudaStream_t s) {
    if (M == 0) return;
    // E > 32: two warps per observer (one per 32 excitations, adjacent in the
    // block so the second reads the pair data from L1) or one warp with two
    // excitations per lane (default; measured faster, FFTPIM_SWEEP_HALVES=1 for the other)
    static const bool halves = [] {
        const char* e = getenv("FFTPIM_SWEEP_HALVES");
        return e && e[0] == '1';
    }();
    const bool two = E > 32;
    if (two && halves) {
        const int blocks = nblk(M * 64, 256);
        if (ncomp == 3)
            k_corr_sweep<3, false, true><<<blocks, 256, 0, s>>>(ptr, pair_src, comp, P, qt, E, omega, corr, M);
        else
            k_corr_sweep<5, false, true><<<blocks, 256, 0, s>>>(ptr, pair_src, comp, P, qt, E, omega, corr, M);
        fftpim_count_launch();
        return;
    }
    const int blocks = nblk(M * 32, 256);
#define KS(NC)                                                                                              \
    if (two) k_corr_sweep<NC, true, false><<<blocks, 256, 0, s>>>(ptr, pair_src, comp, P, qt, E, omega, corr, M); \
    else k_corr_sweep<NC, false, false><<<blocks, 256, 0, s>>>(ptr, pair_src, comp, P, qt, E, omega, corr, M);
    if (ncomp == 3) {
        KS(3)
    } else {
        KS(5)
    }
#undef KS
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
