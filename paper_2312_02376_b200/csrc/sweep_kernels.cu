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

// Rows in source order (sort_pair_rows): a warp takes TWO consecutive sorted
// observers and merge-joins their pair lists on the packed source value, so a
// charge row (E x 16 B, the kernel's L2 traffic: P x 1 KB per sweep at E = 64) is
// loaded once for both observers when they share the source -- neighbouring
// observers share ~85 % of their sources, so the L2 traffic drops ~1.85x.
// Same products and the same per-row summation order as k_corr_sweep (each
// row's pairs are still taken in list order): bit-identical sums.
#ifndef SWEEP2_MINB
#define SWEEP2_MINB 2
#endif
template <int NC>
__device__ __forceinline__ void sweep_mac(const cplx (*sb)[32], int k, const cplx& q0, const cplx& q1, bool two,
                                          double* s0r, double* s0i, double* s1r, double* s1i) {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        const cplx b = sb[j][k];
        s0r[j] = fma(b.re, q0.re, s0r[j]);
        s0r[j] = fma(-b.im, q0.im, s0r[j]);
        s0i[j] = fma(b.re, q0.im, s0i[j]);
        s0i[j] = fma(b.im, q0.re, s0i[j]);
        if (two) {
            s1r[j] = fma(b.re, q1.re, s1r[j]);
            s1r[j] = fma(-b.im, q1.im, s1r[j]);
            s1i[j] = fma(b.re, q1.im, s1i[j]);
            s1i[j] = fma(b.im, q1.re, s1i[j]);
        }
    }
}

template <int NC, bool TWO, bool FULL>
__global__ void __launch_bounds__(256, SWEEP2_MINB)
    k_corr_sweep2(const int64_t* __restrict__ ptr, const int* __restrict__ psrc, const cplx* __restrict__ comp,
                  int64_t P, const cplx* __restrict__ qt3, int64_t N, int E, const cplx* __restrict__ omega,
                  cplx* __restrict__ corr, int64_t M) {
    constexpr int NS = NC + 2;
    // per warp and row: two staged 32-pair blocks (the products of a step run one
    // step behind its loads, so they may still read the block before the newest)
    extern __shared__ __align__(16) unsigned char sweep2_smem[];
    typedef cplx (*SB)[2][2][NC][32];
    typedef int (*SV)[2][2][32];
    SB s_b = reinterpret_cast<SB>(sweep2_smem);
    SV s_v = reinterpret_cast<SV>(sweep2_smem + sizeof(cplx) * 8 * 2 * 2 * NC * 32);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t i0 = 2 * w;
    if (i0 >= M) return;
    const int e0 = lane, e1 = lane + 32;
    const bool ok0 = e0 < E, ok1 = TWO && e1 < E;
    const int64_t NE = N * E;
    double ar[2][NC], ai[2][NC], br[2][NC], bi[2][NC];   // [row][component]: excitation e0 (a), e1 (b)
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j = 0; j < NC; ++j) ar[r][j] = ai[r][j] = br[r][j] = bi[r][j] = 0.0;
    int64_t nb[2], pe[2];   // next pair to stage, end of the row
    nb[0] = ptr[i0];
    pe[0] = ptr[i0 + 1];
    nb[1] = i0 + 1 < M ? ptr[i0 + 1] : 0;
    pe[1] = i0 + 1 < M ? ptr[i0 + 2] : 0;
    int k[2] = {0, 0}, cnt[2] = {0, 0}, buf[2] = {1, 1};
    // one merge step: which rows take part (bit r of t), where their pair sits
    // (buffer * 32 + index), and the loads of the shared charge row
    auto fetch = [&](int& t, int& at0, int& at1, cplx& q0, cplx& q1) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (k[r] == cnt[r] && nb[r] < pe[r]) {   // refill (warp-uniform)
                const int c = (int)min((int64_t)32, pe[r] - nb[r]);
                buf[r] ^= 1;
                __syncwarp();
                if (lane < c) {
                    s_v[wid][r][buf[r]][lane] = psrc[nb[r] + lane];
#pragma unroll
                    for (int j = 0; j < NC; ++j) s_b[wid][r][buf[r]][j][lane] = comp[(int64_t)j * P + nb[r] + lane];
                }
                __syncwarp();
                nb[r] += c;
                k[r] = 0;
                cnt[r] = c;
            }
        }
        const bool h0 = k[0] < cnt[0], h1 = k[1] < cnt[1];
        t = 0;
        q0 = q1 = mk(0.0);
        if (!h0 && !h1) return;
        const int v0 = h0 ? s_v[wid][0][buf[0]][k[0]] : 0, v1 = h1 ? s_v[wid][1][buf[1]][k[1]] : 0;
        // rows are sorted by the packed value as signed ints (sort_pair_rows); any
        // order is still correct (every step consumes a pair), only less shared
        const bool t0 = h0 && (!h1 || v0 <= v1), t1 = h1 && (!h0 || v1 <= v0);
        const int v = t0 ? v0 : v1;
        const cplx* qrow = qt3 + (int64_t)((unsigned)v >> 30) * NE + (int64_t)(v & 0x3fffffff) * E;
        if (FULL || ok0) q0 = qrow[e0];
        if (TWO && (FULL || ok1)) q1 = qrow[e1];
        at0 = buf[0] * 32 + k[0];
        at1 = buf[1] * 32 + k[1];
        t = (t0 ? 1 : 0) | (t1 ? 2 : 0);
        k[0] += t0 ? 1 : 0;
        k[1] += t1 ? 1 : 0;
    };
    int tA, a0, a1;
    cplx qa0, qa1;
    fetch(tA, a0, a1, qa0, qa1);
    while (tA) {
        int tB, b0 = 0, b1 = 0;
        cplx qb0, qb1;
        fetch(tB, b0, b1, qb0, qb1);   // the next step's loads fly during this step's products
        if (tA & 1) sweep_mac<NC>(s_b[wid][0][a0 >> 5], a0 & 31, qa0, qa1, TWO, ar[0], ai[0], br[0], bi[0]);
        if (tA & 2) sweep_mac<NC>(s_b[wid][1][a1 >> 5], a1 & 31, qa0, qa1, TWO, ar[1], ai[1], br[1], bi[1]);
        tA = tB;
        a0 = b0;
        a1 = b1;
        qa0 = qb0;
        qa1 = qb1;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int64_t i = i0 + r;
        if (i >= M) break;
        if (FULL || ok0) {
            double re = 0.0, im = 0.0;
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                const cplx wv = omega[(int64_t)e0 * NS + j + 1];
                re += wv.re * ar[r][j] - wv.im * ai[r][j];
                im += wv.re * ai[r][j] + wv.im * ar[r][j];
            }
            corr[i * E + e0] = cplx{re, im};
        }
        if (TWO && (FULL || ok1)) {
            double re = 0.0, im = 0.0;
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                const cplx wv = omega[(int64_t)e1 * NS + j + 1];
                re += wv.re * br[r][j] - wv.im * bi[r][j];
                im += wv.re * bi[r][j] + wv.im * br[r][j];
            }
            corr[i * E + e1] = cplx{re, im};
        }
    }
}

// Asynchronous charge rows (opt-in, measured slower at C5: 248 vs 177 ms): the idea was that
// k_corr_sweep is bound by the latency of the charge row loads (1 KB per pair from L2, two pairs in flight per warp; FP64 pipe 56 %
// busy).  Here every lane copies its own 16-byte slices of the next SWEEP_D
// pairs' charge rows into a private shared-memory ring with cp.async (no
// registers held, no cross-lane hazard: a lane reads back only what it copied),
// waits for the oldest group and multiplies.  The staged pair blocks are double
// buffered so the ring runs across 32-pair blocks without draining.  Same
// products in the same order: bit-identical sums.
#ifndef SWEEP_D
#define SWEEP_D 8
#endif
#ifndef SWEEP3_MINB
#define SWEEP3_MINB 2
#endif
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int NC, bool TWO, bool FULL>
__global__ void __launch_bounds__(256, SWEEP3_MINB)
    k_corr_sweep3(const int64_t* __restrict__ ptr, const int* __restrict__ psrc, const cplx* __restrict__ comp,
                  int64_t P, const cplx* __restrict__ qt3, int64_t N, int E, const cplx* __restrict__ omega,
                  cplx* __restrict__ corr, int64_t M) {
    constexpr int NS = NC + 2, NQ = TWO ? 2 : 1;
    extern __shared__ __align__(16) unsigned char sweep3_smem[];
    typedef cplx (*SB)[2][NC][32];
    typedef cplx (*SQ)[SWEEP_D][NQ][32];
    typedef int (*SV)[2][32];
    SB s_b = reinterpret_cast<SB>(sweep3_smem);
    SQ s_q = reinterpret_cast<SQ>(sweep3_smem + sizeof(cplx) * 8 * 2 * NC * 32);
    SV s_v = reinterpret_cast<SV>(sweep3_smem + sizeof(cplx) * 8 * (2 * NC + SWEEP_D * NQ) * 32);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (i >= M) return;
    const int e0 = lane, e1 = lane + 32;
    const bool ok0 = e0 < E, ok1 = TWO && e1 < E;
    const int64_t NE = N * E;
    double s0r[NC], s0i[NC], s1r[NC], s1i[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) s0r[k] = s0i[k] = s1r[k] = s1i[k] = 0.0;
    const int64_t p0 = ptr[i];
    const int len = (int)(ptr[i + 1] - p0);
    auto stage = [&](int b) {   // pair block b of this row -> buffer b & 1
        const int c = min(32, len - 32 * b);
        if (lane < c) {
            const int64_t p = p0 + 32 * b + lane;
            s_v[wid][b & 1][lane] = psrc[p];
#pragma unroll
            for (int j = 0; j < NC; ++j) s_b[wid][b & 1][j][lane] = comp[(int64_t)j * P + p];
        }
    };
    auto issue = [&](int m) {   // start the copies of pair m's charge row slices
        if (m < len) {
            const int v = s_v[wid][(m >> 5) & 1][m & 31];
            const cplx* qrow = qt3 + (int64_t)((unsigned)v >> 30) * NE + (int64_t)(v & 0x3fffffff) * E;
            if (FULL || ok0) cp_async16(&s_q[wid][m % SWEEP_D][0][lane], qrow + e0);
            if (TWO && (FULL || ok1)) cp_async16(&s_q[wid][m % SWEEP_D][NQ - 1][lane], qrow + e1);
        }
        cp_async_commit();
    };
    if (len > 0) stage(0);
    __syncwarp();
#pragma unroll
    for (int m = 0; m < SWEEP_D; ++m) issue(m);
    for (int n = 0; n < len; ++n) {
        if ((n & 31) == 0) {
            if (32 * ((n >> 5) + 1) < len) stage((n >> 5) + 1);
            __syncwarp();
        }
        cp_async_wait<SWEEP_D - 1>();
        cplx q0 = s_q[wid][n % SWEEP_D][0][lane], q1 = mk(0.0);
        if (TWO) q1 = s_q[wid][n % SWEEP_D][NQ - 1][lane];
        if (!FULL && !ok0) q0 = mk(0.0);
        if (!FULL && TWO && !ok1) q1 = mk(0.0);
        const int buf = (n >> 5) & 1, k = n & 31;
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            const cplx b = s_b[wid][buf][j][k];
            s0r[j] = fma(b.re, q0.re, s0r[j]);
            s0r[j] = fma(-b.im, q0.im, s0r[j]);
            s0i[j] = fma(b.re, q0.im, s0i[j]);
            s0i[j] = fma(b.im, q0.re, s0i[j]);
            if (TWO) {
                s1r[j] = fma(b.re, q1.re, s1r[j]);
                s1r[j] = fma(-b.im, q1.im, s1r[j]);
                s1i[j] = fma(b.re, q1.im, s1i[j]);
                s1i[j] = fma(b.im, q1.re, s1i[j]);
            }
        }
        issue(n + SWEEP_D);
    }
    cp_async_wait<0>();
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
                       const cplx* qt3, int64_t N, int E, const cplx* omega, cplx* corr, int64_t M, cudaStream_t s,
                       bool sorted_rows) {
    if (M == 0) return;
    const char* e3 = getenv("FFTPIM_SWEEP_ASYNC");   // 1: cp.async ring (measured slower: LSU-bound)
    if (e3 && e3[0] == '1' && ncomp <= 3) {
        const int blocks3 = nblk(M * 32, 256);
#define KS3_ONE(NC, TWO, FULL)                                                                                 \
    {                                                                                                          \
        const size_t sm = sizeof(cplx) * 8 * (2 * NC + SWEEP_D * (TWO ? 2 : 1)) * 32 + sizeof(int) * 8 * 2 * 32; \
        cudaFuncSetAttribute(k_corr_sweep3<NC, TWO, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
        k_corr_sweep3<NC, TWO, FULL><<<blocks3, 256, sm, s>>>(ptr, pair_src, comp, P, qt3, N, E, omega, corr, M); \
    }
#define KS3(NC)                      \
    if (E == 64)                     \
        KS3_ONE(NC, true, true)      \
    else if (E > 32)                 \
        KS3_ONE(NC, true, false)     \
    else if (E == 32)                \
        KS3_ONE(NC, false, true)     \
    else                             \
        KS3_ONE(NC, false, false)
        if (ncomp == 1) {
            KS3(1)
        } else {
            KS3(3)
        }
#undef KS3
#undef KS3_ONE
        fftpim_count_launch();
        return;
    }
    const char* e2 = getenv("FFTPIM_SWEEP_ROWS2");   // 1: two observers per warp, merge-joined (measured slower)
    if (sorted_rows && e2 && e2[0] == '1') {
        const int blocks2 = nblk(((M + 1) / 2) * 32, 256);
#define KS2_ONE(NC, TWO, FULL)                                                                                  \
    {                                                                                                           \
        const size_t sm = sizeof(cplx) * 8 * 2 * 2 * NC * 32 + sizeof(int) * 8 * 2 * 2 * 32;                    \
        cudaFuncSetAttribute(k_corr_sweep2<NC, TWO, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
        k_corr_sweep2<NC, TWO, FULL><<<blocks2, 256, sm, s>>>(ptr, pair_src, comp, P, qt3, N, E, omega, corr, M); \
    }
#define KS2(NC)                      \
    if (E == 64)                     \
        KS2_ONE(NC, true, true)      \
    else if (E > 32)                 \
        KS2_ONE(NC, true, false)     \
    else if (E == 32)                \
        KS2_ONE(NC, false, true)     \
    else                             \
        KS2_ONE(NC, false, false)
        if (ncomp == 1) {
            KS2(1)
        } else if (ncomp == 3) {
            KS2(3)
        } else {
            KS2(5)
        }
#undef KS2
#undef KS2_ONE
        fftpim_count_launch();
        return;
    }
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
