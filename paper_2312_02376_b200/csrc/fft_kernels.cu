// fft_kernels.cu -- the near-zone FFT convolution as pruned, fused column-FFT
// stages (K2, nearzone.py:500-504), replacing full 3D transforms of the
// zero-padded (2n)^3 array:
//
//   S1  z: qg[x][y][0..n2)   -> FFT_{2n2} -> A[x][y][kz]            (x<n0, y<n1)
//   S2  y: A[x][0..n1)[kz]   -> FFT_{2n1} -> B[x][ky][kz]            (x<n0)
//   S3  x: B[0..n0)[ky][kz]  -> FFT_{2n0} -> * khat -> IFFT -> B[x<n0][ky][kz]
//   S4  y: B[x][ky][kz]      -> IFFT      -> A[x][y<n1][kz]
//   S5  z: A[x][y][kz]       -> IFFT      -> ug[x][y][z<n2]
//
// Zero padding is never stored (each column loads its n nonzero inputs and
// keeps its n needed outputs), the spectrum multiply is fused between the x
// transforms, and numpy's 1/M inverse scaling is folded into khat at plan build.
// Each block transforms B columns in shared memory with a mixed-radix Stockham
// autosort FFT (radix 4, 2, 3, 5 specialised; any other radix <= 32 generic)
// using a host-computed twiddle table.  Traffic: ~33 n^3 complex values per
// evaluation instead of ~130 n^3 for full transforms.
#include <cstdlib>

#include <type_traits>

#include "geom.cuh"
#include "kernels.h"

__device__ __forceinline__ cplx twid(const cplx* tw, int t, int sign) {
    const cplx w = tw[t];
    return sign < 0 ? w : cplx{w.re, -w.im};
}

// multiply by exp(sign * i * pi / 2) = sign * i
__device__ __forceinline__ cplx mul_si(cplx a, int sign) {
    return sign < 0 ? cplx{a.im, -a.re} : cplx{-a.im, a.re};
}

// one Stockham pass of radix r over B columns of length L: y <- pass(x)
__device__ __forceinline__ int ilog2_exact(int v) { return (v & (v - 1)) ? -1 : __ffs(v) - 1; }

// XOR swizzle of a column index within its aligned 8-element (128 B) group:
// stride-1, stride-4 and the 4-runs-at-16 patterns of the first Stockham passes
// all land on distinct 16-byte bank slots.
// (identity when L is not a multiple of 8: the last group would be partial)
__device__ __forceinline__ int swz(int i, int L) {
    if (L & 7) return i;
    const int g = i >> 3;
    return i ^ ((g ^ ((g >> 1) & 4)) & 7);
}

// q = v / d, returns v - q*d; shift/mask when d is a power of two (ld >= 0)
__device__ __forceinline__ int divmod(int v, int d, int ld, int* q) {
    if (ld >= 0) {
        *q = v >> ld;
        return v & (d - 1);
    }
    *q = v / d;
    return v - *q * d;
}

// twp: this pass's compact twiddles, twp[(q-1)*p + k] = exp(-2 pi i q k / (p r)),
// so consecutive threads (consecutive k) read consecutive words (no bank conflicts)
// columns live at stride Lp = L + 1 in shared memory (bank-conflict-free column-major access)
__device__ void stockham_pass(const cplx* __restrict__ x, cplx* __restrict__ y, const cplx* __restrict__ tw,
                              const cplx* __restrict__ twp, int L, int B, int r, int p, int sign) {
    const int Lp = L + 1;
    const int m = L / r;
    const int lm = ilog2_exact(m), lp = ilog2_exact(p);   // shift/mask index math when powers of two
    for (int idx = threadIdx.x; idx < B * m; idx += blockDim.x) {
        int b, j, k, jp;
        if (lm >= 0 && lp >= 0) {
            b = idx >> lm;
            j = idx & (m - 1);
            k = j & (p - 1);
            jp = j >> lp;
        } else {
            b = idx / m;
            j = idx - b * m;
            jp = j / p;
            k = j - jp * p;
        }
        const cplx* xb = x + b * Lp;
        cplx* yb = y + b * Lp;
        const int base = jp * p * r + k;
        if (r == 4) {
            cplx a0 = xb[swz(j, L)], a1 = xb[swz(j + m, L)], a2 = xb[swz(j + 2 * m, L)], a3 = xb[swz(j + 3 * m, L)];
            if (k) {
                a1 = a1 * twid(twp, k, sign);
                a2 = a2 * twid(twp, p + k, sign);
                a3 = a3 * twid(twp, 2 * p + k, sign);
            }
            const cplx t0 = a0 + a2, t1 = a0 - a2, t2 = a1 + a3, t3 = mul_si(a1 - a3, sign);
            yb[swz(base, L)] = t0 + t2;
            yb[swz(base + p, L)] = t1 + t3;
            yb[swz(base + 2 * p, L)] = t0 - t2;
            yb[swz(base + 3 * p, L)] = t1 - t3;
        } else if (r == 2) {
            cplx a0 = xb[swz(j, L)], a1 = xb[swz(j + m, L)];
            if (k) a1 = a1 * twid(twp, k, sign);
            yb[swz(base, L)] = a0 + a1;
            yb[swz(base + p, L)] = a0 - a1;
        } else if (r == 3) {
            cplx a0 = xb[swz(j, L)], a1 = xb[swz(j + m, L)], a2 = xb[swz(j + 2 * m, L)];
            if (k) {
                a1 = a1 * twid(twp, k, sign);
                a2 = a2 * twid(twp, p + k, sign);
            }
            const cplx w1 = twid(tw, m, sign), w2 = twid(tw, 2 * m, sign);
            yb[swz(base, L)] = a0 + a1 + a2;
            yb[swz(base + p, L)] = a0 + w1 * a1 + w2 * a2;
            yb[swz(base + 2 * p, L)] = a0 + w2 * a1 + w1 * a2;
        } else {
            cplx a[32];
            for (int q = 0; q < r; ++q) {
                a[q] = xb[swz(j + q * m, L)];
                if (k && q) a[q] = a[q] * twid(twp, (q - 1) * p + k, sign);
            }
            for (int s = 0; s < r; ++s) {
                cplx acc = a[0];
                for (int q = 1; q < r; ++q) acc = acc + a[q] * twid(tw, (int)(((long long)q * s * m) % L), sign);
                yb[swz(base + s * p, L)] = acc;
            }
        }
    }
}

// all passes; returns the buffer holding the result
__device__ cplx* column_fft(cplx* x, cplx* y, const cplx* tw, const cplx* twp, const FftStage& st, int B, int sign) {
    int p = 1, off = 0;
    for (int ri = 0; ri < st.nrad; ++ri) {
        const int r = st.radix[ri];
        stockham_pass(x, y, tw, twp + off, st.L, B, r, p, sign);
        off += (r - 1) * p;
        __syncthreads();
        cplx* t = x;
        x = y;
        y = t;
        p *= r;
    }
    return x;
}

__global__ void __launch_bounds__(256) k_fft_stage(FftStage st) {
    extern __shared__ cplx sm[];
    const int L = st.L, B = st.B, Lp = L + 1;
    cplx* x = sm;
    cplx* y = sm + B * Lp;
    cplx* tw = sm + 2 * B * Lp;
    cplx* twp = tw + L;
    for (int t = threadIdx.x; t < L; t += blockDim.x) tw[t] = st.tw[t];
    for (int t = threadIdx.x; t < st.ntwp; t += blockDim.x) twp[t] = st.twp[t];
    const int c0 = blockIdx.x * B;
    const int nb = min(B, st.nb0 - c0);
    const int64_t in_base = (int64_t)blockIdx.y * st.in_s1 + (int64_t)c0 * st.in_s0;
    const int64_t out_base = (int64_t)blockIdx.y * st.out_s1 + (int64_t)c0 * st.out_s0;
    // load the nonzero inputs; the rest of each column is zero
    const int lL = ilog2_exact(L), lB = ilog2_exact(B), lo = ilog2_exact(st.lout);
    if (st.in_stride == 1) {
        for (int idx = threadIdx.x; idx < B * L; idx += blockDim.x) {
            int b;
            const int i = divmod(idx, L, lL, &b);
            x[b * Lp + swz(i, L)] = (b < nb && i < st.lin) ? st.in[in_base + b * st.in_s0 + i] : mk(0.0);
        }
    } else {
        for (int idx = threadIdx.x; idx < B * L; idx += blockDim.x) {
            int i;
            const int b = divmod(idx, B, lB, &i);
            x[b * Lp + swz(i, L)] = (b < nb && i < st.lin) ? st.in[in_base + b * st.in_s0 + (int64_t)i * st.in_stride] : mk(0.0);
        }
    }
    __syncthreads();
    cplx* r;
    if (st.spec) {
        r = column_fft(x, y, tw, twp, st, B, -1);
        const int64_t sp_base = (int64_t)blockIdx.y * st.spec_s1 + (int64_t)c0 * st.spec_s0;
        for (int idx = threadIdx.x; idx < B * L; idx += blockDim.x) {
            int k;
            const int b = divmod(idx, B, lB, &k);
            if (b < nb) r[b * Lp + swz(k, L)] = r[b * Lp + swz(k, L)] * st.spec[sp_base + b * st.spec_s0 + (int64_t)k * st.spec_stride];
        }
        __syncthreads();
        cplx* o = (r == x) ? y : x;
        r = column_fft(r, o, tw, twp, st, B, +1);
    } else {
        r = column_fft(x, y, tw, twp, st, B, st.sign);
    }
    if (st.out_stride == 1) {
        for (int idx = threadIdx.x; idx < B * st.lout; idx += blockDim.x) {
            int b;
            const int i = divmod(idx, st.lout, lo, &b);
            if (b < nb) st.out[out_base + b * st.out_s0 + i] = r[b * Lp + swz(i, L)];
        }
    } else {
        for (int idx = threadIdx.x; idx < B * st.lout; idx += blockDim.x) {
            int i;
            const int b = divmod(idx, B, lB, &i);
            if (b < nb) st.out[out_base + b * st.out_s0 + (int64_t)i * st.out_stride] = r[b * Lp + swz(i, L)];
        }
    }
}

// ---------------------------------------------------------------------------
// Power-of-two lengths with B = 1024 / L columns per block: the same Stockham
// radix-4 (+ one radix-2) algorithm with every index, pass span and twiddle
// offset known at compile time, so each thread executes straight-line code.
template <int L, int R, int P>
__device__ __forceinline__ void p2_pass(const cplx* __restrict__ x, cplx* __restrict__ y, const cplx* __restrict__ twp,
                                        int sign) {
    constexpr int B = 1024 / L, M = L / R, LP = L + 1;
    constexpr int NB = B * M;   // butterflies in this pass
#pragma unroll
    for (int rep = 0; rep < (NB + 255) / 256; ++rep) {
        const int idx = threadIdx.x + 256 * rep;
        if (NB % 256 != 0 && idx >= NB) break;
        const int b = idx / M, j = idx % M;
        const int k = j % P, jp = j / P;
        const cplx* xb = x + b * LP;
        cplx* yb = y + b * LP;
        const int base = jp * P * R + k;
        if (R == 4) {
            cplx a0 = xb[swz(j, L)], a1 = xb[swz(j + M, L)], a2 = xb[swz(j + 2 * M, L)], a3 = xb[swz(j + 3 * M, L)];
            if (P > 1) {
                a1 = a1 * twid(twp, k, sign);
                a2 = a2 * twid(twp, P + k, sign);
                a3 = a3 * twid(twp, 2 * P + k, sign);
            }
            const cplx t0 = a0 + a2, t1 = a0 - a2, t2 = a1 + a3, t3 = mul_si(a1 - a3, sign);
            yb[swz(base, L)] = t0 + t2;
            yb[swz(base + P, L)] = t1 + t3;
            yb[swz(base + 2 * P, L)] = t0 - t2;
            yb[swz(base + 3 * P, L)] = t1 - t3;
        } else {
            cplx a0 = xb[swz(j, L)], a1 = xb[swz(j + M, L)];
            if (P > 1) a1 = a1 * twid(twp, k, sign);
            yb[swz(base, L)] = a0 + a1;
            yb[swz(base + P, L)] = a0 - a1;
        }
    }
}

// passes while P < L: radix 4 while at least 4 remain, then radix 2
template <int L, int P, int OFF>
__device__ __forceinline__ cplx* p2_passes(cplx* x, cplx* y, const cplx* twp, int sign) {
    if constexpr (P >= L) {
        return x;
    } else {
        constexpr int R = (L / P >= 4) ? 4 : 2;
        p2_pass<L, R, P>(x, y, twp + OFF, sign);
        __syncthreads();
        return p2_passes<L, P * R, OFF + (R - 1) * P>(y, x, twp, sign);
    }
}

template <int L>
__global__ void __launch_bounds__(256) k_fft_stage_p2(FftStage st) {
    constexpr int B = 1024 / L, LP = L + 1;
    extern __shared__ cplx sm[];
    cplx* x = sm;
    cplx* y = sm + B * LP;
    cplx* twp = sm + 2 * B * LP;
    for (int t = threadIdx.x; t < st.ntwp; t += 256) twp[t] = st.twp[t];
    const int c0 = blockIdx.x * B;
    const int nb = min(B, st.nb0 - c0);
    const int64_t in_base = (int64_t)blockIdx.y * st.in_s1 + (int64_t)c0 * st.in_s0;
    const int64_t out_base = (int64_t)blockIdx.y * st.out_s1 + (int64_t)c0 * st.out_s0;
    if (st.in_stride == 1) {
#pragma unroll 4
        for (int idx = threadIdx.x; idx < B * L; idx += 256) {
            const int b = idx / L, i = idx % L;
            x[b * LP + swz(i, L)] = (b < nb && i < st.lin) ? st.in[in_base + b * st.in_s0 + i] : mk(0.0);
        }
    } else {
#pragma unroll 4
        for (int idx = threadIdx.x; idx < B * L; idx += 256) {
            const int i = idx / B, b = idx % B;
            x[b * LP + swz(i, L)] = (b < nb && i < st.lin) ? st.in[in_base + b * st.in_s0 + (int64_t)i * st.in_stride] : mk(0.0);
        }
    }
    __syncthreads();
    cplx* r;
    if (st.spec) {
        r = p2_passes<L, 1, 0>(x, y, twp, -1);
        const int64_t sp_base = (int64_t)blockIdx.y * st.spec_s1 + (int64_t)c0 * st.spec_s0;
#pragma unroll 4
        for (int idx = threadIdx.x; idx < B * L; idx += 256) {
            const int k = idx / B, b = idx % B;
            if (b < nb) r[b * LP + swz(k, L)] = r[b * LP + swz(k, L)] * st.spec[sp_base + b * st.spec_s0 + (int64_t)k * st.spec_stride];
        }
        __syncthreads();
        r = p2_passes<L, 1, 0>(r, r == x ? y : x, twp, +1);
    } else {
        r = p2_passes<L, 1, 0>(x, y, twp, st.sign);
    }
    if (st.out_stride == 1) {
        for (int idx = threadIdx.x; idx < B * st.lout; idx += 256) {
            const int b = idx / st.lout, i = idx - b * st.lout;
            if (b < nb) st.out[out_base + b * st.out_s0 + i] = r[b * LP + swz(i, L)];
        }
    } else {
        for (int idx = threadIdx.x; idx < B * st.lout; idx += 256) {
            const int i = idx / B, b = idx % B;
            if (b < nb) st.out[out_base + b * st.out_s0 + (int64_t)i * st.out_stride] = r[b * LP + swz(i, L)];
        }
    }
}

template <int L>
static bool p2_launch(const FftStage& st, cudaStream_t s) {
    if (st.L != L || st.B != 1024 / L) return false;
    const size_t smem = (size_t)(2 * (1024 / L) * (L + 1) + st.ntwp) * sizeof(cplx);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_fft_stage_p2<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 4096);
        configured = true;
    }
    dim3 grid((st.nb0 + st.B - 1) / st.B, st.nb1);
    k_fft_stage_p2<L><<<grid, 256, smem, s>>>(st);
    return true;
}

static bool launch_fft_stage_p2(const FftStage& st, cudaStream_t s) {
    return p2_launch<16>(st, s) || p2_launch<32>(st, s) || p2_launch<64>(st, s) || p2_launch<128>(st, s) ||
           p2_launch<256>(st, s) || p2_launch<512>(st, s) || p2_launch<1024>(st, s);
}

// ---------------------------------------------------------------------------
// Register-resident column FFTs, L = E * T with E = 16 values per thread and
// T = L / 16 threads per column (L = 64, 128, 256), E = 32 and T = 16 for L = 512.  Thread t of a column holds
// x[t + T j] (j < E); the transform is the two-level split
//   X[k1 + E k2] = sum_t w_T^{t k2} w_L^{t k1} sum_j x[t + T j] w_E^{j k1}
// -- an E-point DFT in registers, the twiddle, one shared-memory exchange and
// E/T T-point DFTs in registers, leaving X[(t + T s) + E k2] in a[s T + k2].
// The inverse runs the same split backwards and returns x[t + T n1] to a[n1],
// the layout the column was loaded in, so the fused x stage (forward, spectrum
// multiply, inverse) needs exactly two exchanges and no other shared traffic.
// Global access: z stages (unit stride along the transform) put a column's T
// threads on consecutive lanes; x/y stages put consecutive columns (unit
// stride apart) on consecutive lanes.
__constant__ double c_cos32[32] = {
    1.0, 0.9807852804032304, 0.9238795325112867, 0.8314696123025452, 0.7071067811865476, 0.5555702330196023,
    0.38268343236508984, 0.19509032201612833, 0.0, -0.19509032201612833, -0.38268343236508984, -0.5555702330196023,
    -0.7071067811865476, -0.8314696123025452, -0.9238795325112867, -0.9807852804032304, -1.0, -0.9807852804032304,
    -0.9238795325112867, -0.8314696123025452, -0.7071067811865476, -0.5555702330196023, -0.38268343236508984,
    -0.19509032201612833, -0.0, 0.19509032201612833, 0.38268343236508984, 0.5555702330196023, 0.7071067811865476,
    0.8314696123025452, 0.9238795325112867, 0.9807852804032304};
__constant__ double c_sin32[32] = {
    0.0, 0.19509032201612833, 0.38268343236508984, 0.5555702330196023, 0.7071067811865476, 0.8314696123025452,
    0.9238795325112867, 0.9807852804032304, 1.0, 0.9807852804032304, 0.9238795325112867, 0.8314696123025452,
    0.7071067811865476, 0.5555702330196023, 0.38268343236508984, 0.19509032201612833, -0.0, -0.19509032201612833,
    -0.38268343236508984, -0.5555702330196023, -0.7071067811865476, -0.8314696123025452, -0.9238795325112867,
    -0.9807852804032304, -1.0, -0.9807852804032304, -0.9238795325112867, -0.8314696123025452, -0.7071067811865476,
    -0.5555702330196023, -0.38268343236508984, -0.19509032201612833};

// exp(SIGN * 2 pi i e / 32)
template <int SIGN>
__device__ __forceinline__ cplx w32(int e) {
    e &= 31;
    return cplx{c_cos32[e], SIGN < 0 ? -c_sin32[e] : c_sin32[e]};
}

// one Stockham pass of radix R (span P) over N register values, x -> y
template <int N, int R, int P, int SIGN>
__device__ __forceinline__ void rpass(const cplx (&x)[N], cplx (&y)[N]) {
    constexpr int M = N / R, S = 32 / (R * P);   // w_{RP}^{qk} = w_32^{qkS}
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const int k = j % P, base = (j / P) * P * R + k;
        if (R == 4) {
            cplx a0 = x[j], a1 = x[j + M], a2 = x[j + 2 * M], a3 = x[j + 3 * M];
            if (k) {
                a1 = a1 * w32<SIGN>(k * S);
                a2 = a2 * w32<SIGN>(2 * k * S);
                a3 = a3 * w32<SIGN>(3 * k * S);
            }
            const cplx t0 = a0 + a2, t1 = a0 - a2, t2 = a1 + a3, t3 = mul_si(a1 - a3, SIGN);
            y[base] = t0 + t2;
            y[base + P] = t1 + t3;
            y[base + 2 * P] = t0 - t2;
            y[base + 3 * P] = t1 - t3;
        } else {
            cplx a0 = x[j], a1 = x[j + M];
            if (k) a1 = a1 * w32<SIGN>(k * S);
            y[base] = a0 + a1;
            y[base + P] = a0 - a1;
        }
    }
}

// natural-order N-point DFT (N | 32) of a register array, in place
template <int N, int SIGN, int P = 1>
__device__ __forceinline__ void dft_reg(cplx (&a)[N]) {
    if constexpr (P < N) {
        constexpr int R = (N / P >= 4) ? 4 : 2;
        cplx b[N];
        rpass<N, R, P, SIGN>(a, b);
#pragma unroll
        for (int i = 0; i < N; ++i) a[i] = b[i];
        dft_reg<N, SIGN, P * R>(a);
    }
}

// In-place radix-2 decimation in frequency on a register array (N | 32), then a
// compile-time bit-reversal renaming: natural order in and out.  Each butterfly
// overwrites its own two inputs, so the live set stays ~N values (the Stockham
// passes above keep input and output arrays live together); FFTPIM_FFT_IP=1
// selects it for the L = 512 (E = 32) register kernel.
template <int N>
__host__ __device__ constexpr int bitrev_c(int k) {
    int r = 0;
    for (int m = 1; m < N; m <<= 1) {
        r = (r << 1) | (k & 1);
        k >>= 1;
    }
    return r;
}
template <int N, int SIGN>
__device__ __forceinline__ void dft_reg_ip(cplx (&a)[N]) {
#pragma unroll
    for (int h = N / 2; h >= 1; h >>= 1) {
#pragma unroll
        for (int b = 0; b < N; b += 2 * h) {
#pragma unroll
            for (int j = 0; j < h; ++j) {
                const cplx u = a[b + j], v = a[b + j + h];
                a[b + j] = u + v;
                const cplx d = u - v;
                // w_{2h}^j = w_32^(j * 16 / h)
                const int e = j * (16 / h);
                if (e == 0)
                    a[b + j + h] = d;
                else if (e == 8)
                    a[b + j + h] = mul_si(d, SIGN);
                else
                    a[b + j + h] = d * w32<SIGN>(e);
            }
        }
    }
    cplx t[N];
#pragma unroll
    for (int k = 0; k < N; ++k) t[k] = a[bitrev_c<N>(k)];
#pragma unroll
    for (int k = 0; k < N; ++k) a[k] = t[k];
}

// w_L^{SIGN m}, m < L, from the plan's table exp(-2 pi i m / L)
template <int SIGN>
__device__ __forceinline__ cplx twl(const cplx* __restrict__ tw, int m) {
    const double2 w = __ldg(reinterpret_cast<const double2*>(tw) + m);
    return SIGN < 0 ? cplx{w.x, w.y} : cplx{w.x, -w.y};
}

// values per thread: 16 for L <= 256, 32 for L = 512 (T = L / E threads per
// column; the second level needs T | E)
template <int L>
struct RegE {
    static constexpr int E = L <= 256 ? 16 : 32;
};

// TS: stride into the twiddle table (1: tw has L entries; 3: tw is the table
// of a length-3L transform, w_L^m = tw[3 m])
struct RegNoOp {
    __device__ __forceinline__ void operator()() const {}
};

// `mid` runs right after the exchange barrier, when the first-level values have
// left the registers: the fused x stage issues its spectrum loads there, so their
// DRAM latency overlaps the second-level DFTs
template <int L, int SIGN, int TS = 1, bool IP = false, class Mid = RegNoOp>
__device__ __forceinline__ void reg_fwd(cplx (&a)[RegE<L>::E], cplx* buf, int t, const cplx* tw, Mid mid = Mid()) {
    constexpr int E = RegE<L>::E, T = L / E;
    if constexpr (IP)
        dft_reg_ip<E, SIGN>(a);
    else
        dft_reg<E, SIGN>(a);
#pragma unroll
    for (int k1 = 1; k1 < E; ++k1) a[k1] = a[k1] * twl<SIGN>(tw, ((t * k1) & (L - 1)) * TS);
#pragma unroll
    for (int k1 = 0; k1 < E; ++k1) buf[k1 * (T + 1) + t] = a[k1];
    __syncthreads();
    mid();
#pragma unroll
    for (int s = 0; s < E / T; ++s) {
        cplx b[T];
        const cplx* row = buf + (t + T * s) * (T + 1);
#pragma unroll
        for (int u = 0; u < T; ++u) b[u] = row[u];
        dft_reg<T, SIGN>(b);
#pragma unroll
        for (int k2 = 0; k2 < T; ++k2) a[s * T + k2] = b[k2];
    }
}

// inverse of the layout reg_fwd leaves (unnormalised, sign +1)
template <int L, int TS = 1, bool IP = false>
__device__ __forceinline__ void reg_inv(cplx (&a)[RegE<L>::E], cplx* buf, int t, const cplx* tw) {
    constexpr int E = RegE<L>::E, T = L / E;
    __syncthreads();   // buf reuse
#pragma unroll
    for (int s = 0; s < E / T; ++s) {
        const int k1 = t + T * s;
        cplx b[T];
#pragma unroll
        for (int k2 = 0; k2 < T; ++k2) b[k2] = a[s * T + k2];
        dft_reg<T, +1>(b);
        cplx* row = buf + k1 * (T + 1);
#pragma unroll
        for (int n2 = 0; n2 < T; ++n2) row[n2] = n2 ? b[n2] * twl<+1>(tw, ((k1 * n2) & (L - 1)) * TS) : b[n2];
    }
    __syncthreads();
#pragma unroll
    for (int k1 = 0; k1 < E; ++k1) a[k1] = buf[k1 * (T + 1) + t];
    if constexpr (IP)
        dft_reg_ip<E, +1>(a);
    else
        dft_reg<E, +1>(a);
}

#define RF_THREADS 128
#ifndef FFT_SPEC_EARLY   // fused x stage: spectrum loads issued before the second-level DFTs
#define FFT_SPEC_EARLY 0   // measured slower at C4 (x stage 1.55-1.57 vs 1.39-1.49 ms: 176 B of spills at 255 registers), C2 equal
#endif
#ifndef FFT_PF_FOLDED   // L2 prefetch of the spectrum rows also when the table is read at folded columns
#define FFT_PF_FOLDED 0   // measured slower at C4 (x stage 1.41 -> 1.64 ms)
#endif
#ifndef RF_MINB512
#define RF_MINB512 3
#endif
template <int L, bool ZC, bool IP = false>
__global__ void __launch_bounds__(RF_THREADS, (L == 512 && IP) ? RF_MINB512 : 1) k_fft_reg(FftStage st) {
    constexpr int E = RegE<L>::E, T = L / E, CPB = RF_THREADS / T, CS = E * (T + 1) + 1;
    extern __shared__ cplx xs[];
    const int c = ZC ? threadIdx.x / T : threadIdx.x % CPB;
    const int t = ZC ? threadIdx.x % T : threadIdx.x / CPB;
    const int col = blockIdx.x * CPB + c;
    const bool okc = col < st.nb0;
    bool pf = st.spec && st.spec_s0 == 1;
    int64_t pf_col = (int64_t)blockIdx.x * CPB;
    const int pf_n = min(CPB, st.nb0 - (int)blockIdx.x * CPB);
    if (pf && (st.fold_y | st.fold_z)) {
        // folded table: the block's columns map to a contiguous (possibly reversed)
        // run of folded columns when they stay inside one ky row and on one side of the fold
        auto fold = [&](int cc) {
            int ky = cc / st.spec_L2, kz = cc - ky * st.spec_L2;
            if (st.fold_y && 2 * ky > st.fold_y) ky = st.fold_y - ky;
            if (st.fold_z && 2 * kz > st.fold_z) kz = st.fold_z - kz;
            return (int64_t)ky * st.spec_L2 + kz;
        };
        const int c0 = (int)blockIdx.x * CPB;
        const int64_t f0 = fold(c0), f1 = fold(c0 + pf_n - 1);
        pf = (f1 - f0 == pf_n - 1) || (f0 - f1 == pf_n - 1);
        pf_col = f0 < f1 ? f0 : f1;
        static_assert(FFT_PF_FOLDED == 0 || FFT_PF_FOLDED == 1, "");
        if (!FFT_PF_FOLDED) pf = false;
    }
    if (pf) {
        // pull this block's spectrum rows (CPB consecutive columns per k) into L2
        // now; they are read after the forward transform
        const int ncols = pf_n;
        const cplx* sp0 = st.spec + (int64_t)blockIdx.y * st.spec_s1 + pf_col;
        for (int k = threadIdx.x; k < L; k += RF_THREADS)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sp0 + (int64_t)k * st.spec_stride),
                         "r"(ncols * (int)sizeof(cplx))
                         : "memory");
    }
    const cplx* __restrict__ in = st.in + (int64_t)blockIdx.y * st.in_s1 + (int64_t)col * st.in_s0;
    cplx a[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const int i = t + T * j;
        a[j] = (okc && i < st.lin) ? in[(int64_t)i * st.in_stride] : mk(0.0);
    }
    cplx* buf = xs + c * CS;
    cplx* out = st.out + (int64_t)blockIdx.y * st.out_s1 + (int64_t)col * st.out_s0;
    if (st.spec) {
        int64_t fcol = col;
        if (st.fold_y | st.fold_z) {
            int ky = col / st.spec_L2, kz = col - ky * st.spec_L2;
            if (st.fold_y && 2 * ky > st.fold_y) ky = st.fold_y - ky;
            if (st.fold_z && 2 * kz > st.fold_z) kz = st.fold_z - kz;
            fcol = (int64_t)ky * st.spec_L2 + kz;
        }
        const cplx* sp = st.spec + (int64_t)blockIdx.y * st.spec_s1 + fcol * st.spec_s0;
#if FFT_SPEC_EARLY
        cplx kh[E];
        reg_fwd<L, -1, 1, IP>(a, buf, t, st.tw, [&]() {
            if (okc) {
#pragma unroll
                for (int s = 0; s < E / T; ++s)
#pragma unroll
                    for (int k2 = 0; k2 < T; ++k2) kh[s * T + k2] = sp[(int64_t)(t + T * s + E * k2) * st.spec_stride];
            }
        });
        if (okc) {
#pragma unroll
            for (int j = 0; j < E; ++j) a[j] = a[j] * kh[j];
        }
#else
        reg_fwd<L, -1, 1, IP>(a, buf, t, st.tw);
        if (okc) {
#pragma unroll
            for (int s = 0; s < E / T; ++s)
#pragma unroll
                for (int k2 = 0; k2 < T; ++k2)
                    a[s * T + k2] = a[s * T + k2] * sp[(int64_t)(t + T * s + E * k2) * st.spec_stride];
        }
#endif
        reg_inv<L, 1, IP>(a, buf, t, st.tw);
#pragma unroll
        for (int n1 = 0; n1 < E; ++n1) {
            const int i = t + T * n1;
            if (okc && i < st.lout) out[(int64_t)i * st.out_stride] = a[n1];
        }
        return;
    }
    if (st.sign < 0)
        reg_fwd<L, -1, 1, IP>(a, buf, t, st.tw);
    else
        reg_fwd<L, +1, 1, IP>(a, buf, t, st.tw);
#pragma unroll
    for (int s = 0; s < E / T; ++s)
#pragma unroll
        for (int k2 = 0; k2 < T; ++k2) {
            const int k = t + T * s + E * k2;
            if (okc && k < st.lout) out[(int64_t)k * st.out_stride] = a[s * T + k2];
        }
}

template <int L>
static bool reg_launch(const FftStage& st, cudaStream_t s) {
    if (st.L != L) return false;
    constexpr int E = RegE<L>::E, T = L / E, CPB = RF_THREADS / T, CS = E * (T + 1) + 1;
    const size_t smem = (size_t)CPB * CS * sizeof(cplx);
    static bool configured = false;
    static const bool ip = [] {   // in-place E-point register DFTs (fewer live registers)
        const char* e = getenv("FFTPIM_FFT_IP");
        return e && e[0] == '1';
    }();
    if (!configured) {
        cudaFuncSetAttribute(k_fft_reg<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_fft_reg<L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_fft_reg<L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_fft_reg<L, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    dim3 grid((st.nb0 + CPB - 1) / CPB, st.nb1);
    if (ip) {
        if (st.in_stride == 1)
            k_fft_reg<L, true, true><<<grid, RF_THREADS, smem, s>>>(st);
        else
            k_fft_reg<L, false, true><<<grid, RF_THREADS, smem, s>>>(st);
        return true;
    }
    if (st.in_stride == 1)
        k_fft_reg<L, true><<<grid, RF_THREADS, smem, s>>>(st);
    else
        k_fft_reg<L, false><<<grid, RF_THREADS, smem, s>>>(st);
    return true;
}

// ---------------------------------------------------------------------------
// L = 3 M (M = 32 .. 256: L = 96, 192, 384, 768) register-resident column FFTs
// by one radix-3 split in frequency:
//   X[3k + r] = FFT_M(y_r)[k],   y_r[n] = w_L^(s n r) sum_m x[n + m M] w_3^(s m r)
// A column has 3 T threads (T = M / 16): thread (r, t) builds y_r[t + T j]
// (j < 16) from its three input rows and runs group r's M-point register FFT
// (reg_fwd with the L table at stride 3).  The inverse of the fused x stage
// runs the group FFTs backwards (reg_inv) and recombines the groups through
// shared memory:  x[n + m M] = sum_r w_3^(m r) w_L^(n r) z_r[n].
#define RF3_THREADS 192
template <int SIGN>
__device__ __forceinline__ cplx w3pow(int e) {   // exp(SIGN 2 pi i e / 3)
    const double h = 0.86602540378443864676;
    switch (e % 3) {
        case 0: return cplx{1.0, 0.0};
        case 1: return cplx{-0.5, SIGN < 0 ? -h : h};
        default: return cplx{-0.5, SIGN < 0 ? h : -h};
    }
}

template <int M, int SIGN>
__device__ __forceinline__ void reg3_split(cplx (&a)[16], const cplx* __restrict__ in, int64_t stride, int lin,
                                           bool okc, int r, int t, const cplx* tw) {
    constexpr int L = 3 * M, T = M / 16;
    const cplx w1 = w3pow<SIGN>(r), w2 = w3pow<SIGN>(2 * r);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int n = t + T * j;
        const cplx v0 = (okc && n < lin) ? in[(int64_t)n * stride] : mk(0.0);
        const cplx v1 = (okc && n + M < lin) ? in[(int64_t)(n + M) * stride] : mk(0.0);
        const cplx v2 = (okc && n + 2 * M < lin) ? in[(int64_t)(n + 2 * M) * stride] : mk(0.0);
        const cplx y = v0 + w1 * v1 + w2 * v2;
        a[j] = r ? y * twl<SIGN>(tw, (n * r) % L) : y;
    }
}

template <int M, bool ZC>
__global__ void __launch_bounds__(RF3_THREADS) k_fft_reg3(FftStage st) {
    constexpr int L = 3 * M, E = 16, T = M / E, TPC = 3 * T, CPB = RF3_THREADS / TPC, CS = E * (T + 1) + 1;
    constexpr int COLS = 3 * CS > L ? 3 * CS : L;   // shared words per column
    extern __shared__ cplx xs[];
    const int c = ZC ? threadIdx.x / TPC : threadIdx.x % CPB;
    const int u = ZC ? threadIdx.x % TPC : threadIdx.x / CPB;
    const int r = u / T, t = u % T;
    const int col = blockIdx.x * CPB + c;
    const bool okc = col < st.nb0;
    const cplx* __restrict__ in = st.in + (int64_t)blockIdx.y * st.in_s1 + (int64_t)col * st.in_s0;
    cplx* out = st.out + (int64_t)blockIdx.y * st.out_s1 + (int64_t)col * st.out_s0;
    cplx* cbuf = xs + c * COLS;
    cplx* buf = cbuf + r * CS;
    cplx a[E];
    if (st.spec) {
        reg3_split<M, -1>(a, in, st.in_stride, st.lin, okc, r, t, st.tw);
        reg_fwd<M, -1, 3>(a, buf, t, st.tw);
        int64_t fcol = col;
        if (st.fold_y | st.fold_z) {   // even khat along y / z: read the folded column
            int ky = col / st.spec_L2, kz = col - ky * st.spec_L2;
            if (st.fold_y && 2 * ky > st.fold_y) ky = st.fold_y - ky;
            if (st.fold_z && 2 * kz > st.fold_z) kz = st.fold_z - kz;
            fcol = (int64_t)ky * st.spec_L2 + kz;
        }
        const cplx* sp = st.spec + (int64_t)blockIdx.y * st.spec_s1 + fcol * st.spec_s0;
        if (okc) {
#pragma unroll
            for (int s2 = 0; s2 < E / T; ++s2)
#pragma unroll
                for (int k2 = 0; k2 < T; ++k2)
                    a[s2 * T + k2] = a[s2 * T + k2] * sp[(int64_t)(3 * (t + T * s2 + E * k2) + r) * st.spec_stride];
        }
        reg_inv<M, 3>(a, buf, t, st.tw);
        // recombine: thread (m, t) produces x[n + m M] from the three groups' z_r[n]
        __syncthreads();
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const int n = t + T * j;
            cbuf[r * M + n] = r ? a[j] * twl<+1>(st.tw, (n * r) % L) : a[j];
        }
        __syncthreads();
        const cplx w1 = w3pow<+1>(r), w2 = w3pow<+1>(2 * r);
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const int n = t + T * j, i = n + r * M;
            if (okc && i < st.lout) out[(int64_t)i * st.out_stride] = cbuf[n] + w1 * cbuf[M + n] + w2 * cbuf[2 * M + n];
        }
        return;
    }
    if (st.sign < 0) {
        reg3_split<M, -1>(a, in, st.in_stride, st.lin, okc, r, t, st.tw);
        reg_fwd<M, -1, 3>(a, buf, t, st.tw);
    } else {
        reg3_split<M, +1>(a, in, st.in_stride, st.lin, okc, r, t, st.tw);
        reg_fwd<M, +1, 3>(a, buf, t, st.tw);
    }
#pragma unroll
    for (int s2 = 0; s2 < E / T; ++s2)
#pragma unroll
        for (int k2 = 0; k2 < T; ++k2) {
            const int k = 3 * (t + T * s2 + E * k2) + r;
            if (okc && k < st.lout) out[(int64_t)k * st.out_stride] = a[s2 * T + k2];
        }
}

template <int M>
static bool reg3_launch(const FftStage& st, cudaStream_t s) {
    if (st.L != 3 * M) return false;
    constexpr int L = 3 * M, T = M / 16, TPC = 3 * T, CPB = RF3_THREADS / TPC, CS = 16 * (T + 1) + 1;
    constexpr int COLS = 3 * CS > L ? 3 * CS : L;
    const size_t smem = (size_t)CPB * COLS * sizeof(cplx);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_fft_reg3<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_fft_reg3<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    dim3 grid((st.nb0 + CPB - 1) / CPB, st.nb1);
    if (st.in_stride == 1)
        k_fft_reg3<M, true><<<grid, RF3_THREADS, smem, s>>>(st);
    else
        k_fft_reg3<M, false><<<grid, RF3_THREADS, smem, s>>>(st);
    return true;
}

// ---------------------------------------------------------------------------
// L = 512 as 8 x 8 x 8 (E = 8 values per thread, 64 threads per column): three
// register radix-8 levels with two shared-memory exchanges per direction.
// n = t + 64 j (t = t1 + 8 t2), k = ka + 8 m1 + 64 m2:
//   A: thread t:          DFT_8 over j  -> ka,  x w_512^(t ka)
//   B: thread (ka, t1):   DFT_8 over t2 -> m1,  x w_64^(t1 m1)
//   C: thread (ka, m1):   DFT_8 over t1 -> m2
// The fused x stage multiplies by the spectrum in layout C and runs the three
// levels backwards (conjugate twiddles) to the loading layout.  8 complex values
// per thread instead of 32: ~64 registers, six times the resident warps of the
// E = 32 kernel, at twice its shared-memory exchanges.
#define R8_NT 256
template <bool ZC>
__global__ void __launch_bounds__(R8_NT) k_fft_r8x3(FftStage st) {
    constexpr int CPB = R8_NT / 64, AS = 65, BS = 9;   // row strides of the two exchange layouts
    extern __shared__ cplx xs8[];
    const int c = ZC ? threadIdx.x / 64 : threadIdx.x % CPB;
    const int t = ZC ? threadIdx.x % 64 : threadIdx.x / CPB;
    const int col = blockIdx.x * CPB + c;
    const bool okc = col < st.nb0;
    cplx* buf = xs8 + c * (8 * AS > 64 * BS ? 8 * AS : 64 * BS);
    const cplx* __restrict__ in = st.in + (int64_t)blockIdx.y * st.in_s1 + (int64_t)col * st.in_s0;
    cplx* out = st.out + (int64_t)blockIdx.y * st.out_s1 + (int64_t)col * st.out_s0;
    const int hi = t >> 3, lo = t & 7;   // level B/C thread coordinates (ka, t1) / (ka, m1)
    cplx a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int i = t + 64 * j;
        a[j] = (okc && i < st.lin) ? in[(int64_t)i * st.in_stride] : mk(0.0);
    }
    auto forward = [&](auto sgn) {
        constexpr int SG = decltype(sgn)::value;
        dft_reg<8, SG>(a);                                   // A
#pragma unroll
        for (int ka = 1; ka < 8; ++ka) a[ka] = a[ka] * twl<SG>(st.tw, t * ka);
#pragma unroll
        for (int ka = 0; ka < 8; ++ka) buf[ka * AS + t] = a[ka];
        __syncthreads();
#pragma unroll
        for (int t2 = 0; t2 < 8; ++t2) a[t2] = buf[hi * AS + lo + 8 * t2];
        dft_reg<8, SG>(a);                                   // B (ka = hi, t1 = lo)
#pragma unroll
        for (int m1 = 1; m1 < 8; ++m1) a[m1] = a[m1] * twl<SG>(st.tw, 8 * lo * m1);
        __syncthreads();
#pragma unroll
        for (int m1 = 0; m1 < 8; ++m1) buf[(hi * 8 + m1) * BS + lo] = a[m1];
        __syncthreads();
#pragma unroll
        for (int t1 = 0; t1 < 8; ++t1) a[t1] = buf[(hi * 8 + lo) * BS + t1];
        dft_reg<8, SG>(a);                                   // C (ka = hi, m1 = lo) -> m2
    };
    // layout C: value m2 of thread (ka = hi, m1 = lo) is X[hi + 8 lo + 64 m2]
    if (st.spec) {
        forward(std::integral_constant<int, -1>());
        int64_t fcol = col;
        if (st.fold_y | st.fold_z) {
            int ky = col / st.spec_L2, kz = col - ky * st.spec_L2;
            if (st.fold_y && 2 * ky > st.fold_y) ky = st.fold_y - ky;
            if (st.fold_z && 2 * kz > st.fold_z) kz = st.fold_z - kz;
            fcol = (int64_t)ky * st.spec_L2 + kz;
        }
        const cplx* sp = st.spec + (int64_t)blockIdx.y * st.spec_s1 + fcol * st.spec_s0;
        if (okc) {
#pragma unroll
            for (int m2 = 0; m2 < 8; ++m2) a[m2] = a[m2] * sp[(int64_t)(hi + 8 * lo + 64 * m2) * st.spec_stride];
        }
        dft_reg<8, +1>(a);                                   // C^-1: m2 -> t1
        __syncthreads();
#pragma unroll
        for (int t1 = 0; t1 < 8; ++t1) buf[(hi * 8 + lo) * BS + t1] = a[t1];
        __syncthreads();
#pragma unroll
        for (int m1 = 0; m1 < 8; ++m1) a[m1] = buf[(hi * 8 + m1) * BS + lo];   // thread (ka, t1)
#pragma unroll
        for (int m1 = 1; m1 < 8; ++m1) a[m1] = a[m1] * twl<+1>(st.tw, 8 * lo * m1);
        dft_reg<8, +1>(a);                                   // B^-1: m1 -> t2
        __syncthreads();
#pragma unroll
        for (int t2 = 0; t2 < 8; ++t2) buf[hi * AS + lo + 8 * t2] = a[t2];
        __syncthreads();
#pragma unroll
        for (int ka = 0; ka < 8; ++ka) a[ka] = buf[ka * AS + t];   // thread t
#pragma unroll
        for (int ka = 1; ka < 8; ++ka) a[ka] = a[ka] * twl<+1>(st.tw, t * ka);
        dft_reg<8, +1>(a);                                   // A^-1: ka -> j
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int i = t + 64 * j;
            if (okc && i < st.lout) out[(int64_t)i * st.out_stride] = a[j];
        }
        return;
    }
    if (st.sign < 0)
        forward(std::integral_constant<int, -1>());
    else
        forward(std::integral_constant<int, +1>());
#pragma unroll
    for (int m2 = 0; m2 < 8; ++m2) {
        const int k = hi + 8 * lo + 64 * m2;
        if (okc && k < st.lout) out[(int64_t)k * st.out_stride] = a[m2];
    }
}

static bool r8x3_launch(const FftStage& st, cudaStream_t s) {
    if (st.L != 512) return false;
    constexpr int CPB = R8_NT / 64;
    const size_t smem = (size_t)CPB * (8 * 65 > 64 * 9 ? 8 * 65 : 64 * 9) * sizeof(cplx);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_fft_r8x3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_fft_r8x3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    dim3 grid((st.nb0 + CPB - 1) / CPB, st.nb1);
    if (st.in_stride == 1)
        k_fft_r8x3<true><<<grid, R8_NT, smem, s>>>(st);
    else
        k_fft_r8x3<false><<<grid, R8_NT, smem, s>>>(st);
    return true;
}

static bool launch_fft_stage_reg(const FftStage& st, cudaStream_t s) {
    static const bool off = [] {
        const char* e = getenv("FFTPIM_FFT_REG");
        return e && e[0] == '0';
    }();
    if (off) return false;
    static const bool r512 = [] {
        const char* e = getenv("FFTPIM_FFT_REG512");
        return !(e && e[0] == '0');
    }();
    static const bool r3 = [] {
        const char* e = getenv("FFTPIM_FFT_REG3");
        return !(e && e[0] == '0');
    }();
    static const bool r8 = [] {   // L = 512 as 8 x 8 x 8: FFTPIM_FFT_R8=1 (measured 2x slower at C4 than
        const char* e = getenv("FFTPIM_FFT_R8");   // the E = 32 two-level kernel: shared-memory bound)
        return e && e[0] == '1';
    }();
    return reg_launch<64>(st, s) || reg_launch<128>(st, s) || reg_launch<256>(st, s) ||
           (r512 && r8 && r8x3_launch(st, s)) || (r512 && reg_launch<512>(st, s)) ||
           (r3 && (reg3_launch<32>(st, s) || reg3_launch<64>(st, s) || reg3_launch<128>(st, s) ||
                   reg3_launch<256>(st, s)));
}

size_t fft_stage_smem(const FftStage& st) { return (size_t)(2 * st.B * (st.L + 1) + st.L + st.ntwp) * sizeof(cplx); }

void launch_fft_stage(const FftStage& st, cudaStream_t s) {
    if (launch_fft_stage_reg(st, s) || launch_fft_stage_p2(st, s)) {
        fftpim_count_launch();
        return;
    }
    const size_t smem = fft_stage_smem(st);
    static size_t configured = 48 * 1024;
    if (smem > configured) {
        cudaFuncSetAttribute(k_fft_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    dim3 grid((st.nb0 + st.B - 1) / st.B, st.nb1);
    k_fft_stage<<<grid, 256, smem, s>>>(st);
    fftpim_count_launch();
}
