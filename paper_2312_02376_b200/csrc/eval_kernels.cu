// eval_kernels.cu -- the hot path, SolvePlan.evaluate (solver.py:24-25):
//   K0  q -> sorted order
//   K1  near projection, owner-computes gather per grid node (grids.py:167-181)
//   K2  spectrum multiply between the cuFFT passes (nearzone.py:500-504)
//   K5a far projection, per-warp private grids in shared memory (farzone.py:156)
//   K5b far grid superposition sum (farzone.py:157-158)
//   K3+K4+K5c fused observer pass: near interpolation, correction matvec and far
//       interpolation in one warp per observer (grids.py:183-188, nearzone.py:506-524,
//       farzone.py:159)
// Every reduction has a fixed order: results are bitwise reproducible run to run.
#include <cub/block/block_radix_sort.cuh>

#include "geom.cuh"
#include "kernels.h"

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

__device__ __forceinline__ cplx warp_sum(cplx v) {
    for (int o = 16; o > 0; o >>= 1) {
        v.re += __shfl_xor_sync(0xffffffffu, v.re, o);
        v.im += __shfl_xor_sync(0xffffffffu, v.im, o);
    }
    return v;
}

// ---------------------------------------------------------------- K0
__global__ void k_permute_q(const cplx* __restrict__ q, const int* __restrict__ perm, int64_t n,
                            cplx* __restrict__ qs) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) qs[i] = q[perm[i]];
}
// NPSP plans (real coefficients) also keep the real parts and flag any charge
// with a nonzero imaginary part: real charges let K4 gather 8 B per pair
// instead of 16 (bit-identical: the imaginary products are exact zeros)
__global__ void k_permute_q_r(const cplx* __restrict__ q, const int* __restrict__ perm, int64_t n,
                              cplx* __restrict__ qs, double* __restrict__ qre, int* flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const cplx v = q[perm[i]];
    qs[i] = v;
    qre[i] = v.re;
    if (v.im != 0.0) *flag = 1;
}
void launch_permute_q(const EvalArgs& a, cudaStream_t s) {
    if (a.N == 0) return;
    if (a.q_re) {
        cudaMemsetAsync(a.q_flag, 0, sizeof(int), s);
        k_permute_q_r<<<nblk(a.N, 256), 256, 0, s>>>(a.q, a.src_perm, a.N, a.q_sorted, a.q_re, a.q_flag);
    } else {
        k_permute_q<<<nblk(a.N, 256), 256, 0, s>>>(a.q, a.src_perm, a.N, a.q_sorted);
    }
    fftpim_count_launch();
}

// ---------------------------------------------------------------- K1
// One thread per element of the zero-padded (2n)^3 buffer: padding slots write
// 0, grid nodes gather the points whose stencil covers them.  Points are
// sorted by stencil start, so for fixed (x, y) start offsets the candidate z
// starts form one contiguous CSR range.
template <int W>
__global__ void __launch_bounds__(256) k_near_project(EvalArgs a) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const StencilGeom& g = a.g;
    if (t >= (int64_t)a.knx * g.n[1] * g.n[2]) return;
    const int z = (int)(t % g.n[2]), y = (int)((t / g.n[2]) % g.n[1]),
              x = (int)(t / ((int64_t)g.n[1] * g.n[2])) + a.kx0;
    cplx acc = mk(0.0);
    {
        const int wx = g.w[0], wy = g.w[1], wz = g.w[2];
        const int zlo = max(z - (wz - 1), 0), zhi = min(z, g.nc[2] - 1);
        for (int ia = 0; ia < wx; ++ia) {
            const int sx = x - ia;
            if (sx < 0 || sx >= g.nc[0] || zlo > zhi) continue;
            // all W candidate ranges of this x offset loaded before any point is touched
            int r0[W], r1[W];
#pragma unroll
            for (int ib = 0; ib < W; ++ib) {
                const int sy = y - ib;
                const bool ok = ib < wy && sy >= 0 && sy < g.nc[1];
                const int k0 = ok ? (sx * g.nc[1] + sy) * g.nc[2] : 0;
                r0[ib] = ok ? a.cell_start[k0 + zlo] : 0;
                r1[ib] = ok ? a.cell_start[k0 + zhi + 1] : 0;
            }
#pragma unroll
            for (int ib = 0; ib < W; ++ib) {
                for (int p = r0[ib]; p < r1[ib]; ++p) {
                    const double* w = a.src_w + (int64_t)p * 3 * W;
                    const int ic = z - a.src_start[3 * (int64_t)p + 2];
                    const double wgt = (w[ia] * w[W + ib]) * w[2 * W + ic];
                    const cplx qv = a.q_sorted[p];
                    acc.re += wgt * qv.re;
                    acc.im += wgt * qv.im;
                }
            }
        }
    }
    a.k1_out[((int64_t)(x - a.kx0) * a.go1 + y) * a.go2 + z] = acc;
}

bool launch_near_project_tiled(const EvalArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- K1 as a fixed sparse operator
// The projection weights depend only on the source positions, so the plan can
// hold K1 as a sliced-ELL matrix over the grid nodes (rows).  Within each window
// of K1E_WIN consecutive rows the rows are ordered by decreasing length
// (k1_row), so the 32 rows of a slice have nearly equal lengths; entry k of slot
// t (= sorted position) lives at off[t / 32] + 128 (k / 4) + 4 (t % 32) + k % 4
// (int32 source index, fp64 weight product): groups of four entries per lane,
// one 16-byte index load and two 16-byte weight loads per group, the warp's
// loads contiguous.  Each row lists its points in the gather K1's
// order (ia, ib, ascending point) with the same weight expression, so the
// evaluation sums are bit-identical to k_near_project's.
#define K1E_WIN 256
template <int W, bool FILL>
__global__ void __launch_bounds__(256) k_k1_rows(EvalArgs a, int* cnt, const int* row_of, const int64_t* off,
                                                 const int* remap, int* idx, double* wgt) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const StencilGeom& g = a.g;
    if (t >= (int64_t)a.knx * g.n[1] * g.n[2]) return;
    const int64_t r = FILL ? row_of[t] : t;
    const int z = (int)(r % g.n[2]), y = (int)((r / g.n[2]) % g.n[1]),
              x = (int)(r / ((int64_t)g.n[1] * g.n[2])) + a.kx0;
    const int64_t base = FILL ? off[t >> 5] + 4 * (t & 31) : 0;
    int n = 0;
    const int wx = g.w[0], wy = g.w[1], wz = g.w[2];
    const int zlo = max(z - (wz - 1), 0), zhi = min(z, g.nc[2] - 1);
    for (int ia = 0; ia < wx; ++ia) {
        const int sx = x - ia;
        if (sx < 0 || sx >= g.nc[0] || zlo > zhi) continue;
        for (int ib = 0; ib < wy; ++ib) {
            const int sy = y - ib;
            if (sy < 0 || sy >= g.nc[1]) continue;
            const int k0 = (sx * g.nc[1] + sy) * g.nc[2];
            const int p0 = a.cell_start[k0 + zlo], p1 = a.cell_start[k0 + zhi + 1];
            if (FILL) {
                for (int p = p0; p < p1; ++p) {
                    const double* w = a.src_w + (int64_t)p * 3 * W;
                    const int ic = z - a.src_start[3 * (int64_t)p + 2];
                    const int64_t e = base + 128 * (int64_t)(n >> 2) + (n & 3);
                    idx[e] = remap ? remap[p] : p;
                    wgt[e] = (w[ia] * w[W + ib]) * w[2 * W + ic];
                    ++n;
                }
            } else {
                n += p1 - p0;
            }
        }
    }
    if (!FILL) cnt[t] = n;
}

// per window: rows by decreasing length (stable), lengths moved along
__global__ void __launch_bounds__(K1E_WIN) k_k1_window_sort(const int* __restrict__ cnt_row, int64_t rows,
                                                           int* cnt_sorted, int* row_of) {
    using Sort = cub::BlockRadixSort<int, K1E_WIN, 1, int>;
    __shared__ typename Sort::TempStorage tmp;
    const int64_t r = (int64_t)blockIdx.x * K1E_WIN + threadIdx.x;
    int key[1] = {r < rows ? cnt_row[r] : -1};
    int val[1] = {(int)r};
    Sort(tmp).SortDescending(key, val);
    const int64_t o = (int64_t)blockIdx.x * K1E_WIN + threadIdx.x;
    if (o < rows) {
        cnt_sorted[o] = key[0];
        row_of[o] = val[0];
    }
}

// 32 * (longest row of the slice rounded up to 4), slice s; entry nslices is 0
// (exclusive scan)
__global__ void k_k1_slice_slots(const int* __restrict__ cnt, int64_t rows, int64_t nslices, int64_t* slots) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s > nslices) return;
    int m = 0;
    if (s < nslices)
        for (int l = 0; l < 32 && 32 * s + l < rows; ++l) m = max(m, cnt[32 * s + l]);
    slots[s] = 32 * (int64_t)((m + 3) & ~3);
}

void launch_k1_count(const EvalArgs& a, int* cnt_row, int* cnt_sorted, int* row_of, int64_t* slots,
                     cudaStream_t s) {
    const int64_t rows = (int64_t)a.knx * a.g.n[1] * a.g.n[2];
    const int b = nblk(rows, 256);
    switch (a.g.order + 1) {
        case 2: k_k1_rows<2, false><<<b, 256, 0, s>>>(a, cnt_row, nullptr, nullptr, nullptr, nullptr, nullptr); break;
        case 3: k_k1_rows<3, false><<<b, 256, 0, s>>>(a, cnt_row, nullptr, nullptr, nullptr, nullptr, nullptr); break;
        case 4: k_k1_rows<4, false><<<b, 256, 0, s>>>(a, cnt_row, nullptr, nullptr, nullptr, nullptr, nullptr); break;
        case 5: k_k1_rows<5, false><<<b, 256, 0, s>>>(a, cnt_row, nullptr, nullptr, nullptr, nullptr, nullptr); break;
        case 6: k_k1_rows<6, false><<<b, 256, 0, s>>>(a, cnt_row, nullptr, nullptr, nullptr, nullptr, nullptr); break;
        default: k_k1_rows<7, false><<<b, 256, 0, s>>>(a, cnt_row, nullptr, nullptr, nullptr, nullptr, nullptr); break;
    }
    k_k1_window_sort<<<nblk(rows, K1E_WIN), K1E_WIN, 0, s>>>(cnt_row, rows, cnt_sorted, row_of);
    const int64_t nsl = (rows + 31) / 32;
    k_k1_slice_slots<<<nblk(nsl + 1, 256), 256, 0, s>>>(cnt_sorted, rows, nsl, slots);
    fftpim_count_launch(3);
}

void launch_k1_fill(const EvalArgs& a, const int* row_of, const int64_t* off, const int* remap, int* idx,
                    double* wgt, cudaStream_t s) {
    const int b = nblk((int64_t)a.knx * a.g.n[1] * a.g.n[2], 256);
    switch (a.g.order + 1) {
        case 2: k_k1_rows<2, true><<<b, 256, 0, s>>>(a, nullptr, row_of, off, remap, idx, wgt); break;
        case 3: k_k1_rows<3, true><<<b, 256, 0, s>>>(a, nullptr, row_of, off, remap, idx, wgt); break;
        case 4: k_k1_rows<4, true><<<b, 256, 0, s>>>(a, nullptr, row_of, off, remap, idx, wgt); break;
        case 5: k_k1_rows<5, true><<<b, 256, 0, s>>>(a, nullptr, row_of, off, remap, idx, wgt); break;
        case 6: k_k1_rows<6, true><<<b, 256, 0, s>>>(a, nullptr, row_of, off, remap, idx, wgt); break;
        default: k_k1_rows<7, true><<<b, 256, 0, s>>>(a, nullptr, row_of, off, remap, idx, wgt); break;
    }
    fftpim_count_launch();
}

// one thread per slot (grid node).  Every lane of a slice runs the slice's
// longest row rounded up to 4 (windows are sorted by decreasing length, so the
// slice's first slot holds it); padding entries are (index 0, weight 0) and add
// exact zeros.  The loads are volatile asm so they issue in program order: all
// index and weight loads of a two-group chunk, then its eight gathers.
__device__ __forceinline__ int4 ld_cs_i4(const int* p) {
    int4 v;
    asm volatile("ld.global.cs.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_cs_d2(const double* p) {
    double2 v;
    asm volatile("ld.global.cs.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_d2(const cplx* p) {
    double2 v;
    asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

#ifndef K1E_THREADS
#define K1E_THREADS 128
#endif
#ifndef K1E_MINB
#define K1E_MINB 8
#endif
#ifndef K1_PF
#define K1_PF 1
#endif
__global__ void __launch_bounds__(K1E_THREADS, K1E_MINB) k_k1_spmv(EvalArgs a) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int n1 = a.g.n[1], n2 = a.g.n[2];
    if (t >= (int64_t)a.knx * n1 * n2) return;
    const int G = (a.k1_cnt[t & ~(int64_t)31] + 3) >> 2;   // groups of four
    const int64_t r = a.k1_row[t];
    const int64_t base = a.k1_off[t >> 5] + 4 * (t & 31);
    const int* ix = a.k1_idx + base;
    const double* wt = a.k1_wgt + base;
    const cplx* q = a.k1_q;
    double ar = 0.0, ai = 0.0;
    int g = 0;
#if K1_PF
    // the next pair of groups' indices and weights are in flight while this
    // pair's q gathers complete (same entry order: identical sums)
    int4 i0, i1;
    double2 w0, w1, w2, w3;
    if (G >= 2) {
        i0 = ld_cs_i4(ix);
        i1 = ld_cs_i4(ix + 128);
        w0 = ld_cs_d2(wt);
        w1 = ld_cs_d2(wt + 2);
        w2 = ld_cs_d2(wt + 128);
        w3 = ld_cs_d2(wt + 128 + 2);
    }
    for (; g + 2 <= G; g += 2) {
        int4 j0 = i0, j1 = i1;
        double2 x0 = w0, x1 = w1, x2 = w2, x3 = w3;
        if (g + 4 <= G) {
            j0 = ld_cs_i4(ix + 128 * (g + 2));
            j1 = ld_cs_i4(ix + 128 * (g + 3));
            x0 = ld_cs_d2(wt + 128 * (g + 2));
            x1 = ld_cs_d2(wt + 128 * (g + 2) + 2);
            x2 = ld_cs_d2(wt + 128 * (g + 3));
            x3 = ld_cs_d2(wt + 128 * (g + 3) + 2);
        }
        const double2 v0 = ld_d2(q + i0.x), v1 = ld_d2(q + i0.y), v2 = ld_d2(q + i0.z), v3 = ld_d2(q + i0.w);
        const double2 v4 = ld_d2(q + i1.x), v5 = ld_d2(q + i1.y), v6 = ld_d2(q + i1.z), v7 = ld_d2(q + i1.w);
        ar += w0.x * v0.x; ai += w0.x * v0.y;
        ar += w0.y * v1.x; ai += w0.y * v1.y;
        ar += w1.x * v2.x; ai += w1.x * v2.y;
        ar += w1.y * v3.x; ai += w1.y * v3.y;
        ar += w2.x * v4.x; ai += w2.x * v4.y;
        ar += w2.y * v5.x; ai += w2.y * v5.y;
        ar += w3.x * v6.x; ai += w3.x * v6.y;
        ar += w3.y * v7.x; ai += w3.y * v7.y;
        i0 = j0;
        i1 = j1;
        w0 = x0;
        w1 = x1;
        w2 = x2;
        w3 = x3;
    }
#else
    for (; g + 2 <= G; g += 2) {
        const int4 i0 = ld_cs_i4(ix + 128 * g), i1 = ld_cs_i4(ix + 128 * (g + 1));
        const double2 w0 = ld_cs_d2(wt + 128 * g), w1 = ld_cs_d2(wt + 128 * g + 2);
        const double2 w2 = ld_cs_d2(wt + 128 * (g + 1)), w3 = ld_cs_d2(wt + 128 * (g + 1) + 2);
        const double2 v0 = ld_d2(q + i0.x), v1 = ld_d2(q + i0.y), v2 = ld_d2(q + i0.z), v3 = ld_d2(q + i0.w);
        const double2 v4 = ld_d2(q + i1.x), v5 = ld_d2(q + i1.y), v6 = ld_d2(q + i1.z), v7 = ld_d2(q + i1.w);
        ar += w0.x * v0.x; ai += w0.x * v0.y;
        ar += w0.y * v1.x; ai += w0.y * v1.y;
        ar += w1.x * v2.x; ai += w1.x * v2.y;
        ar += w1.y * v3.x; ai += w1.y * v3.y;
        ar += w2.x * v4.x; ai += w2.x * v4.y;
        ar += w2.y * v5.x; ai += w2.y * v5.y;
        ar += w3.x * v6.x; ai += w3.x * v6.y;
        ar += w3.y * v7.x; ai += w3.y * v7.y;
    }
#endif
    if (g < G) {
        const int4 i0 = ld_cs_i4(ix + 128 * g);
        const double2 w0 = ld_cs_d2(wt + 128 * g), w1 = ld_cs_d2(wt + 128 * g + 2);
        const double2 v0 = ld_d2(q + i0.x), v1 = ld_d2(q + i0.y), v2 = ld_d2(q + i0.z), v3 = ld_d2(q + i0.w);
        ar += w0.x * v0.x; ai += w0.x * v0.y;
        ar += w0.y * v1.x; ai += w0.y * v1.y;
        ar += w1.x * v2.x; ai += w1.x * v2.y;
        ar += w1.y * v3.x; ai += w1.y * v3.y;
    }
    const int z = (int)(r % n2), y = (int)((r / n2) % n1), xl = (int)(r / ((int64_t)n1 * n2));
    a.k1_out[((int64_t)xl * a.go1 + y) * a.go2 + z] = cplx{ar, ai};
}

void launch_near_project(const EvalArgs& a, cudaStream_t s) {
    if (a.k1_rec && launch_k1_lines_g(a, a.k1_rec, s)) return;
    if (a.k1_pos && launch_k1_lines(a, a.k1_pos, s)) return;
    if (a.k1_off) {
        k_k1_spmv<<<nblk((int64_t)a.knx * a.g.n[1] * a.g.n[2], K1E_THREADS), K1E_THREADS, 0, s>>>(a);
        fftpim_count_launch();
        return;
    }
    if (launch_near_project_tiled(a, s)) return;
    const int W = a.g.order + 1;
    const int b = nblk((int64_t)a.knx * a.g.n[1] * a.g.n[2], 256);
    switch (W) {
        case 2: k_near_project<2><<<b, 256, 0, s>>>(a); break;
        case 3: k_near_project<3><<<b, 256, 0, s>>>(a); break;
        case 4: k_near_project<4><<<b, 256, 0, s>>>(a); break;
        case 5: k_near_project<5><<<b, 256, 0, s>>>(a); break;
        case 6: k_near_project<6><<<b, 256, 0, s>>>(a); break;
        default: k_near_project<7><<<b, 256, 0, s>>>(a); break;
    }
    fftpim_count_launch();
}

// Tiled K1: a block owns a TX x TY x TZ tile of grid nodes (one thread each) and
// first stages every point whose stencil can reach the tile -- the sorted points
// of the start-cell columns (sx, sy) in the tile's reach, each a contiguous run
// -- into shared memory (weights, z start, q) with coalesced loads.  The
// per-node gather then reads shared memory only, in the same order as
// k_near_project (ia, ib, ascending point), so both produce identical bits.
// Tiles whose reach holds more than the staging capacity gather from global.
#define K1_TX 4
#define K1_TY 8
#define K1_TZ 8
template <int W>
struct K1Tile {
    static constexpr int RX = K1_TX + W - 1, RY = K1_TY + W - 1, RZ = K1_TZ + W - 1;
    static constexpr int NCOL = RX * RY;
    static constexpr int CAP = W <= 4 ? 512 : 768;
};

template <int W>
__global__ void __launch_bounds__(256) k_near_project_tiled(EvalArgs a) {
    using T = K1Tile<W>;
    extern __shared__ double k1s[];
    double* sw = k1s;                                   // CAP x 3W weights
    double* sq = sw + T::CAP * 3 * W;                   // CAP x 2 (q)
    int* sz = reinterpret_cast<int*>(sq + T::CAP * 2);  // CAP z starts
    int* cs = sz + T::CAP;                              // NCOL x (RZ + 1) local cell starts
    int* coff = cs + T::NCOL * (T::RZ + 1);             // NCOL + 1 column offsets
    int* cbase = coff + T::NCOL + 1;                    // NCOL global first index
    const StencilGeom& g = a.g;
    const int x0 = a.kx0 + blockIdx.x * K1_TX, y0 = blockIdx.y * K1_TY, z0 = blockIdx.z * K1_TZ;
    const int sx0 = x0 - (W - 1), sy0 = y0 - (W - 1), sz0 = z0 - (W - 1);
    // column ranges (cells sz0 .. sz0 + RZ - 1, clipped)
    const int zl = max(sz0, 0), zh = min(sz0 + T::RZ - 1, g.nc[2] - 1);
    for (int c = threadIdx.x; c < T::NCOL; c += blockDim.x) {
        const int sx = sx0 + c / T::RY, sy = sy0 + c % T::RY;
        int lo = 0, hi = 0;
        if (sx >= 0 && sx < g.nc[0] && sy >= 0 && sy < g.nc[1] && zl <= zh) {
            const int k0 = (sx * g.nc[1] + sy) * g.nc[2];
            lo = a.cell_start[k0 + zl];
            hi = a.cell_start[k0 + zh + 1];
            for (int j = 0; j <= T::RZ; ++j) {
                const int zc = min(max(sz0 + j, zl), zh + 1);
                cs[c * (T::RZ + 1) + j] = a.cell_start[k0 + zc] - lo;
            }
        } else {
            for (int j = 0; j <= T::RZ; ++j) cs[c * (T::RZ + 1) + j] = 0;
        }
        cbase[c] = lo;
        coff[c + 1] = hi - lo;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        coff[0] = 0;
        for (int c = 0; c < T::NCOL; ++c) coff[c + 1] += coff[c];
    }
    __syncthreads();
    const int total = coff[T::NCOL];
    const bool staged = total <= T::CAP;
    if (staged) {
        for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
            int lo = 0, hi = T::NCOL;   // column of idx: coff[lo] <= idx < coff[lo+1]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (coff[mid] <= idx) lo = mid; else hi = mid;
            }
            const int64_t p = cbase[lo] + (idx - coff[lo]);
            const double* w = a.src_w + p * 3 * W;
#pragma unroll
            for (int j = 0; j < 3 * W; ++j) sw[idx * 3 * W + j] = w[j];
            const cplx qv = a.q_sorted[p];
            sq[2 * idx] = qv.re;
            sq[2 * idx + 1] = qv.im;
            sz[idx] = a.src_start[3 * p + 2];
        }
    }
    __syncthreads();
    const int x = x0 + threadIdx.x / (K1_TY * K1_TZ), y = y0 + (threadIdx.x / K1_TZ) % K1_TY, z = z0 + threadIdx.x % K1_TZ;
    if (x >= a.kx0 + a.knx || y >= g.n[1] || z >= g.n[2]) return;
    cplx acc = mk(0.0);
    const int zlo = max(z - (W - 1), 0), zhi = min(z, g.nc[2] - 1);
    for (int ia = 0; ia < W; ++ia) {
        const int sx = x - ia;
        if (sx < 0 || sx >= g.nc[0] || zlo > zhi) continue;
        for (int ib = 0; ib < W; ++ib) {
            const int sy = y - ib;
            if (sy < 0 || sy >= g.nc[1]) continue;
            const int c = (sx - sx0) * T::RY + (sy - sy0);
            if (staged) {
                const int* cc = cs + c * (T::RZ + 1);
                const int p0 = coff[c] + cc[zlo - sz0], p1 = coff[c] + cc[zhi + 1 - sz0];
                for (int p = p0; p < p1; ++p) {
                    const double* w = sw + p * 3 * W;
                    const double wgt = (w[ia] * w[W + ib]) * w[2 * W + (z - sz[p])];
                    acc.re += wgt * sq[2 * p];
                    acc.im += wgt * sq[2 * p + 1];
                }
            } else {
                const int k0 = (sx * g.nc[1] + sy) * g.nc[2];
                const int p0 = a.cell_start[k0 + zlo], p1 = a.cell_start[k0 + zhi + 1];
                for (int p = p0; p < p1; ++p) {
                    const double* w = a.src_w + (int64_t)p * 3 * W;
                    const int ic = z - a.src_start[3 * (int64_t)p + 2];
                    const double wgt = (w[ia] * w[W + ib]) * w[2 * W + ic];
                    const cplx qv = a.q_sorted[p];
                    acc.re += wgt * qv.re;
                    acc.im += wgt * qv.im;
                }
            }
        }
    }
    a.k1_out[((int64_t)(x - a.kx0) * a.go1 + y) * a.go2 + z] = acc;
}

template <int W>
static size_t k1_tiled_smem() {
    using T = K1Tile<W>;
    return (size_t)T::CAP * (3 * W + 2) * sizeof(double) + (size_t)T::CAP * sizeof(int) +
           (size_t)(T::NCOL * (T::RZ + 1) + 2 * T::NCOL + 1) * sizeof(int);
}

template <int W>
static void k1_tiled_launch(const EvalArgs& a, cudaStream_t s) {
    const size_t smem = k1_tiled_smem<W>();
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_near_project_tiled<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    dim3 grid((a.knx + K1_TX - 1) / K1_TX, (a.g.n[1] + K1_TY - 1) / K1_TY, (a.g.n[2] + K1_TZ - 1) / K1_TZ);
    k_near_project_tiled<W><<<grid, K1_TX * K1_TY * K1_TZ, smem, s>>>(a);
}

// Tap-major K1 (point-centric, deterministic): a block owns a TX x TY x TZ tile
// of stencil-start cells, one thread per cell holding its first points' stencil
// weights in registers.  For each of the (order+1)^3 taps in a fixed order every
// thread adds its cell's contribution to node cell+tap of the block's extended
// node tile in shared memory -- distinct cells hit distinct nodes for a fixed
// tap, and a barrier separates taps, so there are no races and no atomics.  The
// overlapping extended tiles are then summed per node in fixed block order.
#define K1T_TX 4
#define K1T_TY 4
#define K1T_TZ 16
#define K1T_REG 2
template <int W>
struct K1Taps {
    static constexpr int EX = K1T_TX + W - 1, EY = K1T_TY + W - 1, EZ = K1T_TZ + W - 1;
    static constexpr int NODES = EX * EY * EZ;
};

template <int W>
__global__ void __launch_bounds__(K1T_TX * K1T_TY * K1T_TZ) k_near_project_taps(EvalArgs a) {
    using T = K1Taps<W>;
    __shared__ cplx tile[T::NODES];
    const StencilGeom& g = a.g;
    for (int n = threadIdx.x; n < T::NODES; n += blockDim.x) tile[n] = mk(0.0);
    const int lx = threadIdx.x / (K1T_TY * K1T_TZ), ly = (threadIdx.x / K1T_TZ) % K1T_TY, lz = threadIdx.x % K1T_TZ;
    const int cx = a.kx0 - (W - 1) + blockIdx.x * K1T_TX + lx;   // start cells of the slab's reach
    const int cy = blockIdx.y * K1T_TY + ly, cz = blockIdx.z * K1T_TZ + lz;
    int p0 = 0, p1 = 0;
    if (cx >= 0 && cx < g.nc[0] && cy < g.nc[1] && cz < g.nc[2]) {
        const int k = (cx * g.nc[1] + cy) * g.nc[2] + cz;
        p0 = a.cell_start[k];
        p1 = a.cell_start[k + 1];
    }
    double w[K1T_REG][3 * W];
    cplx qv[K1T_REG];
    const int nreg = min(p1 - p0, K1T_REG);
#pragma unroll
    for (int r = 0; r < K1T_REG; ++r) {
        if (r < nreg) {
            const double* src = a.src_w + (int64_t)(p0 + r) * 3 * W;
#pragma unroll
            for (int j = 0; j < 3 * W; ++j) w[r][j] = src[j];
            qv[r] = a.q_sorted[p0 + r];
        }
    }
    __syncthreads();
#pragma unroll
    for (int ia = 0; ia < W; ++ia)
#pragma unroll
        for (int ib = 0; ib < W; ++ib)
#pragma unroll
            for (int ic = 0; ic < W; ++ic) {
                if (p1 > p0) {
                    cplx acc = mk(0.0);
#pragma unroll
                    for (int r = 0; r < K1T_REG; ++r)
                        if (r < nreg) {
                            const double wgt = (w[r][ia] * w[r][W + ib]) * w[r][2 * W + ic];
                            acc.re += wgt * qv[r].re;
                            acc.im += wgt * qv[r].im;
                        }
                    for (int p = p0 + K1T_REG; p < p1; ++p) {   // crowded cells: from L1/L2
                        const double* wp = a.src_w + (int64_t)p * 3 * W;
                        const double wgt = (wp[ia] * wp[W + ib]) * wp[2 * W + ic];
                        const cplx qp = a.q_sorted[p];
                        acc.re += wgt * qp.re;
                        acc.im += wgt * qp.im;
                    }
                    cplx& dst = tile[((lx + ia) * T::EY + (ly + ib)) * T::EZ + (lz + ic)];
                    dst = dst + acc;
                }
                __syncthreads();
            }
    cplx* out = a.k1_scratch + ((int64_t)(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * T::NODES;
    for (int n = threadIdx.x; n < T::NODES; n += blockDim.x) out[n] = tile[n];
}

// node (x, y, z) = sum of the extended tiles covering it, blocks in fixed order
template <int W>
__global__ void __launch_bounds__(256) k_near_project_combine(EvalArgs a, int gx, int gy, int gz) {
    using T = K1Taps<W>;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const StencilGeom& g = a.g;
    if (t >= (int64_t)a.knx * g.n[1] * g.n[2]) return;
    const int z = (int)(t % g.n[2]), y = (int)((t / g.n[2]) % g.n[1]), xl = (int)(t / ((int64_t)g.n[1] * g.n[2]));
    // block bx covers (slab-local, shifted by order) x in [bx*TX, bx*TX + EX)
    const int xs = xl + (W - 1);
    cplx acc = mk(0.0);
    for (int bx = max(0, (xs - T::EX + K1T_TX) / K1T_TX); bx <= min(gx - 1, xs / K1T_TX); ++bx) {
        const int ox = xs - bx * K1T_TX;
        if (ox >= T::EX) continue;
        for (int by = max(0, (y - T::EY + K1T_TY) / K1T_TY); by <= min(gy - 1, y / K1T_TY); ++by) {
            const int oy = y - by * K1T_TY;
            if (oy >= T::EY) continue;
            for (int bz = max(0, (z - T::EZ + K1T_TZ) / K1T_TZ); bz <= min(gz - 1, z / K1T_TZ); ++bz) {
                const int oz = z - bz * K1T_TZ;
                if (oz >= T::EZ) continue;
                acc = acc + a.k1_scratch[((int64_t)(bz * gy + by) * gx + bx) * T::NODES + (ox * T::EY + oy) * T::EZ + oz];
            }
        }
    }
    a.k1_out[((int64_t)xl * a.go1 + y) * a.go2 + z] = acc;
}

template <int W>
static void k1_taps_launch(const EvalArgs& a, cudaStream_t s) {
    // cells reaching the slab's planes: [kx0 - order, kx0 + knx) in x
    const int gx = (a.knx + W - 1 + K1T_TX - 1) / K1T_TX;
    const int gy = (a.g.nc[1] + K1T_TY - 1) / K1T_TY, gz = (a.g.nc[2] + K1T_TZ - 1) / K1T_TZ;
    k_near_project_taps<W><<<dim3(gx, gy, gz), K1T_TX * K1T_TY * K1T_TZ, 0, s>>>(a);
    const int64_t nodes = (int64_t)a.knx * a.g.n[1] * a.g.n[2];
    k_near_project_combine<W><<<nblk(nodes, 256), 256, 0, s>>>(a, gx, gy, gz);
}

int64_t k1_scratch_elems(const StencilGeom& g, int knx) {
    const int W = g.order + 1;
    const int gx = (knx + W - 1 + K1T_TX - 1) / K1T_TX;
    const int gy = (g.nc[1] + K1T_TY - 1) / K1T_TY, gz = (g.nc[2] + K1T_TZ - 1) / K1T_TZ;
    const int64_t nodes = (int64_t)(K1T_TX + W - 1) * (K1T_TY + W - 1) * (K1T_TZ + W - 1);
    return (int64_t)gx * gy * gz * nodes;
}

bool launch_near_project_tiled(const EvalArgs& a, cudaStream_t s) {
    if (a.g.n[0] < 2 || a.g.n[1] < 2 || a.g.n[2] < 2) return false;   // single-plane axes: global path
    if (a.k1_scratch) {
        switch (a.g.order + 1) {
            case 3: k1_taps_launch<3>(a, s); break;
            case 4: k1_taps_launch<4>(a, s); break;
            case 5: k1_taps_launch<5>(a, s); break;
            default: return false;
        }
        fftpim_count_launch(2);
        return true;
    }
    switch (a.g.order + 1) {
        case 3: k1_tiled_launch<3>(a, s); break;
        case 4: k1_tiled_launch<4>(a, s); break;
        case 5: k1_tiled_launch<5>(a, s); break;
        default: return false;
    }
    fftpim_count_launch();
    return true;
}

__global__ void k_axpy(cplx* __restrict__ acc, const cplx* __restrict__ x, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) acc[i] = acc[i] + x[i];
}
void launch_axpy(cplx* acc, const cplx* x, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    k_axpy<<<nblk(n, 256), 256, 0, s>>>(acc, x, n);
    fftpim_count_launch();
}

// ---------------------------------------------------------------- K2
__global__ void k_spectrum_mul(cplx* __restrict__ work, const cplx* __restrict__ khat, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) work[i] = work[i] * khat[i];
}
void launch_spectrum_mul(const EvalArgs& a, cudaStream_t s) {
    k_spectrum_mul<<<nblk(a.n_fft, 256), 256, 0, s>>>(a.work, a.khat, a.n_fft);
    fftpim_count_launch();
}

// ---------------------------------------------------------------- K5a
// Each warp takes a contiguous chunk of the (cell-sorted) points; lane l owns
// the stencil taps l, l + 32, ... and accumulates w * q in registers while the
// far stencil start stays the same (consecutive sorted points share it for runs
// of ~10 near cells), flushing the run into the warp's private copy of the far
// source grid in shared memory when the start changes (lanes own distinct
// taps, so no collisions; a warp barrier orders consecutive flushes).  Warps
// are summed in order, blocks in order by k_far_reduce: fixed order throughout.
// Point data is staged in shared memory in warp-sized batches with one
// coalesced load per lane.
template <int WF>
__global__ void __launch_bounds__(256) k_far_project(EvalArgs a) {
    extern __shared__ double smem_d[];
    const int nfy = a.fs.n[1], nfz = a.fs.n[2];
    const int nf = a.fs.n[0] * nfy * nfz;
    const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    cplx* sgrid = reinterpret_cast<cplx*>(smem_d);
    constexpr int REC = 3 * WF + 2;                       // weights + q per staged point
    constexpr int TPL = (WF * WF * WF + 31) / 32;         // taps per lane
    double* stage = smem_d + 2 * (size_t)nf * warps + warp * (32 * REC);
    int* sstart = reinterpret_cast<int*>(smem_d + 2 * (size_t)nf * warps + warps * 32 * REC) + warp * 96;
    for (int t = threadIdx.x; t < nf * warps; t += blockDim.x) sgrid[t] = mk(0.0);
    __syncthreads();
    cplx* mine = sgrid + warp * nf;
    const int wfx = a.fs.w[0], wfy = a.fs.w[1], wfz = a.fs.w[2];
    // this lane's taps; taps beyond a single-plane axis are skipped (they would
    // alias another lane's node)
    int ta[TPL], tb[TPL], tc[TPL];
    bool tok[TPL];
#pragma unroll
    for (int t = 0; t < TPL; ++t) {
        const int tp = lane + 32 * t;
        tc[t] = tp % WF;
        tb[t] = (tp / WF) % WF;
        ta[t] = tp / (WF * WF);
        tok[t] = tp < WF * WF * WF && ta[t] < wfx && tb[t] < wfy && tc[t] < wfz;
    }
    double accr[TPL], acci[TPL];
#pragma unroll
    for (int t = 0; t < TPL; ++t) accr[t] = acci[t] = 0.0;
    int c0 = -1, c1 = 0, c2 = 0;   // far stencil start of the open run
    auto flush = [&]() {
#pragma unroll
        for (int t = 0; t < TPL; ++t) {
            if (!tok[t]) continue;
            cplx& d = mine[((c0 + ta[t]) * nfy + (c1 + tb[t])) * nfz + (c2 + tc[t])];
            d.re += accr[t];
            d.im += acci[t];
            accr[t] = acci[t] = 0.0;
        }
        __syncwarp();
    };
    const int64_t stride = (int64_t)gridDim.x * warps * 32;
    // the next batch's weights, charge and starts are loaded into registers while
    // this batch is accumulated (one global round trip per batch, overlapped)
    double nw[3 * WF], nq[2];
    int ns[3];
    auto fetch = [&](int64_t p) {
        if (p < a.far_n) {
            const double* w = a.src_fw + p * 3 * WF;
#pragma unroll
            for (int j = 0; j < 3 * WF; ++j) nw[j] = __ldg(w + j);
            const double2 qv = __ldg(reinterpret_cast<const double2*>(a.far_q + p));
            nq[0] = qv.x;
            nq[1] = qv.y;
            ns[0] = __ldg(a.src_fstart + 3 * p);
            ns[1] = __ldg(a.src_fstart + 3 * p + 1);
            ns[2] = __ldg(a.src_fstart + 3 * p + 2);
        }
    };
    int64_t base = ((int64_t)blockIdx.x * warps + warp) * 32;
    fetch(base + lane);
    for (; base < a.far_n; base += stride) {
        const int64_t p = base + lane;
        __syncwarp();
        if (p < a.far_n) {
#pragma unroll
            for (int j = 0; j < 3 * WF; ++j) stage[lane * REC + j] = nw[j];
            stage[lane * REC + 3 * WF] = nq[0];
            stage[lane * REC + 3 * WF + 1] = nq[1];
            sstart[lane * 3] = ns[0];
            sstart[lane * 3 + 1] = ns[1];
            sstart[lane * 3 + 2] = ns[2];
        }
        __syncwarp();
        fetch(base + stride + lane);
        const int cnt = (int)min((int64_t)32, a.far_n - base);
        for (int j = 0; j < cnt; ++j) {
            const double* r = stage + j * REC;
            const int s0 = sstart[3 * j], s1 = sstart[3 * j + 1], s2 = sstart[3 * j + 2];
            if (s0 != c0 || s1 != c1 || s2 != c2) {   // warp-uniform
                if (c0 >= 0) flush();
                c0 = s0;
                c1 = s1;
                c2 = s2;
            }
            const double qre = r[3 * WF], qim = r[3 * WF + 1];
#pragma unroll
            for (int t = 0; t < TPL; ++t) {
                const double wgt = (r[ta[t]] * r[WF + tb[t]]) * r[2 * WF + tc[t]];
                accr[t] += wgt * qre;
                acci[t] += wgt * qim;
            }
        }
    }
    if (c0 >= 0) flush();
    __syncthreads();
    for (int t = threadIdx.x; t < nf; t += blockDim.x) {
        cplx s = mk(0.0);
        for (int k = 0; k < warps; ++k) s = s + sgrid[k * nf + t];
        a.far_partial[(int64_t)blockIdx.x * nf + t] = s;
    }
}

// one warp per far node, fixed-order sum over the block partials
__global__ void k_far_reduce(const cplx* __restrict__ partial, int blocks, int nf, cplx* __restrict__ qg) {
    const int lane = threadIdx.x & 31;
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (t >= nf) return;
    cplx s = mk(0.0);
    for (int b = lane; b < blocks; b += 32) s = s + partial[(int64_t)b * nf + t];
    s = warp_sum(s);
    if (lane == 0) qg[t] = s;
}

size_t far_project_smem(int nf, int warps, int order) {
    const int WF = order + 1;
    return (size_t)nf * warps * sizeof(cplx) + (size_t)warps * 32 * (3 * WF + 2) * sizeof(double) +
           (size_t)warps * 96 * sizeof(int);
}

template <int WF>
static void far_project_launch(const EvalArgs& a, size_t smem, cudaStream_t s) {
    static size_t configured = 48 * 1024;
    if (smem > configured) {
        cudaFuncSetAttribute(k_far_project<WF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    k_far_project<WF><<<a.far_blocks, 32 * a.far_warps, smem, s>>>(a);
}

void launch_far_project(const EvalArgs& a, cudaStream_t s) {
    if (a.far_pos && launch_far_project_win(a, a.far_pos, a.far_slots, a.far_win, s)) return;
    const int nf = a.fs.n[0] * a.fs.n[1] * a.fs.n[2];
    const size_t smem = far_project_smem(nf, a.far_warps, a.fs.order);
    switch (a.fs.order + 1) {
        case 2: far_project_launch<2>(a, smem, s); break;
        case 3: far_project_launch<3>(a, smem, s); break;
        case 4: far_project_launch<4>(a, smem, s); break;
        case 5: far_project_launch<5>(a, smem, s); break;
        case 6: far_project_launch<6>(a, smem, s); break;
        default: far_project_launch<7>(a, smem, s); break;
    }
    k_far_reduce<<<nblk((int64_t)nf * 32, 256), 256, 0, s>>>(a.far_partial, a.far_blocks, nf, a.far_qg);
    fftpim_count_launch(2);
}

// ---------------------------------------------------------------- K5b
// ug[o] = sum_s K[o - s + (n-1)] qg[s].  One block per observer-grid (x, y)
// column; the source grid is staged in shared memory, each thread sums a fixed
// strided subset of sources for every z output, then a fixed-order block reduce.
#define FAR_SUM_MAXZ 32
__global__ void __launch_bounds__(256) k_far_sum(EvalArgs a) {
    extern __shared__ cplx sq[];
    const int nx = a.fs.n[0], ny = a.fs.n[1], nz = a.fs.n[2];
    const int nf = nx * ny * nz;
    const int ky = 2 * ny - 1, kz = 2 * nz - 1;
    const int ox = blockIdx.x / ny, oy = blockIdx.x % ny;
    for (int t = threadIdx.x; t < nf; t += blockDim.x) sq[t] = a.far_qg[t];
    __syncthreads();
    // thread t: output oz = t % nz, source columns c = t / nz, t / nz + groups, ...
    const int groups = blockDim.x / nz;
    const int oz = threadIdx.x % nz, grp = threadIdx.x / nz;
    cplx acc = mk(0.0);
    const int nsc = nx * ny;   // source columns
    if (grp < groups) {
        for (int c = grp; c < nsc; c += groups) {
            const int sx = c / ny, sy = c % ny;
            const cplx* krow = a.far_kernel + ((int64_t)(ox - sx + nx - 1) * ky + (oy - sy + ny - 1)) * kz + oz + nz - 1;
            const cplx* qcol = sq + c * nz;
            for (int sz = 0; sz < nz; ++sz) acc = acc + krow[-sz] * qcol[sz];
        }
    }
    __shared__ cplx red[256];
    red[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < nz) {
        cplx v = mk(0.0);
        for (int g = 0; g < groups; ++g) v = v + red[g * nz + threadIdx.x];
        a.far_ug[(ox * ny + oy) * nz + threadIdx.x] = v;
    }
}

void launch_far_sum(const EvalArgs& a, cudaStream_t s) {
    const int nf = a.fs.n[0] * a.fs.n[1] * a.fs.n[2];
    k_far_sum<<<a.fs.n[0] * a.fs.n[1], 256, (size_t)nf * sizeof(cplx), s>>>(a);
    fftpim_count_launch();
}

