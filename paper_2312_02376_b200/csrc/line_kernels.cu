// line_kernels.cu -- K1 near projection (grids.py:167-181, via nearzone.py:499)
// as an owner-computes line sweep with stencils computed from the sorted
// positions: the only per-point inputs are 24 B of position and 16 B of charge.
//
// A block owns a TY x TZ tile of grid lines along x (one (y, z) pair per line)
// and a chunk of XC output planes.  It sweeps the stencil-start planes sx of
// the chunk's reach in ascending order.  For each plane it stages every point
// whose start cell lies in the tile's reach -- (TY + W - 1) rows of cells
// (sx, sy, z0 - W + 1 .. z0 + TZ - 1), each ONE contiguous run of the
// cell-sorted point order -- into shared memory with its three axis stencils
// (computed once per staging).  Each thread owns R consecutive z lines at one
// y and keeps, per line, a window of W registers for the nodes sx .. sx + W - 1:
// a point of row sy = y - ib adds q * wy[ib] * wz[z - sz] * wx[ia] to window
// slot ia.  After plane sx node x = sx is complete (it only receives from
// planes x - W + 1 .. x), is stored once, and the window shifts.  No atomics,
// no halo merge; every node's sum runs in a fixed order (planes ascending,
// staging pieces, rows, points ascending), so the result is bitwise
// reproducible.
//
// Stencils: start = rint(t - order/2) clipped, w_j = prod_{i!=j}(rel - i) /
// prod_{i!=j}(j - i) with the reference's operation order (grids.py:123-139).
// The two divisions (t = (x - o)/h and num/den) use a reciprocal product plus
// one FMA remainder correction, which returns the correctly rounded quotient:
// the starts and weights equal the plan's stored ones bit for bit
// (tools/div_check.c checks the correction against true division on 1e9
// samples; tests/test_gpu_paths.py compares the projections).
#include "geom.cuh"
#include "kernels.h"

// RN(x / d) given rcp = RN(1 / d)
__device__ __forceinline__ double div_rcp(double x, double d, double rcp) {
    const double q0 = __dmul_rn(x, rcp);
    const double r = __fma_rn(-q0, d, x);
    return __fma_rn(r, rcp, q0);
}

template <int W>
struct LagrangeDen {
    double den[W], rcp[W];
    __device__ __forceinline__ LagrangeDen() {
#pragma unroll
        for (int j = 0; j < W; ++j) {
            double d = 1.0;
#pragma unroll
            for (int i = 0; i < W; ++i)
                if (i != j) d *= (double)(j - i);
            den[j] = d;
            rcp[j] = 1.0 / d;
        }
    }
};

// axis stencil of width W (order W - 1) on an axis with n > 1 planes; for
// n == 1 the stencil is the single plane (weight 1, the rest 0)
template <int W>
__device__ __forceinline__ int fast_stencil(double x, int n, double origin, double h, double rcp_h,
                                            const LagrangeDen<W>& L, double* w) {
    if (n == 1) {
        w[0] = 1.0;
#pragma unroll
        for (int j = 1; j < W; ++j) w[j] = 0.0;
        return 0;
    }
    const double t = div_rcp(__dsub_rn(x, origin), h, rcp_h);
    int s = (int)rint(__dsub_rn(t, (W - 1) / 2.0));
    s = max(0, min(s, n - W));
    const double rel = __dsub_rn(t, (double)s);
#pragma unroll
    for (int j = 0; j < W; ++j) {
        double num = 1.0;
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (i != j) num = __dmul_rn(num, __dsub_rn(rel, (double)i));
        w[j] = div_rcp(num, L.den[j], L.rcp[j]);
    }
    return s;
}

#define K1L_TY 16
#define K1L_TZ 32
#define K1L_R 4
#define K1L_NT (K1L_TY * (K1L_TZ / K1L_R))

template <int W>
struct K1Lines {
    static constexpr int ROWS = K1L_TY + W - 1;
    static constexpr int CELLS = K1L_TZ + W - 1;
    static constexpr int REC = (2 + 3 * W + 1 + 1) & ~1;   // q, wx, wy, wz, sz; even -> 16 B records
};

template <int W>
size_t k1_lines_smem(int cap) {
    using T = K1Lines<W>;
    return (size_t)cap * T::REC * sizeof(double) + (size_t)(T::ROWS * (T::CELLS + 1) + T::ROWS + 1) * sizeof(int);
}

template <int W>
__global__ void __launch_bounds__(K1L_NT, 2) k_k1_lines(EvalArgs a, const double* __restrict__ pos, int xc,
                                                        int cap, double rh0, double rh1, double rh2) {
    using T = K1Lines<W>;
    constexpr int ROWS = T::ROWS, CELLS = T::CELLS, REC = T::REC, R = K1L_R;
    extern __shared__ double k1l_smem[];
    double* rec = k1l_smem;                                       // cap x REC
    int* lcs = reinterpret_cast<int*>(rec + (size_t)cap * REC);  // ROWS x (CELLS + 1) global point starts
    int* soff = lcs + ROWS * (CELLS + 1);                         // ROWS + 1 staged row offsets
    const StencilGeom& g = a.g;
    const LagrangeDen<W> L;
    const int tid = threadIdx.x;
    const int ly = tid / (K1L_TZ / R), lzg = tid % (K1L_TZ / R);
    const int y0 = blockIdx.y * K1L_TY, z0 = blockIdx.x * K1L_TZ;
    const int y = y0 + ly, zb = z0 + lzg * R;
    const int xo0 = a.kx0 + blockIdx.z * xc;
    const int xo1 = min(xo0 + xc, a.kx0 + a.knx);
    const int wx0 = g.w[0];
    const int sx_lo = max(xo0 - (wx0 - 1), 0);
    const int sx_hi = min(xo1 - 1, g.nc[0] - 1);
    const int nc1 = g.nc[1], nc2 = g.nc[2];

    double wr[R][W], wi[R][W];
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
        for (int ia = 0; ia < W; ++ia) wr[j][ia] = wi[j][ia] = 0.0;

    auto store = [&](int x, int slot) {
        if (x < xo0 || x >= xo1 || y >= g.n[1]) return;
        cplx* dst = a.k1_out + ((int64_t)(x - a.kx0) * a.go1 + y) * a.go2;
#pragma unroll
        for (int j = 0; j < R; ++j)
            if (zb + j < g.n[2]) {
#pragma unroll
                for (int ia = 0; ia < W; ++ia)
                    if (ia == slot) dst[zb + j] = cplx{wr[j][ia], wi[j][ia]};
            }
    };

    for (int sx = sx_lo; sx <= sx_hi; ++sx) {
        // global point range of every reach cell: row r = sy - (y0 - W + 1),
        // cell c = sz - (z0 - W + 1); cells past the axis clamp to the row end
        for (int e = tid; e < ROWS * (CELLS + 1); e += K1L_NT) {
            const int r = e / (CELLS + 1), c = e - r * (CELLS + 1);
            const int sy = y0 - (W - 1) + r;
            int v = 0;
            if (sy >= 0 && sy < nc1) {
                const int sz = min(max(z0 - (W - 1) + c, 0), nc2);
                v = a.cell_start[((int64_t)sx * nc1 + sy) * nc2 + sz];
            }
            lcs[e] = v;
        }
        __syncthreads();
        if (tid < 32) {
            int len = tid < ROWS ? lcs[tid * (CELLS + 1) + CELLS] - lcs[tid * (CELLS + 1)] : 0;
            int inc = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, inc, o);
                if (tid >= o) inc += v;
            }
            if (tid < ROWS) soff[tid + 1] = inc;
            if (tid == 0) soff[0] = 0;
        }
        __syncthreads();
        const int total = soff[ROWS];
        for (int p0 = 0; p0 < total; p0 += cap) {
            const int pc = min(cap, total - p0);
            for (int e = tid; e < pc; e += K1L_NT) {
                const int idx = p0 + e;
                int r = 0;
#pragma unroll 1
                while (r + 1 < ROWS && soff[r + 1] <= idx) ++r;
                const int64_t gi = lcs[r * (CELLS + 1)] + (idx - soff[r]);
                double* rp = rec + (size_t)e * REC;
                const cplx qv = a.q_sorted[gi];
                rp[0] = qv.re;
                rp[1] = qv.im;
                fast_stencil<W>(pos[3 * gi], g.n[0], g.origin[0], g.h[0], rh0, L, rp + 2);
                fast_stencil<W>(pos[3 * gi + 1], g.n[1], g.origin[1], g.h[1], rh1, L, rp + 2 + W);
                const int sz = fast_stencil<W>(pos[3 * gi + 2], g.n[2], g.origin[2], g.h[2], rh2, L, rp + 2 + 2 * W);
                rp[2 + 3 * W] = (double)sz;
            }
            __syncthreads();
#pragma unroll 1
            for (int ib = 0; ib < W; ++ib) {
                const int r = ly + (W - 1) - ib;
                const int* row = lcs + r * (CELLS + 1);
                const int base = soff[r] - row[0] - p0;
                const int b0 = max(base + row[lzg * R], 0);
                const int b1 = min(base + row[lzg * R + R + W - 1], pc);
#pragma unroll 1
                for (int k = b0; k < b1; ++k) {
                    const double* rp = rec + (size_t)k * REC;
                    const double2 qv = *reinterpret_cast<const double2*>(rp);
                    double wx[W];
#pragma unroll
                    for (int ia = 0; ia < W; ++ia) wx[ia] = rp[2 + ia];
                    const double wy = rp[2 + W + ib];
                    const int sz = (int)rp[2 + 3 * W];
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const int ic = zb + j - sz;
                        const double wz = (unsigned)ic < (unsigned)W ? rp[2 + 2 * W + ic] : 0.0;
                        const double t = wy * wz;
                        const double cr = qv.x * t, ci = qv.y * t;
#pragma unroll
                        for (int ia = 0; ia < W; ++ia) {
                            wr[j][ia] = fma(cr, wx[ia], wr[j][ia]);
                            wi[j][ia] = fma(ci, wx[ia], wi[j][ia]);
                        }
                    }
                }
            }
            __syncthreads();
        }
        // node sx has all its planes: store it, shift the windows
        store(sx, 0);
#pragma unroll
        for (int j = 0; j < R; ++j) {
#pragma unroll
            for (int ia = 0; ia + 1 < W; ++ia) {
                wr[j][ia] = wr[j][ia + 1];
                wi[j][ia] = wi[j][ia + 1];
            }
            wr[j][W - 1] = wi[j][W - 1] = 0.0;
        }
    }
    // nodes past the last start plane (x > nc0 - 1) or past the chunk's sweep
#pragma unroll
    for (int ia = 0; ia + 1 < W; ++ia) store(sx_hi + 1 + ia, ia);
}

template <int W>
static void k1_lines_launch(const EvalArgs& a, const double* pos, cudaStream_t s) {
    static int cap = 0;
    static size_t smem = 0;
    if (!cap) {
        cap = 448;
        if (const char* e = getenv("FFTPIM_K1L_CAP")) cap = std::max(64, atoi(e));
        smem = k1_lines_smem<W>(cap);
        cudaFuncSetAttribute(k_k1_lines<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    const int gz = (a.g.n[2] + K1L_TZ - 1) / K1L_TZ, gy = (a.g.n[1] + K1L_TY - 1) / K1L_TY;
    // chunks of >= 2 (W - 1) planes (the warm-up planes are redone per chunk),
    // enough chunks for ~4 blocks per SM
    int xc = (int)(((int64_t)a.knx * gy * gz + 591) / 592);
    xc = std::max(xc, 2 * (W - 1));
    if (const char* e = getenv("FFTPIM_K1L_XC")) xc = std::max(1, atoi(e));
    xc = std::min(xc, std::max(a.knx, 1));
    const int gx = (a.knx + xc - 1) / xc;
    const double rh0 = a.g.h[0] > 0 ? 1.0 / a.g.h[0] : 0.0, rh1 = a.g.h[1] > 0 ? 1.0 / a.g.h[1] : 0.0,
                 rh2 = a.g.h[2] > 0 ? 1.0 / a.g.h[2] : 0.0;
    k_k1_lines<W><<<dim3(gz, gy, gx), K1L_NT, smem, s>>>(a, pos, xc, cap, rh0, rh1, rh2);
}

bool launch_k1_lines(const EvalArgs& a, const double* pos, cudaStream_t s) {
    if (a.knx <= 0) return true;
    switch (a.g.order + 1) {
        case 3: k1_lines_launch<3>(a, pos, s); break;
        case 4: k1_lines_launch<4>(a, pos, s); break;
        case 5: k1_lines_launch<5>(a, pos, s); break;
        case 6: k1_lines_launch<6>(a, pos, s); break;
        default: return false;
    }
    fftpim_count_launch();
    return true;
}

// ---- K1 line sweep, independent threads (no staging, no block barriers).
// Same lines, windows and summation order as k_k1_lines, but each thread reads
// the points of its rows straight from the plan's per-point stencil records
// (rec[i] = wx[W], wy[W], wz[W], start z; 16-byte aligned, sorted order) through
// L1: no shared memory and no barriers, so the dependent cell-start -> record
// loads of one thread overlap with the other warps' arithmetic.
template <int W>
__global__ void __launch_bounds__(K1L_NT) k_k1_lines_g(EvalArgs a, const double* __restrict__ rec, int xc) {
    constexpr int R = K1L_R, RECW = (3 * W + 2) & ~1;
    const StencilGeom& g = a.g;
    const int tid = threadIdx.x;
    const int ly = tid / (K1L_TZ / R), lzg = tid % (K1L_TZ / R);
    const int y = blockIdx.y * K1L_TY + ly, zb = blockIdx.x * K1L_TZ + lzg * R;
    const int xo0 = a.kx0 + blockIdx.z * xc;
    const int xo1 = min(xo0 + xc, a.kx0 + a.knx);
    const int sx_lo = max(xo0 - (g.w[0] - 1), 0);
    const int sx_hi = min(xo1 - 1, g.nc[0] - 1);
    const int nc1 = g.nc[1], nc2 = g.nc[2];
    const int zlo = max(zb - (W - 1), 0), zhi = min(zb + R, nc2);   // start cells [zlo, zhi)
    const bool live = y < g.n[1] && zb < g.n[2];
    double wr[R][W], wi[R][W];
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
        for (int ia = 0; ia < W; ++ia) wr[j][ia] = wi[j][ia] = 0.0;
    auto store = [&](int x, int slot) {
        if (!live || x < xo0 || x >= xo1) return;
        cplx* dst = a.k1_out + ((int64_t)(x - a.kx0) * a.go1 + y) * a.go2;
#pragma unroll
        for (int j = 0; j < R; ++j)
            if (zb + j < g.n[2]) {
#pragma unroll
                for (int ia = 0; ia < W; ++ia)
                    if (ia == slot) dst[zb + j] = cplx{wr[j][ia], wi[j][ia]};
            }
    };
    const cplx* __restrict__ qs = a.q_sorted;
    for (int sx = sx_lo; sx <= sx_hi; ++sx) {
        if (live && zlo < zhi) {
            int b0[W], b1[W];
#pragma unroll
            for (int ib = 0; ib < W; ++ib) {
                const int sy = y - ib;
                b0[ib] = b1[ib] = 0;
                if (sy >= 0 && sy < nc1) {
                    const int64_t k = ((int64_t)sx * nc1 + sy) * nc2;
                    b0[ib] = __ldg(a.cell_start + k + zlo);
                    b1[ib] = __ldg(a.cell_start + k + zhi);
                }
            }
#pragma unroll
            for (int ib = 0; ib < W; ++ib) {
#pragma unroll 1
                for (int k = b0[ib]; k < b1[ib]; ++k) {
                    const double2* rp = reinterpret_cast<const double2*>(rec + (int64_t)k * RECW);
                    double r[RECW];
#pragma unroll
                    for (int e = 0; e < RECW / 2; ++e) {
                        const double2 v = __ldg(rp + e);
                        r[2 * e] = v.x;
                        r[2 * e + 1] = v.y;
                    }
                    const double2 qv = __ldg(reinterpret_cast<const double2*>(qs + k));
                    const double wy = r[W + ib];
                    const int sz = (int)r[3 * W];
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const int ic = zb + j - sz;
                        double wz = 0.0;
#pragma unroll
                        for (int c = 0; c < W; ++c) wz = ic == c ? r[2 * W + c] : wz;
                        const double t = wy * wz;
                        const double cr = qv.x * t, ci = qv.y * t;
#pragma unroll
                        for (int ia = 0; ia < W; ++ia) {
                            wr[j][ia] = fma(cr, r[ia], wr[j][ia]);
                            wi[j][ia] = fma(ci, r[ia], wi[j][ia]);
                        }
                    }
                }
            }
        }
        store(sx, 0);
#pragma unroll
        for (int j = 0; j < R; ++j) {
#pragma unroll
            for (int ia = 0; ia + 1 < W; ++ia) {
                wr[j][ia] = wr[j][ia + 1];
                wi[j][ia] = wi[j][ia + 1];
            }
            wr[j][W - 1] = wi[j][W - 1] = 0.0;
        }
    }
#pragma unroll
    for (int ia = 0; ia + 1 < W; ++ia) store(sx_hi + 1 + ia, ia);
}

template <int W>
static void k1_lines_g_launch(const EvalArgs& a, const double* rec, cudaStream_t s) {
    const int gz = (a.g.n[2] + K1L_TZ - 1) / K1L_TZ, gy = (a.g.n[1] + K1L_TY - 1) / K1L_TY;
    int xc = (int)(((int64_t)a.knx * gy * gz + 1183) / 1184);   // ~8 blocks per SM
    xc = std::max(xc, 2 * (W - 1));
    if (const char* e = getenv("FFTPIM_K1L_XC")) xc = std::max(1, atoi(e));
    xc = std::min(xc, std::max(a.knx, 1));
    k_k1_lines_g<W><<<dim3(gz, gy, (a.knx + xc - 1) / xc), K1L_NT, 0, s>>>(a, rec, xc);
}

bool launch_k1_lines_g(const EvalArgs& a, const double* rec, cudaStream_t s) {
    if (a.knx <= 0) return true;
    switch (a.g.order + 1) {
        case 3: k1_lines_g_launch<3>(a, rec, s); break;
        case 4: k1_lines_g_launch<4>(a, rec, s); break;
        case 5: k1_lines_g_launch<5>(a, rec, s); break;
        case 6: k1_lines_g_launch<6>(a, rec, s); break;
        default: return false;
    }
    fftpim_count_launch();
    return true;
}

// per-point stencil records for k_k1_lines_g: wx, wy, wz (the plan's bit-exact
// weights) and the z start, (3W + 2) & ~1 doubles per point
__global__ void k_stencil_records(const double* __restrict__ w, const int* __restrict__ start, int64_t n, int W,
                                  int recw, double* __restrict__ rec) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double* r = rec + i * recw;
    for (int j = 0; j < 3 * W; ++j) r[j] = w[i * 3 * W + j];
    r[3 * W] = (double)start[3 * i + 2];
    for (int j = 3 * W + 1; j < recw; ++j) r[j] = 0.0;
}
int stencil_record_width(int W) { return (3 * W + 2) & ~1; }
void launch_stencil_records(const double* w, const int* start, int64_t n, int W, double* rec, cudaStream_t s) {
    if (n == 0) return;
    k_stencil_records<<<(int)((n + 255) / 256), 256, 0, s>>>(w, start, n, W, stencil_record_width(W), rec);
    fftpim_count_launch();
}

// sorted positions pos_s[i] = pos[perm[i]] (plan build)
__global__ void k_gather_pos(const double* __restrict__ pos, const int* __restrict__ perm, int64_t n,
                             double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p = perm[i];
    out[3 * i] = pos[3 * p];
    out[3 * i + 1] = pos[3 * p + 1];
    out[3 * i + 2] = pos[3 * p + 2];
}
void launch_gather_pos(const double* pos, const int* perm, int64_t n, double* out, cudaStream_t s) {
    if (n == 0) return;
    k_gather_pos<<<(int)((n + 255) / 256), 256, 0, s>>>(pos, perm, n, out);
    fftpim_count_launch();
}

// ------------------------------------------------------------- K3 + K5c + fix-up
// The observer pass of corr_kernels.cu (k_observers: LPO lanes per observer,
// far grid staged in shared memory, the observer's K4 segments, fixed xor
// tree) with the near and far stencils computed from the observer's sorted
// position instead of read from the plan: lanes 0..2 of an observer each
// compute one axis (both grids) into a shared-memory record, so an observer
// costs 24 B of position instead of 3 (W + WF) weights and 6 starts.
struct ObsPosArgs {
    const double* pos;          // (M, 3) observer positions, sorted order (slab: own range)
    double rn[3], rf[3];        // 1 / spacing of the near and far observer grids
};

__device__ __forceinline__ cplx corr_row_sum(const EvalArgs& a, int64_t i) {
    const int64_t p0 = a.pair_ptr[i], p1 = a.pair_ptr[i + 1];
    if (p0 == p1) return mk(0.0);
    const int64_t span = (p1 - 1) / CORR_TILE - p0 / CORR_TILE + 1;
    const cplx* sv = a.seg_val + a.seg_first[i];
    cplx s = sv[0];
    for (int64_t j = 1; j < span; ++j) s = s + sv[j];
    return s;
}

#ifndef OBSP_MINB
#define OBSP_MINB 3
#endif
template <int W, int WF, int MODE, int LPO>
__global__ void __launch_bounds__(256, OBSP_MINB) k_observers_pos(EvalArgs a, ObsPosArgs o) {
    extern __shared__ double obs_smem[];
    constexpr int OPB = 256 / LPO;                  // observers per block
    constexpr int RECD = 3 * W + 3 * WF;
    const bool far = (a.parts & FFTPIM_FAR) && MODE != 2;
    const bool near = (a.parts & FFTPIM_NEAR) && MODE != 1;
    const int nfx = a.fo.n[0], nfy = a.fo.n[1], nfz = a.fo.n[2];
    const int nf = far ? nfx * nfy * nfz : 0;
    cplx* sfar = reinterpret_cast<cplx*>(obs_smem);
    double* recs = obs_smem + 2 * nf;
    int* rst = reinterpret_cast<int*>(recs + OPB * RECD);
    if (far)
        for (int t = threadIdx.x; t < nf; t += blockDim.x) sfar[t] = a.far_ug[t];
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t i = gt / LPO;
    const int sub = (int)(gt % LPO);
    const int lo = threadIdx.x / LPO;
    const bool active = i < a.M;
    const int64_t ii = active ? i : a.M - 1;
    double* rec = recs + lo * RECD;
    int* st = rst + lo * 6;
    {
        const LagrangeDen<W> Ln;
        const LagrangeDen<WF> Lf;
        for (int ax = sub; ax < 3; ax += LPO) {
            const double x = o.pos[3 * ii + ax];
            if (near) st[ax] = fast_stencil<W>(x, a.g.n[ax], a.g.origin[ax], a.g.h[ax], o.rn[ax], Ln, rec + ax * W);
            if (far)
                st[3 + ax] = fast_stencil<WF>(x, a.fo.n[ax], a.fo.origin[ax], a.fo.h[ax], o.rf[ax], Lf,
                                              rec + 3 * W + ax * WF);
        }
    }
    __syncthreads();
    double ar = 0.0, ai = 0.0;
    if ((a.parts & FFTPIM_NEAR) && MODE != 2 && active && sub == LPO - 1 && a.sw_e >= 0) {
        const cplx c = a.sw_corr ? a.sw_corr[i * a.sw_E + a.sw_e] : corr_row_sum(a, i);
        ar = c.re;
        ai = c.im;
    }
    if (MODE == 2 && active && sub == LPO - 1) {
        const cplx c = a.obs_pre[i];
        ar = c.re;
        ai = c.im;
    }
    if (near) {
        const double* w = rec;
        const int c1 = a.gi1, c2 = a.gi2;
        const int m0 = a.g.n[0] - 1, m1 = a.g.n[1] - 1, m2 = a.g.n[2] - 1;
        const int s0 = st[0], s1 = st[1], s2 = st[2];
        constexpr int ET = (W * W + LPO - 1) / LPO;
        double wyz[ET];
        int off[ET];
#pragma unroll
        for (int t = 0; t < ET; ++t) {
            const int e = sub + LPO * t;
            const bool ok = e < W * W;
            const int ib = ok ? e / W : 0, ic = ok ? e % W : 0;
            wyz[t] = ok ? w[W + ib] * w[2 * W + ic] : 0.0;
            off[t] = min(s1 + ib, m1) * c2 + min(s2 + ic, m2);
        }
#pragma unroll
        for (int ia = 0; ia < W; ++ia) {
            const double wxa = w[ia];
            const cplx* plane = a.interp_grid + (int64_t)(min(s0 + ia, m0) - a.gx0) * c1 * c2;
#pragma unroll
            for (int t = 0; t < ET; ++t) {
                const cplx v = plane[off[t]];
                const double wgt = wxa * wyz[t];
                ar += wgt * v.re;
                ai += wgt * v.im;
            }
        }
    }
    if (far) {
        const double* w = rec + 3 * W;
        const int s0 = st[3], s1 = st[4], s2 = st[5];
        constexpr int ET = (WF * WF + LPO - 1) / LPO;
        double wyz[ET];
        int off[ET];
#pragma unroll
        for (int t = 0; t < ET; ++t) {
            const int e = sub + LPO * t;
            const bool ok = e < WF * WF;
            const int ib = ok ? e / WF : 0, ic = ok ? e % WF : 0;
            wyz[t] = ok ? w[WF + ib] * w[2 * WF + ic] : 0.0;
            off[t] = min(s1 + ib, nfy - 1) * nfz + min(s2 + ic, nfz - 1);
        }
#pragma unroll
        for (int ia = 0; ia < WF; ++ia) {
            const double wxa = w[ia];
            const cplx* plane = sfar + min(s0 + ia, nfx - 1) * nfy * nfz;
#pragma unroll
            for (int t = 0; t < ET; ++t) {
                const cplx v = plane[off[t]];
                const double wgt = wxa * wyz[t];
                ar += wgt * v.re;
                ai += wgt * v.im;
            }
        }
    }
#pragma unroll
    for (int d = 1; d < LPO; d <<= 1) {   // fixed xor tree over the observer's lanes
        ar += __shfl_xor_sync(0xffffffffu, ar, d);
        ai += __shfl_xor_sync(0xffffffffu, ai, d);
    }
    if (active && sub == 0) {
        if (MODE == 1)
            a.obs_pre[i] = cplx{ar, ai};
        else
            a.u[a.obs_perm[i]] = cplx{ar, ai};
    }
}

template <int W, int WF, int MODE, int LPO>
static void obsp_launch(const EvalArgs& a, const ObsPosArgs& o, cudaStream_t s) {
    const bool far = (a.parts & FFTPIM_FAR) && MODE != 2;
    const size_t nf = far ? (size_t)a.fo.n[0] * a.fo.n[1] * a.fo.n[2] : 0;
    const size_t smem = nf * sizeof(cplx) + (size_t)(256 / LPO) * ((3 * W + 3 * WF) * sizeof(double) + 6 * sizeof(int));
    static size_t configured = 48 * 1024;
    if (smem > configured) {
        cudaFuncSetAttribute(k_observers_pos<W, WF, MODE, LPO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        configured = smem;
    }
    k_observers_pos<W, WF, MODE, LPO><<<(int)((a.M * LPO + 255) / 256), 256, smem, s>>>(a, o);
}

template <int W, int MODE, int LPO>
static bool obsp_far(const EvalArgs& a, const ObsPosArgs& o, cudaStream_t s) {
    switch (a.fo.order + 1) {
        case 3: obsp_launch<W, 3, MODE, LPO>(a, o, s); return true;
        case 4: obsp_launch<W, 4, MODE, LPO>(a, o, s); return true;
        case 5: obsp_launch<W, 5, MODE, LPO>(a, o, s); return true;
        default: return false;
    }
}

template <int MODE, int LPO>
static bool obsp_near(const EvalArgs& a, const ObsPosArgs& o, cudaStream_t s) {
    switch (a.g.order + 1) {
        case 3: return obsp_far<3, MODE, LPO>(a, o, s);
        case 4: return obsp_far<4, MODE, LPO>(a, o, s);
        case 5: return obsp_far<5, MODE, LPO>(a, o, s);
        case 6: return obsp_far<6, MODE, LPO>(a, o, s);
        default: return false;
    }
}

// false: orders outside 2..5 (near) / 2..4 (far) -- the caller uses k_observers
bool launch_observers_pos(const EvalArgs& a, const double* pos, cudaStream_t s, int mode) {
    if (a.M == 0) return true;
    ObsPosArgs o;
    o.pos = pos;
    for (int ax = 0; ax < 3; ++ax) {
        o.rn[ax] = a.g.h[ax] > 0 ? 1.0 / a.g.h[ax] : 0.0;
        o.rf[ax] = a.fo.h[ax] > 0 ? 1.0 / a.fo.h[ax] : 0.0;
    }
    const bool lpo4 = a.M <= 16384 || a.g.order >= 4;
    bool ok;
    if (mode == 1)
        ok = lpo4 ? obsp_near<1, 4>(a, o, s) : obsp_near<1, 2>(a, o, s);
    else if (mode == 2)
        ok = lpo4 ? obsp_near<2, 4>(a, o, s) : obsp_near<2, 2>(a, o, s);
    else
        ok = lpo4 ? obsp_near<0, 4>(a, o, s) : obsp_near<0, 2>(a, o, s);
    if (ok) fftpim_count_launch();
    return ok;
}
