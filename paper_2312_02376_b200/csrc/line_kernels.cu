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

#ifndef K1L_TY
#define K1L_TY 16
#endif
#ifndef K1L_TZ
#define K1L_TZ 32
#endif
#ifndef K1L_R
#define K1L_R 4     // z lines per thread
#endif
#ifndef K1L_MINB
#define K1L_MINB 3  // resident blocks per SM the register budget is set for
#endif
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
    return (size_t)cap * T::REC * sizeof(double) + (size_t)(2 * T::ROWS * (T::CELLS + 1) + T::ROWS + 1) * sizeof(int);
}

#ifndef K1L_PF
#define K1L_PF 3   // staged points per thread per piece held in flight (cap <= K1L_PF * K1L_NT)
#endif
template <int W>
__global__ void __launch_bounds__(K1L_NT, K1L_MINB) k_k1_lines(EvalArgs a, const double* __restrict__ pos, int xc,
                                                        int n_items, int cap, double rh0, double rh1, double rh2) {
    using T = K1Lines<W>;
    constexpr int ROWS = T::ROWS, CELLS = T::CELLS, REC = T::REC, R = K1L_R, LCS = ROWS * (CELLS + 1);
    constexpr int LPT = (LCS + K1L_NT - 1) / K1L_NT;   // cell starts per thread
    extern __shared__ double k1l_smem[];
    double* rec = k1l_smem;                                       // cap x REC
    int* lcs2 = reinterpret_cast<int*>(rec + (size_t)cap * REC);  // 2 x ROWS x (CELLS + 1) global point starts
    int* soff = lcs2 + 2 * LCS;                                   // ROWS + 1 staged row offsets
    const StencilGeom& g = a.g;
    const LagrangeDen<W> L;
    const int tid = threadIdx.x;
    const int ly = tid / (K1L_TZ / R), lzg = tid % (K1L_TZ / R);
    const int gz = (g.n[2] + K1L_TZ - 1) / K1L_TZ, gy = (g.n[1] + K1L_TY - 1) / K1L_TY;
    const int nc1 = g.nc[1], nc2 = g.nc[2];
    // cell starts of plane sx for this thread's entries of the reach
    auto load_lcs = [&](int sx, int y0, int z0, int (&v)[LPT]) {
#pragma unroll
        for (int u = 0; u < LPT; ++u) {
            const int e = tid + u * K1L_NT;
            v[u] = 0;
            if (e < LCS && sx >= 0 && sx < g.nc[0]) {
                const int r = e / (CELLS + 1), c = e - r * (CELLS + 1);
                const int sy = y0 - (W - 1) + r;
                if (sy >= 0 && sy < nc1) {
                    const int sz = min(max(z0 - (W - 1) + c, 0), nc2);
                    v[u] = __ldg(a.cell_start + ((int64_t)sx * nc1 + sy) * nc2 + sz);
                }
            }
        }
    };
    auto put_lcs = [&](int* dst, const int (&v)[LPT]) {
#pragma unroll
        for (int u = 0; u < LPT; ++u) {
            const int e = tid + u * K1L_NT;
            if (e < LCS) dst[e] = v[u];
        }
    };
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int tz = item % gz, ty = (item / gz) % gy, tx = item / (gz * gy);
        const int y0 = ty * K1L_TY, z0 = tz * K1L_TZ;
        const int y = y0 + ly, zb = z0 + lzg * R;
        const int xo0 = a.kx0 + tx * xc;
        const int xo1 = min(xo0 + xc, a.kx0 + a.knx);
        const int sx_lo = max(xo0 - (g.w[0] - 1), 0);
        const int sx_hi = min(xo1 - 1, g.nc[0] - 1);
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
        {
            int v[LPT];
            load_lcs(sx_lo, y0, z0, v);
            __syncthreads();   // previous item's last readers of lcs2 / soff / rec
            put_lcs(lcs2 + (sx_lo & 1) * LCS, v);
        }
        for (int sx = sx_lo; sx <= sx_hi; ++sx) {
            const int* lcs = lcs2 + (sx & 1) * LCS;
            __syncthreads();
            if (tid < 32) {   // staged row offsets (ROWS <= 32)
                const int len = tid < ROWS ? lcs[tid * (CELLS + 1) + CELLS] - lcs[tid * (CELLS + 1)] : 0;
                int inc = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, inc, o);
                    if (tid >= o) inc += t;
                }
                if (tid < ROWS) soff[tid + 1] = inc;
                if (tid == 0) soff[0] = 0;
            }
            __syncthreads();
            const int total = soff[ROWS];
            // the next plane's cell starts are in flight during this plane
            int nxt[LPT];
            load_lcs(sx + 1, y0, z0, nxt);
            for (int p0 = 0; p0 < total; p0 += cap) {
                const int pc = min(cap, total - p0);
                // all loads of this thread's staged points first, then the stencils
                int64_t gi[K1L_PF];
                double px[K1L_PF], py[K1L_PF], pz[K1L_PF];
                double2 qq[K1L_PF];
#pragma unroll
                for (int u = 0; u < K1L_PF; ++u) {
                    const int e = tid + u * K1L_NT;
                    gi[u] = -1;
                    if (e < pc) {
                        const int idx = p0 + e;
                        int lo = 0, hi = ROWS;   // soff[lo] <= idx < soff[lo + 1]
#pragma unroll
                        for (int st = 0; st < 5; ++st) {
                            const int mid = (lo + hi) >> 1;
                            if (hi - lo > 1) {
                                if (soff[mid] <= idx) lo = mid; else hi = mid;
                            }
                        }
                        gi[u] = lcs[lo * (CELLS + 1)] + (idx - soff[lo]);
                        px[u] = __ldg(pos + 3 * gi[u]);
                        py[u] = __ldg(pos + 3 * gi[u] + 1);
                        pz[u] = __ldg(pos + 3 * gi[u] + 2);
                        qq[u] = __ldg(reinterpret_cast<const double2*>(a.q_sorted + gi[u]));
                    }
                }
                if (p0) __syncthreads();   // the previous piece's readers of rec
#pragma unroll
                for (int u = 0; u < K1L_PF; ++u) {
                    if (gi[u] < 0) continue;
                    double* rp = rec + (size_t)(tid + u * K1L_NT) * REC;
                    rp[0] = qq[u].x;
                    rp[1] = qq[u].y;
                    fast_stencil<W>(px[u], g.n[0], g.origin[0], g.h[0], rh0, L, rp + 2);
                    fast_stencil<W>(py[u], g.n[1], g.origin[1], g.h[1], rh1, L, rp + 2 + W);
                    // the z start rides in the record's last slot as an int (no F2I in the point loop)
                    *reinterpret_cast<int*>(rp + 2 + 3 * W) = fast_stencil<W>(pz[u], g.n[2], g.origin[2], g.h[2], rh2, L, rp + 2 + 2 * W);
                }
                __syncthreads();
                // this thread's point ranges of the W rows it reads, flattened
                // into one loop (less lane divergence than W separate loops)
                int b0[W], pre[W + 1];
                pre[0] = 0;
#pragma unroll
                for (int ib = 0; ib < W; ++ib) {
                    const int r = ly + (W - 1) - ib;
                    const int* row = lcs + r * (CELLS + 1);
                    const int base = soff[r] - row[0] - p0;
                    b0[ib] = max(base + row[lzg * R], 0);
                    pre[ib + 1] = pre[ib] + max(min(base + row[lzg * R + R + W - 1], pc) - b0[ib], 0);
                }
#pragma unroll 1
                for (int t = 0; t < pre[W]; ++t) {
                    int ib = 0;
#pragma unroll
                    for (int u = 1; u < W; ++u) ib += t >= pre[u];
                    int k = b0[0] + t;
#pragma unroll
                    for (int u = 1; u < W; ++u)
                        if (ib == u) k = b0[u] + (t - pre[u]);
                    const double* rp = rec + (size_t)k * REC;
                    const double2 qv = *reinterpret_cast<const double2*>(rp);
                    double wx[W];
#pragma unroll
                    for (int ia = 0; ia < W; ++ia) wx[ia] = rp[2 + ia];
                    const double wy = rp[2 + W + ib];
                    const int sz = *reinterpret_cast<const int*>(rp + 2 + 3 * W);
                    const double qyr = qv.x * wy, qyi = qv.y * wy;
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const int ic = zb + j - sz;
                        const double wz = (unsigned)ic < (unsigned)W ? rp[2 + 2 * W + ic] : 0.0;
                        const double cr = qyr * wz, ci = qyi * wz;
#pragma unroll
                        for (int ia = 0; ia < W; ++ia) {
                            wr[j][ia] = fma(cr, wx[ia], wr[j][ia]);
                            wi[j][ia] = fma(ci, wx[ia], wi[j][ia]);
                        }
                    }
                }
            }
            put_lcs(lcs2 + ((sx + 1) & 1) * LCS, nxt);
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
}

template <int W>
static void k1_lines_launch(const EvalArgs& a, const double* pos, cudaStream_t s) {
    static int cap = 0, per_sm = 0;
    static size_t smem = 0;
    if (!cap) {
        cap = K1L_PF * K1L_NT;
        if (const char* e = getenv("FFTPIM_K1L_CAP")) cap = std::max(64, std::min(cap, atoi(e)));
        smem = k1_lines_smem<W>(cap);
        cudaFuncSetAttribute(k_k1_lines<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_k1_lines<W>, K1L_NT, smem);
        per_sm = std::max(per_sm, 1);
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int slots = sms * per_sm;
    const int gz = (a.g.n[2] + K1L_TZ - 1) / K1L_TZ, gy = (a.g.n[1] + K1L_TY - 1) / K1L_TY;
    // chunk length: minimise rounds x planes swept per item (W - 1 warm-up planes each)
    int xc = std::max(a.knx, 1), best = 1 << 30;
    for (int c = std::min(2 * (W - 1), a.knx); c <= a.knx; ++c) {
        const int items = gz * gy * ((a.knx + c - 1) / c);
        const int rounds = (items + slots - 1) / slots;
        const int cost = rounds * (c + W - 1);
        if (cost < best) {
            best = cost;
            xc = c;
        }
    }
    if (const char* e = getenv("FFTPIM_K1L_XC")) xc = std::max(1, atoi(e));
    xc = std::max(1, std::min(xc, std::max(a.knx, 1)));
    const int items = gz * gy * ((a.knx + xc - 1) / xc);
    const double rh0 = a.g.h[0] > 0 ? 1.0 / a.g.h[0] : 0.0, rh1 = a.g.h[1] > 0 ? 1.0 / a.g.h[1] : 0.0,
                 rh2 = a.g.h[2] > 0 ? 1.0 / a.g.h[2] : 0.0;
    k_k1_lines<W><<<std::min(items, slots), K1L_NT, smem, s>>>(a, pos, xc, items, cap, rh0, rh1, rh2);
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

// ------------------------------------------------------------- K3 on grid tiles
// Observer pass for the near interpolation (+ far interpolation and the K4
// row fix-up, or the precomputed far/fix-up term of the split schedule): a
// block owns a TX x TY x TZ tile of observer stencil-start cells -- TX * TY rows,
// each ONE contiguous run of the cell-sorted observers -- and first copies
// the (TX + W - 1) x (TY + W - 1) x (TZ + W - 1) grid nodes those observers can
// reach (coalesced z runs) plus the far observer grid into shared memory.
// Each thread then takes observers, computes their near and far stencils from
// the sorted position and gathers the 125 (or W^3) taps from the tile:
// consecutive lanes take consecutive observers of a row, whose taps are
// consecutive tile words.  The K4 row fix-up is the same fixed-order segment
// sum as k_observers; every sum has a fixed order.
#define K3T_TX 4
#define K3T_TY 4
#define K3T_TZ 32
#define K3T_NT 256
template <int W>
struct K3Tile {
    static constexpr int EX = K3T_TX + W - 1, EY = K3T_TY + W - 1, EZ = K3T_TZ + W - 1;
    static constexpr int NODES = EX * EY * EZ;
    static constexpr int ROWS = K3T_TX * K3T_TY;
};

#ifndef K3T_MINB
#define K3T_MINB 4
#endif
template <int W, int WF, int MODE>
__global__ void __launch_bounds__(K3T_NT, K3T_MINB) k_observers_tile(EvalArgs a, ObsPosArgs o, const int* __restrict__ ocs,
                                                             int64_t i0, int tsx0, int tnx) {
    using T = K3Tile<W>;
    extern __shared__ double k3t_smem[];
    cplx* tile = reinterpret_cast<cplx*>(k3t_smem);                 // NODES
    cplx* sfar = tile + T::NODES;                                    // far grid (MODE 0)
    const bool far = MODE == 0 && (a.parts & FFTPIM_FAR);
    const int nfx = a.fo.n[0], nfy = a.fo.n[1], nfz = a.fo.n[2];
    const int nf = far ? nfx * nfy * nfz : 0;
    int* rbeg = reinterpret_cast<int*>(sfar + nf);                   // ROWS + 1 (row starts, staged order)
    int* rglo = rbeg + T::ROWS + 1;                                  // ROWS (global first observer)
    const StencilGeom& g = a.g;
    const int gz = (g.nc[2] + K3T_TZ - 1) / K3T_TZ, gy = (g.nc[1] + K3T_TY - 1) / K3T_TY;
    const int bz = blockIdx.x % gz, by = (blockIdx.x / gz) % gy, bx = blockIdx.x / (gz * gy);
    const int sx0 = tsx0 + bx * K3T_TX, sy0 = by * K3T_TY, sz0 = bz * K3T_TZ;
    const int nc1 = g.nc[1], nc2 = g.nc[2];
    const int sxe = min(tsx0 + tnx, g.nc[0]);
    if (threadIdx.x < 32) {
        const int r = threadIdx.x;
        int lo = 0, len = 0;
        if (r < T::ROWS) {
            const int sx = sx0 + r / K3T_TY, sy = sy0 + r % K3T_TY;
            if (sx < sxe && sy < nc1) {
                const int64_t k = ((int64_t)sx * nc1 + sy) * nc2;
                lo = ocs[k + sz0];
                len = ocs[k + min(sz0 + K3T_TZ, nc2)] - lo;
            }
        }
        int inc = len;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, d);
            if (r >= d) inc += t;
        }
        if (r < T::ROWS) {
            rbeg[r + 1] = inc;
            rglo[r] = lo;
        }
        if (r == 0) rbeg[0] = 0;
    }
    // grid tile: nodes (sx0 + ex, sy0 + ey, sz0 + ez), clipped to the grid
    {
        const int m0 = g.n[0], m1 = g.n[1], m2 = g.n[2];
        // all of a thread's node loads are issued before the first store (one exposed
        // global latency per block instead of one per node)
        constexpr int NLD = (T::NODES + K3T_NT - 1) / K3T_NT;
        cplx v[NLD];
#pragma unroll
        for (int u = 0; u < NLD; ++u) {
            const int e = threadIdx.x + u * K3T_NT;
            const int ez = e % T::EZ, ey = (e / T::EZ) % T::EY, ex = e / (T::EZ * T::EY);
            const int x = sx0 + ex, y = sy0 + ey, z = sz0 + ez;
            v[u] = mk(0.0);
            if (e < T::NODES && x < m0 && x < sxe + W - 1 && y < m1 && z < m2)
                v[u] = a.interp_grid[((int64_t)(x - a.gx0) * a.gi1 + y) * a.gi2 + z];
        }
#pragma unroll
        for (int u = 0; u < NLD; ++u) {
            const int e = threadIdx.x + u * K3T_NT;
            if (e < T::NODES) tile[e] = v[u];
        }
        if (far)
            for (int t = threadIdx.x; t < nf; t += K3T_NT) sfar[t] = a.far_ug[t];
    }
    __syncthreads();
    const int total = rbeg[T::ROWS];
    const LagrangeDen<W> Ln;
    const LagrangeDen<WF> Lf;
    // (loading a thread's first observer position before the tile loads was measured slower:
    // 1.81 vs 1.73 ms at C4 -- the extra barrier and 80 B of spills outweigh the hidden latency)
    for (int k = threadIdx.x; k < total; k += K3T_NT) {
        int r = 0;
#pragma unroll
        for (int st = 0; st < 4; ++st) {   // ROWS = 16: rbeg[r] <= k < rbeg[r + 1]
            const int step = 8 >> st;
            if (rbeg[r + step] <= k) r += step;
        }
        const int64_t ig = rglo[r] + (k - rbeg[r]);   // global sorted observer
        const int64_t i = ig - i0;                    // this plan's (shard's) observer
        const double px = o.pos[3 * i], py = o.pos[3 * i + 1], pz = o.pos[3 * i + 2];
        double ar = 0.0, ai = 0.0;
        if (MODE == 2) {
            const cplx c = a.obs_pre[i];
            ar = c.re;
            ai = c.im;
        } else if ((a.parts & FFTPIM_NEAR) && a.sw_e >= 0) {
            const cplx c = a.sw_corr ? a.sw_corr[i * a.sw_E + a.sw_e] : corr_row_sum(a, i);
            ar = c.re;
            ai = c.im;
        }
        if (a.parts & FFTPIM_NEAR) {
            // per x plane an independent partial (W accumulator chains in flight),
            // summed in plane order
            double wx[W], wy[W], wz[W];
            const int s0 = fast_stencil<W>(px, g.n[0], g.origin[0], g.h[0], o.rn[0], Ln, wx) - sx0;
            const int s1 = fast_stencil<W>(py, g.n[1], g.origin[1], g.h[1], o.rn[1], Ln, wy) - sy0;
            const int s2 = fast_stencil<W>(pz, g.n[2], g.origin[2], g.h[2], o.rn[2], Ln, wz) - sz0;
            double pr[W], pi[W];
#pragma unroll
            for (int ia = 0; ia < W; ++ia) {
                pr[ia] = pi[ia] = 0.0;
#pragma unroll
                for (int ib = 0; ib < W; ++ib) {
                    const cplx* row = tile + ((s0 + ia) * T::EY + (s1 + ib)) * T::EZ + s2;
                    const double wxy = wx[ia] * wy[ib];
#pragma unroll
                    for (int ic = 0; ic < W; ++ic) {
                        const cplx v = row[ic];
                        const double wgt = wxy * wz[ic];
                        pr[ia] += wgt * v.re;
                        pi[ia] += wgt * v.im;
                    }
                }
            }
#pragma unroll
            for (int ia = 0; ia < W; ++ia) {
                ar += pr[ia];
                ai += pi[ia];
            }
        }
        if (far) {
            double wx[WF], wy[WF], wz[WF];
            const int s0 = fast_stencil<WF>(px, a.fo.n[0], a.fo.origin[0], a.fo.h[0], o.rf[0], Lf, wx);
            const int s1 = fast_stencil<WF>(py, a.fo.n[1], a.fo.origin[1], a.fo.h[1], o.rf[1], Lf, wy);
            const int s2 = fast_stencil<WF>(pz, a.fo.n[2], a.fo.origin[2], a.fo.h[2], o.rf[2], Lf, wz);
#pragma unroll
            for (int ia = 0; ia < WF; ++ia) {
#pragma unroll
                for (int ib = 0; ib < WF; ++ib) {
                    const int xx = min(s0 + ia, nfx - 1), yy = min(s1 + ib, nfy - 1);
                    const cplx* row = sfar + (xx * nfy + yy) * nfz;
                    const double wxy = wx[ia] * wy[ib];
#pragma unroll
                    for (int ic = 0; ic < WF; ++ic) {
                        const cplx v = row[min(s2 + ic, nfz - 1)];
                        const double wgt = wxy * wz[ic];
                        ar += wgt * v.re;
                        ai += wgt * v.im;
                    }
                }
            }
        }
        if (a.u_sorted)   // overlap schedule: K4 is still running, k_finish_corr adds its row sums
            a.u_sorted[i] = cplx{ar, ai};
        else
            a.u[a.obs_perm[i]] = cplx{ar, ai};
    }
}

// u (caller order) = interpolated potentials (sorted order) + the K4 row sums
__global__ void k_finish_corr(EvalArgs a) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= a.M) return;
    const cplx c = corr_row_sum(a, i);
    const cplx v = a.u_sorted[i];
    a.u[a.obs_perm[i]] = cplx{v.re + c.re, v.im + c.im};
}

void launch_finish_corr(const EvalArgs& a, cudaStream_t s) {
    if (a.M == 0) return;
    k_finish_corr<<<(int)((a.M + 255) / 256), 256, 0, s>>>(a);
    fftpim_count_launch();
}

template <int W, int WF, int MODE>
static void obs_tile_launch(const EvalArgs& a, const ObsPosArgs& o, const int* ocs, int64_t i0, cudaStream_t s) {
    using T = K3Tile<W>;
    const bool far = MODE == 0 && (a.parts & FFTPIM_FAR);
    const size_t nf = far ? (size_t)a.fo.n[0] * a.fo.n[1] * a.fo.n[2] : 0;
    const size_t smem = (T::NODES + nf) * sizeof(cplx) + (2 * T::ROWS + 1) * sizeof(int);
    static size_t configured = 48 * 1024;
    if (smem > configured) {
        cudaFuncSetAttribute(k_observers_tile<W, WF, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    const int tsx0 = a.kx0, tnx = std::min(a.knx, a.g.nc[0] - a.kx0);
    if (tnx <= 0) return;
    const int gz = (a.g.nc[2] + K3T_TZ - 1) / K3T_TZ, gy = (a.g.nc[1] + K3T_TY - 1) / K3T_TY;
    const int gx = (tnx + K3T_TX - 1) / K3T_TX;
    k_observers_tile<W, WF, MODE><<<gx * gy * gz, K3T_NT, smem, s>>>(a, o, ocs, i0, tsx0, tnx);
}

template <int W, int MODE>
static bool obs_tile_far(const EvalArgs& a, const ObsPosArgs& o, const int* ocs, int64_t i0, cudaStream_t s) {
    switch (a.fo.order + 1) {
        case 3: obs_tile_launch<W, 3, MODE>(a, o, ocs, i0, s); return true;
        case 4: obs_tile_launch<W, 4, MODE>(a, o, ocs, i0, s); return true;
        case 5: obs_tile_launch<W, 5, MODE>(a, o, ocs, i0, s); return true;
        default: return false;
    }
}

template <int MODE>
static bool obs_tile_near(const EvalArgs& a, const ObsPosArgs& o, const int* ocs, int64_t i0, cudaStream_t s) {
    switch (a.g.order + 1) {
        case 3: return obs_tile_far<3, MODE>(a, o, ocs, i0, s);
        case 4: return obs_tile_far<4, MODE>(a, o, ocs, i0, s);
        case 5: return obs_tile_far<5, MODE>(a, o, ocs, i0, s);
        case 6: return obs_tile_far<6, MODE>(a, o, ocs, i0, s);
        default: return false;
    }
}

// mode 0 (fused) and 2 (near + obs_pre) on grid tiles; false: not applicable
// (mode 1, single-plane axes, orders outside the instantiated set)
bool launch_observers_tile(const EvalArgs& a, const double* pos, const int* ocs, int64_t i0, cudaStream_t s,
                           int mode) {
    if (mode == 1 || !ocs) return false;
    if (a.g.n[0] < 2 || a.g.n[1] < 2 || a.g.n[2] < 2) return false;
    if (a.M == 0) return true;
    ObsPosArgs o;
    o.pos = pos;
    for (int ax = 0; ax < 3; ++ax) {
        o.rn[ax] = a.g.h[ax] > 0 ? 1.0 / a.g.h[ax] : 0.0;
        o.rf[ax] = a.fo.h[ax] > 0 ? 1.0 / a.fo.h[ax] : 0.0;
    }
    const bool ok = mode == 2 ? obs_tile_near<2>(a, o, ocs, i0, s) : obs_tile_near<0>(a, o, ocs, i0, s);
    if (ok) fftpim_count_launch();
    return ok;
}

// ------------------------------------------------------------- K5a on windows
// Far projection (farzone.py:156, grids.py:167-181 on the 10^3 far source grid)
// from the sorted positions.  A warp takes a chunk of consecutive sorted points;
// their far stencil starts span few far cells (the points are sorted by near
// cell), so the warp first finds the bounding window of its chunk's far nodes
// and accumulates into a private copy of just that window in shared memory
// (lane l owns taps l, l + 32, ... and sums runs of points with the same start in
// registers, flushing on a start change).  A chunk whose window exceeds the
// shared capacity accumulates straight into its own global slot (private, L2).
// The chunk windows are then summed per far node in a fixed order
// (k_far_windows_reduce): no atomics, bitwise reproducible.
#define FPW_WARPS 8
#define FPW_CAP 400       // window entries per warp in shared memory: 400 (2 blocks per SM) or 256 (3 blocks)
struct FarWinArgs {
    const double* pos;          // sorted positions of the projected points
    const cplx* q;              // their sorted charges
    int64_t n;                  // points
    int chunk;                  // points per warp chunk
    int nchunks;
    int cap;                    // shared-memory window entries per warp
    cplx* slots;                // (nchunks, nf) windows
    int* win;                   // (nchunks, 6): x0, y0, z0, ex, ey, ez
    double rf[3];
};

template <int WF>
__global__ void __launch_bounds__(32 * FPW_WARPS) k_far_project_win(EvalArgs a, FarWinArgs f) {
    constexpr int TPL = (WF * WF * WF + 31) / 32;
    constexpr int REC = 3 * WF + 2;
    extern __shared__ __align__(16) double fpw_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * FPW_WARPS + warp;
    if (c >= f.nchunks) return;
    cplx* wgrid = reinterpret_cast<cplx*>(fpw_smem) + warp * f.cap;
    double* stage = fpw_smem + 2 * FPW_WARPS * f.cap + warp * 32 * REC;
    int* sst = reinterpret_cast<int*>(fpw_smem + 2 * FPW_WARPS * f.cap + FPW_WARPS * 32 * REC) + warp * 32 * 3;
    const StencilGeom& fs = a.fs;
    const int nfx = fs.n[0], nfy = fs.n[1], nfz = fs.n[2];
    const int nf = nfx * nfy * nfz;
    const int64_t p0 = (int64_t)c * f.chunk, p1 = min(p0 + f.chunk, f.n);
    const LagrangeDen<WF> L;
    // pass 1: bounding window of the chunk's far stencil starts
    int lo[3] = {1 << 30, 1 << 30, 1 << 30}, hi[3] = {-1, -1, -1};
    for (int64_t p = p0 + lane; p < p1; p += 32) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            double w[WF];
            const int s = fast_stencil<WF>(__ldg(f.pos + 3 * p + ax), fs.n[ax], fs.origin[ax], fs.h[ax], f.rf[ax], L, w);
            lo[ax] = min(lo[ax], s);
            hi[ax] = max(hi[ax], s);
        }
    }
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
        for (int o = 16; o; o >>= 1) {
            lo[ax] = min(lo[ax], __shfl_xor_sync(0xffffffffu, lo[ax], o));
            hi[ax] = max(hi[ax], __shfl_xor_sync(0xffffffffu, hi[ax], o));
        }
    int ext[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) ext[ax] = min(hi[ax] + fs.w[ax], fs.n[ax]) - lo[ax];
    const int wn = ext[0] * ext[1] * ext[2];
    const bool in_smem = wn <= f.cap;
    cplx* dst = in_smem ? wgrid : f.slots + (int64_t)c * nf;
    for (int t = lane; t < wn; t += 32) dst[t] = mk(0.0);
    if (lane < 3) {
        f.win[6 * c + lane] = lo[lane];
        f.win[6 * c + 3 + lane] = ext[lane];
    }
    // this lane's taps (taps past a single-plane axis are skipped)
    int ta[TPL], tb[TPL], tc[TPL];
    bool tok[TPL];
#pragma unroll
    for (int t = 0; t < TPL; ++t) {
        const int tp = lane + 32 * t;
        tc[t] = tp % WF;
        tb[t] = (tp / WF) % WF;
        ta[t] = tp / (WF * WF);
        tok[t] = tp < WF * WF * WF && ta[t] < fs.w[0] && tb[t] < fs.w[1] && tc[t] < fs.w[2];
    }
    double accr[TPL], acci[TPL];
#pragma unroll
    for (int t = 0; t < TPL; ++t) accr[t] = acci[t] = 0.0;
    int c0 = -1, c1 = 0, c2 = 0;
    auto flush = [&]() {
#pragma unroll
        for (int t = 0; t < TPL; ++t) {
            if (!tok[t]) continue;
            cplx& d = dst[((c0 - lo[0] + ta[t]) * ext[1] + (c1 - lo[1] + tb[t])) * ext[2] + (c2 - lo[2] + tc[t])];
            d.re += accr[t];
            d.im += acci[t];
            accr[t] = acci[t] = 0.0;
        }
        __syncwarp();
    };
    __syncwarp();
    // pass 2: batches of 32 points, stencils computed by the loading lane; the next
    // batch's position and charge are in flight while this batch is processed
    double nx[3] = {0.0, 0.0, 0.0};
    double2 nq = make_double2(0.0, 0.0);
    if (p0 + lane < p1) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) nx[ax] = __ldg(f.pos + 3 * (p0 + lane) + ax);
        nq = __ldg(reinterpret_cast<const double2*>(f.q + p0 + lane));
    }
    for (int64_t base = p0; base < p1; base += 32) {
        const int64_t p = base + lane;
        const double cx[3] = {nx[0], nx[1], nx[2]};
        const double2 qv = nq;
        if (p + 32 < p1) {
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) nx[ax] = __ldg(f.pos + 3 * (p + 32) + ax);
            nq = __ldg(reinterpret_cast<const double2*>(f.q + p + 32));
        }
        __syncwarp();
        if (p < p1) {
            double* r = stage + lane * REC;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax)
                sst[lane * 3 + ax] = fast_stencil<WF>(cx[ax], fs.n[ax], fs.origin[ax], fs.h[ax], f.rf[ax], L, r + ax * WF);
            r[3 * WF] = qv.x;
            r[3 * WF + 1] = qv.y;
        }
        __syncwarp();
        const int cnt = (int)min((int64_t)32, p1 - base);
        for (int j = 0; j < cnt; ++j) {
            const double* r = stage + j * REC;
            const int s0 = sst[3 * j], s1 = sst[3 * j + 1], s2 = sst[3 * j + 2];
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
    if (in_smem) {
        cplx* out = f.slots + (int64_t)c * nf;
        for (int t = lane; t < wn; t += 32) out[t] = wgrid[t];
    }
}

// Plan-time bounding windows of the chunks (the positions never change): pass 1
// of k_far_project_win once, so that the evaluation kernel below starts at pass 2.
template <int WF>
__global__ void __launch_bounds__(256) k_far_win_bounds(StencilGeom fs, FarWinArgs f) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * 8 + warp;
    if (c >= f.nchunks) return;
    const int64_t p0 = (int64_t)c * f.chunk, p1 = min(p0 + f.chunk, f.n);
    const LagrangeDen<WF> L;
    int lo[3] = {1 << 30, 1 << 30, 1 << 30}, hi[3] = {-1, -1, -1};
    for (int64_t p = p0 + lane; p < p1; p += 32) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            double w[WF];
            const int s = fast_stencil<WF>(__ldg(f.pos + 3 * p + ax), fs.n[ax], fs.origin[ax], fs.h[ax], f.rf[ax], L, w);
            lo[ax] = min(lo[ax], s);
            hi[ax] = max(hi[ax], s);
        }
    }
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
        for (int o = 16; o; o >>= 1) {
            lo[ax] = min(lo[ax], __shfl_xor_sync(0xffffffffu, lo[ax], o));
            hi[ax] = max(hi[ax], __shfl_xor_sync(0xffffffffu, hi[ax], o));
        }
    if (lane < 3) {
        f.win[6 * c + lane] = lo[lane];
        f.win[6 * c + 3 + lane] = min(hi[lane] + fs.w[lane], fs.n[lane]) - lo[lane];
    }
}

// k_far_project_win with the windows read from the plan (no pass 1) and the
// batch of 32 staged points split into runs of equal stencil starts by one
// ballot: the inner loop over a run has no data-dependent branch, so the
// shared-memory loads of the following points are in flight while a point's
// products retire.  Same chunks, runs and summation order as k_far_project_win:
// the far grid is bit-identical.
template <int WF>
__global__ void __launch_bounds__(32 * FPW_WARPS) k_far_project_win2(EvalArgs a, FarWinArgs f) {
    constexpr int TPL = (WF * WF * WF + 31) / 32;
    constexpr int REC = 3 * WF + 2;
    extern __shared__ __align__(16) double fpw_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * FPW_WARPS + warp;
    if (c >= f.nchunks) return;
    cplx* wgrid = reinterpret_cast<cplx*>(fpw_smem) + warp * f.cap;
    double* stage = fpw_smem + 2 * FPW_WARPS * f.cap + warp * 32 * REC;
    const StencilGeom& fs = a.fs;
    const int nf = fs.n[0] * fs.n[1] * fs.n[2];
    const int64_t p0 = (int64_t)c * f.chunk, p1 = min(p0 + f.chunk, f.n);
    const LagrangeDen<WF> L;
    const int lo0 = __ldg(f.win + 6 * c), lo1 = __ldg(f.win + 6 * c + 1), lo2 = __ldg(f.win + 6 * c + 2);
    const int ext0 = __ldg(f.win + 6 * c + 3), ext1 = __ldg(f.win + 6 * c + 4), ext2 = __ldg(f.win + 6 * c + 5);
    const int wn = ext0 * ext1 * ext2;
    const bool in_smem = wn <= f.cap;
    cplx* dst = in_smem ? wgrid : f.slots + (int64_t)c * nf;
    for (int t = lane; t < wn; t += 32) dst[t] = mk(0.0);
    // this lane's taps: word offsets into a staged record and into the window
    int oa[TPL], ob[TPL], oc[TPL], od[TPL];
    bool tok[TPL];
#pragma unroll
    for (int t = 0; t < TPL; ++t) {
        const int tp = lane + 32 * t;
        const int tc = tp % WF, tb = (tp / WF) % WF, ta = tp / (WF * WF);
        tok[t] = tp < WF * WF * WF && ta < fs.w[0] && tb < fs.w[1] && tc < fs.w[2];
        oa[t] = tok[t] ? ta : 0;
        ob[t] = tok[t] ? WF + tb : WF;
        oc[t] = tok[t] ? 2 * WF + tc : 2 * WF;
        od[t] = (ta * ext1 + tb) * ext2 + tc;
    }
    double accr[TPL], acci[TPL];
#pragma unroll
    for (int t = 0; t < TPL; ++t) accr[t] = acci[t] = 0.0;
    int c0 = -1, c1 = 0, c2 = 0;
    auto flush = [&]() {
        const int base = ((c0 - lo0) * ext1 + (c1 - lo1)) * ext2 + (c2 - lo2);
#pragma unroll
        for (int t = 0; t < TPL; ++t) {
            if (!tok[t]) continue;
            cplx& d = dst[base + od[t]];
            d.re += accr[t];
            d.im += acci[t];
            accr[t] = acci[t] = 0.0;
        }
        __syncwarp();
    };
    __syncwarp();
    for (int64_t base = p0; base < p1; base += 32) {
        const int64_t p = base + lane;
        const int cnt = (int)min((int64_t)32, p1 - base);
        int s0 = c0, s1 = c1, s2 = c2;
        __syncwarp();
        if (p < p1) {
            double* r = stage + lane * REC;
            s0 = fast_stencil<WF>(__ldg(f.pos + 3 * p), fs.n[0], fs.origin[0], fs.h[0], f.rf[0], L, r);
            s1 = fast_stencil<WF>(__ldg(f.pos + 3 * p + 1), fs.n[1], fs.origin[1], fs.h[1], f.rf[1], L, r + WF);
            s2 = fast_stencil<WF>(__ldg(f.pos + 3 * p + 2), fs.n[2], fs.origin[2], fs.h[2], f.rf[2], L, r + 2 * WF);
            const double2 qv = __ldg(reinterpret_cast<const double2*>(f.q + p));
            r[3 * WF] = qv.x;
            r[3 * WF + 1] = qv.y;
        }
        // run heads: a staged point whose start differs from its predecessor's
        // (lane 0: from the start carried over from the previous batch)
        int q0 = __shfl_up_sync(0xffffffffu, s0, 1), q1 = __shfl_up_sync(0xffffffffu, s1, 1),
            q2 = __shfl_up_sync(0xffffffffu, s2, 1);
        if (lane == 0) {
            q0 = c0;
            q1 = c1;
            q2 = c2;
        }
        const unsigned heads = __ballot_sync(0xffffffffu, lane < cnt && (s0 != q0 || s1 != q1 || s2 != q2));
        __syncwarp();
        int j = 0;
        while (j < cnt) {
            if ((heads >> j) & 1u) {
                if (c0 >= 0) flush();
                c0 = __shfl_sync(0xffffffffu, s0, j);
                c1 = __shfl_sync(0xffffffffu, s1, j);
                c2 = __shfl_sync(0xffffffffu, s2, j);
            }
            const unsigned rest = j < 31 ? heads & (0xffffffffu << (j + 1)) : 0u;
            const int e = rest ? __ffs(rest) - 1 : cnt;
#pragma unroll 4
            for (int k = j; k < e; ++k) {
                const double* r = stage + k * REC;
                const double qre = r[3 * WF], qim = r[3 * WF + 1];
#pragma unroll
                for (int t = 0; t < TPL; ++t) {
                    const double wgt = (r[oa[t]] * r[ob[t]]) * r[oc[t]];
                    accr[t] += wgt * qre;
                    acci[t] += wgt * qim;
                }
            }
            j = e;
        }
    }
    if (c0 >= 0) flush();
    if (in_smem) {
        cplx* out = f.slots + (int64_t)c * nf;
        for (int t = lane; t < wn; t += 32) out[t] = wgrid[t];
    }
}

// Order-3 far stencils (4^3 = 64 taps), four staged points per warp step: the warp
// splits into four groups of 8 lanes, group g takes point a + 4 r + g of a run
// [a, b) of equal stencil starts, and a lane owns the 8 taps (ta = 0..3,
// tb = 2 h, 2 h + 1, tc) with h = (lane & 7) >> 2, tc = lane & 3: five
// shared-memory loads (two 16-byte wx pairs, one wy pair, wz, q) feed 32 FP64
// instructions, ~10 instructions per point instead of ~25.  At the end of a run
// the four groups' sums are added by two shuffle steps in a fixed order and
// group g adds the taps ta = g to the window.  Windows, chunks and runs as in
// k_far_project_win2; the sums differ from k_far_project_win's in the last bits
// only (another fixed order).
__global__ void __launch_bounds__(32 * FPW_WARPS) k_far_project_win4(EvalArgs a, FarWinArgs f) {
    constexpr int WF = 4, REC = 3 * WF + 2;
    extern __shared__ __align__(16) double fpw_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * FPW_WARPS + warp;
    if (c >= f.nchunks) return;
    cplx* wgrid = reinterpret_cast<cplx*>(fpw_smem) + warp * f.cap;
    double* stage = fpw_smem + 2 * FPW_WARPS * f.cap + warp * 32 * REC;
    const StencilGeom& fs = a.fs;
    const int nf = fs.n[0] * fs.n[1] * fs.n[2];
    const int64_t p0 = (int64_t)c * f.chunk, p1 = min(p0 + f.chunk, f.n);
    const LagrangeDen<WF> L;
    const int lo0 = __ldg(f.win + 6 * c), lo1 = __ldg(f.win + 6 * c + 1), lo2 = __ldg(f.win + 6 * c + 2);
    const int ext0 = __ldg(f.win + 6 * c + 3), ext1 = __ldg(f.win + 6 * c + 4), ext2 = __ldg(f.win + 6 * c + 5);
    const int wn = ext0 * ext1 * ext2;
    const bool in_smem = wn <= f.cap;
    cplx* dst = in_smem ? wgrid : f.slots + (int64_t)c * nf;
    for (int t = lane; t < wn; t += 32) dst[t] = mk(0.0);
    const int grp = lane >> 3, h = (lane & 7) >> 2, tc = lane & 3;
    // taps this lane adds to the window at a run end: ta = grp, tb = 2 h + j
    int od[2];
    bool tok[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int tb = 2 * h + j;
        tok[j] = grp < fs.w[0] && tb < fs.w[1] && tc < fs.w[2];
        od[j] = (grp * ext1 + tb) * ext2 + tc;
    }
    double accr[4][2], acci[4][2];
#pragma unroll
    for (int ta = 0; ta < 4; ++ta)
#pragma unroll
        for (int j = 0; j < 2; ++j) accr[ta][j] = acci[ta][j] = 0.0;
    int c0 = -1, c1 = 0, c2 = 0;
    auto flush = [&]() {
        const int base = ((c0 - lo0) * ext1 + (c1 - lo1)) * ext2 + (c2 - lo2);
#pragma unroll
        for (int ta = 0; ta < 4; ++ta)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                double vr = accr[ta][j], vi = acci[ta][j];
                vr += __shfl_xor_sync(0xffffffffu, vr, 8);
                vi += __shfl_xor_sync(0xffffffffu, vi, 8);
                vr += __shfl_xor_sync(0xffffffffu, vr, 16);
                vi += __shfl_xor_sync(0xffffffffu, vi, 16);
                if (ta == grp && tok[j]) {
                    cplx& d = dst[base + od[j]];
                    d.re += vr;
                    d.im += vi;
                }
                accr[ta][j] = acci[ta][j] = 0.0;
            }
        __syncwarp();
    };
    __syncwarp();
    for (int64_t base = p0; base < p1; base += 32) {
        const int64_t p = base + lane;
        const int cnt = (int)min((int64_t)32, p1 - base);
        int s0 = c0, s1 = c1, s2 = c2;
        __syncwarp();
        if (p < p1) {
            double* r = stage + lane * REC;
            s0 = fast_stencil<WF>(__ldg(f.pos + 3 * p), fs.n[0], fs.origin[0], fs.h[0], f.rf[0], L, r);
            s1 = fast_stencil<WF>(__ldg(f.pos + 3 * p + 1), fs.n[1], fs.origin[1], fs.h[1], f.rf[1], L, r + WF);
            s2 = fast_stencil<WF>(__ldg(f.pos + 3 * p + 2), fs.n[2], fs.origin[2], fs.h[2], f.rf[2], L, r + 2 * WF);
            const double2 qv = __ldg(reinterpret_cast<const double2*>(f.q + p));
            r[3 * WF] = qv.x;
            r[3 * WF + 1] = qv.y;
        }
        int q0 = __shfl_up_sync(0xffffffffu, s0, 1), q1 = __shfl_up_sync(0xffffffffu, s1, 1),
            q2 = __shfl_up_sync(0xffffffffu, s2, 1);
        if (lane == 0) {
            q0 = c0;
            q1 = c1;
            q2 = c2;
        }
        const unsigned heads = __ballot_sync(0xffffffffu, lane < cnt && (s0 != q0 || s1 != q1 || s2 != q2));
        __syncwarp();
        int j = 0;
        while (j < cnt) {
            if ((heads >> j) & 1u) {
                if (c0 >= 0) flush();
                c0 = __shfl_sync(0xffffffffu, s0, j);
                c1 = __shfl_sync(0xffffffffu, s1, j);
                c2 = __shfl_sync(0xffffffffu, s2, j);
            }
            const unsigned rest = j < 31 ? heads & (0xffffffffu << (j + 1)) : 0u;
            const int e = rest ? __ffs(rest) - 1 : cnt;
            for (int k = j + grp; k < e; k += 4) {
                const double* r = stage + k * REC;
                const double2 wx01 = *reinterpret_cast<const double2*>(r);
                const double2 wx23 = *reinterpret_cast<const double2*>(r + 2);
                const double2 wy = *reinterpret_cast<const double2*>(r + WF + 2 * h);
                const double wz = r[2 * WF + tc];
                const double2 qv = *reinterpret_cast<const double2*>(r + 3 * WF);
                const double wx[4] = {wx01.x, wx01.y, wx23.x, wx23.y};
#pragma unroll
                for (int ta = 0; ta < 4; ++ta) {
                    const double w0 = (wx[ta] * wy.x) * wz, w1 = (wx[ta] * wy.y) * wz;
                    accr[ta][0] += w0 * qv.x;
                    acci[ta][0] += w0 * qv.y;
                    accr[ta][1] += w1 * qv.x;
                    acci[ta][1] += w1 * qv.y;
                }
            }
            __syncwarp();
            j = e;
        }
    }
    if (c0 >= 0) flush();
    if (in_smem) {
        cplx* out = f.slots + (int64_t)c * nf;
        for (int t = lane; t < wn; t += 32) out[t] = wgrid[t];
    }
}

// far node t: sum of the chunk windows covering it, chunks in a fixed tree order
__global__ void __launch_bounds__(256) k_far_windows_reduce(FarWinArgs f, int nfx, int nfy, int nfz, cplx* qg) {
    const int t = blockIdx.x;
    const int x = t / (nfy * nfz), y = (t / nfz) % nfy, z = t % nfz;
    const int nf = nfx * nfy * nfz;
    cplx s = mk(0.0);
    for (int c = threadIdx.x; c < f.nchunks; c += blockDim.x) {
        const int* w = f.win + 6 * c;
        const int lx = x - w[0], ly = y - w[1], lz = z - w[2];
        if (lx >= 0 && lx < w[3] && ly >= 0 && ly < w[4] && lz >= 0 && lz < w[5])
            s = s + f.slots[(int64_t)c * nf + (lx * w[4] + ly) * w[5] + lz];
    }
    __shared__ cplx red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) qg[t] = red[0];
}

// points per warp chunk for `slots` resident warps (one wave, equal chunks)
static int far_chunk_for(int64_t n, int slots) {
    int64_t c = (n + slots - 1) / slots;
    c = std::max<int64_t>(256, std::min<int64_t>(4096, c));
    return (int)((c + 31) / 32 * 32);
}

// Plan build: choose the chunk length and the shared-memory window capacity, and
// compute the chunk windows of the n sorted points.  First choice: one wave of
// 3 blocks x 8 warps per SM with 256-entry windows (more resident warps hide the
// dependent FP64 chains); if a chunk's window is larger, 2 blocks per SM with
// 400-entry windows (larger windows accumulate in their global slot).
// FFTPIM_FAR_CAP=400 forces the second choice.
void far_win_setup(const StencilGeom& fs, const double* pos, int64_t n, int* win, int* chunk_out, int* cap_out,
                   cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const int forced = [] {
        const char* e = getenv("FFTPIM_FAR_CAP");
        return e ? atoi(e) : 0;
    }();
    *chunk_out = far_chunk_for(n, sms * 2 * FPW_WARPS);
    *cap_out = FPW_CAP;
    if (!pos || !win || n <= 0) return;
    for (int attempt = forced == FPW_CAP ? 1 : 0; attempt < 2; ++attempt) {
        FarWinArgs f;
        f.pos = pos;
        f.q = nullptr;
        f.n = n;
        f.chunk = far_chunk_for(n, sms * (attempt == 0 ? 3 : 2) * FPW_WARPS);
        f.nchunks = (int)((n + f.chunk - 1) / f.chunk);
        f.cap = attempt == 0 ? 256 : FPW_CAP;
        f.slots = nullptr;
        f.win = win;
        for (int ax = 0; ax < 3; ++ax) f.rf[ax] = fs.h[ax] > 0 ? 1.0 / fs.h[ax] : 0.0;
        const int blocks = (f.nchunks + 7) / 8;
        switch (fs.order + 1) {
            case 3: k_far_win_bounds<3><<<blocks, 256, 0, s>>>(fs, f); break;
            case 4: k_far_win_bounds<4><<<blocks, 256, 0, s>>>(fs, f); break;
            case 5: k_far_win_bounds<5><<<blocks, 256, 0, s>>>(fs, f); break;
            default: return;
        }
        fftpim_count_launch();
        *chunk_out = f.chunk;
        *cap_out = f.cap;
        if (attempt == 1) return;
        std::vector<int> h((size_t)f.nchunks * 6);
        cudaMemcpyAsync(h.data(), win, h.size() * sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        int worst = 0;
        for (int c = 0; c < f.nchunks; ++c) worst = std::max(worst, h[6 * c + 3] * h[6 * c + 4] * h[6 * c + 5]);
        if (worst <= f.cap) return;
    }
}

// upper bound of the chunk count over both choices (slot allocation)
int64_t far_win_max_chunks(int64_t n) { return (n + 255) / 256 + 1; }

bool launch_far_project_win(const EvalArgs& a, const double* pos, cplx* slots, int* win, cudaStream_t s) {
    if (!pos || !slots || a.far_chunk <= 0) return false;
    FarWinArgs f;
    f.pos = pos;
    f.q = a.far_q;
    f.n = a.far_n;
    f.chunk = a.far_chunk;
    f.nchunks = (int)((a.far_n + f.chunk - 1) / f.chunk);
    f.cap = a.far_cap;
    f.slots = slots;
    f.win = win;
    for (int ax = 0; ax < 3; ++ax) f.rf[ax] = a.fs.h[ax] > 0 ? 1.0 / a.fs.h[ax] : 0.0;
    const int WF = a.fs.order + 1;
    const size_t smem = (size_t)FPW_WARPS * (f.cap * sizeof(cplx) + 32 * (3 * WF + 2) * sizeof(double) +
                                             32 * 3 * sizeof(int));
    const int blocks = (f.nchunks + FPW_WARPS - 1) / FPW_WARPS;
    // FFTPIM_FAR_WIN2=1: plan-time windows + ballot-split runs (k_far_project_win2).  Bit-identical, 30 %
    // fewer instructions, but measured slower on one B200 (C4 1.02 vs 0.97 ms, C5 0.32 vs 0.27 ms, C3 0.19 vs
    // 0.16 ms): the kernel is bound by the dependent FP64 chains per point, not by the per-point branch
    static const bool v2 = [] {
        const char* e = getenv("FFTPIM_FAR_WIN2");
        return e && e[0] == '1';
    }();
    auto go = [&](auto kern, auto kern2) {
        static size_t configured = 48 * 1024;
        if (smem > configured) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            configured = smem;
        }
        if (f.nchunks <= 0) return;
        if (v2)
            kern2<<<blocks, 32 * FPW_WARPS, smem, s>>>(a, f);
        else
            kern<<<blocks, 32 * FPW_WARPS, smem, s>>>(a, f);
    };
    // FFTPIM_FAR_WIN4=1: order-3 stencils, four points per warp step (k_far_project_win4).  Measured 2.2x slower
    // than the general kernel (C4 2.12 vs 0.97 ms, C5 0.55-0.62 vs 0.27 ms, C3 0.37-0.40 vs 0.16 ms): runs of equal
    // starts are ~13 points, so the 128 shuffles of the group reduction per run outweigh the shorter point loop
    static const bool v4 = [] {
        const char* e = getenv("FFTPIM_FAR_WIN4");
        return e && e[0] == '1';
    }();
    if (WF == 4 && v4 && !v2) {
        static size_t configured4 = 48 * 1024;
        if (smem > configured4) {
            cudaFuncSetAttribute(k_far_project_win4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            configured4 = smem;
        }
        if (f.nchunks > 0) k_far_project_win4<<<blocks, 32 * FPW_WARPS, smem, s>>>(a, f);
        const int nf4 = a.fs.n[0] * a.fs.n[1] * a.fs.n[2];
        k_far_windows_reduce<<<nf4, 256, 0, s>>>(f, a.fs.n[0], a.fs.n[1], a.fs.n[2], a.far_qg);
        fftpim_count_launch(2);
        return true;
    }
    switch (WF) {
        case 3: go(k_far_project_win<3>, k_far_project_win2<3>); break;
        case 4: go(k_far_project_win<4>, k_far_project_win2<4>); break;
        case 5: go(k_far_project_win<5>, k_far_project_win2<5>); break;
        default: return false;
    }
    const int nf = a.fs.n[0] * a.fs.n[1] * a.fs.n[2];
    k_far_windows_reduce<<<nf, 256, 0, s>>>(f, a.fs.n[0], a.fs.n[1], a.fs.n[2], a.far_qg);
    fftpim_count_launch(2);
    return true;
}

// observers per K3 tile (TX x TY x TZ stencil-start cells), max over tiles
__global__ void k_max_tile_count(StencilGeom g, const int* __restrict__ ocs, int* out) {
    const int gz = (g.nc[2] + K3T_TZ - 1) / K3T_TZ, gy = (g.nc[1] + K3T_TY - 1) / K3T_TY;
    const int gx = (g.nc[0] + K3T_TX - 1) / K3T_TX;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)gx * gy * gz) return;
    const int bz = (int)(t % gz), by = (int)((t / gz) % gy), bx = (int)(t / ((int64_t)gz * gy));
    int n = 0;
    for (int r = 0; r < K3T_TX * K3T_TY; ++r) {
        const int sx = bx * K3T_TX + r / K3T_TY, sy = by * K3T_TY + r % K3T_TY;
        if (sx >= g.nc[0] || sy >= g.nc[1]) continue;
        const int64_t k = ((int64_t)sx * g.nc[1] + sy) * g.nc[2];
        n += ocs[k + min((bz + 1) * K3T_TZ, g.nc[2])] - ocs[k + bz * K3T_TZ];
    }
    atomicMax(out, n);
}
int64_t launch_max_tile_count(const StencilGeom& g, const int* ocs, cudaStream_t s) {
    int* d = nullptr;
    cudaMallocAsync(&d, sizeof(int), s);
    cudaMemsetAsync(d, 0, sizeof(int), s);
    const int64_t tiles = (int64_t)((g.nc[0] + K3T_TX - 1) / K3T_TX) * ((g.nc[1] + K3T_TY - 1) / K3T_TY) *
                          ((g.nc[2] + K3T_TZ - 1) / K3T_TZ);
    k_max_tile_count<<<(int)((tiles + 255) / 256), 256, 0, s>>>(g, ocs, d);
    int h = 0;
    cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFreeAsync(d, s);
    fftpim_count_launch();
    return h;
}
