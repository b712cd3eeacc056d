// build_kernels.cu -- device-side plan build:
//   point sorting by near stencil cell, Lagrange stencils (grids.py:110-217),
//   near kernel table + circulant embedding (nearzone.py:127-147, 212-235),
//   correction pair discovery and coefficients (nearzone.py:303-487),
//   far kernel series with per-point adaptive truncation (pgf.py:166-462).
#include "geom.cuh"
#include "kernels.h"

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// ---------------------------------------------------------------------------
// points and stencils
// ---------------------------------------------------------------------------
__global__ void k_cell_keys(const double* __restrict__ pos, int64_t n, StencilGeom g, int* keys,
                            DevStatus* st) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int s[3];
    double w[FFTPIM_MAX_W];
    for (int a = 0; a < 3; ++a) {
        if (!axis_stencil(pos[3 * i + a], g.n[a], g.origin[a], g.h[a], g.order, g.margin[a], &s[a], w))
            set_status(st, FFTPIM_DOMAIN, 10 + a, i, a);
    }
    keys[i] = cell_key(g, s[0], s[1], s[2]);
}

void launch_cell_keys(const double* pos, int64_t n, const StencilGeom& g, int* keys, DevStatus* st,
                      cudaStream_t s) {
    if (n == 0) return;
    k_cell_keys<<<nblk(n, 256), 256, 0, s>>>(pos, n, g, keys, st);
    fftpim_count_launch();
}

// start[c] = first sorted index with key >= c  (CSR from sorted keys, no atomics)
__global__ void k_csr_from_sorted(const int* __restrict__ keys, int64_t n, int64_t ncells, int* start) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    int64_t lo = (i == 0) ? 0 : (int64_t)keys[i - 1] + 1;
    int64_t hi = (i == n) ? ncells : (int64_t)keys[i];
    for (int64_t c = lo; c <= hi; ++c) start[c] = (int)i;
}

void launch_csr_from_sorted(const int* keys, int64_t n, int64_t ncells, int* start, cudaStream_t s) {
    k_csr_from_sorted<<<nblk(n + 1, 256), 256, 0, s>>>(keys, n, ncells, start);
    fftpim_count_launch();
}

__global__ void k_stencils(const double* __restrict__ pos, const int* __restrict__ perm, int64_t n,
                           StencilGeom g, double* w, int* start, DevStatus* st, int where) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t p = perm ? perm[i] : i;
    const int W = g.order + 1;
    for (int a = 0; a < 3; ++a) {
        double wl[FFTPIM_MAX_W];
        int sa;
        if (!axis_stencil(pos[3 * p + a], g.n[a], g.origin[a], g.h[a], g.order, g.margin[a], &sa, wl))
            set_status(st, FFTPIM_DOMAIN, where, p, a);
        start[3 * i + a] = sa;
        for (int j = 0; j < W; ++j) w[(3 * i + a) * W + j] = (j < g.w[a]) ? wl[j] : 0.0;
    }
}

void launch_stencils(const double* pos, const int* perm, int64_t n, const StencilGeom& g, double* w,
                     int* start, DevStatus* st, int where, cudaStream_t s) {
    if (n == 0) return;
    k_stencils<<<nblk(n, 128), 128, 0, s>>>(pos, perm, n, g, w, start, st, where);
    fftpim_count_launch();
}

__global__ void k_rank(const int* __restrict__ perm, int64_t n, int* rank) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) rank[perm[i]] = (int)i;
}

void launch_rank(const int* perm, int64_t n, int* rank, cudaStream_t s) {
    if (n == 0) return;
    k_rank<<<nblk(n, 256), 256, 0, s>>>(perm, n, rank);
    fftpim_count_launch();
}

__global__ void k_iota(int* p, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = (int)i;
}
void launch_iota(int* p, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    k_iota<<<nblk(n, 256), 256, 0, s>>>(p, n);
    fftpim_count_launch();
}

__global__ void k_fill_u8(unsigned char* p, int64_t n, unsigned char v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
void launch_fill_u8(unsigned char* p, int64_t n, unsigned char v, cudaStream_t s) {
    if (n == 0) return;
    k_fill_u8<<<nblk(n, 256), 256, 0, s>>>(p, n, v);
    fftpim_count_launch();
}

// ---------------------------------------------------------------------------
// near kernel table, embedded for the zero-padded circulant (nearzone.py:127-147)
// ---------------------------------------------------------------------------
// slot e of a doubled axis -> displacement index; false for the zero slot n
__device__ __forceinline__ bool embed_disp(int e, int n, int* idx) {
    if (n == 1) {
        *idx = 0;
        return true;
    }
    if (e < n) {
        *idx = e;
        return true;
    }
    if (e == n) return false;
    *idx = e - 2 * n;
    return true;
}

__global__ void k_embed_table(cplx* out, int c0, int c1, int c2, int n0, int n1, int n2, double h0,
                              double h1, double h2, ImageSet im) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t total = (int64_t)c0 * c1 * c2;
    if (t >= total) return;
    int ez = (int)(t % c2), ey = (int)((t / c2) % c1), ex = (int)(t / ((int64_t)c1 * c2));
    int ix, iy, iz;
    cplx v = mk(0.0);
    if (embed_disp(ex, n0, &ix) && embed_disp(ey, n1, &iy) && embed_disp(ez, n2, &iz) &&
        !(ix == 0 && iy == 0 && iz == 0)) {   // centre zeroed (nearzone.py:229-230)
        bool bad = false;
        v = image_sum(im, (double)ix * h0, (double)iy * h1, (double)iz * h2, im.sing_tol, true, &bad);
    }
    out[t] = v;
}

void launch_embed_table(cplx* out, const int cdims[3], const int dims[3], const double h[3],
                        const ImageSet& im, cudaStream_t s) {
    int64_t total = (int64_t)cdims[0] * cdims[1] * cdims[2];
    k_embed_table<<<nblk(total, 128), 128, 0, s>>>(out, cdims[0], cdims[1], cdims[2], dims[0], dims[1],
                                                   dims[2], h[0], h[1], h[2], im);
    fftpim_count_launch();
}

// nearzone.py:281-287 -- image terms zeroed during tabulation (|d - off|^2 <= tol^2)
__global__ void k_count_coincident(int m0, int m1, int m2, int n0, int n1, int n2, double h0, double h1,
                                   double h2, ImageSet im, unsigned long long* cnt) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t total = (int64_t)m0 * m1 * m2;
    unsigned long long local = 0;
    if (t < total) {
        int iz = (int)(t % m2), iy = (int)((t / m2) % m1), ix = (int)(t / ((int64_t)m1 * m2));
        double px = (double)(ix - (n0 - 1 > 0 ? n0 - 1 : 0)) * h0;
        double py = (double)(iy - (n1 - 1 > 0 ? n1 - 1 : 0)) * h1;
        double pz = (double)(iz - (n2 - 1 > 0 ? n2 - 1 : 0)) * h2;
        double tol2 = im.sing_tol * im.sing_tol;
        for (int i = 0; i < im.count; ++i) {
            double dx = px - im.off[i][0], dy = py - im.off[i][1], dz = pz - im.off[i][2];
            if (dot3(dx, dy, dz) <= tol2) ++local;
        }
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(cnt, local);
}

void launch_count_coincident(const int dims[3], const double h[3], const ImageSet& im,
                             unsigned long long* cnt, cudaStream_t s) {
    int m[3];
    for (int a = 0; a < 3; ++a) m[a] = dims[a] > 1 ? 2 * dims[a] - 1 : 1;
    int64_t total = (int64_t)m[0] * m[1] * m[2];
    k_count_coincident<<<nblk(total, 256), 256, 0, s>>>(m[0], m[1], m[2], dims[0], dims[1], dims[2], h[0],
                                                        h[1], h[2], im, cnt);
    fftpim_count_launch();
}

__global__ void k_scale(cplx* a, int64_t n, double f) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = a[i] * f;
}
void launch_scale(cplx* a, int64_t n, double f, cudaStream_t s) {
    k_scale<<<nblk(n, 256), 256, 0, s>>>(a, n, f);
    fftpim_count_launch();
}

// ---------------------------------------------------------------------------
// wrapped source copies and source boxes (nearzone.py:310-352)
// ---------------------------------------------------------------------------
__global__ void k_wrap_flags(const double* __restrict__ pos, int64_t n, int c0, int c1, int c2, double lo0,
                             double lo1, double lo2, double hi0, double hi1, double hi2,
                             unsigned char* flags) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c[3] = {c0, c1, c2};
    const double lo[3] = {lo0, lo1, lo2}, hi[3] = {hi0, hi1, hi2};
    bool keep = true;
    for (int a = 0; a < 3; ++a) {
        double x = pos[3 * i + a];
        if (c[a] < 0) keep = keep && (x >= lo[a]);
        if (c[a] > 0) keep = keep && (x <= hi[a]);
    }
    flags[i] = keep ? 1 : 0;
}

void launch_wrap_flags(const double* pos, int64_t n, const int code[3], const double lo[3],
                       const double hi[3], unsigned char* flags, cudaStream_t s) {
    if (n == 0) return;
    k_wrap_flags<<<nblk(n, 256), 256, 0, s>>>(pos, n, code[0], code[1], code[2], lo[0], lo[1], lo[2], hi[0],
                                              hi[1], hi[2], flags);
    fftpim_count_launch();
}

__global__ void k_aug_keys(const double* __restrict__ pos, const int* __restrict__ aug_orig,
                           const unsigned char* __restrict__ aug_code, int64_t A, PairGeom pg, int* keys) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= A) return;
    int o = aug_orig[k], c = aug_code[k];
    int b[3];
    for (int a = 0; a < 3; ++a) {
        double x = __dadd_rn(pos[3 * (int64_t)o + a], pg.shift[c][a]);
        b[a] = box_id(x, pg.h[a], pg.nb[a], pg.max_pad, pg.dims[a] > 1);
    }
    keys[k] = (b[0] * pg.ext[1] + b[1]) * pg.ext[2] + b[2];
}

void launch_aug_keys(const double* pos, const int* aug_orig, const unsigned char* aug_code, int64_t A,
                     const PairGeom& pg, int* keys, cudaStream_t s) {
    if (A == 0) return;
    k_aug_keys<<<nblk(A, 256), 256, 0, s>>>(pos, aug_orig, aug_code, A, pg, keys);
    fftpim_count_launch();
}

// ---------------------------------------------------------------------------
// correction pairs: one warp per observer (sorted order).  Candidates come from
// contiguous box ranges (x, y offsets outer, the z run of boxes contiguous in
// the sorted source list), visited in the reference's order (nearzone.py:374-393
// + the stable sort by observer at :465-478), so the per-observer pair order
// equals the reference's.
// ---------------------------------------------------------------------------
struct Cand {
    bool keep;
    int orig;
    int code;
    double d[3];
};

__device__ __forceinline__ Cand candidate(const PairGeom& pg, const PairArgs& a, int k, double ox, double oy,
                                          double oz) {
    Cand c;
    int aug = a.box_order[k];
    c.orig = a.aug_orig[aug];
    c.code = a.aug_code[aug];
    const double* sp = a.src_pos + 3 * (int64_t)c.orig;
    double o[3] = {ox, oy, oz};
    double e[3];
    for (int ax = 0; ax < 3; ++ax) {
        double xa = __dadd_rn(sp[ax], pg.shift[c.code][ax]);
        c.d[ax] = __dsub_rn(o[ax], xa);
        e[ax] = __dmul_rn(c.d[ax], pg.inv_h[ax]);
    }
    c.keep = dot3(e[0], e[1], e[2]) <= pg.r2_keep;       // nearzone.py:364, 396
    return c;
}

__global__ void __launch_bounds__(256) k_pairs_count(PairGeom pg, PairArgs a) {
    __shared__ int smin[27 * 3], smax[27 * 3];
    __shared__ unsigned long long s_self, s_wrap;
    for (int t = threadIdx.x; t < 81; t += blockDim.x) {
        smin[t] = INT_MAX;
        smax[t] = INT_MIN;
    }
    if (threadIdx.x == 0) s_self = s_wrap = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    unsigned long long my_self = 0, my_wrap = 0;
    if (i < a.M) {
        const int m = a.obs_perm[i];
        const double ox = a.obs_pos[3 * (int64_t)m], oy = a.obs_pos[3 * (int64_t)m + 1],
                     oz = a.obs_pos[3 * (int64_t)m + 2];
        int ob[3];
        const double o3[3] = {ox, oy, oz};
        for (int ax = 0; ax < 3; ++ax) ob[ax] = box_id(o3[ax], pg.h[ax], pg.nb[ax], pg.max_pad, pg.dims[ax] > 1);
        const int so[3] = {a.obs_start[3 * i], a.obs_start[3 * i + 1], a.obs_start[3 * i + 2]};
        int count = 0;
        const double tol2 = pg.sing_tol * pg.sing_tol;
        for (int dx = -pg.jr[0]; dx <= pg.jr[0]; ++dx) {
            int tx = ob[0] + dx;
            if (tx < 0 || tx >= pg.ext[0]) continue;
            for (int dy = -pg.jr[1]; dy <= pg.jr[1]; ++dy) {
                int ty = ob[1] + dy;
                if (ty < 0 || ty >= pg.ext[1]) continue;
                int zlo = max(ob[2] - pg.jr[2], 0), zhi = min(ob[2] + pg.jr[2], pg.ext[2] - 1);
                if (zlo > zhi) continue;
                int f0 = (tx * pg.ext[1] + ty) * pg.ext[2];
                int c0 = a.box_start[f0 + zlo], c1 = a.box_start[f0 + zhi + 1];
                for (int base = c0; base < c1; base += 32) {
                    int k = base + lane;
                    bool keep = false;
                    Cand c;
                    if (k < c1) {
                        c = candidate(pg, a, k, ox, oy, oz);
                        keep = c.keep;
                    }
                    unsigned mask = __ballot_sync(0xffffffffu, keep);
                    count += __popc(mask);
                    if (keep) {
                        bool self = pg.same_points && c.orig == m && c.code == 0;
                        my_self += self;
                        my_wrap += (c.code != 0);
                        if (!self && dot3(c.d[0], c.d[1], c.d[2]) <= tol2)
                            set_status(a.st, FFTPIM_DOMAIN, 30, m, c.orig);   // nearzone.py:405-416
                        int r = a.src_rank[c.orig];
                        for (int ax = 0; ax < 3; ++ax) {
                            int d0 = so[ax] - a.src_start[3 * (int64_t)r + ax] - (a.wdt[ax] - 1);
                            atomicMin(&smin[c.code * 3 + ax], d0);
                            atomicMax(&smax[c.code * 3 + ax], d0);
                        }
                    }
                }
            }
        }
        if (lane == 0) a.counts[i] = (int64_t)count;
    }
    for (int o = 16; o > 0; o >>= 1) {
        my_self += __shfl_down_sync(0xffffffffu, my_self, o);
        my_wrap += __shfl_down_sync(0xffffffffu, my_wrap, o);
    }
    if (lane == 0) {
        if (my_self) atomicAdd(&s_self, my_self);
        if (my_wrap) atomicAdd(&s_wrap, my_wrap);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 81; t += blockDim.x) {
        if (smin[t] != INT_MAX) atomicMin(&a.d0min[t], smin[t]);
        if (smax[t] != INT_MIN) atomicMax(&a.d0max[t], smax[t]);
    }
    if (threadIdx.x == 0) {
        if (s_self) atomicAdd(&a.tallies[0], s_self);
        if (s_wrap) atomicAdd(&a.tallies[1], s_wrap);
    }
}

void launch_pairs_count(const PairGeom& pg, const PairArgs& a, cudaStream_t s) {
    if (a.M == 0) return;
    k_pairs_count<<<nblk(a.M * 32, 256), 256, 0, s>>>(pg, a);
    fftpim_count_launch();
}

// coefficient of one kept pair (nearzone.py:405-457)
__device__ cplx pair_coefficient(const PairGeom& pg, const ImageSet& im, const CodeTables& tabs,
                                 const PairArgs& a, int64_t i, int m, const Cand& c, bool* bad) {
    const bool self = pg.same_points && c.orig == m && c.code == 0;
    cplx direct = mk(0.0);
    if (!self) direct = image_sum(im, c.d[0], c.d[1], c.d[2], pg.sing_tol, false, bad);
    const int r = a.src_rank[c.orig];
    const int W = a.W;
    double C[3][2 * FFTPIM_MAX_W - 1];
    int d0[3];
    for (int ax = 0; ax < 3; ++ax) {
        const int w = a.wdt[ax];
        const double* wo = a.obs_w + (3 * i + ax) * W;
        const double* ws = a.src_w + (3 * (int64_t)r + ax) * W;
        for (int u = 0; u < 2 * w - 1; ++u) C[ax][u] = 0.0;
        for (int p = 0; p < w; ++p)
            for (int q = 0; q < w; ++q) C[ax][p - q + w - 1] += wo[p] * ws[q];   // nearzone.py:150-157
        d0[ax] = a.obs_start[3 * i + ax] - a.src_start[3 * (int64_t)r + ax] - (w - 1) - tabs.lo[c.code][ax];
    }
    const cplx* T = a.tables + tabs.offset[c.code];
    const int ly = tabs.len[c.code][1], lz = tabs.len[c.code][2];
    const int ux = 2 * a.wdt[0] - 1, uy = 2 * a.wdt[1] - 1, uz = 2 * a.wdt[2] - 1;
    cplx g = mk(0.0);
    for (int u = 0; u < ux; ++u) {
        cplx gy = mk(0.0);
        for (int v = 0; v < uy; ++v) {
            const cplx* row = T + ((int64_t)(d0[0] + u) * ly + (d0[1] + v)) * lz + d0[2];
            cplx gz = mk(0.0);
            for (int w = 0; w < uz; ++w) gz = gz + C[2][w] * row[w];
            gy = gy + C[1][v] * gz;
        }
        g = g + C[0][u] * gy;
    }
    return cplx{pg.phase_re[c.code], pg.phase_im[c.code]} * (direct - g);   // nearzone.py:456-457
}

__global__ void __launch_bounds__(128) k_pairs_fill(PairGeom pg, ImageSet im, CodeTables tabs, PairArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (i >= a.M) return;
    const int m = a.obs_perm[i];
    const double ox = a.obs_pos[3 * (int64_t)m], oy = a.obs_pos[3 * (int64_t)m + 1],
                 oz = a.obs_pos[3 * (int64_t)m + 2];
    const double o3[3] = {ox, oy, oz};
    int ob[3];
    for (int ax = 0; ax < 3; ++ax) ob[ax] = box_id(o3[ax], pg.h[ax], pg.nb[ax], pg.max_pad, pg.dims[ax] > 1);
    int64_t out = a.pair_ptr[i];
    bool bad = false;
    for (int dx = -pg.jr[0]; dx <= pg.jr[0]; ++dx) {
        int tx = ob[0] + dx;
        if (tx < 0 || tx >= pg.ext[0]) continue;
        for (int dy = -pg.jr[1]; dy <= pg.jr[1]; ++dy) {
            int ty = ob[1] + dy;
            if (ty < 0 || ty >= pg.ext[1]) continue;
            int zlo = max(ob[2] - pg.jr[2], 0), zhi = min(ob[2] + pg.jr[2], pg.ext[2] - 1);
            if (zlo > zhi) continue;
            int f0 = (tx * pg.ext[1] + ty) * pg.ext[2];
            int c0 = a.box_start[f0 + zlo], c1 = a.box_start[f0 + zhi + 1];
            for (int base = c0; base < c1; base += 32) {
                int k = base + lane;
                bool keep = false;
                Cand c;
                if (k < c1) {
                    c = candidate(pg, a, k, ox, oy, oz);
                    keep = c.keep;
                }
                unsigned mask = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    int64_t slot = out + __popc(mask & ((1u << lane) - 1u));
                    cplx v = pair_coefficient(pg, im, tabs, a, i, m, c, &bad);
                    a.pair_src[slot] = a.src_rank[c.orig];
                    if (a.pair_codeid) a.pair_codeid[slot] = (unsigned char)c.code;
                    if (a.coef_r)
                        a.coef_r[slot] = v.re;
                    else
                        a.coef[slot] = v;
                }
                out += __popc(mask);
            }
        }
    }
    if (bad) set_status(a.st, FFTPIM_DOMAIN, 31, m, -1);
}

void launch_pairs_fill(const PairGeom& pg, const ImageSet& im, const CodeTables& tabs, const PairArgs& a,
                       cudaStream_t s) {
    if (a.M == 0) return;
    k_pairs_fill<<<nblk(a.M * 32, 128), 128, 0, s>>>(pg, im, tabs, a);
    fftpim_count_launch();
}

// per-code window tables of G_near(idx*h - c*L), centre zeroed for c = 0
// (nearzone.py:229-230 for the main table, :439-451 for the displaced ones)
__global__ void k_code_tables(CodeTables tabs, int ncodes, PairGeom pg, ImageSet im, cplx* tables,
                              int64_t total) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= total) return;
    int c = 0;
    while (c + 1 < ncodes && t >= tabs.offset[c + 1]) ++c;
    int64_t l = t - tabs.offset[c];
    const int lx = tabs.len[c][0], ly = tabs.len[c][1], lz = tabs.len[c][2];
    if (lx == 0) return;
    int iz = (int)(l % lz), iy = (int)((l / lz) % ly), ix = (int)(l / ((int64_t)ly * lz));
    int idx[3] = {ix + tabs.lo[c][0], iy + tabs.lo[c][1], iz + tabs.lo[c][2]};
    cplx v = mk(0.0);
    if (!(c == 0 && idx[0] == 0 && idx[1] == 0 && idx[2] == 0)) {
        double p[3];
        for (int a = 0; a < 3; ++a) p[a] = __dsub_rn((double)idx[a] * pg.h[a], pg.shift[c][a]);
        bool bad = false;
        v = image_sum(im, p[0], p[1], p[2], im.sing_tol, true, &bad);
    }
    tables[t] = v;
}

void launch_code_tables(const CodeTables& tabs, int ncodes, const PairGeom& pg, const ImageSet& im,
                        cplx* tables, int64_t total, cudaStream_t s) {
    if (total == 0) return;
    k_code_tables<<<nblk(total, 128), 128, 0, s>>>(tabs, ncodes, pg, im, tables, total);
    fftpim_count_launch();
}

// ---------------------------------------------------------------------------
// far kernel: G_total - G_near(i_d) per difference point, one thread per point,
// layer-by-layer with the reference's stopping rule (pgf.py:166-195)
// ---------------------------------------------------------------------------
#include "series.cuh"

__global__ void k_far_series(const double* __restrict__ axes, int kd0, int kd1, int kd2, FarSeriesParams fp,
                             ImageSet im, GLTable gl, cplx* out, DevStatus* st) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t total = (int64_t)kd0 * kd1 * kd2;
    if (t >= total) return;
    int iz = (int)(t % kd2), iy = (int)((t / kd2) % kd1), ix = (int)(t / ((int64_t)kd1 * kd2));
    double x = axes[ix], y = axes[kd0 + iy], z = axes[kd0 + kd1 + iz];
    Drive d = fp.npsp ? lattice_series(fp, gl, x, y, z, fp.zmin, fp.zmax, st, t) : spectral_series(fp, gl, x, y, z, st, t);
    if (!d.done) set_status(st, FFTPIM_NOT_CONVERGED, 47, t, d.terms);   // farzone.py:115-119
    bool bad = false;
    cplx near = image_sum(im, x, y, z, im.sep_tol, false, &bad);     // pgf.py:461 (no drop)
    if (bad) set_status(st, FFTPIM_DOMAIN, 48, t, 0);
    out[t] = d.total - near;
    atomicMax(&st->kernel_terms, (int)(d.terms > 2147483647LL ? 2147483647LL : d.terms));
}

void launch_far_series(const double* axes, const int kd[3], const FarSeriesParams& fp, const ImageSet& im,
                       const GLTable& gl, cplx* out, DevStatus* st, cudaStream_t s) {
    int64_t total = (int64_t)kd[0] * kd[1] * kd[2];
    k_far_series<<<nblk(total, 64), 64, 0, s>>>(axes, kd[0], kd[1], kd[2], fp, im, gl, out, st);
    fftpim_count_launch();
}
