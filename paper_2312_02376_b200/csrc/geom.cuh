// geom.cuh -- device helpers shared by the plan-build and evaluation kernels:
// Lagrange stencils, padded box ids and the truncated image sum G_near.
// Discrete decisions (stencil starts, box ids, the pair-keep test) use
// explicitly rounded operations (no FMA contraction) so they reproduce the
// reference's numpy arithmetic bit for bit.
#pragma once
#include "plan.cuh"

#define FOUR_PI_D (4.0 * M_PI)

// grids.py:110-140 -- start = rint(t - q/2) clipped to [0, n-1-q]; w_j =
// prod_{i!=j} (rel - i) / prod_{i!=j} (j - i).  Returns false outside the hull.
__device__ __forceinline__ bool axis_stencil(double x, int n, double origin, double h, int order,
                                             double margin, int* start, double* w) {
    if (n == 1) {
        *start = 0;
        w[0] = 1.0;
        return true;
    }
    double t = __ddiv_rn(__dsub_rn(x, origin), h);
    double slack = __dadd_rn(__ddiv_rn(margin, h), 1e-9);
    bool ok = !(t < -slack) && !(t > __dadd_rn((double)(n - 1), slack));
    double s = rint(__dsub_rn(t, order / 2.0));
    int si = (int)s;
    if (si < 0) si = 0;
    if (si > n - 1 - order) si = n - 1 - order;
    *start = si;
    double rel = __dsub_rn(t, (double)si);
    for (int j = 0; j <= order; ++j) {
        double num = 1.0, den = 1.0;
        for (int i = 0; i <= order; ++i) {
            if (i == j) continue;
            num = __dmul_rn(num, __dsub_rn(rel, (double)i));
            den = den * (double)(j - i);
        }
        w[j] = __ddiv_rn(num, den);
    }
    return ok;
}

// flat cell key of a stencil start triple
__device__ __forceinline__ int cell_key(const StencilGeom& g, int sx, int sy, int sz) {
    return (sx * g.nc[1] + sy) * g.nc[2] + sz;
}

// nearzone.py:181-191 -- floor(x/h) clipped to [-pad, nb-1+pad], + pad
__device__ __forceinline__ int box_id(double x, double h, int nb, int pad, int active) {
    if (!active) return 0;
    double f = floor(__ddiv_rn(x, h));
    long long b = (long long)f;
    if (b < -pad) b = -pad;
    if (b > nb - 1 + pad) b = nb - 1 + pad;
    return (int)(b + pad);
}

// sum of squares in numpy einsum order, no FMA
__device__ __forceinline__ double dot3(double a, double b, double c) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c));
}

// pgf.py:126-154 -- sum_i ph_i e^{-j k0 r_i} / (4 pi r_i), r_i = |p - off_i|.
// drop: coincident terms (r <= tol) contribute zero; otherwise they set *bad.
__device__ __forceinline__ cplx image_sum(const ImageSet& im, double px, double py, double pz,
                                          double tol, bool drop, bool* bad) {
    cplx acc = mk(0.0);
    // -1j * k0 = (k0.im, -k0.re)
    const double cre = im.k0_im, cim = -im.k0_re;
    for (int i = 0; i < im.count; ++i) {
        double dx = __dsub_rn(px, im.off[i][0]);
        double dy = __dsub_rn(py, im.off[i][1]);
        double dz = __dsub_rn(pz, im.off[i][2]);
        double r = sqrt(dot3(dx, dy, dz));
        if (r <= tol) {
            if (!drop) *bad = true;
            continue;
        }
        cplx e = cexp_(cplx{cre * r, cim * r});
        cplx t = cplx{im.ph_re[i], im.ph_im[i]} * e;
        acc = acc + t / (FOUR_PI_D * r);
    }
    return acc;
}

__device__ __forceinline__ void set_status(DevStatus* st, int code, int where, long long a,
                                           long long b) {
    if (atomicCAS(&st->code, 0, code) == 0) {
        st->where = where;
        st->a = a;
        st->b = b;
    }
}
