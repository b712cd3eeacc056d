// series.cuh -- the reference's adaptive periodic-Green's-function series on
// the device (pgf.py:166-195 driver, :215-295 spectral, :328-425 lattice),
// one point per thread.  Shared by the far-kernel tabulation (K7,
// build_kernels.cu) and the brute-force direct evaluator (direct_kernels.cu).
#pragma once
#include "geom.cuh"
#include "kernels.h"

struct Drive {
    cplx total;
    long long terms;
    int quiet;
    bool done;
};

__device__ __forceinline__ bool drive_step(Drive& d, cplx layer, long long cnt, const FarSeriesParams& fp) {
    d.total = d.total + layer;
    d.terms += cnt;
    double ref = cabs_(d.total);
    if (!(ref > 1e-300)) ref = 1e-300;
    bool small = cabs_(layer) <= fp.tol * ref;
    d.quiet = small ? d.quiet + 1 : 0;
    if (d.quiet >= fp.consecutive) {
        d.done = true;
        return false;
    }
    return d.terms < fp.max_terms;
}

__device__ inline double log_trig(double y, double a, double ly, bool* bad) {
    // pgf.py:317-325
    double e = exp(-2.0 * M_PI * a / ly);
    double t = 1.0 - 2.0 * e * cos(2.0 * M_PI * y / ly) + e * e;
    if (t <= 0.0) *bad = true;
    return log(t);
}

// zmin, zmax: z extrema over the batch the reference evaluates together (the 3D
// lead's image range, pgf.py:394-397)
__device__ inline Drive lattice_series(const FarSeriesParams& fp, const GLTable& gl, double x, double y, double z,
                                       double zmin, double zmax, DevStatus* st, long long pt) {
    Drive d{mk(0.0), 0, 0, false};
    const double lx = fp.L[0], ly = fp.L[1], lz = fp.L[2], cut = fp.cutoff;
    bool bad = false;
    if (fp.dim == 1) {
        double rho = hypot(y, z);
        if (rho <= fp.sep) {
            set_status(st, FFTPIM_SEPARATION, 40, pt, 0);
            return d;
        }
        d.total = mk(-log(rho) / (2.0 * M_PI * lx));
        d.terms = 1;
        for (int m = 1; m < 200000; ++m) {
            double arg = 2.0 * m * M_PI * rho / lx;
            double v = arg <= cut ? k0_real(arg, gl) : 0.0;
            v = v * (cos(2.0 * m * M_PI * x / lx) / (M_PI * lx));
            if (!drive_step(d, mk(v), 1, fp)) break;
        }
        return d;
    }
    if (fp.dim == 2) {
        double az = fabs(z);
        d.total = mk(-az / (2.0 * lx * ly) - log_trig(y, az, ly, &bad) / (4.0 * M_PI * lx));
        d.terms = 1;
        for (int m = 1; m < 200000; ++m) {
            double smax = cut * lx / (2.0 * M_PI * m);
            long long nlo = (long long)floor((-smax - y) / ly), nhi = (long long)ceil((smax - y) / ly);
            double acc = 0.0;
            long long cnt = 0;
            for (long long n = nlo; n <= nhi; ++n) {
                double t = n * ly + y;
                double s2 = t * t + z * z;
                if (s2 <= fp.sep * fp.sep) bad = true;
                double arg = 2.0 * m * M_PI * sqrt(s2) / lx;
                if (arg <= cut) {
                    acc += k0_real(arg, gl);
                    ++cnt;
                }
            }
            acc = acc * (cos(2.0 * m * M_PI * x / lx) / (M_PI * lx));
            if (!drive_step(d, mk(acc), cnt > 0 ? cnt : 1, fp)) break;
        }
    } else {
        double az = fabs(z);
        double lead = (z * z - az * lz) / (2.0 * lx * ly * lz);
        double reach = cut * ly / (2.0 * M_PI);
        long long klo = (long long)floor((-reach - zmax) / lz), khi = (long long)ceil((reach - zmin) / lz);
        for (long long k = klo; k <= khi; ++k) lead = lead - log_trig(y, fabs(k * lz + z), ly, &bad) / (4.0 * M_PI * lx);
        d.total = mk(lead);
        d.terms = 1;
        for (int m = 1; m < 200000; ++m) {
            double smax = cut * lx / (2.0 * M_PI * m);
            long long nlo = (long long)floor((-smax - y) / ly), nhi = (long long)ceil((smax - y) / ly);
            long long zlo = (long long)floor((-smax - z) / lz), zhi = (long long)ceil((smax - z) / lz);
            double acc = 0.0;
            long long cnt = 0;
            for (long long n = nlo; n <= nhi; ++n) {
                double t = n * ly + y;
                double uy = t * t;
                for (long long k = zlo; k <= zhi; ++k) {
                    double tz = k * lz + z;
                    double s2 = uy + tz * tz;
                    if (s2 <= fp.sep * fp.sep) bad = true;
                    double arg = 2.0 * m * M_PI * sqrt(s2) / lx;
                    if (arg <= cut) {
                        acc += k0_real(arg, gl);
                        ++cnt;
                    }
                }
            }
            acc = acc * (cos(2.0 * m * M_PI * x / lx) / (M_PI * lx));
            if (!drive_step(d, mk(acc), cnt > 0 ? cnt : 1, fp)) break;
        }
    }
    if (bad) set_status(st, FFTPIM_DOMAIN, 41, pt, 0);
    return d;
}

__device__ inline Drive spectral_series(const FarSeriesParams& fp, const GLTable& gl, double x, double y, double z,
                                 DevStatus* st, long long pt) {
    Drive d{mk(0.0), 0, 0, false};
    const double lx = fp.L[0], ly = fp.L[1], lz = fp.L[2];
    const cplx k0{fp.k0_re, fp.k0_im};
    const cplx k0sq = k0 * k0;
    const cplx kx0{fp.ks_re[0], fp.ks_im[0]}, ky0{fp.ks_re[1], fp.ks_im[1]}, kz0{fp.ks_re[2], fp.ks_im[2]};
    if (fp.dim == 1) {
        double rho = hypot(y, z);
        if (rho <= fp.sep) {
            set_status(st, FFTPIM_SEPARATION, 42, pt, 0);
            return d;
        }
        for (int s = 0; s < 200000; ++s) {
            cplx acc = mk(0.0);
            int nm = s == 0 ? 1 : 2;
            for (int t = 0; t < nm; ++t) {
                int m = t == 0 ? s : -s;
                cplx km = kx0 + mk(2.0 * M_PI * m / lx);
                cplx kr = csqrt_lower(k0sq - km * km);
                if (cabs_(kr) < fp.wood) {
                    set_status(st, FFTPIM_WOOD_ANOMALY, 43, m, 0);
                    return d;
                }
                cplx h = h0c(kr * rho, gl);
                cplx e = cexp_mj(km * x);
                acc = acc + (e * h) / cplx{0.0, 4.0 * lx};
            }
            if (!drive_step(d, acc, nm, fp)) break;
        }
        return d;
    }
    const bool three = fp.dim == 3;
    const double az = fabs(z);
    for (int s = 0; s < 200000; ++s) {
        cplx acc = mk(0.0);
        int cnt = s == 0 ? 1 : 8 * s;
        for (int t = 0; t < cnt; ++t) {
            int m, n;   // shell order of pgf.py:202-212
            if (s == 0) {
                m = 0;
                n = 0;
            } else if (t < 2 * (2 * s + 1)) {
                m = -s + t / 2;
                n = (t & 1) ? -s : s;
            } else {
                int r = t - 2 * (2 * s + 1);
                m = (r & 1) ? -s : s;
                n = -s + 1 + r / 2;
            }
            cplx kx = kx0 + mk(2.0 * M_PI * m / lx);
            cplx ky = ky0 + mk(2.0 * M_PI * n / ly);
            cplx kz = csqrt_lower(k0sq - kx * kx - ky * ky);
            if (cabs_(kz) < fp.wood) {
                set_status(st, FFTPIM_WOOD_ANOMALY, 44, m, n);
                return d;
            }
            cplx f = cexp_mj(kz * az);
            if (three) {
                cplx ea = cexp_mj((kz - kz0) * lz), eb = cexp_mj((kz + kz0) * lz);
                if (fmax(cabs_(ea), cabs_(eb)) > 1.0 + 1e-12) {
                    set_status(st, FFTPIM_NOT_CONVERGED, 45, m, n);
                    return d;
                }
                cplx one = mk(1.0);
                if (fmin(cabs_(one - ea), cabs_(one - eb)) < 1e-8) {
                    set_status(st, FFTPIM_WOOD_ANOMALY, 46, m, n);
                    return d;
                }
                cplx ca = ea / (one - ea), cb = eb / (one - eb);
                f = f + ca * cexp_mj(kz * z) + cb * cexp_mj(-(kz * z));
            }
            cplx ph = cexp_mj(kx * x + ky * y);
            acc = acc + ph * f / ((cplx{0.0, 2.0} * kz) * lx * ly);
        }
        if (!drive_step(d, acc, cnt, fp)) break;
    }
    return d;
}

