// cmath.cuh -- fp64 complex arithmetic and the special functions the FFT-PIM
// plan build needs on device: the Im<=0 square root, K0 and H0^(2).
//
// Algorithms follow the reference's in-repo special functions
// (/root/reference/pkg/src/perisum/special.py:40-203) regime by regime, so the
// far-kernel series truncates after the same layers (hard part 4);
// values agree to ~1e-13 relative, not bit-for-bit.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#define FP_HD __host__ __device__ __forceinline__

struct __align__(16) cplx {   // 16-byte aligned: one 128-bit load or store per value
    double re, im;
};

FP_HD cplx mk(double r, double i = 0.0) { return cplx{r, i}; }
FP_HD cplx operator+(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }
FP_HD cplx operator-(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }
FP_HD cplx operator-(cplx a) { return cplx{-a.re, -a.im}; }
FP_HD cplx operator*(cplx a, cplx b) {
    return cplx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
FP_HD cplx operator*(cplx a, double s) { return cplx{a.re * s, a.im * s}; }
FP_HD cplx operator*(double s, cplx a) { return cplx{a.re * s, a.im * s}; }
FP_HD cplx operator/(cplx a, double s) { return cplx{a.re / s, a.im / s}; }
FP_HD double cabs_(cplx a) { return hypot(a.re, a.im); }
// Smith's algorithm (numpy's complex division is also scaled)
FP_HD cplx operator/(cplx a, cplx b) {
    if (fabs(b.re) >= fabs(b.im)) {
        if (b.re == 0.0 && b.im == 0.0) return cplx{a.re / 0.0, a.im / 0.0};
        double r = b.im / b.re, den = b.re + b.im * r;
        return cplx{(a.re + a.im * r) / den, (a.im - a.re * r) / den};
    }
    double r = b.re / b.im, den = b.re * r + b.im;
    return cplx{(a.re * r + a.im) / den, (a.im * r - a.re) / den};
}
FP_HD cplx operator/(double s, cplx b) { return cplx{s, 0.0} / b; }
FP_HD cplx cexp_(cplx a) {
    double e = exp(a.re), s, c;
    sincos(a.im, &s, &c);
    return cplx{e * c, e * s};
}
// exp(-j * a) for complex a
FP_HD cplx cexp_mj(cplx a) { return cexp_(cplx{a.im, -a.re}); }
FP_HD cplx clog_(cplx a) { return cplx{log(cabs_(a)), atan2(a.im, a.re)}; }
// principal square root (branch cut on the negative real axis, Re >= 0)
FP_HD cplx csqrt_(cplx z) {
    if (z.re == 0.0 && z.im == 0.0) return cplx{0.0, z.im};
    double m = cabs_(z);
    if (z.re >= 0.0) {
        double t = sqrt(0.5 * (m + z.re));
        return cplx{t, z.im / (2.0 * t)};
    }
    double t = sqrt(0.5 * (m - z.re));
    return cplx{fabs(z.im) / (2.0 * t), copysign(t, z.im)};
}
// w*w = z with Im w <= 0 (special.py:40-50)
FP_HD cplx csqrt_lower(cplx z) {
    cplx w = csqrt_(z);
    if (w.im > 0.0) w = -w;
    return w;
}

#define EULER_GAMMA_D 0.5772156649015328606065121
#define FFTPIM_GL_N 64

struct GLTable {
    double node[FFTPIM_GL_N];
    double weight[FFTPIM_GL_N];
};

// ---------------- K0 on Re w >= 0 (special.py:66-124) ----------------------
FP_HD double k0_real_small(double w) {
    double q = 0.25 * (w * w), t = 1.0, i0 = 1.0, acc = 0.0, h = 0.0;
    for (int k = 1; k < 20; ++k) {
        t = t * q / (double)(k * k);
        i0 = i0 + t;
        h += 1.0 / k;
        acc = acc + h * t;
    }
    return acc - (log(0.5 * w) + EULER_GAMMA_D) * i0;
}
FP_HD double k0_real_mid(double w, const GLTable& gl) {
    double acc = 0.0;
    for (int i = 0; i < FFTPIM_GL_N; ++i) acc = acc + gl.weight[i] / sqrt(gl.node[i] + 2.0 * w);
    return exp(-w) * acc;
}
FP_HD double k0_real_large(double w) {
    double t = 1.0, acc = 1.0;
    for (int k = 0; k < 30; ++k) {
        t = t * (-((double)((2 * k + 1) * (2 * k + 1))) / (8.0 * (k + 1))) / w;
        acc = acc + t;
        if (fabs(t) < 1e-18) break;
    }
    return exp(-w) * (sqrt(M_PI / (2.0 * w)) * acc);
}
FP_HD double k0_real(double w, const GLTable& gl) {
    double r = fabs(w);
    if (r <= 2.0) return k0_real_small(w);
    if (r > 16.0) return k0_real_large(w);
    return k0_real_mid(w, gl);
}

FP_HD cplx k0_small(cplx w) {
    cplx q = 0.25 * (w * w), t = mk(1.0), i0 = mk(1.0), acc = mk(0.0);
    double h = 0.0;
    for (int k = 1; k < 20; ++k) {
        t = t * q / (double)(k * k);
        i0 = i0 + t;
        h += 1.0 / k;
        acc = acc + h * t;
    }
    cplx lg = clog_(0.5 * w);
    lg.re += EULER_GAMMA_D;
    return acc - lg * i0;
}
FP_HD cplx k0_mid(cplx w, const GLTable& gl) {
    cplx acc = mk(0.0);
    for (int i = 0; i < FFTPIM_GL_N; ++i) {
        cplx s = csqrt_(cplx{gl.node[i] + 2.0 * w.re, 2.0 * w.im});
        acc = acc + gl.weight[i] / s;
    }
    return cexp_(-w) * acc;
}
FP_HD cplx k0_large(cplx w) {
    cplx t = mk(1.0), acc = mk(1.0);
    for (int k = 0; k < 30; ++k) {
        t = t * (-((double)((2 * k + 1) * (2 * k + 1))) / (8.0 * (k + 1))) / w;
        acc = acc + t;
        if (cabs_(t) < 1e-18) break;
    }
    return cexp_(-w) * (csqrt_(M_PI / (2.0 * w)) * acc);
}
FP_HD cplx k0c(cplx w, const GLTable& gl) {
    double r = cabs_(w);
    if (r <= 2.0) return k0_small(w);
    if (r > 16.0) return k0_large(w);
    return k0_mid(w, gl);
}

// ---------------- H0^(2) (special.py:140-203) -------------------------------
FP_HD cplx h0_small(cplx z) {
    cplx mq = -0.25 * (z * z), t = mk(1.0), j0 = mk(1.0), acc = mk(0.0);
    double h = 0.0;
    for (int k = 1; k < 40; ++k) {
        t = t * mq / (double)(k * k);
        j0 = j0 + t;
        h += 1.0 / k;
        acc = acc - h * t;
    }
    cplx lg = clog_(0.5 * z);
    lg.re += EULER_GAMMA_D;
    cplx y0 = (2.0 / M_PI) * (lg * j0 + acc);
    return cplx{j0.re + y0.im, j0.im - y0.re};  // j0 - 1j*y0
}
FP_HD cplx h0_large(cplx z) {
    cplx t = mk(1.0), acc = mk(1.0);
    double last = INFINITY;
    for (int k = 0; k < 40; ++k) {
        t = t * cplx{0.0, (double)((2 * k + 1) * (2 * k + 1)) / (8.0 * (k + 1))} / z;
        double m = cabs_(t);
        if (!(m < last)) break;
        acc = acc + t;
        last = m;
    }
    cplx pre = csqrt_(2.0 / (M_PI * z));
    return pre * cexp_mj(cplx{z.re - 0.25 * M_PI, z.im}) * acc;
}
FP_HD cplx h0c(cplx z, const GLTable& gl) {
    double r = cabs_(z);
    bool lower = z.im <= 0.0;
    if (r <= 4.0 || (!lower && r <= 8.0)) return h0_small(z);
    if (lower) return cplx{0.0, 2.0 / M_PI} * k0c(cplx{-z.im, z.re}, gl);  // (2j/pi) K0(jz)
    return h0_large(z);
}
