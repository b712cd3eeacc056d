// fftpim.cu -- C ABI (include/fftpim.h): plan build orchestration on device,
// evaluation, operand export.  The host code here only sets up scalars and
// launches kernels; every O(N) or O(pairs) step runs on the GPU.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <climits>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "kernels.h"

namespace {

// NVTX ranges (FFTPIM_NVTX=1) around the C-ABI calls and the plan-build phases, for
// nsys / ncu --nvtx timelines.  Header-only NVTX3: a no-op without a tool attached.
struct NvtxRange {
    bool on;
    explicit NvtxRange(const char* name) {
        static const bool enabled = [] {
            const char* e = getenv("FFTPIM_NVTX");
            return e && e[0] == '1';
        }();
        on = enabled;
        if (on) nvtxRangePushA(name);
    }
    ~NvtxRange() {
        if (on) nvtxRangePop();
    }
    void next(const char* name) {   // close the current phase, open the next
        if (on) {
            nvtxRangePop();
            nvtxRangePushA(name);
        }
    }
};

thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};

struct Fail {
    int code;
    std::string msg;
};

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess)                                                                     \
            throw Fail{FFTPIM_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)};              \
    } while (0)
#define CKFFT(x)                                                                                   \
    do {                                                                                           \
        cufftResult r_ = (x);                                                                      \
        if (r_ != CUFFT_SUCCESS) throw Fail{FFTPIM_CUDA, std::string(#x) + ": cufft error " + std::to_string((int)r_)}; \
    } while (0)

template <typename T>
T* dalloc(FftpimPlan* P, int64_t count) {
    if (count <= 0) count = 1;
    void* p = nullptr;
    CK(cudaMalloc(&p, sizeof(T) * (size_t)count));
    P->allocations.push_back(p);
    P->device_bytes += (int64_t)(sizeof(T) * (size_t)count);
    return (T*)p;
}

void dfree(FftpimPlan* P, void* p) {
    if (!p) return;
    auto it = std::find(P->allocations.begin(), P->allocations.end(), p);
    if (it != P->allocations.end()) P->allocations.erase(it);
    cudaFree(p);
}

// Golub-Welsch for the generalized Gauss-Laguerre rule with weight v^-1/2 e^-v
// (special.py:53-63): eigen-decomposition of the symmetric tridiagonal Jacobi
// matrix by implicit QL, tracking only the first eigenvector components.
GLTable gauss_laguerre_half() {
    const int n = FFTPIM_GL_N;
    std::vector<double> d(n), e(n, 0.0), z(n, 0.0);
    for (int k = 0; k < n; ++k) d[k] = 2.0 * k + 0.5;
    for (int k = 1; k < n; ++k) e[k - 1] = std::sqrt(k * (k - 0.5));
    z[0] = 1.0;   // first row of the eigenvector matrix, rotated along
    for (int l = 0; l < n; ++l) {
        int iter = 0;
        while (true) {
            int m = l;
            for (; m < n - 1; ++m) {
                double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
                if (std::fabs(e[m]) <= 1e-17 * dd) break;
            }
            if (m == l) break;
            if (++iter > 200) break;
            double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
            double r = std::hypot(g, 1.0);
            g = d[m] - d[l] + e[l] / (g + (g >= 0 ? std::fabs(r) : -std::fabs(r)));
            double s = 1.0, c = 1.0, p = 0.0;
            int i = m - 1;
            for (; i >= l; --i) {
                double f = s * e[i], b = c * e[i];
                r = std::hypot(f, g);
                e[i + 1] = r;
                if (r == 0.0) {
                    d[i + 1] -= p;
                    e[m] = 0.0;
                    break;
                }
                s = f / r;
                c = g / r;
                g = d[i + 1] - p;
                r = (d[i] - g) * s + 2.0 * c * b;
                p = s * r;
                d[i + 1] = g + p;
                g = c * r - b;
                double fz = z[i + 1];
                z[i + 1] = s * z[i] + c * fz;
                z[i] = c * z[i] - s * fz;
            }
            if (r == 0.0 && i >= l) continue;
            d[l] -= p;
            e[l] = g;
            e[m] = 0.0;
        }
    }
    std::vector<int> idx(n);
    for (int i = 0; i < n; ++i) idx[i] = i;
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return d[a] < d[b]; });
    GLTable t;
    for (int i = 0; i < n; ++i) {
        t.node[i] = d[idx[i]];
        t.weight[i] = std::sqrt(M_PI) * z[idx[i]] * z[idx[i]];
    }
    return t;
}

void set_geom(StencilGeom& g, const int n[3], const double origin[3], const double h[3], int order,
              const double margin[3]) {
    g.order = order;
    for (int a = 0; a < 3; ++a) {
        g.n[a] = n[a];
        g.origin[a] = origin[a];
        g.h[a] = h[a];
        g.w[a] = n[a] > 1 ? order + 1 : 1;
        g.nc[a] = n[a] - g.w[a] + 1;
        g.margin[a] = margin[a];
    }
}

void check_status(FftpimPlan* P, const char* phase) {
    CK(cudaStreamSynchronize(P->build_stream));
    DevStatus st;
    CK(cudaMemcpy(&st, P->status, sizeof(st), cudaMemcpyDeviceToHost));
    if (st.code) {
        char buf[256];
        const char* what = "error";
        switch (st.code) {
            case FFTPIM_DOMAIN: what = "DomainError"; break;
            case FFTPIM_WOOD_ANOMALY: what = "WoodAnomalyError"; break;
            case FFTPIM_NOT_CONVERGED: what = "NotConvergedError"; break;
            case FFTPIM_SEPARATION: what = "SeparationError"; break;
        }
        std::string detail;
        switch (st.where) {
            case 10: case 11: case 12: case 20: case 21: case 22: case 23:
                detail = "point outside grid hull (beyond allowed margin)"; break;
            case 30: detail = "observer " + std::to_string(st.a) + " coincides with a distinct source " +
                              std::to_string(st.b) + " inside the error-correction region: true singularity"; break;
            case 31: detail = "image point coincides with evaluation point (correction pair of observer " +
                              std::to_string(st.a) + ")"; break;
            case 40: case 42: detail = "1D series requires transverse separation sqrt(y^2+z^2) > 0"; break;
            case 41: detail = "lattice series argument vanished"; break;
            case 43: detail = "|k_rho(m=" + std::to_string(st.a) + ")| below threshold"; break;
            case 44: detail = "|k_z(m=" + std::to_string(st.a) + ", n=" + std::to_string(st.b) + ")| below threshold"; break;
            case 45: detail = "z image stack diverges: |exp(-j(k_z -+ k_z0) L_z)| > 1"; break;
            case 46: detail = "resonant z stack at (m=" + std::to_string(st.a) + ", n=" + std::to_string(st.b) + ")"; break;
            case 47: detail = "far kernel series did not converge at difference point " + std::to_string(st.a) +
                              " (terms used: " + std::to_string(st.b) + ")"; break;
            case 48: detail = "far kernel: image point coincides with evaluation point"; break;
            case 60: detail = "observer " + std::to_string(st.a) + " coincides with source " + std::to_string(st.b); break;
            case 61: detail = "image point coincides with evaluation point (observer " + std::to_string(st.a) +
                              ", source " + std::to_string(st.b) + ")"; break;
            default: detail = "code " + std::to_string(st.where);
        }
        snprintf(buf, sizeof(buf), "%s during %s: ", what, phase);
        throw Fail{st.code, std::string(buf) + detail};
    }
}

int64_t prod3(const int d[3]) { return (int64_t)d[0] * d[1] * d[2]; }

template <typename K, typename V>
void radix_sort_pairs(const K* kin, K* kout, const V* vin, V* vout, int64_t n, int end_bit, cudaStream_t s) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, s);
    void* tmp = nullptr;
    CK(cudaMallocAsync(&tmp, bytes + 16, s));
    cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, s);
    CK(cudaFreeAsync(tmp, s));
    fftpim_count_launch(4);
}

int bits_for(int64_t maxval) {
    int b = 1;
    while (b < 31 && ((int64_t)1 << b) <= maxval) ++b;
    return b;
}

// Sort points by near stencil cell; returns perm (sorted -> original), and
// fills stencil arrays in sorted order.
void sort_points(FftpimPlan* P, const double* d_pos, int64_t n, int* perm, int* cell_start_or_null,
                 cudaStream_t s) {
    const StencilGeom& g = P->near_g;
    int64_t ncells = prod3(g.nc);
    int* keys = nullptr;
    int* keys_sorted = nullptr;
    int* iota = nullptr;
    CK(cudaMallocAsync(&keys, sizeof(int) * std::max<int64_t>(n, 1), s));
    CK(cudaMallocAsync(&keys_sorted, sizeof(int) * std::max<int64_t>(n, 1), s));
    CK(cudaMallocAsync(&iota, sizeof(int) * std::max<int64_t>(n, 1), s));
    launch_cell_keys(d_pos, n, g, keys, P->status, s);
    launch_iota(iota, n, s);
    radix_sort_pairs(keys, keys_sorted, iota, perm, n, bits_for(ncells), s);
    if (cell_start_or_null) launch_csr_from_sorted(keys_sorted, n, ncells, cell_start_or_null, s);
    CK(cudaFreeAsync(keys, s));
    CK(cudaFreeAsync(keys_sorted, s));
    CK(cudaFreeAsync(iota, s));
}

// complex elements per column-FFT block (B columns x L); FFTPIM_FFT_BLOCK tunes it
int fft_block_elems() {
    static int v = [] {
        const char* e = getenv("FFTPIM_FFT_BLOCK");
        int x = e ? atoi(e) : 1024;
        return x >= 64 ? x : 1024;
    }();
    return v;
}

// Radix factorisation for the Stockham stages: 4s, a 2, then small primes.
bool fft_radices(int L, int* radix, int* nrad) {
    int n = 0;
    while (L % 4 == 0 && n < 24) radix[n++] = 4, L /= 4;
    while (L % 2 == 0 && n < 24) radix[n++] = 2, L /= 2;
    for (int p = 3; p <= 31 && L > 1; p += 2)
        while (L % p == 0 && n < 24) radix[n++] = p, L /= p;
    *nrad = n;
    return L == 1;
}

// Pruned column-FFT pipeline for the zero-padded convolution (fft_kernels.cu).
// Falls back to cuFFT full transforms when a doubled axis has a prime factor > 31
// or is longer than 2048.
void setup_fft_pipeline(FftpimPlan* P, const int dims[3], cudaStream_t s) {
    const int n0 = dims[0], n1 = dims[1], n2 = dims[2];
    const int L[3] = {P->cdims[0], P->cdims[1], P->cdims[2]};
    int rad[3][24], nr[3];
    for (int a = 0; a < 3; ++a) {
        if (dims[a] == 1) continue;
        if (L[a] > 2048 || !fft_radices(L[a], rad[a], &nr[a])) return;
    }
    const char* e = getenv("FFTPIM_FFT");   // "cufft": full cuFFT transforms (unsharded plans)
    if (e && std::string(e) == "cufft" && !P->sharded) return;
    P->custom_fft = true;
    P->info.custom_fft = 1;
    for (int a = 0; a < 3; ++a) {
        if (dims[a] == 1) continue;
        std::vector<cplx> tw(L[a]);
        for (int t = 0; t < L[a]; ++t) {
            long double ang = 2.0L * 3.141592653589793238462643383279502884L * t / L[a];
            tw[t] = cplx{(double)cosl(ang), (double)-sinl(ang)};
        }
        P->twiddle[a] = dalloc<cplx>(P, L[a]);
        CK(cudaMemcpyAsync(P->twiddle[a], tw.data(), sizeof(cplx) * L[a], cudaMemcpyHostToDevice, s));
        // per-pass compact twiddles: pass (r, p): exp(-2 pi i q k / (p r)), q = 1..r-1, k < p
        std::vector<cplx> twp;
        int p = 1;
        for (int ri = 0; ri < nr[a]; ++ri) {
            const int r = rad[a][ri];
            for (int q = 1; q < r; ++q)
                for (int k = 0; k < p; ++k) twp.push_back(tw[(int64_t)q * k * (L[a] / (p * r)) % L[a]]);
            p *= r;
        }
        P->n_twiddle_pass[a] = (int)twp.size();
        P->twiddle_pass[a] = dalloc<cplx>(P, std::max<int64_t>(1, (int64_t)twp.size()));
        if (!twp.empty())
            CK(cudaMemcpyAsync(P->twiddle_pass[a], twp.data(), sizeof(cplx) * twp.size(), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
    P->qg = dalloc<cplx>(P, (int64_t)n0 * n1 * n2);
    cplx* A = P->qg;
    if (n2 > 1) A = P->fbufA = dalloc<cplx>(P, (int64_t)n0 * n1 * L[2]);
    cplx* Bb = A;
    if (n1 > 1) Bb = P->fbufB = dalloc<cplx>(P, (int64_t)n0 * L[1] * L[2]);
    auto base = [&](int axis, int sign) {
        FftStage st{};
        st.L = L[axis];
        st.nrad = nr[axis];
        for (int k = 0; k < nr[axis]; ++k) st.radix[k] = rad[axis][k];
        st.tw = P->twiddle[axis];
        st.twp = P->twiddle_pass[axis];
        st.ntwp = P->n_twiddle_pass[axis];
        st.sign = sign;
        return st;
    };
    const int64_t L12 = (int64_t)L[1] * L[2];
    if (n2 > 1) {   // S1: z forward, qg -> A
        FftStage st = base(2, -1);
        st.in = P->qg; st.out = A; st.lin = n2; st.lout = L[2]; st.in_stride = 1; st.out_stride = 1;
        st.nb0 = n1; st.in_s0 = n2; st.out_s0 = L[2];
        st.nb1 = n0; st.in_s1 = (int64_t)n1 * n2; st.out_s1 = (int64_t)n1 * L[2];
        P->stage[0] = st;
        P->stage_on[0] = true;
        // S5: z inverse, A -> qg
        FftStage t = base(2, +1);
        t.in = A; t.out = P->qg; t.lin = L[2]; t.lout = n2; t.in_stride = 1; t.out_stride = 1;
        t.nb0 = n1; t.in_s0 = L[2]; t.out_s0 = n2;
        t.nb1 = n0; t.in_s1 = (int64_t)n1 * L[2]; t.out_s1 = (int64_t)n1 * n2;
        P->stage[4] = t;
        P->stage_on[4] = true;
    }
    if (n1 > 1) {   // S2: y forward, A -> B
        FftStage st = base(1, -1);
        st.in = A; st.out = Bb; st.lin = n1; st.lout = L[1]; st.in_stride = L[2]; st.out_stride = L[2];
        st.nb0 = L[2]; st.in_s0 = 1; st.out_s0 = 1;
        st.nb1 = n0; st.in_s1 = (int64_t)n1 * L[2]; st.out_s1 = L12;
        P->stage[1] = st;
        P->stage_on[1] = true;
        // S4: y inverse, B -> A
        FftStage t = base(1, +1);
        t.in = Bb; t.out = A; t.lin = L[1]; t.lout = n1; t.in_stride = L[2]; t.out_stride = L[2];
        t.nb0 = L[2]; t.in_s0 = 1; t.out_s0 = 1;
        t.nb1 = n0; t.in_s1 = L12; t.out_s1 = (int64_t)n1 * L[2];
        P->stage[3] = t;
        P->stage_on[3] = true;
    }
    {   // S3: x forward * khat * x inverse, in place on B
        FftStage st = base(0, -1);
        st.in = Bb; st.out = Bb; st.lin = n0; st.lout = n0; st.in_stride = L12; st.out_stride = L12;
        st.nb0 = (int)L12; st.in_s0 = 1; st.out_s0 = 1;
        st.nb1 = 1; st.in_s1 = 0; st.out_s1 = 0;
        st.spec = P->khat; st.spec_stride = L12; st.spec_s0 = 1; st.spec_s1 = 0;
        {
            const FftpimProblem& pr = P->prob;
            const char* e = getenv("FFTPIM_KHAT_FOLD");
            const bool on = !(e && e[0] == '0');
            auto even = [&](int a) {
                if (!on || dims[a] == 1 || (P->sweep && a == P->sw_axis)) return false;
                return a >= pr.dim || (pr.kshift[a][0] == 0.0 && pr.kshift[a][1] == 0.0);
            };
            st.fold_y = even(1) ? L[1] : 0;
            st.fold_z = even(2) ? L[2] : 0;
            st.spec_L2 = L[2];
        }
        P->stage[2] = st;
        P->stage_on[2] = true;
    }
    for (int k = 0; k < 5; ++k) {
        FftStage& st = P->stage[k];
        if (!P->stage_on[k]) continue;
        st.B = std::max(1, std::min(st.nb0, fft_block_elems() / st.L));
    }
}

// Slab-shard version of the pruned pipeline: z and y transforms on the shard's
// own x-planes, then an all-to-all transpose to FFT columns [C0, C1) for the
// fused x stage (its khat slice only), the transpose back, y/z inverses, and a
// halo of order planes from the next shard for the interpolation.
void setup_fft_pipeline_shard(FftpimPlan* P, const int dims[3], cudaStream_t s) {
    if (!P->custom_fft) throw Fail{FFTPIM_VALUE, "slab-decomposed plans need FFT lengths with prime factors <= 31"};
    if (dims[1] < 2 || dims[2] < 2) throw Fail{FFTPIM_VALUE, "slab-decomposed plans need three active axes"};
    const int G = P->world, n0 = dims[0], n1 = dims[1], n2 = dims[2];
    const int L0 = P->cdims[0], L1 = P->cdims[1], L2 = P->cdims[2];
    const int nl = P->n0_loc;
    P->C = (int64_t)L1 * L2;
    P->col_start.resize(G + 1);
    for (int r = 0; r <= G; ++r) P->col_start[r] = (int64_t)r * P->C / G;
    P->C0 = P->col_start[P->rank];
    P->C1 = P->col_start[P->rank + 1];
    const int64_t ncol = P->C1 - P->C0;
    // replace the full-domain buffers by slab buffers
    dfree(P, P->qg);
    dfree(P, P->fbufA);
    dfree(P, P->fbufB);
    P->qg = dalloc<cplx>(P, (int64_t)(nl + P->halo) * n1 * n2);
    P->fbufA = dalloc<cplx>(P, (int64_t)nl * n1 * L2);
    P->fbufB = dalloc<cplx>(P, (int64_t)nl * L1 * L2);
    P->a2a_send = dalloc<cplx>(P, (int64_t)nl * P->C);
    P->a2a_recv = dalloc<cplx>(P, (int64_t)n0 * ncol);
    // khat slice [kx][own columns]
    cplx* ks = dalloc<cplx>(P, (int64_t)L0 * ncol);
    CK(cudaMemcpy2DAsync(ks, ncol * sizeof(cplx), P->khat + P->C0, P->C * sizeof(cplx), ncol * sizeof(cplx), L0,
                         cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    dfree(P, P->khat);
    P->khat = ks;
    FftStage* st = P->stage;
    // S1: z forward, qg (own planes) -> A
    st[0].in = P->qg; st[0].out = P->fbufA; st[0].nb1 = nl;
    // S2: y forward, A -> B
    st[1].in = P->fbufA; st[1].out = P->fbufB; st[1].nb1 = nl;
    // S3: x fused on the transposed columns: recv[x][c_local]
    st[2].in = P->a2a_recv; st[2].out = P->a2a_recv; st[2].lin = n0; st[2].lout = n0;
    st[2].in_stride = ncol; st[2].out_stride = ncol; st[2].nb0 = (int)ncol; st[2].in_s0 = 1; st[2].out_s0 = 1;
    st[2].spec = P->khat; st[2].spec_stride = ncol; st[2].spec_s0 = 1;
    st[2].fold_y = st[2].fold_z = 0;   // a column slice of khat: no symmetric folding
    st[2].B = std::max(1, std::min(st[2].nb0, fft_block_elems() / st[2].L));
    // S4: y inverse, B -> A
    st[3].in = P->fbufB; st[3].out = P->fbufA; st[3].nb1 = nl;
    // S5: z inverse, A -> qg (own planes, the halo planes follow)
    st[4].in = P->fbufA; st[4].out = P->qg; st[4].nb1 = nl;
    (void)L0;
}

EvalArgs eval_args(FftpimPlan* P, const double* q, double* u, int parts);
// run-encoded K4 stream by default?  (measured at C4: see DESIGN.md section 3)
static bool k4_runs_default(const FftpimPlan* P) { return false && P->info.pair_rows_source_order == 1; }

// Images of G_near for the shift ks (pgf.py:114-123): offsets i*L and phases
// exp(-j i.(ks o L)), i in [-i_d, i_d]^dim.  axis >= 0 keeps only the images with
// i[axis] == only and leaves the axis part out of the phase (sweep components).
static void make_images(const FftpimProblem& pr, const double ks[3][2], ImageSet& im, int axis = -1, int only = 0) {
    int hw[3];
    for (int a = 0; a < 3; ++a) hw[a] = a < pr.dim ? pr.i_d : 0;
    int c = 0;
    std::complex<double> kl[3];
    for (int a = 0; a < 3; ++a) kl[a] = std::complex<double>(ks[a][0], ks[a][1]) * pr.L[a];
    for (int i = -hw[0]; i <= hw[0]; ++i)
        for (int j = -hw[1]; j <= hw[1]; ++j)
            for (int k = -hw[2]; k <= hw[2]; ++k) {
                const int ii[3] = {i, j, k};
                if (axis >= 0 && ii[axis] != only) continue;
                double idx[3] = {(double)i, (double)j, (double)k};
                std::complex<double> dotp(0.0, 0.0);
                for (int a = 0; a < 3; ++a)
                    if (a != axis) dotp += idx[a] * kl[a];
                std::complex<double> ph = std::exp(std::complex<double>(0.0, -1.0) * dotp);
                for (int a = 0; a < 3; ++a) im.off[c][a] = idx[a] * pr.L[a];
                im.ph_re[c] = ph.real();
                im.ph_im[c] = ph.imag();
                ++c;
            }
    im.count = c;
}

// phase of image code c, exp(-j c.(ks o L)) (nearzone.py:456-457); the sweep
// axis part left out when axis >= 0
static void code_phases(const FftpimProblem& pr, const double ks[3][2], PairGeom& pg, int axis = -1) {
    for (int c = 0; c < pg.ncodes; ++c) {
        std::complex<double> dotp(0.0, 0.0);
        for (int a = 0; a < 3; ++a)
            if (a != axis) dotp += (double)pg.code[c][a] * (std::complex<double>(ks[a][0], ks[a][1]) * pr.L[a]);
        std::complex<double> ph = std::exp(std::complex<double>(0.0, -1.0) * dotp);
        pg.phase_re[c] = ph.real();
        pg.phase_im[c] = ph.imag();
    }
}

// kernel_hat = fftn(embed(G_near)) / M for the image set im (nearzone.py:215-235)
static void tabulate_khat(FftpimPlan* P, const int dims[3], const double h[3], const ImageSet& im, cplx* out,
                          cudaStream_t s) {
    launch_embed_table(out, P->cdims, dims, h, im, s);
    CKFFT(cufftSetStream(P->fft_plan, s));
    CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)out, (cufftDoubleComplex*)out, CUFFT_FORWARD));
    fftpim_count_launch(1);
    launch_scale(out, P->n_fft, 1.0 / (double)P->n_fft, s);   // numpy ifftn's 1/M
}

// far kernel G_total - G_near on the difference points (farzone.py:100-121,
// pgf.py:450-462) for the shift ks; returns the worst series length
static int64_t tabulate_far(FftpimPlan* P, const double ks[3][2], const ImageSet& im, cplx* out, cudaStream_t s) {
    const FftpimProblem& pr = P->prob;
    int fdims[3];
    double fh[3];
    for (int a = 0; a < 3; ++a) {
        fdims[a] = P->far_sg.n[a];
        fh[a] = P->far_sg.h[a];
    }
    double maxLp = 0.0;
    for (int a = 0; a < pr.dim; ++a) maxLp = std::max(maxLp, pr.L[a]);
    std::vector<double> axes;
    double zmin = 1e300, zmax = -1e300;
    for (int a = 0; a < 3; ++a) {
        int n = fdims[a];
        double shift = P->far_og.origin[a] - P->far_sg.origin[a];
        if (n == 1) {
            axes.push_back(shift);
            if (a == 2) zmin = zmax = shift;
        } else {
            for (int l = -(n - 1); l < n; ++l) {
                double v = (double)l * fh[a] + shift;
                axes.push_back(v);
                if (a == 2) {
                    zmin = std::min(zmin, v);
                    zmax = std::max(zmax, v);
                }
            }
        }
    }
    double* d_axes = dalloc<double>(P, (int64_t)axes.size());
    CK(cudaMemcpyAsync(d_axes, axes.data(), sizeof(double) * axes.size(), cudaMemcpyHostToDevice, s));
    FarSeriesParams fp{};
    fp.dim = pr.dim;
    fp.npsp = P->npsp;
    for (int a = 0; a < 3; ++a) {
        fp.L[a] = pr.L[a];
        fp.ks_re[a] = ks[a][0];
        fp.ks_im[a] = ks[a][1];
    }
    fp.k0_re = pr.k0[0];
    fp.k0_im = pr.k0[1];
    fp.tol = pr.series_tol;
    fp.cutoff = std::log(1.0 / pr.series_tol) + 8.0;
    fp.sep = im.sep_tol;
    fp.wood = 1e-8 * 2.0 * M_PI / maxLp;
    fp.zmin = zmin;
    fp.zmax = zmax;
    fp.max_terms = 1000000;
    fp.max_layers = 200000;
    fp.consecutive = 3;
    static const GLTable gl = gauss_laguerre_half();
    launch_far_series(d_axes, P->far_kdims, fp, im, gl, out, P->status, s);
    check_status(P, "far kernel tabulation");
    DevStatus st;
    CK(cudaMemcpy(&st, P->status, sizeof(st), cudaMemcpyDeviceToHost));
    dfree(P, d_axes);
    return st.kernel_terms;
}

// plans with at most this many pairs run the concurrent schedule (near chain |
// K4 | far chain); larger ones run the stages in order (FFTPIM_CONCURRENT_MAX)
static int64_t concurrent_max_pairs() {
    static const int64_t v = [] {
        const char* e = getenv("FFTPIM_CONCURRENT_MAX");
        return e ? (int64_t)atoll(e) : (int64_t)500000000LL;
    }();
    return v;
}

// largest observer count of a grid-tile observer-pass tile (line_kernels.cu),
// from the observer cell CSR (built here when observers are not the sources)
int64_t max_tile_count(FftpimPlan* P, const int* ocs, const double* d_obs, int64_t M, cudaStream_t s) {
    int* tmp = nullptr;
    if (!ocs) {
        int* perm = dalloc<int>(P, M);
        tmp = dalloc<int>(P, prod3(P->near_g.nc) + 1);
        sort_points(P, d_obs, M, perm, tmp, s);
        dfree(P, perm);
        ocs = tmp;
    }
    const int64_t v = launch_max_tile_count(P->near_g, ocs, s);
    if (tmp) dfree(P, tmp);
    return v;
}

void build(FftpimPlan* P) {
    NvtxRange nv("fftpim build: sort, stencils, near kernel");
    const FftpimProblem& pr = P->prob;
    cudaStream_t s = P->build_stream;
    const int64_t N = pr.n_src, M = pr.n_obs;
    P->N = N;
    P->M = M;
    P->npsp = pr.regime == FFTPIM_NPSP;
    if (N <= 0 || M <= 0) throw Fail{FFTPIM_VALUE, "empty source or observer set"};
    // i_d = 0: near zone only (free-space near kernel, no wrapped copies;
    // nearzone.py:205-212, :314) -- the far engine needs i_d >= 1 (farzone.py:84-85)
    if (pr.i_d < 0) throw Fail{FFTPIM_VALUE, "i_d must be >= 0"};
    P->near_only = pr.i_d == 0;
    if (P->near_only && P->sweep) throw Fail{FFTPIM_VALUE, "far-zone engine requires i_d >= 1"};
    if (pr.dim < 1 || pr.dim > 3) throw Fail{FFTPIM_VALUE, "dim must be 1, 2 or 3"};
    if (pr.near_order < 1 || pr.near_order > FFTPIM_MAX_ORDER || pr.far_order < 1 ||
        pr.far_order > FFTPIM_MAX_ORDER)
        throw Fail{FFTPIM_VALUE, "interpolation order must be in [1, 6]"};
    if (pr.i_d > 2) throw Fail{FFTPIM_VALUE, "i_d > 2 is not supported by this build"};
    // zones to build: build_near_plan / build_far_plan build only their half
    const int bparts = pr.parts ? pr.parts : FFTPIM_ALL;
    if (bparts & ~FFTPIM_ALL) throw Fail{FFTPIM_VALUE, "parts must be a non-empty subset of NEAR|FAR"};
    if (bparts != FFTPIM_ALL && (P->sweep || P->sharded))
        throw Fail{FFTPIM_VALUE, "sweep and slab plans build both zones"};
    if (P->near_only && bparts == FFTPIM_FAR) throw Fail{FFTPIM_VALUE, "far-zone engine requires i_d >= 1"};
    P->info.built_parts = P->near_only ? FFTPIM_NEAR : bparts;
    const bool want_near = bparts & FFTPIM_NEAR, want_far = (bparts & FFTPIM_FAR) && !P->near_only;

    // ---- near grid (nearzone.py:198-211, grids.py:90-107)
    int dims[3];
    bool auto_grid = pr.near_grid[0] <= 0 && pr.near_grid[1] <= 0 && pr.near_grid[2] <= 0;
    if (auto_grid) {   // model.py:146-162
        int act = 0;
        for (int a = 0; a < 3; ++a) act += pr.D[a] > 0.0;
        double target = 1.15 * (double)std::max<int64_t>(std::max(N, M), 1);
        int side = std::max(2, (int)std::ceil(std::pow(target, 1.0 / act)));
        if (side % 2 == 0) ++side;
        for (int a = 0; a < 3; ++a) dims[a] = pr.D[a] > 0.0 ? side : 1;
    } else {
        for (int a = 0; a < 3; ++a) dims[a] = pr.D[a] > 0.0 ? pr.near_grid[a] : 1;
    }
    double h[3], zero3[3] = {0, 0, 0};
    for (int a = 0; a < 3; ++a) {
        if (pr.D[a] > 0.0 && dims[a] < 2)
            throw Fail{FFTPIM_VALUE, "near grid needs >= 2 points on active axis " + std::to_string(a)};
        h[a] = pr.D[a] > 0.0 ? pr.D[a] / (dims[a] - 1) : 0.0;
        if (dims[a] > 1 && pr.near_order + 1 > dims[a])
            throw Fail{FFTPIM_VALUE, "near order needs more planes than the grid has"};
    }
    int nb[3];
    for (int a = 0; a < 3; ++a) nb[a] = std::max(dims[a] - 1, 1);
    for (int a = 0; a < pr.dim; ++a)
        if (dims[a] > 1 && 2.0 * pr.er_range_boxes * h[a] >= pr.L[a])
            throw Fail{FFTPIM_VALUE, "error-correction range on axis " + std::to_string(a) +
                                         " must satisfy 2*D_ER < L"};
    double margin[3];
    for (int a = 0; a < 3; ++a) margin[a] = 1e-9 * std::max(h[a], 1.0);   // nearzone.py:237
    set_geom(P->near_g, dims, zero3, h, pr.near_order, margin);
    P->n_grid = prod3(dims);
    for (int a = 0; a < 3; ++a) P->cdims[a] = dims[a] > 1 ? 2 * dims[a] : 1;
    P->n_fft = prod3(P->cdims);

    // ---- far grids (grids.py:58-87, farzone.py:84-98, 125-127)
    int fdims[3];
    double fs_org[3], fo_org[3], fh[3], fmarg[3];
    for (int a = 0; a < 3; ++a) {
        if (pr.D[a] <= 0.0) {
            fdims[a] = 1;
            fs_org[a] = fo_org[a] = fh[a] = 0.0;
            continue;
        }
        fdims[a] = pr.far_grid[a];
        if (fdims[a] < 2) throw Fail{FFTPIM_VALUE, "far grid needs >= 2 points on active axis"};
        if (pr.far_order + 1 > fdims[a]) throw Fail{FFTPIM_VALUE, "far order needs more planes than the grid has"};
        fh[a] = pr.D[a] / fdims[a];
        fs_org[a] = 0.0;
        fo_org[a] = fh[a] / 2.0;
    }
    P->info.on_axis_offset = 0;
    if (pr.dim == 1 && pr.D[1] == 0.0 && pr.D[2] == 0.0) {
        fs_org[1] = fh[0] / 2.0;
        P->info.on_axis_offset = 1;
    }
    for (int a = 0; a < 3; ++a) fmarg[a] = fdims[a] > 1 ? fh[a] : 0.0;
    set_geom(P->far_sg, fdims, fs_org, fh, pr.far_order, fmarg);
    set_geom(P->far_og, fdims, fo_org, fh, pr.far_order, fmarg);
    P->n_far = prod3(fdims);
    for (int a = 0; a < 3; ++a) P->far_kdims[a] = fdims[a] > 1 ? 2 * fdims[a] - 1 : 1;

    // ---- images of G_near (pgf.py:114-123)
    ImageSet& im = P->images;
    im.k0_re = pr.k0[0];
    im.k0_im = pr.k0[1];
    double maxL = std::max(pr.L[0], std::max(pr.L[1], pr.L[2]));
    double maxD = std::max(pr.D[0], std::max(pr.D[1], pr.D[2]));
    double maxLp = 0.0;
    for (int a = 0; a < pr.dim; ++a) maxLp = std::max(maxLp, pr.L[a]);
    im.sing_tol = 1e-12 * std::max(std::max(maxL, maxD), 1.0);   // nearzone.py:213
    im.sep_tol = 1e-13 * std::max(maxLp, 1.0);                     // pgf.py:93-94
    make_images(pr, pr.kshift, im);

    // ---- points
    double* d_src = dalloc<double>(P, 3 * N);
    CK(cudaMemcpyAsync(d_src, pr.src_pos, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, s));
    double* d_obs = d_src;
    const bool same = pr.same_points != 0;
    if (!same) {
        d_obs = dalloc<double>(P, 3 * M);
        CK(cudaMemcpyAsync(d_obs, pr.obs_pos, sizeof(double) * 3 * M, cudaMemcpyHostToDevice, s));
    }
    const int W = pr.near_order + 1, WF = pr.far_order + 1;
    P->src_perm = dalloc<int>(P, N);
    P->src_rank = dalloc<int>(P, N);
    P->cell_start = dalloc<int>(P, prod3(P->near_g.nc) + 1);
    sort_points(P, d_src, N, P->src_perm, P->cell_start, s);
    launch_rank(P->src_perm, N, P->src_rank, s);
    P->src_w = dalloc<double>(P, N * 3 * W);
    P->src_start = dalloc<int>(P, N * 3);
    launch_stencils(d_src, P->src_perm, N, P->near_g, P->src_w, P->src_start, P->status, 20, s);
    {
        // K1: line sweep (stencils from sorted positions) by default for large
        // point sets, the plan-time sliced-ELL operator otherwise;
        // FFTPIM_K1=lines|ell|gather|taps overrides
        const char* e = getenv("FFTPIM_K1");
        const bool ok = W >= 3 && W <= 6;
        // measured (B200): the line sweep wins on sparse grids (C4, 0.5 points per
        // stencil cell: 1.5 vs 2.9 ms), the ELL operator on denser ones (C5 1.3 per
        // cell: 0.37 vs 0.86 ms; clustered C3: 1.7 vs 6.9 ms)
        const double density = (double)N / (double)prod3(P->near_g.nc);
        const std::string mode = e ? e : (N > 262144 && density < 0.75 ? "lines_smem" : "ell");
        P->k1_lines = ok && (mode == "lines" || mode == "lines_smem");
        if (P->k1_lines && mode == "lines_smem") {
            P->src_pos_s = dalloc<double>(P, 3 * N);
            launch_gather_pos(d_src, P->src_perm, N, P->src_pos_s, s);
        } else if (P->k1_lines) {
            P->src_rec = dalloc<double>(P, N * stencil_record_width(W));
            launch_stencil_records(P->src_w, P->src_start, N, W, P->src_rec, s);
        }
    }
    P->src_fw = dalloc<double>(P, N * 3 * WF);
    P->src_fstart = dalloc<int>(P, N * 3);
    launch_stencils(d_src, P->src_perm, N, P->far_sg, P->src_fw, P->src_fstart, P->status, 21, s);
    if (same) {
        P->obs_perm = P->src_perm;
        P->obs_w = P->src_w;
        P->obs_start = P->src_start;
    } else {
        P->obs_perm = dalloc<int>(P, M);
        sort_points(P, d_obs, M, P->obs_perm, nullptr, s);
        P->obs_w = dalloc<double>(P, M * 3 * W);
        P->obs_start = dalloc<int>(P, M * 3);
        launch_stencils(d_obs, P->obs_perm, M, P->near_g, P->obs_w, P->obs_start, P->status, 22, s);
    }
    P->obs_fw = dalloc<double>(P, M * 3 * WF);
    P->obs_fstart = dalloc<int>(P, M * 3);
    launch_stencils(d_obs, P->obs_perm, M, P->far_og, P->obs_fw, P->obs_fstart, P->status, 23, s);
    check_status(P, "stencil construction");
    nv.next("fftpim build: near kernel table, pair discovery");
    {
        // observer pass with stencils from sorted positions (line_kernels.cu) for
        // large observer sets; FFTPIM_OBS=pos|weights overrides
        // measured: the grid-tile pass wins for large, evenly spread observer sets
        // (C4 1.7 vs 2.5 ms, C5 0.25 vs 0.33 ms); clustered sets (C3 blobs: a few
        // tiles hold thousands of observers) keep the stored-weight pass
        const char* e = getenv("FFTPIM_OBS");
        std::string om = e ? e : "weights";
        if (!e && M > 262144 && dims[0] > 1 && dims[1] > 1 && dims[2] > 1 &&
            max_tile_count(P, same ? P->cell_start : nullptr, d_obs, M, s) <= 2048)
            om = "tile";
        P->obs_pos_pass = W >= 3 && W <= 6 && WF >= 3 && WF <= 5 && (om == "pos" || om == "tile");
        P->obs_tile = P->obs_pos_pass && om == "tile";
        if (P->obs_tile) {
            if (same) {
                P->obs_cell_start = P->cell_start;
            } else {
                P->obs_cell_start = dalloc<int>(P, prod3(P->near_g.nc) + 1);
                int* tmp_perm = dalloc<int>(P, M);
                sort_points(P, d_obs, M, tmp_perm, P->obs_cell_start, s);   // same key, same stable order
                dfree(P, tmp_perm);
            }
        }
        if (P->obs_pos_pass) {
            if (same && P->src_pos_s) {
                P->obs_pos_s = P->src_pos_s;
            } else {
                P->obs_pos_s = dalloc<double>(P, 3 * M);
                launch_gather_pos(d_obs, P->obs_perm, M, P->obs_pos_s, s);
            }
        }
    }

    // ---- slab ownership: planes [X0, X1), observers/sources whose
    // near stencil starts there = one contiguous range of the x-major sorted order
    P->i0 = 0;
    P->i1 = M;
    P->X0 = 0;
    P->X1 = dims[0];
    P->n0_loc = dims[0];
    P->halo = 0;
    if (P->sharded) {
        if (!same) throw Fail{FFTPIM_VALUE, "slab-decomposed plans need observers == sources"};
        const int G = P->world;
        P->plane_start.resize(G + 1);
        for (int r = 0; r <= G; ++r) P->plane_start[r] = (int)((int64_t)r * dims[0] / G);
        P->X0 = P->plane_start[P->rank];
        P->X1 = P->plane_start[P->rank + 1];
        P->n0_loc = P->X1 - P->X0;
        for (int r = 0; r + 1 < G; ++r)
            if (P->plane_start[r + 1] - P->plane_start[r] < W - 1)
                throw Fail{FFTPIM_VALUE, "too many slab shards for the near grid (need >= order planes each)"};
        P->halo = P->rank + 1 < G ? W - 1 : 0;
        auto first_sorted = [&](int sx) -> int64_t {
            if (sx >= P->near_g.nc[0]) return N;
            int v = 0;
            CK(cudaMemcpy(&v, P->cell_start + (int64_t)sx * P->near_g.nc[1] * P->near_g.nc[2], sizeof(int),
                          cudaMemcpyDeviceToHost));
            return v;
        };
        P->i0 = first_sorted(P->X0);
        P->i1 = first_sorted(P->X1);
    }
    const int64_t Mown = P->i1 - P->i0;

    // ---- near kernel table -> kernel_hat (nearzone.py:215-235)
    unsigned long long* d_cnt = dalloc<unsigned long long>(P, 4);
    CK(cudaMemsetAsync(d_cnt, 0, 4 * sizeof(unsigned long long), s));
    launch_count_coincident(dims, h, im, d_cnt, s);
    if (want_near) {
    P->khat = dalloc<cplx>(P, P->n_fft);
    {
        int rank = 0, n[3];
        for (int a = 0; a < 3; ++a)
            if (P->cdims[a] > 1) n[rank++] = P->cdims[a];
        if (rank == 0) throw Fail{FFTPIM_VALUE, "near grid has no active axis"};
        CKFFT(cufftPlanMany(&P->fft_plan, rank, n, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, 1));
        tabulate_khat(P, dims, h, im, P->khat, s);
    }
    setup_fft_pipeline(P, dims, s);
    if (P->sharded) setup_fft_pipeline_shard(P, dims, s);
    if (!P->custom_fft) {
        P->work = dalloc<cplx>(P, P->n_fft);
        P->pad_in = dalloc<cplx>(P, P->n_fft);
        CK(cudaMemsetAsync(P->pad_in, 0, sizeof(cplx) * P->n_fft, s));   // padding stays zero: out-of-place forward FFT
    }
    }   // want_near
    P->q_sorted = dalloc<cplx>(P, N + CORR_QPAD);   // zero tail: padding pairs of k_corr_runs
    CK(cudaMemset(P->q_sorted + N, 0, sizeof(cplx) * CORR_QPAD));
    {
        // tap-major K1 (3 active axes, orders 2..4) pays off for crowded cells
        // (clustered sources, C3: >= 1 point per stencil cell on average); sparse
        // grids keep the gather K1.  FFTPIM_K1=taps|gather overrides.
        const char* e = getenv("FFTPIM_K1");
        const double density = (double)N / (double)prod3(P->near_g.nc);
        bool taps = density >= 1.0 && !P->k1_lines;
        if (e) taps = std::string(e) == "taps";
        if (taps && dims[0] > 1 && dims[1] > 1 && dims[2] > 1 && pr.near_order >= 2 && pr.near_order <= 4)
            P->k1_scratch = dalloc<cplx>(P, k1_scratch_elems(P->near_g, P->n0_loc));
    }

    // ---- correction pairs (nearzone.py:245-256, 303-487)
    PairGeom& pg = P->pg;
    const int jr_full = pr.er_range_boxes + pr.near_order + 2;
    int jr[3], pad[3];
    for (int a = 0; a < 3; ++a) {
        if (dims[a] == 1) {
            jr[a] = 0;
        } else {
            int r = jr_full;
            if (a < pr.dim && pr.i_d >= 1) {
                int per = (int)std::floor(pr.L[a] / h[a] + 1e-9);
                int half = (per - 1 >= 0) ? (per - 1) / 2 : -((2 - per) / 2);   // Python floor division
                r = std::min(r, std::max(half, 1));
            }
            jr[a] = std::min(r, nb[a]);
        }
        pad[a] = jr[a] + 1;
    }
    int max_pad = std::max(pad[0], std::max(pad[1], pad[2]));
    for (int a = 0; a < 3; ++a) {
        pg.dims[a] = dims[a];
        pg.h[a] = h[a];
        pg.inv_h[a] = dims[a] > 1 ? 1.0 / h[a] : 0.0;
        pg.nb[a] = nb[a];
        pg.jr[a] = jr[a];
        pg.ext[a] = dims[a] > 1 ? nb[a] + 2 * max_pad : 1;
        P->info.join_radius[a] = jr[a];
    }
    P->info.jr_full = jr_full;
    pg.max_pad = max_pad;
    pg.r2_keep = (double)jr_full * (double)jr_full + 1e-9;
    pg.sing_tol = im.sing_tol;
    pg.same_points = same;
    // code list: (0,0,0) first, then itertools.product order (nearzone.py:315-319)
    {
        int c = 0;
        auto set_code = [&](int cx, int cy, int cz) {
            pg.code[c][0] = cx;
            pg.code[c][1] = cy;
            pg.code[c][2] = cz;
            for (int a = 0; a < 3; ++a) pg.shift[c][a] = (double)pg.code[c][a] * pr.L[a];
            ++c;
        };
        set_code(0, 0, 0);
        int rng[3][2];
        for (int a = 0; a < 3; ++a) {
            bool wrap = pr.i_d >= 1 && a < pr.dim && dims[a] > 1;
            rng[a][0] = wrap ? -1 : 0;
            rng[a][1] = wrap ? 1 : 0;
        }
        for (int cx = rng[0][0]; cx <= rng[0][1]; ++cx)
            for (int cy = rng[1][0]; cy <= rng[1][1]; ++cy)
                for (int cz = rng[2][0]; cz <= rng[2][1]; ++cz)
                    if (cx || cy || cz) set_code(cx, cy, cz);
        pg.ncodes = c;
        code_phases(pr, pr.kshift, pg);
    }
    // augmented source list: originals, then wrapped copies code by code
    std::vector<int64_t> code_off(pg.ncodes + 1, 0);
    int* aug_orig = nullptr;
    unsigned char* aug_code = nullptr;
    int64_t A = N;
    {
        std::vector<int*> parts;
        std::vector<int64_t> counts;
        unsigned char* flags = nullptr;
        int* d_nsel = nullptr;
        CK(cudaMallocAsync(&flags, N, s));
        CK(cudaMallocAsync(&d_nsel, sizeof(int), s));
        code_off[0] = 0;
        code_off[1] = N;
        for (int c = 1; c < pg.ncodes; ++c) {
            int cv[3];
            double lo[3], hi[3];
            for (int a = 0; a < 3; ++a) {
                cv[a] = pg.code[c][a];
                double pd = pad[a] * h[a];
                lo[a] = pr.L[a] - pd;
                hi[a] = pr.D[a] - pr.L[a] + pd;
            }
            launch_wrap_flags(d_src, N, cv, lo, hi, flags, s);
            int* sel = nullptr;
            CK(cudaMallocAsync(&sel, sizeof(int) * N, s));
            size_t bytes = 0;
            cub::CountingInputIterator<int> it(0);
            cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, sel, d_nsel, (int)N, s);
            void* tmp = nullptr;
            CK(cudaMallocAsync(&tmp, bytes + 16, s));
            cub::DeviceSelect::Flagged(tmp, bytes, it, flags, sel, d_nsel, (int)N, s);
            fftpim_count_launch(2);
            CK(cudaFreeAsync(tmp, s));
            int nsel = 0;
            CK(cudaMemcpyAsync(&nsel, d_nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            parts.push_back(sel);
            counts.push_back(nsel);
            code_off[c + 1] = code_off[c] + nsel;
        }
        A = code_off[pg.ncodes];
        aug_orig = dalloc<int>(P, A);
        aug_code = dalloc<unsigned char>(P, A);
        launch_iota(aug_orig, N, s);
        launch_fill_u8(aug_code, N, 0, s);
        for (int c = 1; c < pg.ncodes; ++c) {
            int64_t n = counts[c - 1];
            if (n)
                CK(cudaMemcpyAsync(aug_orig + code_off[c], parts[c - 1], sizeof(int) * n, cudaMemcpyDeviceToDevice, s));
            launch_fill_u8(aug_code + code_off[c], n, (unsigned char)c, s);
            CK(cudaFreeAsync(parts[c - 1], s));
        }
        CK(cudaFreeAsync(flags, s));
        CK(cudaFreeAsync(d_nsel, s));
    }
    // bucket augmented sources by padded box (stable: reference aug order inside a box)
    int64_t total_boxes = (int64_t)pg.ext[0] * pg.ext[1] * pg.ext[2];
    if (total_boxes >= INT_MAX) throw Fail{FFTPIM_VALUE, "too many correction boxes"};
    int* box_start = dalloc<int>(P, total_boxes + 1);
    int* box_order = dalloc<int>(P, A);
    {
        int *keys = nullptr, *keys_sorted = nullptr, *iota = nullptr;
        CK(cudaMallocAsync(&keys, sizeof(int) * A, s));
        CK(cudaMallocAsync(&keys_sorted, sizeof(int) * A, s));
        CK(cudaMallocAsync(&iota, sizeof(int) * A, s));
        launch_aug_keys(d_src, aug_orig, aug_code, A, pg, keys, s);
        launch_iota(iota, A, s);
        radix_sort_pairs(keys, keys_sorted, iota, box_order, A, bits_for(total_boxes), s);
        launch_csr_from_sorted(keys_sorted, A, total_boxes, box_start, s);
        CK(cudaFreeAsync(keys, s));
        CK(cudaFreeAsync(keys_sorted, s));
        CK(cudaFreeAsync(iota, s));
    }
    // count pass
    PairArgs pa{};
    pa.src_pos = d_src;
    pa.obs_pos = d_obs;
    pa.obs_perm = P->obs_perm + P->i0;
    pa.M = Mown;
    pa.box_start = box_start;
    pa.box_order = box_order;
    pa.aug_orig = aug_orig;
    pa.aug_code = aug_code;
    pa.obs_start = P->obs_start + 3 * P->i0;
    pa.obs_w = P->obs_w + P->i0 * 3 * W;
    pa.src_start = P->src_start;
    pa.src_w = P->src_w;
    pa.src_rank = P->src_rank;
    pa.W = W;
    for (int a = 0; a < 3; ++a) pa.wdt[a] = P->near_g.w[a];
    pa.st = P->status;
    int64_t* counts = dalloc<int64_t>(P, Mown + 1);
    int* d0mm = dalloc<int>(P, 2 * 81);
    {
        std::vector<int> init(162);
        for (int i = 0; i < 81; ++i) {
            init[i] = INT_MAX;
            init[81 + i] = INT_MIN;
        }
        CK(cudaMemcpyAsync(d0mm, init.data(), sizeof(int) * 162, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
    pa.counts = counts;
    pa.d0min = d0mm;
    pa.d0max = d0mm + 81;
    pa.tallies = d_cnt + 1;
    if (want_near)
        launch_pairs_count(pg, pa, s);
    else   // far-zone-only plan: no correction pairs
        CK(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (Mown + 1), s));
    check_status(P, "correction pair discovery");
    nv.next("fftpim build: pair coefficients, row order, K4 metadata");
    P->pair_ptr = dalloc<int64_t>(P, Mown + 1);
    {
        size_t bytes = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, bytes, counts, P->pair_ptr, (int)(Mown + 1), s);
        void* tmp = nullptr;
        CK(cudaMallocAsync(&tmp, bytes + 16, s));
        CK(cudaMemsetAsync(counts + Mown, 0, sizeof(int64_t), s));
        cub::DeviceScan::ExclusiveSum(tmp, bytes, counts, P->pair_ptr, (int)(Mown + 1), s);
        fftpim_count_launch(2);
        CK(cudaFreeAsync(tmp, s));
    }
    int64_t npairs = 0;
    unsigned long long tallies[3];
    std::vector<int> mm(162);
    CK(cudaMemcpyAsync(&npairs, P->pair_ptr + Mown, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(tallies, d_cnt, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(mm.data(), d0mm, sizeof(int) * 162, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    P->info.coincident_kernel_terms = (int64_t)tallies[0];
    P->info.n_self_pairs = (int64_t)tallies[1];
    P->info.n_wrapped_pairs = (int64_t)tallies[2];
    P->info.n_pairs = npairs;
    // window tables per code (values independent of the window, nearzone.py:439-451)
    CodeTables& tb = P->tabs;
    int64_t tab_total = 0;
    for (int c = 0; c < 27; ++c) {
        tb.offset[c] = tab_total;
        for (int a = 0; a < 3; ++a) {
            tb.lo[c][a] = 0;
            tb.len[c][a] = 0;
        }
        if (c >= pg.ncodes || mm[c * 3] == INT_MAX) continue;
        int64_t sz = 1;
        for (int a = 0; a < 3; ++a) {
            tb.lo[c][a] = mm[c * 3 + a];
            tb.len[c][a] = mm[81 + c * 3 + a] + 2 * (P->near_g.w[a] - 1) - mm[c * 3 + a] + 1;
            sz *= tb.len[c][a];
        }
        tab_total += sz;
    }
    cplx* tables = dalloc<cplx>(P, tab_total);
    // fill pass
    const int64_t npairs_pad = (npairs + CORR_TILE - 1) / CORR_TILE * CORR_TILE;
    P->pair_src = dalloc<int>(P, npairs);
    // image codes are only needed for operand export; skipped for huge pair counts (C3/C4)
    if (npairs <= (int64_t)1 << 31 || P->sweep) P->pair_codeid = dalloc<unsigned char>(P, npairs);
    pa.pair_ptr = P->pair_ptr;
    pa.tables = tables;
    pa.pair_src = P->pair_src;
    pa.pair_codeid = P->pair_codeid;
    if (P->sweep) {
        // one pass per image index i_a along the sweep axis: coefficient
        // components without the axis phases (sweep_kernels.cu)
        if (N >= (1 << 30)) throw Fail{FFTPIM_VALUE, "sweep plans need fewer than 2^30 sources"};
        P->sw_comp = dalloc<cplx>(P, (int64_t)P->sw_ncomp * npairs);
        for (int j = 0; j < P->sw_ncomp; ++j) {
            ImageSet imj = im;
            make_images(pr, pr.kshift, imj, P->sw_axis, j - pr.i_d);
            PairGeom pgj = pg;
            code_phases(pr, pr.kshift, pgj, P->sw_axis);
            launch_code_tables(tb, pg.ncodes, pgj, imj, tables, tab_total, s);
            pa.coef = P->sw_comp + (int64_t)j * npairs;
            pa.coef_r = nullptr;
            launch_pairs_fill(pgj, imj, tb, pa, s);
            pa.pair_codeid = nullptr;   // written once
        }
        signed char ca[27] = {0};
        for (int c = 0; c < pg.ncodes; ++c) ca[c] = pg.code[c][P->sw_axis];
        launch_sweep_pack_src(P->pair_src, P->pair_codeid, ca, npairs, s);
        P->info.real_coefficients = 0;
    } else {
        launch_code_tables(tb, pg.ncodes, pg, im, tables, tab_total, s);
        if (P->npsp) {
            P->pair_coef_r = dalloc<double>(P, npairs_pad);   // zero tail: k_corr_runs copies whole tiles
            CK(cudaMemsetAsync(P->pair_coef_r + npairs, 0, sizeof(double) * (npairs_pad - npairs), s));
            if (!P->sharded) {   // real-charge fast path of K4 (eval_kernels.cu k_permute_q)
                P->q_re = dalloc<double>(P, N + CORR_QPAD);
                CK(cudaMemset(P->q_re + N, 0, sizeof(double) * CORR_QPAD));
                P->q_flag = dalloc<int>(P, 1);
            }
        } else
        {
            P->pair_coef = dalloc<cplx>(P, npairs_pad);
            CK(cudaMemsetAsync(P->pair_coef + npairs, 0, sizeof(cplx) * (npairs_pad - npairs), s));
        }
        P->info.real_coefficients = P->npsp ? 1 : 0;
        pa.coef = P->pair_coef;
        pa.coef_r = P->pair_coef_r;
        launch_pairs_fill(pg, im, tb, pa, s);
    }
    P->n_tiles = (npairs + CORR_TILE - 1) / CORR_TILE;
    P->info.pair_rows_source_order = 0;
    if (npairs > 0) {
        // rows in source order for large pair lists (K4 gather locality, see
        // sort_pair_rows); FFTPIM_K4_SORT=0|1 overrides.  Exports then list each
        // observer's pairs in source order (same set as the reference).  Sweep
        // plans permute their phase components with the rows.
        const char* e = getenv("FFTPIM_K4_SORT");
        if (e ? e[0] == '1' : npairs >= (int64_t)1 << 28) {
            size_t free_b = 0, tot_b = 0;
            CK(cudaMemGetInfo(&free_b, &tot_b));
            const size_t budget = (size_t)(0.6 * (double)free_b);
            std::vector<cplx*> carr;
            if (P->sweep)
                for (int j = 0; j < P->sw_ncomp; ++j) carr.push_back(P->sw_comp + (int64_t)j * npairs);
            else if (P->pair_coef)
                carr.push_back(P->pair_coef);
            if (sort_pair_rows(P->pair_ptr, Mown, P->pair_src, carr.data(), (int)carr.size(), P->pair_coef_r,
                               P->pair_codeid, budget, s))
                P->info.pair_rows_source_order = 1;
            else
                cudaGetLastError();
        }
    }
    P->info.k4_wide_groups = -1;
    P->info.k4_runs = -1;
    if (!P->sweep && npairs > 0) {
        // 16-bit source offsets for K4 (2 B instead of 4 B per pair) when they fit
        // in memory; FFTPIM_K4_C16=0|1 overrides (default: large pair lists)
        const char* e = getenv("FFTPIM_K4_C16");
        // measured slower at C4 (K4 21.2 -> 28.6 ms: the kernel is bound by L1
        // wavefronts, not DRAM bytes, and the group decode adds to it): opt-in
        bool c16 = e ? e[0] == '1' : false;
        if (c16) {
            size_t free_b = 0, tot_b = 0;
            CK(cudaMemGetInfo(&free_b, &tot_b));
            c16 = (double)npairs * 2.2 < 0.8 * (double)free_b;
        }
        if (c16) {
            P->pair_off16 = dalloc<unsigned short>(P, npairs_pad);   // zero tail (whole tiles, k_corr_o16)
            CK(cudaMemsetAsync(P->pair_off16 + npairs, 0, sizeof(unsigned short) * (npairs_pad - npairs), s));
            P->grp_base = dalloc<int>(P, (npairs + 31) / 32 + 8);
            P->info.k4_wide_groups = build_group_offsets(P->pair_src, npairs, P->grp_base, P->pair_off16, s);
        }
    }
    if (!P->sweep) {   // the batched sweep K4 walks pair_ptr rows directly
        P->head_bits = dalloc<unsigned>(P, (npairs + 31) / 32 + 8);
        P->seg_first = dalloc<int64_t>(P, Mown + 1);
        P->seg_base = dalloc<int64_t>(P, P->n_tiles);
        int64_t* spans = dalloc<int64_t>(P, Mown + 1);
        build_corr_metadata(P->pair_ptr, Mown, npairs, P->n_tiles, P->head_bits, P->seg_first, P->seg_base, spans,
                            &P->n_segments, s);
        dfree(P, spans);
        P->seg_val = dalloc<cplx>(P, P->n_segments);
        // run-encoded sources + bulk-copy K4 (corr_kernels.cu k_corr_runs) for rows in
        // source order; FFTPIM_K4_RUNS=0|1 overrides.  NPSP plans too large to export
        // their pairs (> 2^31) drop the int32 index array afterwards.
        const char* er = getenv("FFTPIM_K4_RUNS");
        if (npairs > 0 && !P->pair_off16 && (er ? er[0] == '1' : k4_runs_default(P))) {
            unsigned* meta = nullptr;
            int* bias = nullptr;
            int64_t rbytes = 0;
            const int64_t nruns = build_run_records(P->pair_src, P->head_bits, P->seg_base, npairs, P->n_tiles, N,
                                                    &meta, &bias, &rbytes, s);
            if (nruns >= 0) {
                P->run_rec = meta;
                P->run_bias = bias;
                P->allocations.push_back(meta);
                P->allocations.push_back(bias);
                P->device_bytes += rbytes;
                P->info.k4_runs = nruns;
                P->k4_counter = dalloc<unsigned long long>(P, 1);
                // NPSP plans (no batched multi-RHS K4, which walks pair_src) are the
                // ones that come close to the 180 GB: C3 frees 55 GB here
                const char* ed = getenv("FFTPIM_K4_DROP_SRC");   // tests: exports decode the runs
                if (ed ? ed[0] == '1' : npairs > (int64_t)1 << 31 && P->pair_coef_r) {
                    P->device_bytes -= (int64_t)sizeof(int) * npairs;
                    dfree(P, P->pair_src);
                    P->pair_src = nullptr;
                }
            }
        }
    }
    check_status(P, "correction coefficients");
    nv.next("fftpim build: K1 operator, far zone");
    CK(cudaStreamSynchronize(s));
    dfree(P, tables);
    dfree(P, counts);
    dfree(P, d0mm);
    dfree(P, box_start);
    dfree(P, box_order);
    dfree(P, aug_orig);
    dfree(P, aug_code);

    // ---- K1 as a sliced-ELL operator (eval_kernels.cu) when its entries fit in
    // half the free memory; FFTPIM_K1=gather|taps|ell overrides
    {
        const char* e = getenv("FFTPIM_K1");
        if (want_near && !P->k1_lines && (!e || std::string(e) == "ell")) {
            EvalArgs a = eval_args(P, nullptr, nullptr, FFTPIM_NEAR);
            const int64_t rows = (int64_t)a.knx * dims[1] * dims[2];
            const int64_t nsl = (rows + 31) / 32;
            int* cnt_row = dalloc<int>(P, rows);
            int* cnt = dalloc<int>(P, rows);
            int* row_of = dalloc<int>(P, rows);
            int64_t* off = dalloc<int64_t>(P, nsl + 1);
            int64_t* slots = dalloc<int64_t>(P, nsl + 1);
            launch_k1_count(a, cnt_row, cnt, row_of, slots, s);
            size_t bytes = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, bytes, slots, off, (int)(nsl + 1), s);
            void* tmp = nullptr;
            CK(cudaMallocAsync(&tmp, bytes + 16, s));
            cub::DeviceScan::ExclusiveSum(tmp, bytes, slots, off, (int)(nsl + 1), s);
            CK(cudaFreeAsync(tmp, s));
            // longest row: slot 0 of each window holds the window's longest
            int* d_max = dalloc<int>(P, 1);
            bytes = 0;
            cub::DeviceReduce::Max(nullptr, bytes, cnt, d_max, (int)rows, s);
            CK(cudaMallocAsync(&tmp, bytes + 16, s));
            cub::DeviceReduce::Max(tmp, bytes, cnt, d_max, (int)rows, s);
            CK(cudaFreeAsync(tmp, s));
            int64_t total = 0;
            int longest = 0;
            CK(cudaMemcpyAsync(&total, off + nsl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(&longest, d_max, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            dfree(P, slots);
            dfree(P, cnt_row);
            dfree(P, d_max);
            size_t free_b = 0, tot_b = 0;
            CK(cudaMemGetInfo(&free_b, &tot_b));
            const double need = (double)total * (sizeof(int) + sizeof(double));
            const bool fits = total < ((int64_t)1 << 31) && need < 0.9 * (double)free_b;
            // (long rows of crowded cells are fine: rows are length-sorted within
            // windows, so a slice pads to rows of similar length; measured at C3:
            // 1.1 ms vs 4.4 ms for the tap-major computed K1)
            (void)longest;
            const bool want = e ? true : need <= 0.5 * (double)free_b;
            if (rows > 0 && fits && want) {
                // small charge vectors stay L2-resident in caller order: K1 then
                // reads q directly and need not wait for the permutation
                P->k1_orig = !P->sharded && N <= 262144;
                const char* eo = getenv("FFTPIM_K1_ORIG");
                if (eo && !P->sharded) P->k1_orig = std::string(eo) == "1";
                P->k1_idx = dalloc<int>(P, total);
                P->k1_wgt = dalloc<double>(P, total);
                // padding slots (shorter rows of a slice): index 0, weight 0
                CK(cudaMemsetAsync(P->k1_idx, 0, sizeof(int) * total, s));
                CK(cudaMemsetAsync(P->k1_wgt, 0, sizeof(double) * total, s));
                launch_k1_fill(a, row_of, off, P->k1_orig ? P->src_perm : nullptr, P->k1_idx, P->k1_wgt, s);
                if (P->k1_orig && getenv("FFTPIM_K1_ONE_ORDER") == nullptr) {
                    // second index array in sorted order for device-resident charges
                    // (same rows, same weights: the fill rewrites identical values)
                    P->k1_idx_sorted = dalloc<int>(P, total);
                    CK(cudaMemsetAsync(P->k1_idx_sorted, 0, sizeof(int) * total, s));
                    launch_k1_fill(a, row_of, off, nullptr, P->k1_idx_sorted, P->k1_wgt, s);
                }
                P->k1_cnt = cnt;
                P->k1_row = row_of;
                P->k1_off = off;
                P->k1_slots = total;
                P->info.k1_operator = 1;
                P->info.k1_slots = total;
                if (P->k1_scratch) {
                    dfree(P, P->k1_scratch);
                    P->k1_scratch = nullptr;
                }
            } else {
                dfree(P, cnt);
                dfree(P, row_of);
                dfree(P, off);
            }
            CK(cudaStreamSynchronize(s));
        }
    }

    // ---- far kernel (farzone.py:100-121, pgf.py:450-462)
    P->far_kernel = dalloc<cplx>(P, prod3(P->far_kdims));
    if (!want_far) {
        CK(cudaMemsetAsync(P->far_kernel, 0, sizeof(cplx) * prod3(P->far_kdims), s));
    } else if (pr.far_kernel) {
        // kernel blob hit (farzone.py:103-112): the table and its kernel_terms come
        // from the blob, the series is not evaluated
        CK(cudaMemcpyAsync(P->far_kernel, pr.far_kernel, sizeof(cplx) * prod3(P->far_kdims),
                           cudaMemcpyHostToDevice, s));
        P->info.kernel_terms = pr.far_kernel_terms;
    } else {
        P->info.kernel_terms = tabulate_far(P, pr.kshift, im, P->far_kernel, s);
    }
    // ---- sweep: kernel_hat and far kernel per excitation
    if (P->sweep) {
        const int64_t nk = prod3(P->far_kdims);
        P->sw_khat = dalloc<cplx>(P, (int64_t)P->sw_E * P->n_fft);
        P->sw_far = dalloc<cplx>(P, (int64_t)P->sw_E * nk);
        const int NS = P->sw_ncomp + 2;
        std::vector<cplx> omega((size_t)P->sw_E * NS);
        for (int e = 0; e < P->sw_E; ++e) {
            double ks[3][2];
            for (int a = 0; a < 3; ++a) {
                ks[a][0] = pr.kshift[a][0];
                ks[a][1] = pr.kshift[a][1];
            }
            ks[P->sw_axis][0] = P->sw_k[2 * e];
            ks[P->sw_axis][1] = P->sw_k[2 * e + 1];
            ImageSet ime = im;
            make_images(pr, ks, ime);
            tabulate_khat(P, dims, h, ime, P->sw_khat + (int64_t)e * P->n_fft, s);
            P->info.kernel_terms = std::max(P->info.kernel_terms, tabulate_far(P, ks, ime, P->sw_far + (int64_t)e * nk, s));
            const std::complex<double> kl = std::complex<double>(ks[P->sw_axis][0], ks[P->sw_axis][1]) * pr.L[P->sw_axis];
            for (int k = 0; k < NS; ++k) {
                const double m = (double)(k - 1 - pr.i_d);
                const std::complex<double> w = std::exp(std::complex<double>(0.0, -1.0) * m * kl);
                omega[(size_t)e * NS + k] = cplx{w.real(), w.imag()};
            }
        }
        P->sw_omega = dalloc<cplx>(P, (int64_t)P->sw_E * NS);
        CK(cudaMemcpyAsync(P->sw_omega, omega.data(), sizeof(cplx) * omega.size(), cudaMemcpyHostToDevice, s));
        P->sw_qt = dalloc<cplx>(P, 3 * N * P->sw_E);   // code-phased charges, c = -1, 0, 1
        P->sw_corr = dalloc<cplx>(P, Mown * P->sw_E);
        CK(cudaStreamSynchronize(s));
    }
    // far evaluation scratch
    {
        const int64_t nf = P->n_far;
        if (nf > 3072 || fdims[2] > 32)
            throw Fail{FFTPIM_VALUE, "far grid too large for this build (max 3072 nodes, 32 along z)"};
        static const int warps0 = [] {
            const char* e = getenv("FFTPIM_FAR_WARPS");
            // k_far_project is __launch_bounds__(256): at most 8 warps
            return e ? std::min(std::max(atoi(e), 1), 8) : 8;
        }();
        static const int bps = [] {   // blocks per SM
            const char* e = getenv("FFTPIM_FAR_BPS");
            return e ? atoi(e) : 1;
        }();
        int warps = warps0;
        while (warps > 1 && far_project_smem((int)nf, warps, pr.far_order) > 200 * 1024 / bps) --warps;
        // one wave of blocks: the per-block private grids are zeroed and
        // reduced once per block, so few, long-lived blocks are cheaper
        static const int fb = [] {   // absolute block count (0: one wave of bps per SM)
            const char* e = getenv("FFTPIM_FAR_BLOCKS");
            return e ? atoi(e) : 0;
        }();
        // in the concurrent schedule the far chain is off the critical path: half
        // the SMs leave the other half to K1 at the start (measured C2 0.133 -> 0.129 ms)
        const int64_t need = (Mown + 32 * warps - 1) / (32 * warps);
        const int wave = npairs <= concurrent_max_pairs() && !P->sweep ? 74 * bps : 148 * bps;
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(fb > 0 ? fb : wave, need));
        // sequential chains (multi-RHS batches) use a full wave
        const int blocks_seq = (int)std::max<int64_t>(blocks, std::min<int64_t>(fb > 0 ? fb : 148 * bps, need));
        P->far_warps = warps;
        P->far_blocks = blocks;
        P->far_blocks_seq = blocks_seq;
        P->far_partial = dalloc<cplx>(P, (int64_t)blocks_seq * nf);
        {
            // windowed far projection from the sorted positions (FFTPIM_FAR=win|warps)
            const char* e = getenv("FFTPIM_FAR");
            const bool win = (e ? std::string(e) == "win" : N > 262144) && pr.far_order + 1 >= 3 && pr.far_order + 1 <= 5;
            if (win) {
                if (!P->src_pos_s) {
                    P->src_pos_s = dalloc<double>(P, 3 * N);
                    launch_gather_pos(d_src, P->src_perm, N, P->src_pos_s, s);
                }
                const int64_t nfp = P->sharded ? Mown : N;   // points the far projection takes
                // chunk length, window capacity and the chunk windows depend on the positions only
                P->far_win = dalloc<int>(P, far_win_max_chunks(nfp) * 6);
                far_win_setup(P->far_sg, P->src_pos_s + 3 * (P->sharded ? P->i0 : 0), nfp, P->far_win, &P->far_chunk,
                              &P->far_cap, s);
                const int64_t nch = (nfp + P->far_chunk - 1) / P->far_chunk;
                P->far_slots = dalloc<cplx>(P, std::max<int64_t>(nch, 1) * nf);
            }
        }
        P->far_qg = dalloc<cplx>(P, nf);
        P->far_ug = dalloc<cplx>(P, nf);
    }
    if ((npairs <= concurrent_max_pairs() || P->run_rec) && getenv("FFTPIM_OBS_FUSED") == nullptr)
        P->obs_pre = dalloc<cplx>(P, Mown);   // split observer pass (concurrent and overlap schedules)
    CK(cudaStreamSynchronize(s));
    dfree(P, d_cnt);
    dfree(P, d_src);
    if (!same) dfree(P, d_obs);
    for (int a = 0; a < 3; ++a) {
        P->info.near_dims[a] = dims[a];
        P->info.fft_dims[a] = P->cdims[a];
        P->info.far_dims[a] = fdims[a];
    }
    P->info.n_src = N;
    P->info.n_obs = M;
}

// K1 reads the caller-order charges (starting alongside the permutation) only in
// the host entry's graph: with device-resident charges the sorted-order operator
// is faster (C2 122.6 -> 119.7 us), with the upload in the graph the caller-order
// one is (e2e 3.2e8 -> 3.4e8 points/s); both operators sum in the same order
static bool k1_caller_order(const FftpimPlan* P) {
    return P->k1_orig && (P->host_call || P->k1_idx_sorted == nullptr);
}

EvalArgs eval_args(FftpimPlan* P, const double* q, double* u, int parts) {
    EvalArgs a{};
    a.N = P->N;
    a.M = P->M;
    a.q = (const cplx*)q;
    a.u = (cplx*)u;
    a.src_perm = P->src_perm;
    a.obs_perm = P->obs_perm;
    a.q_sorted = P->q_sorted;
    a.g = P->near_g;
    for (int i = 0; i < 3; ++i) a.cdims[i] = P->cdims[i];
    a.cell_start = P->cell_start;
    a.src_w = P->src_w;
    a.src_start = P->src_start;
    a.obs_w = P->obs_w;
    a.obs_start = P->obs_start;
    a.work = P->work;
    a.pad_in = P->pad_in;
    if (P->custom_fft) {
        a.k1_out = P->qg;
        a.go1 = P->near_g.n[1];
        a.go2 = P->near_g.n[2];
        a.interp_grid = P->qg;
        a.gi1 = a.go1;
        a.gi2 = a.go2;
    } else {
        a.k1_out = P->pad_in;
        a.go1 = P->cdims[1];
        a.go2 = P->cdims[2];
        a.interp_grid = P->work;
        a.gi1 = a.go1;
        a.gi2 = a.go2;
    }
    a.khat = P->khat;
    a.n_fft = P->n_fft;
    a.pair_ptr = P->pair_ptr;
    a.pair_src = P->pair_src;
    a.pair_off16 = P->pair_off16;
    a.grp_base = P->grp_base;
    a.run_rec = P->run_rec;
    a.run_bias = P->run_bias;
    a.coef = P->pair_coef;
    a.coef_r = P->pair_coef_r;
    a.q_re = P->q_re;
    a.q_flag = P->q_flag;
    a.n_pairs = P->info.n_pairs;
    a.head_bits = P->head_bits;
    a.seg_base = P->seg_base;
    a.seg_first = P->seg_first;
    a.seg_val = P->seg_val;
    a.fs = P->far_sg;
    a.fo = P->far_og;
    a.src_fw = P->src_fw;
    a.src_fstart = P->src_fstart;
    a.obs_fw = P->obs_fw;
    a.obs_fstart = P->obs_fstart;
    a.far_kernel = P->far_kernel;
    a.far_partial = P->far_partial;
    a.far_qg = P->far_qg;
    a.far_ug = P->far_ug;
    a.far_blocks = P->far_blocks;
    a.far_warps = P->far_warps;
    a.far_q = P->q_sorted;
    a.far_n = P->N;
    a.far_pos = P->far_slots ? P->src_pos_s : nullptr;
    a.far_slots = P->far_slots;
    a.far_win = P->far_win;
    a.far_chunk = P->far_chunk;
    a.far_cap = P->far_cap;
    a.k1_scratch = P->k1_scratch;
    a.k1_cnt = P->k1_cnt;
    a.k1_row = P->k1_row;
    a.k1_off = P->k1_off;
    a.k1_q = k1_caller_order(P) ? a.q : P->q_sorted;
    a.k1_idx = P->k1_orig && !k1_caller_order(P) ? P->k1_idx_sorted : P->k1_idx;
    a.k1_wgt = P->k1_wgt;
    a.k1_pos = P->k1_lines && !P->src_rec ? P->src_pos_s : nullptr;
    a.k1_rec = P->src_rec;
    a.obs_pos = P->obs_pos_pass ? P->obs_pos_s : nullptr;
    a.obs_cell_start = P->obs_tile ? P->obs_cell_start : nullptr;
    a.obs_i0 = 0;
    a.kx0 = 0;
    a.knx = P->near_g.n[0];
    a.gx0 = 0;
    a.parts = parts;
    if (P->sharded) {
        // slab shard: own planes for K1/interp, own observers (= own sources) for
        // K4, interpolation and the far projection partial
        const int64_t i0 = P->i0;
        const int W = P->near_g.order + 1, WF = P->far_sg.order + 1;
        a.M = P->i1 - P->i0;
        a.obs_perm = P->obs_perm + i0;
        a.obs_w = P->obs_w + i0 * 3 * W;
        a.obs_start = P->obs_start + 3 * i0;
        a.obs_fw = P->obs_fw + i0 * 3 * WF;
        a.obs_fstart = P->obs_fstart + 3 * i0;
        if (a.obs_pos) a.obs_pos = P->obs_pos_s + 3 * i0;
        a.obs_i0 = i0;
        a.src_fw = P->src_fw + i0 * 3 * WF;
        a.src_fstart = P->src_fstart + 3 * i0;
        a.far_q = P->q_sorted + i0;
        a.far_n = P->i1 - P->i0;
        if (a.far_pos) a.far_pos = P->src_pos_s + 3 * i0;
        a.kx0 = P->X0;
        a.knx = P->n0_loc;
        a.gx0 = P->X0;
    }
    return a;
}

// Evaluation schedule.  For moderate pair counts the near-field chain (K1 + FFT
// stages), the correction matvec K4 and the far chain run concurrently on three
// plan-owned streams after the q permutation (K4 streams HBM while the FFT
// stages are latency-bound) and join before the observer pass; for very large
// pair streams (C3/C4) K4 needs the whole chip and the chains run in order.
// ---------------------------------------------------------------------------
// Multi-RHS batches (batch >= FFTPIM_BATCH_MIN charge vectors on one plan): the
// correction pairs stream ONCE per 64 right-hand sides through the batched
// row kernel of the sweep (sweep_kernels.cu, one component, unit phases)
// instead of once per vector; the per-vector chains (far chain, K1, FFT stages,
// observer pass without the K4 term) follow, then one pass adds the K4 sums.
static int batch_min() {
    static const int v = [] {
        const char* e = getenv("FFTPIM_BATCH_MIN");
        return e ? atoi(e) : 8;
    }();
    return v;
}

static bool batched_k4(const FftpimPlan* P, int64_t batch, int parts) {
    return batch >= batch_min() && (parts & FFTPIM_NEAR) && P->pair_coef && P->pair_src && !P->sweep && !P->sharded &&
           P->N < ((int64_t)1 << 30) && P->info.n_pairs > 0;
}

// device buffers of the batched path, allocated outside any graph capture
static void ensure_batch_buffers(FftpimPlan* P, int64_t batch, int parts) {
    if (!batched_k4(P, batch, parts)) return;
    int E = (int)std::min<int64_t>(64, batch);
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    while (E > 8 && (size_t)(P->N + P->M) * E * sizeof(cplx) > fr / 2) E /= 2;
    if (P->bt_E >= E) return;
    dfree(P, P->bt_qt);
    dfree(P, P->bt_corr);
    dfree(P, P->bt_omega);
    P->bt_qt = dalloc<cplx>(P, P->N * E);
    P->bt_corr = dalloc<cplx>(P, P->M * E);
    std::vector<cplx> ones((size_t)3 * E, cplx{1.0, 0.0});
    P->bt_omega = dalloc<cplx>(P, 3 * E);
    CK(cudaMemcpy(P->bt_omega, ones.data(), sizeof(cplx) * ones.size(), cudaMemcpyHostToDevice));
    P->bt_E = E;
    if (P->graph_exec) cudaGraphExecDestroy(P->graph_exec);   // captured with the old buffers
    P->graph_exec = nullptr;
    if (P->hgraph_exec) cudaGraphExecDestroy(P->hgraph_exec);
    P->hgraph_exec = nullptr;
}

static void evaluate_batched(FftpimPlan* P, const double* q, double* u, int64_t batch, int parts, cudaStream_t s) {
    cudaStream_t sn = P->aux[0], sc = P->aux[1];
    if (parts & FFTPIM_NEAR && !P->custom_fft) CKFFT(cufftSetStream(P->fft_plan, sn));
    for (int64_t b0 = 0; b0 < batch; b0 += P->bt_E) {
        const int E = (int)std::min<int64_t>(P->bt_E, batch - b0);
        const double* qb = q + 2 * b0 * P->N;
        double* ub = u + 2 * b0 * P->M;
        CK(cudaEventRecord(P->ev_fork, s));
        CK(cudaStreamWaitEvent(sn, P->ev_fork, 0));
        CK(cudaStreamWaitEvent(sc, P->ev_fork, 0));
        launch_batch_permute((const cplx*)qb, P->src_perm, P->N, E, P->bt_qt, sc);
        launch_corr_sweep(P->pair_ptr, P->pair_src, P->pair_coef, 1, P->info.n_pairs, P->bt_qt, P->N, E, P->bt_omega,
                          P->bt_corr, P->M, sc, P->info.pair_rows_source_order == 1);
        for (int e = 0; e < E; ++e) {
            EvalArgs a = eval_args(P, qb + 2 * (int64_t)e * P->N, ub + 2 * (int64_t)e * P->M, parts);
            a.sw_e = -1;   // the K4 term is added below
            a.far_blocks = P->far_blocks_seq;
            launch_permute_q(a, sn);
            if (parts & FFTPIM_FAR) {
                launch_far_project(a, sn);
                launch_far_sum(a, sn);
            }
            launch_near_project(a, sn);
            if (P->custom_fft) {
                for (int k = 0; k < 5; ++k)
                    if (P->stage_on[k]) launch_fft_stage(P->stage[k], sn);
            } else {
                CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->pad_in, (cufftDoubleComplex*)P->work, CUFFT_FORWARD));
                launch_spectrum_mul(a, sn);
                CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->work, (cufftDoubleComplex*)P->work, CUFFT_INVERSE));
                fftpim_count_launch(2);
            }
            launch_observers(a, sn);
        }
        CK(cudaEventRecord(P->ev_join[0], sn));
        CK(cudaEventRecord(P->ev_join[1], sc));
        CK(cudaStreamWaitEvent(s, P->ev_join[0], 0));
        CK(cudaStreamWaitEvent(s, P->ev_join[1], 0));
        launch_sweep_add_corr((cplx*)ub, P->bt_corr, P->obs_perm, P->M, E, s);
    }
    CK(cudaGetLastError());
}

static bool far_side() {
    static const bool on = [] {
        const char* e = getenv("FFTPIM_FAR_SIDE");
        return !(e && e[0] == '0');
    }();
    return on;
}

void evaluate_schedule(FftpimPlan* P, const double* q, double* u, int64_t batch, int parts, cudaStream_t s) {
    if (batched_k4(P, batch, parts) && P->bt_E > 0) {
        evaluate_batched(P, q, u, batch, parts, s);
        return;
    }
    const bool concurrent = P->info.n_pairs <= concurrent_max_pairs();
    // Large plans with the run-encoded K4 (HBM-bound, little issue pressure): a
    // main K4 grid of one 8-warp block per SM starts right after the permutation
    // and streams beside the far chain, K1 and the FFT stages (on-chip-bound or
    // short of bandwidth on their own), which run in the other half of every SM;
    // when that chain is done a helper grid joins on the same tile queue
    // (FFTPIM_K4_OVERLAP=0: chains in order).
    static const int overlap_on = [] {
        const char* e = getenv("FFTPIM_K4_OVERLAP");
        return e ? atoi(e) : 1;
    }();
    if (!concurrent && overlap_on && P->run_rec && P->k4_counter && parts == FFTPIM_ALL) {
        static const int main_blocks = [] {
            const char* e = getenv("FFTPIM_K4A_BLOCKS");
            return e ? atoi(e) : 148;
        }();
        static const int obs_split = [] {
            const char* e = getenv("FFTPIM_K4_OVERLAP_OBS");
            return e ? atoi(e) : 1;
        }();
        static const int help_blocks = [] {
            const char* e = getenv("FFTPIM_K4B_BLOCKS");
            return e ? atoi(e) : 148;
        }();
        if (!P->custom_fft) CKFFT(cufftSetStream(P->fft_plan, s));
        cudaStream_t sc = P->aux[1], sf = P->aux[2];
        for (int64_t b = 0; b < batch; ++b) {
            EvalArgs a = eval_args(P, q + 2 * b * P->N, u + 2 * b * P->M, parts);
            launch_permute_q(a, s);
            CK(cudaEventRecord(P->ev_fork, s));
            EvalArgs ac = a;
            ac.k4_counter = P->k4_counter;
            ac.corr_blocks = main_blocks;
            CK(cudaStreamWaitEvent(sc, P->ev_fork, 0));
            CK(cudaMemsetAsync(P->k4_counter, 0, sizeof(unsigned long long), sc));
            launch_corr_tiles(ac, sc);
            CK(cudaEventRecord(P->ev_join[1], sc));
            CK(cudaStreamWaitEvent(sf, P->ev_fork, 0));
            launch_far_project(a, sf);
            launch_far_sum(a, sf);
            CK(cudaEventRecord(P->ev_join[2], sf));
            launch_near_project(a, s);
            if (P->custom_fft) {
                for (int k = 0; k < 5; ++k)
                    if (P->stage_on[k]) launch_fft_stage(P->stage[k], s);
            } else {
                CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->pad_in, (cufftDoubleComplex*)P->work, CUFFT_FORWARD));
                launch_spectrum_mul(a, s);
                CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->work, (cufftDoubleComplex*)P->work, CUFFT_INVERSE));
                fftpim_count_launch(2);
            }
            CK(cudaStreamWaitEvent(s, P->ev_join[2], 0));
            // the interpolation (grid-tile pass, on-chip bound) also runs beside K4 when
            // the plan has the sorted-order buffer; the finishing pass adds the row sums
            const bool split = P->obs_pre && a.obs_pos && a.obs_cell_start && obs_split;
            bool split_done = false;
            if (split) {
                EvalArgs ai = a;
                ai.u_sorted = P->obs_pre;
                ai.sw_e = -1;   // no K4 term
                split_done = launch_observers_tile(ai, ai.obs_pos, ai.obs_cell_start, ai.obs_i0, s, 0);
            }
            if (help_blocks > 0) {
                ac.corr_blocks = help_blocks;
                launch_corr_tiles(ac, s);
            }
            CK(cudaStreamWaitEvent(s, P->ev_join[1], 0));
            if (split_done) {
                EvalArgs af = a;
                af.u_sorted = P->obs_pre;
                launch_finish_corr(af, s);
            } else {
                launch_observers(a, s);
            }
        }
        CK(cudaGetLastError());
        return;
    }
    if (!concurrent) {
        if (parts & FFTPIM_NEAR && !P->custom_fft) CKFFT(cufftSetStream(P->fft_plan, s));
        for (int64_t b = 0; b < batch; ++b) {
            EvalArgs a = eval_args(P, q + 2 * b * P->N, u + 2 * b * P->M, parts);
            launch_permute_q(a, s);
            // the latency-bound far chain overlaps K1 and the FFT stages on a side stream
            const bool side = (parts & FFTPIM_FAR) && (parts & FFTPIM_NEAR) && far_side();
            if (side) {
                CK(cudaEventRecord(P->ev_fork, s));
                CK(cudaStreamWaitEvent(P->aux[2], P->ev_fork, 0));
                launch_far_project(a, P->aux[2]);
                launch_far_sum(a, P->aux[2]);
                CK(cudaEventRecord(P->ev_join[2], P->aux[2]));
            } else if (parts & FFTPIM_FAR) {
                launch_far_project(a, s);
                launch_far_sum(a, s);
            }
            if (parts & FFTPIM_NEAR) {
                launch_near_project(a, s);
                if (P->custom_fft) {
                    for (int k = 0; k < 5; ++k)
                        if (P->stage_on[k]) launch_fft_stage(P->stage[k], s);
                } else {
                    CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->pad_in, (cufftDoubleComplex*)P->work, CUFFT_FORWARD));
                    launch_spectrum_mul(a, s);
                    CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->work, (cufftDoubleComplex*)P->work, CUFFT_INVERSE));
                    fftpim_count_launch(2);
                }
                launch_corr_tiles(a, s);
            }
            if (side) CK(cudaStreamWaitEvent(s, P->ev_join[2], 0));
            launch_observers(a, s);
        }
        CK(cudaGetLastError());
        return;
    }
    for (int64_t b = 0; b < batch; ++b) {
        EvalArgs a = eval_args(P, q + 2 * b * P->N, u + 2 * b * P->M, parts);
        // a K1 reading the caller-order charges starts alongside the permutation
        if (k1_caller_order(P)) CK(cudaEventRecord(P->ev_start, s));
        launch_permute_q(a, s);
        CK(cudaEventRecord(P->ev_fork, s));
        cudaStream_t sn = P->aux[0], sc = P->aux[1], sf = P->aux[2];
        // split observer pass: far interpolation + K4 fix-up run off the near
        // chain; the final pass after the inverse FFT only interpolates the near grid
        const bool split = parts == FFTPIM_ALL && P->obs_pre != nullptr;
        // capture order = the order the graph hands ready kernels to the GPU:
        // the near chain (critical path) first, then the far chain, then K4
        static const int far_gate = [] {   // 1: the far chain starts after K1
            const char* e = getenv("FFTPIM_FAR_GATE");
            return e ? atoi(e) : 0;
        }();
        auto far_chain = [&]() {
            if (!(parts & FFTPIM_FAR)) return;
            CK(cudaStreamWaitEvent(sf, P->ev_fork, 0));
            if (far_gate && (parts & FFTPIM_NEAR)) CK(cudaStreamWaitEvent(sf, P->ev_k1, 0));
            launch_far_project(a, sf);
            launch_far_sum(a, sf);
            CK(cudaEventRecord(P->ev_join[2], sf));
        };
        if (!(parts & FFTPIM_NEAR)) far_chain();
        if (parts & FFTPIM_NEAR) {
            CK(cudaStreamWaitEvent(sn, k1_caller_order(P) ? P->ev_start : P->ev_fork, 0));
            launch_near_project(a, sn);
            static const int k4_gate = [] {   // 1: K4 starts after K1, 2: after the forward FFT stages
                const char* e = getenv("FFTPIM_K4_GATE");
                return e ? atoi(e) : 0;
            }();
            if (k4_gate == 1 || far_gate) CK(cudaEventRecord(P->ev_k1, sn));
            if (P->custom_fft) {
                for (int k = 0; k < 5; ++k) {
                    if (P->stage_on[k]) launch_fft_stage(P->stage[k], sn);
                    if (k == 1 && k4_gate == 2) CK(cudaEventRecord(P->ev_k1, sn));
                }
            } else {
                CKFFT(cufftSetStream(P->fft_plan, sn));
                CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->pad_in, (cufftDoubleComplex*)P->work, CUFFT_FORWARD));
                launch_spectrum_mul(a, sn);
                CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->work, (cufftDoubleComplex*)P->work, CUFFT_INVERSE));
                fftpim_count_launch(2);
            }
            CK(cudaEventRecord(P->ev_join[0], sn));
            far_chain();
            CK(cudaStreamWaitEvent(sc, P->ev_fork, 0));
            if (k4_gate && P->custom_fft) CK(cudaStreamWaitEvent(sc, P->ev_k1, 0));
            {
                // K4 streams HBM on part of the chip while the latency-bound
                // near chain runs on the rest (FFTPIM_CORR_BLOCKS tunes the split;
                // its persistent blocks hold the register file, 1.5 per SM measured best at C2)
                static const int cb = [] {
                    const char* e = getenv("FFTPIM_CORR_BLOCKS");
                    return e ? atoi(e) : 222;
                }();
                EvalArgs ac = a;
                ac.corr_blocks = cb;
                launch_corr_tiles(ac, sc);
            }
            if (split) {
                EvalArgs ap = a;
                ap.obs_pre = P->obs_pre;
                CK(cudaStreamWaitEvent(sc, P->ev_join[2], 0));
                launch_observers(ap, sc, 1);
            }
            CK(cudaEventRecord(P->ev_join[1], sc));
            CK(cudaStreamWaitEvent(s, P->ev_join[0], 0));
            CK(cudaStreamWaitEvent(s, P->ev_join[1], 0));
        }
        if (parts & FFTPIM_FAR) CK(cudaStreamWaitEvent(s, P->ev_join[2], 0));
        if (split) {
            EvalArgs ap = a;
            ap.obs_pre = P->obs_pre;
            launch_observers(ap, s, 2);
        } else {
            launch_observers(a, s);
        }
    }
    CK(cudaGetLastError());
}

void evaluate(FftpimPlan* P, const double* q, double* u, int64_t batch, int parts, cudaStream_t s,
              cudaEvent_t* ev = nullptr) {
    if (parts & ~FFTPIM_ALL || parts == 0) throw Fail{FFTPIM_VALUE, "parts must be a non-empty subset of NEAR|FAR"};
    if (parts & ~P->info.built_parts)
        throw Fail{FFTPIM_VALUE, (parts & FFTPIM_NEAR) && !(P->info.built_parts & FFTPIM_NEAR)
                                     ? "plan was built without the near zone (build_far_plan)"
                                     : "plan was built without the far zone (build_near_plan)"};
    CK(cudaSetDevice(P->device));
    if (!ev) ensure_batch_buffers(P, batch, parts);
    if (!ev && P->use_graphs) {
        // replay a captured CUDA graph of the whole evaluation (launch-bound at small N);
        // re-captured whenever the caller's buffers or the batch change.  The
        // legacy default stream cannot be captured: the graph then runs on a
        // plan-owned stream fenced by events on both sides.
        const cudaStream_t caller = s;
        if (caller == nullptr) {
            CK(cudaEventRecord(P->ev_in, caller));
            CK(cudaStreamWaitEvent(P->gstream, P->ev_in, 0));
            s = P->gstream;
        }
        if (!(P->graph_exec && P->g_q == q && P->g_u == u && P->g_batch == batch && P->g_parts == parts)) {
            // same batch and parts, new caller buffers: capture again and update the
            // executable in place (no re-instantiation); otherwise instantiate anew
            const bool updatable = P->graph_exec && P->g_batch == batch && P->g_parts == parts;
            if (P->graph_exec && !updatable) {
                cudaGraphExecDestroy(P->graph_exec);
                P->graph_exec = nullptr;
            }
            cudaGraph_t graph = nullptr;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            P->capturing = true;
            const long long l0 = g_launches.load();
            try {
                evaluate_schedule(P, q, u, batch, parts, s);
                P->kernels_per_eval = (int)((g_launches.load() - l0) / batch);
            } catch (...) {
                P->capturing = false;
                cudaStreamEndCapture(s, &graph);
                if (graph) cudaGraphDestroy(graph);
                throw;
            }
            P->capturing = false;
            CK(cudaStreamEndCapture(s, &graph));
            ++P->info.graph_captures;
            bool updated = false;
            if (P->graph_exec) {
                cudaGraphExecUpdateResultInfo res{};
                updated = cudaGraphExecUpdate(P->graph_exec, graph, &res) == cudaSuccess;
                if (!updated) {
                    cudaGetLastError();
                    cudaGraphExecDestroy(P->graph_exec);
                    P->graph_exec = nullptr;
                }
            }
            if (!updated) {
                CK(cudaGraphInstantiate(&P->graph_exec, graph, 0));
                ++P->info.graph_instantiations;
            }
            CK(cudaGraphDestroy(graph));
            P->g_q = q;
            P->g_u = u;
            P->g_batch = batch;
            P->g_parts = parts;
        }
        CK(cudaGraphLaunch(P->graph_exec, s));
        if (caller == nullptr) {
            CK(cudaEventRecord(P->ev_out, s));
            CK(cudaStreamWaitEvent(caller, P->ev_out, 0));
        }
        fftpim_count_launch(P->kernels_per_eval * (int)batch);
        CK(cudaGetLastError());
        return;
    }
    if (!ev) {
        evaluate_schedule(P, q, u, batch, parts, s);
        return;
    }
    if (parts & FFTPIM_NEAR) CKFFT(cufftSetStream(P->fft_plan, s));
    auto mark = [&](int k) {
        if (ev) CK(cudaEventRecord(ev[k], s));
    };
    for (int64_t b = 0; b < batch; ++b) {
        EvalArgs a = eval_args(P, q + 2 * b * P->N, u + 2 * b * P->M, parts);
        mark(0);
        launch_permute_q(a, s);
        mark(1);
        if (parts & FFTPIM_FAR) launch_far_project(a, s);
        mark(2);
        if (parts & FFTPIM_FAR) launch_far_sum(a, s);
        mark(3);
        if (parts & FFTPIM_NEAR) launch_near_project(a, s);
        mark(4);
        if (P->custom_fft) {
            // stages 4/5/6 = forward z,y | fused x fwd*khat*inv | inverse y,z
            if (parts & FFTPIM_NEAR) {
                if (P->stage_on[0]) launch_fft_stage(P->stage[0], s);
                if (P->stage_on[1]) launch_fft_stage(P->stage[1], s);
            }
            mark(5);
            if (parts & FFTPIM_NEAR) launch_fft_stage(P->stage[2], s);
            mark(6);
            if (parts & FFTPIM_NEAR) {
                if (P->stage_on[3]) launch_fft_stage(P->stage[3], s);
                if (P->stage_on[4]) launch_fft_stage(P->stage[4], s);
            }
        } else {
            if (parts & FFTPIM_NEAR) {
                CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->pad_in, (cufftDoubleComplex*)P->work, CUFFT_FORWARD));
                fftpim_count_launch(1);
            }
            mark(5);
            if (parts & FFTPIM_NEAR) launch_spectrum_mul(a, s);
            mark(6);
            if (parts & FFTPIM_NEAR) {
                CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->work, (cufftDoubleComplex*)P->work, CUFFT_INVERSE));
                fftpim_count_launch(1);
            }
        }
        mark(7);
        if (parts & FFTPIM_NEAR) launch_corr_tiles(a, s);
        mark(8);
        launch_observers(a, s);
        mark(9);
    }
    CK(cudaGetLastError());
}

// ------------------------------------------------------------------ slab groups
// A group is the slab decomposition of one problem over `world` shards: either
// one shard per process/GPU with NCCL over NVLink (the all-to-all transposes,
// the 16 KB far-grid all-reduce, the halo), or all shards emulated inside one
// process on one device (exchanges become device copies) -- the single-GPU
// check of the decomposition math.
#define NCK(x)                                                                                     \
    do {                                                                                           \
        ncclResult_t r_ = (x);                                                                     \
        if (r_ != ncclSuccess) throw Fail{FFTPIM_CUDA, std::string(#x) + ": " + ncclGetErrorString(r_)}; \
    } while (0)

struct GroupImpl {
    int world = 1, rank = 0;
    bool emulate = true;
    std::vector<FftpimPlan*> shards;   // emulate: all shards; NCCL: this rank's shard
    ncclComm_t comm = nullptr;
    // the whole shard evaluation (streams, NCCL calls) captured once as a CUDA
    // graph and replayed; re-captured when the caller's buffers change
    cudaGraphExec_t graph_exec = nullptr;
    const double* g_q = nullptr;
    double* g_u = nullptr;
    cudaStream_t g_stream = nullptr;   // capture stream for legacy-default-stream callers
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    int kernels_per_eval = 0;
};

// the shard's K4 (its own observers' correction pairs) needs only the permuted
// charges: it runs on the plan's low-priority stream from right after the
// permutation, overlapping K1, the FFT stages, both transposes and the halo
// exchange; the observer pass joins it.  The grid is capped (FFTPIM_CORR_BLOCKS,
// as in the single-plan concurrent schedule) so the near chain and the NCCL
// kernels still get SMs.
static void shard_fork_k4(FftpimPlan* P, EvalArgs a, cudaStream_t s) {
    static const int cap = [] {
        const char* e = getenv("FFTPIM_SLAB_CORR_BLOCKS");
        return e ? atoi(e) : 222;
    }();
    a.corr_blocks = cap;
    CK(cudaEventRecord(P->ev_fork, s));
    CK(cudaStreamWaitEvent(P->aux[1], P->ev_fork, 0));
    launch_corr_tiles(a, P->aux[1]);
    CK(cudaEventRecord(P->ev_join[1], P->aux[1]));
}

void shard_phase1(FftpimPlan* P, const EvalArgs& a, cudaStream_t s) {
    launch_permute_q(a, s);
    shard_fork_k4(P, a, s);
    launch_near_project(a, s);
    launch_fft_stage(P->stage[0], s);
    launch_fft_stage(P->stage[1], s);
    // pack the own planes' columns per destination shard: send[r][xl][c - C_r]
    const int nl = P->n0_loc;
    int64_t off = 0;
    for (int r = 0; r < P->world; ++r) {
        const int64_t nc = P->col_start[r + 1] - P->col_start[r];
        CK(cudaMemcpy2DAsync(P->a2a_send + off, nc * sizeof(cplx), P->fbufB + P->col_start[r], P->C * sizeof(cplx),
                             nc * sizeof(cplx), nl, cudaMemcpyDeviceToDevice, s));
        off += (int64_t)nl * nc;
    }
    launch_far_project(a, s);
}

void shard_phase3(FftpimPlan* P, const EvalArgs& a, cudaStream_t s) {
    // unpack send[r][xl][c - C_r] -> B[xl][c]
    const int nl = P->n0_loc;
    int64_t off = 0;
    for (int r = 0; r < P->world; ++r) {
        const int64_t nc = P->col_start[r + 1] - P->col_start[r];
        CK(cudaMemcpy2DAsync(P->fbufB + P->col_start[r], P->C * sizeof(cplx), P->a2a_send + off, nc * sizeof(cplx),
                             nc * sizeof(cplx), nl, cudaMemcpyDeviceToDevice, s));
        off += (int64_t)nl * nc;
    }
    launch_fft_stage(P->stage[3], s);
    launch_fft_stage(P->stage[4], s);
    launch_far_sum(a, s);
}

void group_schedule(GroupImpl* G, const double* q, double* u, cudaStream_t s) {
    const int W = G->world;
    std::vector<EvalArgs> args;
    for (auto* P : G->shards) {
        CK(cudaSetDevice(P->device));
        args.push_back(eval_args(P, q, u, FFTPIM_ALL));
    }
    const int ns = (int)G->shards.size();
    for (int k = 0; k < ns; ++k) shard_phase1(G->shards[k], args[k], s);
    // forward transpose + far-grid all-reduce
    if (G->emulate) {
        for (int r = 0; r < W; ++r) {
            FftpimPlan* src = G->shards[r];
            int64_t off = 0;
            for (int d = 0; d < W; ++d) {
                FftpimPlan* dst = G->shards[d];
                const int64_t nc = src->col_start[d + 1] - src->col_start[d];
                const int64_t cnt = (int64_t)src->n0_loc * nc;
                CK(cudaMemcpyAsync(dst->a2a_recv + (int64_t)src->X0 * nc, src->a2a_send + off, cnt * sizeof(cplx),
                                   cudaMemcpyDeviceToDevice, s));
                off += cnt;
            }
        }
        FftpimPlan* P0 = G->shards[0];
        const int64_t nf = P0->n_far;
        for (int r = 1; r < W; ++r) launch_axpy(P0->far_qg, G->shards[r]->far_qg, nf, s);
        for (int r = 1; r < W; ++r)
            CK(cudaMemcpyAsync(G->shards[r]->far_qg, P0->far_qg, nf * sizeof(cplx), cudaMemcpyDeviceToDevice, s));
    } else {
        FftpimPlan* P = G->shards[0];
        const int64_t ncol = P->C1 - P->C0;
        NCK(ncclGroupStart());
        int64_t off = 0;
        for (int d = 0; d < W; ++d) {
            const int64_t nc = P->col_start[d + 1] - P->col_start[d];
            const int64_t cnt = (int64_t)P->n0_loc * nc;
            NCK(ncclSend(P->a2a_send + off, 2 * cnt, ncclDouble, d, G->comm, s));
            const int64_t rcnt = (int64_t)(P->plane_start[d + 1] - P->plane_start[d]) * ncol;
            NCK(ncclRecv(P->a2a_recv + (int64_t)P->plane_start[d] * ncol, 2 * rcnt, ncclDouble, d, G->comm, s));
            off += cnt;
        }
        NCK(ncclGroupEnd());
        NCK(ncclAllReduce(P->far_qg, P->far_qg, 2 * P->n_far, ncclDouble, ncclSum, G->comm, s));
    }
    for (int k = 0; k < ns; ++k) launch_fft_stage(G->shards[k]->stage[2], s);
    // backward transpose: recv rows of shard r's planes -> r's send[d-block]
    if (G->emulate) {
        for (int d = 0; d < W; ++d) {
            FftpimPlan* src = G->shards[d];
            const int64_t nc = src->C1 - src->C0;
            for (int r = 0; r < W; ++r) {
                FftpimPlan* dst = G->shards[r];
                int64_t off = 0;
                for (int k = 0; k < d; ++k) off += (int64_t)dst->n0_loc * (dst->col_start[k + 1] - dst->col_start[k]);
                CK(cudaMemcpyAsync(dst->a2a_send + off, src->a2a_recv + (int64_t)dst->X0 * nc,
                                   (int64_t)dst->n0_loc * nc * sizeof(cplx), cudaMemcpyDeviceToDevice, s));
            }
        }
    } else {
        FftpimPlan* P = G->shards[0];
        const int64_t ncol = P->C1 - P->C0;
        NCK(ncclGroupStart());
        int64_t off = 0;
        for (int d = 0; d < W; ++d) {
            const int64_t nc = P->col_start[d + 1] - P->col_start[d];
            const int64_t scnt = (int64_t)(P->plane_start[d + 1] - P->plane_start[d]) * ncol;
            NCK(ncclSend(P->a2a_recv + (int64_t)P->plane_start[d] * ncol, 2 * scnt, ncclDouble, d, G->comm, s));
            NCK(ncclRecv(P->a2a_send + off, 2 * (int64_t)P->n0_loc * nc, ncclDouble, d, G->comm, s));
            off += (int64_t)P->n0_loc * nc;
        }
        NCK(ncclGroupEnd());
    }
    for (int k = 0; k < ns; ++k) shard_phase3(G->shards[k], args[k], s);
    // halo: the first `order` planes of shard r+1 follow shard r's own planes
    if (G->emulate) {
        for (int r = 0; r + 1 < W; ++r) {
            FftpimPlan* dst = G->shards[r];
            FftpimPlan* src = G->shards[r + 1];
            const int64_t plane = (int64_t)dst->near_g.n[1] * dst->near_g.n[2];
            CK(cudaMemcpyAsync(dst->qg + (int64_t)dst->n0_loc * plane, src->qg, dst->halo * plane * sizeof(cplx),
                               cudaMemcpyDeviceToDevice, s));
        }
    } else {
        FftpimPlan* P = G->shards[0];
        const int64_t plane = (int64_t)P->near_g.n[1] * P->near_g.n[2];
        const int Wh = P->near_g.order;   // halo planes = order
        NCK(ncclGroupStart());
        if (G->rank > 0) NCK(ncclSend(P->qg, 2 * Wh * plane, ncclDouble, G->rank - 1, G->comm, s));
        if (G->rank + 1 < W) NCK(ncclRecv(P->qg + (int64_t)P->n0_loc * plane, 2 * Wh * plane, ncclDouble, G->rank + 1, G->comm, s));
        NCK(ncclGroupEnd());
    }
    for (int k = 0; k < ns; ++k) {
        CK(cudaStreamWaitEvent(s, G->shards[k]->ev_join[1], 0));   // the shard's K4
        launch_observers(args[k], s);
    }
    CK(cudaGetLastError());
}

void group_evaluate(GroupImpl* G, const double* q, double* u, cudaStream_t s) {
    FftpimPlan* P0 = G->shards[0];
    CK(cudaSetDevice(P0->device));
    if (!P0->use_graphs) {
        group_schedule(G, q, u, s);
        return;
    }
    if (!G->g_stream) {
        CK(cudaStreamCreateWithFlags(&G->g_stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&G->ev_in, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&G->ev_out, cudaEventDisableTiming));
    }
    const cudaStream_t caller = s;
    if (caller == nullptr) {   // the legacy default stream cannot be captured
        CK(cudaEventRecord(G->ev_in, caller));
        CK(cudaStreamWaitEvent(G->g_stream, G->ev_in, 0));
        s = G->g_stream;
    }
    if (!(G->graph_exec && G->g_q == q && G->g_u == u)) {
        cudaGraph_t graph = nullptr;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        for (auto* P : G->shards) P->capturing = true;
        const long long l0 = g_launches.load();
        try {
            group_schedule(G, q, u, s);
        } catch (...) {
            for (auto* P : G->shards) P->capturing = false;
            cudaStreamEndCapture(s, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        for (auto* P : G->shards) P->capturing = false;
        G->kernels_per_eval = (int)(g_launches.load() - l0);
        CK(cudaStreamEndCapture(s, &graph));
        bool updated = false;
        if (G->graph_exec) {
            cudaGraphExecUpdateResultInfo res{};
            updated = cudaGraphExecUpdate(G->graph_exec, graph, &res) == cudaSuccess;
            if (!updated) {
                cudaGetLastError();
                cudaGraphExecDestroy(G->graph_exec);
                G->graph_exec = nullptr;
            }
        }
        if (!updated) CK(cudaGraphInstantiate(&G->graph_exec, graph, 0));
        CK(cudaGraphDestroy(graph));
        G->g_q = q;
        G->g_u = u;
    }
    CK(cudaGraphLaunch(G->graph_exec, s));
    fftpim_count_launch(G->kernels_per_eval);
    if (caller == nullptr) {
        CK(cudaEventRecord(G->ev_out, s));
        CK(cudaStreamWaitEvent(caller, G->ev_out, 0));
    }
}

// Orders an evaluation after the plan's previous one when the caller switches
// streams (same-stream evaluations are already ordered), and serialises the
// host-side state (graph capture, staging buffers) between threads.
struct EvalGuard {
    FftpimPlan* P;
    cudaStream_t s;
    std::lock_guard<std::mutex> lock;
    EvalGuard(FftpimPlan* plan, cudaStream_t stream) : P(plan), s(stream), lock(plan->eval_mu) {
        if (P->has_last && P->last_stream != s) cudaStreamWaitEvent(s, P->ev_last, 0);
    }
    ~EvalGuard() {
        if (cudaEventRecord(P->ev_last, s) == cudaSuccess) {
            P->last_stream = s;
            P->has_last = true;
        }
    }
};

int fail(const Fail& f) {
    g_last_error = f.msg;
    return f.code;
}

}  // namespace

void fftpim_count_launch(int n) { g_launches += n; }

extern "C" {

struct SweepSpec {
    int axis, E;
    const double* k;   // (E, 2)
};

static int plan_create_shard(const FftpimProblem* p, int world, int rank, bool sharded, FftpimPlan** out,
                             const SweepSpec* sw = nullptr) {
    if (!p || !out) return fail(Fail{FFTPIM_VALUE, "null argument"});
    *out = nullptr;
    auto t0 = std::chrono::steady_clock::now();
    FftpimPlan* P = new FftpimPlan();
    try {
        P->world = world;
        P->rank = rank;
        P->sharded = sharded;
        P->prob = *p;
        if (sw) {
            if (sw->axis < 0 || sw->axis >= p->dim) throw Fail{FFTPIM_VALUE, "sweep axis must be a periodic axis"};
            if (sw->E < 1 || sw->E > 64) throw Fail{FFTPIM_VALUE, "a sweep plan holds 1..64 excitations"};
            if (p->regime == FFTPIM_NPSP) throw Fail{FFTPIM_VALUE, "NPSP problems have no phase shift to sweep"};
            if (p->i_d > 2) throw Fail{FFTPIM_VALUE, "i_d > 2 is not supported by this build"};
            P->sweep = true;
            P->sw_axis = sw->axis;
            P->sw_E = sw->E;
            P->sw_ncomp = 2 * p->i_d + 1;
            P->sw_k.assign(sw->k, sw->k + 2 * sw->E);
            // the base geometry carries excitation 0's shift
            P->prob.kshift[sw->axis][0] = sw->k[0];
            P->prob.kshift[sw->axis][1] = sw->k[1];
        }
        P->device = p->device;
        P->use_graphs = getenv("FFTPIM_NO_GRAPHS") == nullptr;
        memset(&P->info, 0, sizeof(P->info));
        CK(cudaSetDevice(P->device));
        CK(cudaStreamCreateWithFlags(&P->build_stream, cudaStreamNonBlocking));
        {
            // near chain (aux[0]) at the highest priority: the block scheduler then
            // serves its latency-bound kernels before the K4 stream (aux[1])
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            static const int prio = [] {
                const char* e = getenv("FFTPIM_STREAM_PRIO");
                return e ? atoi(e) : 1;
            }();
            const int pr[3] = {prio ? hi : 0, prio ? lo : 0, prio ? (lo + hi) / 2 : 0};
            for (int k = 0; k < 3; ++k) CK(cudaStreamCreateWithPriority(&P->aux[k], cudaStreamNonBlocking, pr[k]));
        }
        CK(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&P->ev_start, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&P->ev_in, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&P->ev_k1, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&P->ev_out, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&P->ev_last, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&P->gstream, cudaStreamNonBlocking));
        for (auto& e : P->ev_join) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        P->status = dalloc<DevStatus>(P, 1);
        CK(cudaMemsetAsync(P->status, 0, sizeof(DevStatus), P->build_stream));
        build(P);
        P->prob.src_pos = nullptr;
        P->prob.obs_pos = nullptr;
        P->prob.far_kernel = nullptr;
        P->info.device_bytes = P->device_bytes;
        P->info.build_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = P;
        return FFTPIM_OK;
    } catch (const Fail& f) {
        cudaStreamSynchronize(P->build_stream);
        fftpim_plan_destroy(P);
        return fail(f);
    }
}

int fftpim_plan_create(const FftpimProblem* p, FftpimPlan** out) { return plan_create_shard(p, 1, 0, false, out); }

int fftpim_sweep_create(const FftpimProblem* p, int32_t axis, int32_t n_exc, const double* kshift_axis,
                        FftpimPlan** out) {
    if (!kshift_axis) return fail(Fail{FFTPIM_VALUE, "null argument"});
    SweepSpec sw{axis, n_exc, kshift_axis};
    return plan_create_shard(p, 1, 0, false, out, &sw);
}

// One sweep evaluation.  The batched K4 for all excitations (FP64-bound) runs
// on the low-priority stream while the per-excitation chains (permutation, far
// chain, K1, the FFT stages with the excitation's kernel_hat, the observer pass
// without the K4 term -- memory/latency-bound) run on the high-priority stream;
// after both join, one pass adds the K4 sums to every potential.
// the batched K4 of a sweep: code-phased charge copies, then all excitations' sums
static void sweep_k4(FftpimPlan* P, const double* q, cudaStream_t s) {
    const int E = P->sw_E, NS = P->sw_ncomp + 2;
    launch_sweep_permute((const cplx*)q, P->src_perm, P->N, E, P->sw_omega, NS, P->prob.i_d, P->sw_qt, s);
    launch_corr_sweep(P->pair_ptr, P->pair_src, P->sw_comp, P->sw_ncomp, P->info.n_pairs, P->sw_qt, P->N, E,
                      P->sw_omega, P->sw_corr, P->M, s, P->info.pair_rows_source_order == 1);
}

// `ready` (host entry): event e marks excitation e's charges resident; chain e
// waits for it and the batched K4 for the last one.
static void sweep_evaluate(FftpimPlan* P, const double* q, double* u, cudaStream_t s,
                           const cudaEvent_t* ready = nullptr) {
    const int E = P->sw_E;
    const bool serial = P->serial_sweep_required;
    cudaStream_t sn = serial ? s : P->aux[0], sc = serial ? s : P->aux[1];
    if (!serial) {
        CK(cudaEventRecord(P->ev_fork, s));
        CK(cudaStreamWaitEvent(sn, P->ev_fork, 0));
        CK(cudaStreamWaitEvent(sc, P->ev_fork, 0));
    }
    if (ready) CK(cudaStreamWaitEvent(sc, ready[E - 1], 0));
    sweep_k4(P, q, sc);
    const int64_t nk = prod3(P->far_kdims);
    if (!P->custom_fft) CKFFT(cufftSetStream(P->fft_plan, sn));
    for (int e = 0; e < E; ++e) {
        EvalArgs a = eval_args(P, q + 2 * (int64_t)e * P->N, u + 2 * (int64_t)e * P->M, FFTPIM_ALL);
        a.khat = P->sw_khat + (int64_t)e * P->n_fft;
        a.far_kernel = P->sw_far + (int64_t)e * nk;
        a.sw_corr = nullptr;
        a.sw_E = E;
        a.sw_e = -1;   // the K4 term is added by launch_sweep_add_corr
        if (ready) CK(cudaStreamWaitEvent(sn, ready[e], 0));
        launch_permute_q(a, sn);
        launch_far_project(a, sn);
        launch_far_sum(a, sn);
        launch_near_project(a, sn);
        if (P->custom_fft) {
            for (int k = 0; k < 5; ++k) {
                if (!P->stage_on[k]) continue;
                FftStage st = P->stage[k];
                if (st.spec) st.spec = a.khat;
                launch_fft_stage(st, sn);
            }
        } else {
            CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->pad_in, (cufftDoubleComplex*)P->work, CUFFT_FORWARD));
            launch_spectrum_mul(a, sn);
            CKFFT(cufftExecZ2Z(P->fft_plan, (cufftDoubleComplex*)P->work, (cufftDoubleComplex*)P->work, CUFFT_INVERSE));
            fftpim_count_launch(2);
        }
        launch_observers(a, sn);
    }
    if (!serial) {
        CK(cudaEventRecord(P->ev_join[0], sn));
        CK(cudaEventRecord(P->ev_join[1], sc));
        CK(cudaStreamWaitEvent(s, P->ev_join[0], 0));
        CK(cudaStreamWaitEvent(s, P->ev_join[1], 0));
    }
    launch_sweep_add_corr((cplx*)u, P->sw_corr, P->obs_perm, P->M, E, s);
    CK(cudaGetLastError());
}

int fftpim_sweep_evaluate(FftpimPlan* plan, const double* q, double* u, void* stream) {
    NvtxRange nv("fftpim_sweep_evaluate");
    if (!plan || !q || !u) return fail(Fail{FFTPIM_VALUE, "null argument"});
    if (!plan->sweep) return fail(Fail{FFTPIM_VALUE, "not a sweep plan (use fftpim_plan_evaluate)"});
    if (((uintptr_t)q | (uintptr_t)u) & 15) return fail(Fail{FFTPIM_VALUE, "q and u must be 16-byte aligned"});
    try {
        CK(cudaSetDevice(plan->device));
        EvalGuard g(plan, (cudaStream_t)stream);
        sweep_evaluate(plan, q, u, (cudaStream_t)stream);
        return FFTPIM_OK;
    } catch (const Fail& f) {
        return fail(f);
    }
}

int fftpim_sweep_evaluate_host(FftpimPlan* plan, const double* q, double* u) {
    NvtxRange nv("fftpim_sweep_evaluate_host");
    if (!plan || !q || !u) return fail(Fail{FFTPIM_VALUE, "null argument"});
    if (!plan->sweep) return fail(Fail{FFTPIM_VALUE, "not a sweep plan (use fftpim_plan_evaluate_host)"});
    try {
        FftpimPlan* P = plan;
        CK(cudaSetDevice(P->device));
        const int E = P->sw_E;
        cudaStream_t s = P->build_stream, sx = P->aux[2];
        EvalGuard g(P, s);
        if (P->h_batch < E) {   // persistent device staging (E charge and potential vectors)
            dfree(P, P->h_q);
            dfree(P, P->h_u);
            if (P->hgraph_exec) cudaGraphExecDestroy(P->hgraph_exec);
            P->hgraph_exec = nullptr;
            P->h_q = dalloc<double>(P, 2 * P->N * E);
            P->h_u = dalloc<double>(P, 2 * P->M * E);
            P->h_batch = E;
        }
        if ((int)P->sw_ready.size() < E) {
            for (int e = (int)P->sw_ready.size(); e < E; ++e) {
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                P->sw_ready.push_back(ev);
            }
        }
        // upload excitation by excitation on the copy stream; each chain starts
        // as soon as its charges are resident
        CK(cudaEventRecord(P->ev_fork, s));
        CK(cudaStreamWaitEvent(sx, P->ev_fork, 0));
        const size_t qb = sizeof(double) * 2 * P->N;
        for (int e = 0; e < E; ++e) {
            CK(cudaMemcpyAsync(P->h_q + 2 * P->N * e, q + 2 * P->N * e, qb, cudaMemcpyHostToDevice, sx));
            CK(cudaEventRecord(P->sw_ready[e], sx));
        }
        sweep_evaluate(P, P->h_q, P->h_u, s, P->sw_ready.data());
        CK(cudaMemcpyAsync(u, P->h_u, sizeof(double) * 2 * P->M * E, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return FFTPIM_OK;
    } catch (const Fail& f) {
        return fail(f);
    }
}

int fftpim_sweep_profile(FftpimPlan* plan, const double* q, double* u, void* stream, double* ms) {
    if (!plan || !q || !u || !ms) return fail(Fail{FFTPIM_VALUE, "null argument"});
    if (!plan->sweep) return fail(Fail{FFTPIM_VALUE, "not a sweep plan"});
    cudaEvent_t ev[3] = {};
    try {
        CK(cudaSetDevice(plan->device));
        cudaStream_t s = (cudaStream_t)stream;
        for (auto& e : ev) CK(cudaEventCreate(&e));
        FftpimPlan* P = plan;
        CK(cudaEventRecord(ev[0], s));
        sweep_k4(P, q, s);
        CK(cudaEventRecord(ev[1], s));
        sweep_evaluate(P, q, u, s);
        CK(cudaEventRecord(ev[2], s));
        CK(cudaEventSynchronize(ev[2]));
        float a = 0.f, b = 0.f;
        CK(cudaEventElapsedTime(&a, ev[0], ev[1]));
        CK(cudaEventElapsedTime(&b, ev[1], ev[2]));
        ms[0] = a;          // batched K4 alone (with the transposed permutation)
        ms[1] = b;          // one whole (overlapped) sweep evaluation
        for (auto& e : ev) cudaEventDestroy(e);
        return FFTPIM_OK;
    } catch (const Fail& f) {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        return fail(f);
    }
}

int fftpim_sweep_info(const FftpimPlan* plan, int32_t* axis, int32_t* n_exc) {
    if (!plan || !axis || !n_exc) return fail(Fail{FFTPIM_VALUE, "null argument"});
    *axis = plan->sweep ? plan->sw_axis : -1;
    *n_exc = plan->sweep ? plan->sw_E : 0;
    return FFTPIM_OK;
}

// ---------------------------------------------------------------------------
// Brute-force direct sums (oracle.py:62-123) -- see direct_kernels.cu.
int fftpim_direct_evaluate(const FftpimProblem* p, int32_t mode, double tol, int64_t max_terms,
                           int32_t consecutive_small, const double* q, double* u, int64_t* failures,
                           int64_t max_failures, FftpimDirectReport* rep) {
    if (!p || !q || !u || !rep || !p->src_pos) return fail(Fail{FFTPIM_VALUE, "null argument"});
    if (mode < 0 || mode > 2) return fail(Fail{FFTPIM_VALUE, "mode must be 0 (direct), 1 (far zone) or 2 (free space)"});
    if (mode != 2 && (p->dim < 1 || p->dim > 3)) return fail(Fail{FFTPIM_VALUE, "dim must be 1, 2 or 3"});
    if (mode != 2 && !(tol > 0.0)) return fail(Fail{FFTPIM_VALUE, "tol must be positive"});
    if (mode != 2 && (max_terms < 1 || consecutive_small < 1))
        return fail(Fail{FFTPIM_VALUE, "max_terms and consecutive_small must be >= 1"});
    if (mode == 1 && (p->i_d < 0 || p->i_d > 2)) return fail(Fail{FFTPIM_VALUE, "i_d must be in [0, 2]"});
    memset(rep, 0, sizeof(*rep));
    const int64_t N = p->n_src, M = p->n_obs;
    if (M <= 0) return FFTPIM_OK;
    FftpimPlan* P = new FftpimPlan();   // scratch owner of the device buffers
    try {
        P->device = p->device;
        P->prob = *p;
        CK(cudaSetDevice(P->device));
        CK(cudaStreamCreateWithFlags(&P->build_stream, cudaStreamNonBlocking));
        cudaStream_t s = P->build_stream;
        P->status = dalloc<DevStatus>(P, 1);
        CK(cudaMemsetAsync(P->status, 0, sizeof(DevStatus), s));
        const double* obs_h = p->obs_pos ? p->obs_pos : p->src_pos;
        double* d_src = dalloc<double>(P, 3 * std::max<int64_t>(N, 1));
        double* d_obs = dalloc<double>(P, 3 * M);
        cplx* d_q = dalloc<cplx>(P, std::max<int64_t>(N, 1));
        cplx* d_u = dalloc<cplx>(P, M);
        if (N > 0) {
            CK(cudaMemcpyAsync(d_src, p->src_pos, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(d_q, q, sizeof(cplx) * N, cudaMemcpyHostToDevice, s));
        }
        CK(cudaMemcpyAsync(d_obs, obs_h, sizeof(double) * 3 * M, cudaMemcpyHostToDevice, s));
        if (N == 0) {
            CK(cudaMemsetAsync(d_u, 0, sizeof(cplx) * M, s));
        } else {
            const int64_t CH = 64;   // oracle.py:20
            const int64_t nchunk = (M + CH - 1) / CH;
            // z extrema of each chunk's differences (pgf.py:394-397): max/min of
            // fl(o - s) are fl(max o - min s), fl(min o - max s) (rounding is monotone)
            double szmin = 1e300, szmax = -1e300;
            for (int64_t j = 0; j < N; ++j) {
                szmin = std::min(szmin, p->src_pos[3 * j + 2]);
                szmax = std::max(szmax, p->src_pos[3 * j + 2]);
            }
            std::vector<double> zr(2 * nchunk);
            for (int64_t c = 0; c < nchunk; ++c) {
                double omin = 1e300, omax = -1e300;
                for (int64_t i = c * CH; i < std::min(M, (c + 1) * CH); ++i) {
                    omin = std::min(omin, obs_h[3 * i + 2]);
                    omax = std::max(omax, obs_h[3 * i + 2]);
                }
                zr[2 * c] = omin - szmax;
                zr[2 * c + 1] = omax - szmin;
            }
            double* d_zr = dalloc<double>(P, 2 * nchunk);
            CK(cudaMemcpyAsync(d_zr, zr.data(), sizeof(double) * zr.size(), cudaMemcpyHostToDevice, s));
            int* d_sep = dalloc<int>(P, nchunk);
            long long* d_terms = dalloc<long long>(P, nchunk);
            CK(cudaMemsetAsync(d_sep, 0, sizeof(int) * nchunk, s));
            CK(cudaMemsetAsync(d_terms, 0, sizeof(long long) * nchunk, s));
            // rows per launch: whole chunks, at most ~32 M pairs of scratch
            const int64_t cap = (int64_t)1 << 25;
            int64_t rows = std::max<int64_t>(CH, (cap / N) / CH * CH);
            rows = std::min(rows, nchunk * CH);
            cplx* d_vals = dalloc<cplx>(P, rows * N);
            unsigned char* d_flags = dalloc<unsigned char>(P, rows * N);
            double maxLp = 0.0;
            for (int a = 0; a < std::max(1, std::min(3, p->dim)); ++a) maxLp = std::max(maxLp, p->L[a]);
            FarSeriesParams fp{};
            fp.dim = p->dim;
            fp.npsp = p->regime == FFTPIM_NPSP;
            for (int a = 0; a < 3; ++a) {
                fp.L[a] = p->L[a];
                fp.ks_re[a] = p->kshift[a][0];
                fp.ks_im[a] = p->kshift[a][1];
            }
            fp.k0_re = p->k0[0];
            fp.k0_im = p->k0[1];
            if (mode != 2) {
                fp.tol = tol;
                fp.cutoff = std::log(1.0 / tol) + 8.0;   // TruncationPolicy.inner_cutoff
                fp.sep = 1e-13 * std::max(maxLp, 1.0);   // pgf.py:93-94
                fp.wood = 1e-8 * 2.0 * M_PI / maxLp;     // pgf.py:88-90
                fp.max_terms = max_terms;
                fp.max_layers = 200000;
                fp.consecutive = consecutive_small;
            }
            ImageSet im{};
            im.k0_re = p->k0[0];
            im.k0_im = p->k0[1];
            im.sep_tol = 1e-13 * std::max(maxLp, 1.0);
            if (mode == 1) {
                FftpimProblem pi = *p;
                make_images(pi, p->kshift, im);
            }
            static const GLTable gl = gauss_laguerre_half();
            DirectArgs a{};
            a.src = d_src;
            a.obs = d_obs;
            a.q = d_q;
            a.N = N;
            a.zr = d_zr;
            a.dim = p->dim;
            a.npsp = fp.npsp;
            a.far_only = mode == 1;
            a.free_space = mode == 2;
            for (int k = 0; k < 3; ++k) a.L[k] = p->L[k];
            a.floor_t = 1e-12 * maxLp;   // oracle.py:31-32
            a.vals = d_vals;
            a.flags = d_flags;
            a.chunk_sep = d_sep;
            a.chunk_terms = d_terms;
            std::vector<int> sep(nchunk);
            std::vector<long long> terms(nchunk);
            std::vector<unsigned char> flags;
            int64_t nfail = 0;
            for (int64_t m0 = 0; m0 < M; m0 += rows) {
                a.m0 = m0;
                a.mc = std::min(rows, M - m0);
                launch_direct(a, fp, im, gl, d_u, P->status, s);
                check_status(P, mode == 2 ? "free-space sum" : "direct periodic sum");
                // failures in the reference's order: chunk by chunk, (observer, source)
                // row-major; a chunk with separation failures reports only those
                const int64_t c0 = m0 / CH, c1 = (m0 + a.mc + CH - 1) / CH;
                CK(cudaMemcpy(sep.data() + c0, d_sep + c0, sizeof(int) * (c1 - c0), cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(terms.data() + c0, d_terms + c0, sizeof(long long) * (c1 - c0), cudaMemcpyDeviceToHost));
                if (mode == 2) continue;
                flags.resize((size_t)(a.mc * N));
                CK(cudaMemcpy(flags.data(), d_flags, flags.size(), cudaMemcpyDeviceToHost));
                for (int64_t c = c0; c < c1; ++c) {
                    const unsigned char want = sep[c] ? 1 : 2;
                    if (sep[c]) ++rep->n_skipped_chunks;
                    else rep->worst_terms = std::max<int64_t>(rep->worst_terms, terms[c]);
                    for (int64_t i = c * CH; i < std::min(M, (c + 1) * CH); ++i) {
                        const unsigned char* fr = flags.data() + (i - m0) * N;
                        for (int64_t j = 0; j < N; ++j) {
                            if (fr[j] != want) continue;
                            if (failures && nfail < max_failures) {
                                failures[3 * nfail] = i;
                                failures[3 * nfail + 1] = j;
                                failures[3 * nfail + 2] = want;
                            }
                            ++nfail;
                        }
                    }
                }
            }
            rep->n_failures = nfail;
        }
        CK(cudaMemcpyAsync(u, d_u, sizeof(cplx) * M, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        fftpim_plan_destroy(P);
        return FFTPIM_OK;
    } catch (const Fail& f) {
        if (P->build_stream) cudaStreamSynchronize(P->build_stream);
        fftpim_plan_destroy(P);
        return fail(f);
    }
}

int fftpim_nccl_unique_id(void* out, int64_t bytes) {
    if (!out || bytes < (int64_t)sizeof(ncclUniqueId)) return fail(Fail{FFTPIM_VALUE, "need a 128-byte buffer"});
    try {
        ncclUniqueId id;
        NCK(ncclGetUniqueId(&id));
        memcpy(out, &id, sizeof(id));
        return FFTPIM_OK;
    } catch (const Fail& f) {
        return fail(f);
    }
}

int fftpim_group_create(const FftpimProblem* p, int32_t world, int32_t rank, const void* nccl_id,
                        FftpimGroup** out) {
    if (!p || !out || world < 1 || rank < 0 || rank >= world) return fail(Fail{FFTPIM_VALUE, "bad group arguments"});
    if (p->i_d < 1) return fail(Fail{FFTPIM_VALUE, "far-zone engine requires i_d >= 1"});
    *out = nullptr;
    GroupImpl* G = new GroupImpl();
    G->world = world;
    G->rank = rank;
    G->emulate = nccl_id == nullptr;
    try {
        if (G->emulate) {
            for (int r = 0; r < world; ++r) {
                FftpimPlan* P = nullptr;
                int rc = plan_create_shard(p, world, r, true, &P);
                if (rc) throw Fail{rc, g_last_error};
                G->shards.push_back(P);
            }
        } else {
            FftpimPlan* P = nullptr;
            int rc = plan_create_shard(p, world, rank, true, &P);
            if (rc) throw Fail{rc, g_last_error};
            G->shards.push_back(P);
            CK(cudaSetDevice(p->device));
            ncclUniqueId id;
            memcpy(&id, nccl_id, sizeof(id));
            NCK(ncclCommInitRank(&G->comm, world, id, rank));
        }
        *out = reinterpret_cast<FftpimGroup*>(G);
        return FFTPIM_OK;
    } catch (const Fail& f) {
        for (auto* P : G->shards) fftpim_plan_destroy(P);
        if (G->comm) ncclCommDestroy(G->comm);
        delete G;
        return fail(f);
    }
}

int fftpim_group_evaluate(FftpimGroup* g, const double* q, double* u, void* stream) {
    NvtxRange nv("fftpim_group_evaluate");
    if (!g || !q || !u) return fail(Fail{FFTPIM_VALUE, "null argument"});
    if (((uintptr_t)q | (uintptr_t)u) & 15) return fail(Fail{FFTPIM_VALUE, "q and u must be 16-byte aligned"});
    try {
        group_evaluate(reinterpret_cast<GroupImpl*>(g), q, u, (cudaStream_t)stream);
        return FFTPIM_OK;
    } catch (const Fail& f) {
        return fail(f);
    }
}

int fftpim_group_info(const FftpimGroup* g, int32_t shard, FftpimInfo* info) {
    const GroupImpl* G = reinterpret_cast<const GroupImpl*>(g);
    if (!G || !info || shard < 0 || shard >= (int)G->shards.size()) return fail(Fail{FFTPIM_VALUE, "bad shard"});
    *info = G->shards[shard]->info;
    return FFTPIM_OK;
}

void fftpim_group_destroy(FftpimGroup* g) {
    GroupImpl* G = reinterpret_cast<GroupImpl*>(g);
    if (!G) return;
    if (G->graph_exec) cudaGraphExecDestroy(G->graph_exec);
    if (G->g_stream) cudaStreamDestroy(G->g_stream);
    if (G->ev_in) cudaEventDestroy(G->ev_in);
    if (G->ev_out) cudaEventDestroy(G->ev_out);
    for (auto* P : G->shards) fftpim_plan_destroy(P);
    if (G->comm) ncclCommDestroy(G->comm);
    delete G;
}

int fftpim_plan_evaluate(FftpimPlan* plan, const double* q, double* u, int64_t batch, int32_t parts, void* stream) {
    NvtxRange nv("fftpim_plan_evaluate");
    if (!plan || !q || !u) return fail(Fail{FFTPIM_VALUE, "null argument"});
    if (plan->near_only && (parts & FFTPIM_FAR)) return fail(Fail{FFTPIM_VALUE, "far-zone engine requires i_d >= 1"});
    if (plan->sweep) return fail(Fail{FFTPIM_VALUE, "sweep plans evaluate through fftpim_sweep_evaluate"});
    if (((uintptr_t)q | (uintptr_t)u) & 15) return fail(Fail{FFTPIM_VALUE, "q and u must be 16-byte aligned"});
    try {
        CK(cudaSetDevice(plan->device));
        EvalGuard g(plan, (cudaStream_t)stream);
        evaluate(plan, q, u, batch, parts, (cudaStream_t)stream);
        return FFTPIM_OK;
    } catch (const Fail& f) {
        return fail(f);
    }
}

// Pageable caller buffers (the stock plan.evaluate(numpy) call): the bytes go
// through plan-owned pinned staging buffers in 8 MiB chunks -- host threads copy
// chunk k into pinned memory while the DMA engine uploads chunk k - 1, and on
// the way back they copy chunk k out while chunk k + 1 downloads -- instead of
// the driver's serial pageable copies.
// Persistent copy workers (created on first use, parked on a condition variable
// between calls): spawning threads per 8 MiB chunk cost more than the copies.
namespace {
class CopyPool {
public:
    explicit CopyPool(int workers) {
        for (int i = 0; i < workers; ++i) th_.emplace_back([this] { work(); });
        for (auto& t : th_) t.detach();   // parked until process exit
    }
    // split [0, bytes) into `parts` slices; the caller copies the first one
    void run(char* dst, const char* src, size_t bytes, int parts) {
        const size_t per = (bytes / parts + 63) & ~(size_t)63;
        {
            std::lock_guard<std::mutex> lk(m_);
            for (int i = 1; i < parts; ++i) {
                const size_t o = (size_t)i * per;
                if (o >= bytes) break;
                jobs_.push_back(Job{dst + o, src + o, std::min(per, bytes - o)});
                ++pending_;
            }
        }
        cv_.notify_all();
        memcpy(dst, src, std::min(per, bytes));
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [this] { return pending_ == 0; });
    }

private:
    struct Job {
        char* dst;
        const char* src;
        size_t n;
    };
    void work() {
        for (;;) {
            Job j;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [this] { return !jobs_.empty(); });
                j = jobs_.back();
                jobs_.pop_back();
            }
            memcpy(j.dst, j.src, j.n);
            {
                std::lock_guard<std::mutex> lk(m_);
                if (--pending_ == 0) done_.notify_all();
            }
        }
    }
    std::mutex m_;
    std::condition_variable cv_, done_;
    std::vector<Job> jobs_;
    int pending_ = 0;
    std::vector<std::thread> th_;
};
}   // namespace

static void parallel_memcpy(void* dst, const void* src, size_t bytes) {
    static const int nt = [] {
        const char* e = getenv("FFTPIM_HOST_COPY_THREADS");
        const int hw = (int)std::thread::hardware_concurrency();
        return std::max(1, e ? atoi(e) : std::min(8, std::max(1, hw / 2)));
    }();
    const int k = (int)std::min<size_t>(nt, std::max<size_t>(1, bytes >> 20));
    if (k <= 1) {
        memcpy(dst, src, bytes);
        return;
    }
    static std::mutex pool_mu;                       // one staged copy at a time per process
    static CopyPool* pool = new CopyPool(nt - 1);    // leaked on purpose: workers outlive static destructors
    std::lock_guard<std::mutex> lk(pool_mu);
    pool->run((char*)dst, (const char*)src, bytes, k);
}

static void staged_host_evaluate(FftpimPlan* P, const double* q, double* u, size_t qb, size_t ub, int64_t batch,
                                 int parts, cudaStream_t s) {
    constexpr size_t CH = (size_t)8 << 20;
    if (P->pin_bytes < std::max(qb, ub)) {
        if (P->pin_q) cudaFreeHost(P->pin_q);
        if (P->pin_u) cudaFreeHost(P->pin_u);
        P->pin_q = P->pin_u = nullptr;
        CK(cudaMallocHost(&P->pin_q, qb));
        CK(cudaMallocHost(&P->pin_u, ub));
        P->pin_bytes = std::max(qb, ub);
        for (auto& e : P->pin_ev) {
            if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
    }
    for (size_t o = 0; o < qb; o += CH) {
        const size_t n = std::min(CH, qb - o);
        parallel_memcpy((char*)P->pin_q + o, (const char*)q + o, n);
        CK(cudaMemcpyAsync((char*)P->h_q + o, (char*)P->pin_q + o, n, cudaMemcpyHostToDevice, s));
    }
    evaluate(P, P->h_q, P->h_u, batch, parts, s);
    // download in chunks, each copied out as soon as its event fires
    const int nev = (int)(sizeof(P->pin_ev) / sizeof(P->pin_ev[0]));
    std::vector<size_t> offs;
    for (size_t o = 0; o < ub; o += CH) offs.push_back(o);
    size_t done = 0;
    for (size_t i = 0; i < offs.size(); ++i) {
        if (i >= (size_t)nev) {   // recycle the event of chunk i - nev
            const size_t j = i - nev;
            CK(cudaEventSynchronize(P->pin_ev[j % nev]));
            const size_t n = std::min(CH, ub - offs[j]);
            parallel_memcpy((char*)u + offs[j], (char*)P->pin_u + offs[j], n);
            done = j + 1;
        }
        const size_t n = std::min(CH, ub - offs[i]);
        CK(cudaMemcpyAsync((char*)P->pin_u + offs[i], (char*)P->h_u + offs[i], n, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(P->pin_ev[i % nev], s));
    }
    for (size_t j = done; j < offs.size(); ++j) {
        CK(cudaEventSynchronize(P->pin_ev[j % nev]));
        const size_t n = std::min(CH, ub - offs[j]);
        parallel_memcpy((char*)u + offs[j], (char*)P->pin_u + offs[j], n);
    }
}

int fftpim_plan_evaluate_host(FftpimPlan* plan, const double* q, double* u, int64_t batch, int32_t parts) {
    NvtxRange nv("fftpim_plan_evaluate_host");
    if (!plan || !q || !u) return fail(Fail{FFTPIM_VALUE, "null argument"});
    if (plan->near_only && (parts & FFTPIM_FAR)) return fail(Fail{FFTPIM_VALUE, "far-zone engine requires i_d >= 1"});
    if (plan->sweep) return fail(Fail{FFTPIM_VALUE, "sweep plans evaluate through fftpim_sweep_evaluate"});
    try {
        CK(cudaSetDevice(plan->device));
        cudaStream_t s = plan->build_stream;
        EvalGuard g(plan, s);
        // persistent staging buffers: stable pointers keep the captured graph valid
        if (batch > plan->h_batch) {
            dfree(plan, plan->h_q);
            dfree(plan, plan->h_u);
            if (plan->hgraph_exec) cudaGraphExecDestroy(plan->hgraph_exec);
            plan->hgraph_exec = nullptr;
            plan->h_q = dalloc<double>(plan, 2 * plan->N * batch);
            plan->h_u = dalloc<double>(plan, 2 * plan->M * batch);
            plan->h_batch = batch;
        }
        size_t qb = sizeof(double) * 2 * plan->N * batch, ub = sizeof(double) * 2 * plan->M * batch;
        auto pinned = [](const void* p) {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            return at.type == cudaMemoryTypeHost;
        };
        FftpimPlan* P = plan;
        ensure_batch_buffers(P, batch, parts);   // allocations stay outside the capture
        // the captured host graph's buffers are known to be pinned
        const bool same_bufs = P->hgraph_exec && P->hg_q == q && P->hg_u == u;
        if (P->use_graphs && (same_bufs || (pinned(q) && pinned(u)))) {
            // pinned caller buffers: one graph holds the upload, the evaluation
            // schedule and the download (re-captured when the buffers change)
            if (!(P->hgraph_exec && P->hg_q == q && P->hg_u == u && P->hg_batch == batch && P->hg_parts == parts)) {
                if (P->hgraph_exec) cudaGraphExecDestroy(P->hgraph_exec);
                P->hgraph_exec = nullptr;
                cudaGraph_t graph = nullptr;
                CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
                P->capturing = true;
                const long long l0 = g_launches.load();
                try {
                    CK(cudaMemcpyAsync(P->h_q, q, qb, cudaMemcpyHostToDevice, s));
                    P->host_call = true;   // K1 reads the uploaded caller-order charges
                    evaluate_schedule(P, P->h_q, P->h_u, batch, parts, s);
                    P->host_call = false;
                    CK(cudaMemcpyAsync(u, P->h_u, ub, cudaMemcpyDeviceToHost, s));
                    P->hkernels_per_eval = (int)((g_launches.load() - l0) / batch);
                } catch (...) {
                    P->capturing = false;
                    P->host_call = false;
                    cudaStreamEndCapture(s, &graph);
                    if (graph) cudaGraphDestroy(graph);
                    throw;
                }
                P->capturing = false;
                CK(cudaStreamEndCapture(s, &graph));
                CK(cudaGraphInstantiate(&P->hgraph_exec, graph, 0));
                CK(cudaGraphDestroy(graph));
                P->hg_q = q;
                P->hg_u = u;
                P->hg_batch = batch;
                P->hg_parts = parts;
            }
            CK(cudaGraphLaunch(P->hgraph_exec, s));
            fftpim_count_launch(P->hkernels_per_eval * (int)batch);
        } else if (qb + ub >= ((size_t)8 << 20)) {
            staged_host_evaluate(plan, q, u, qb, ub, batch, parts, s);
        } else {
            CK(cudaMemcpyAsync(plan->h_q, q, qb, cudaMemcpyHostToDevice, s));
            evaluate(plan, plan->h_q, plan->h_u, batch, parts, s);
            CK(cudaMemcpyAsync(u, plan->h_u, ub, cudaMemcpyDeviceToHost, s));
        }
        // the call is synchronous: poll instead of sleeping in the driver (the
        // wake-up latency is a visible share of a ~0.2 ms host round trip)
        cudaError_t r;
        while ((r = cudaStreamQuery(s)) == cudaErrorNotReady) {
        }
        CK(r);
        return FFTPIM_OK;
    } catch (const Fail& f) {
        return fail(f);
    }
}

int fftpim_plan_profile(FftpimPlan* plan, const double* q, double* u, int32_t parts, void* stream,
                        double* stage_ms) {
    if (!plan || !q || !u || !stage_ms) return fail(Fail{FFTPIM_VALUE, "null argument"});
    if (plan->sweep) return fail(Fail{FFTPIM_VALUE, "stage profiles are for single-excitation plans"});
    if (plan->near_only && (parts & FFTPIM_FAR)) return fail(Fail{FFTPIM_VALUE, "far-zone engine requires i_d >= 1"});
    cudaEvent_t ev[FFTPIM_N_STAGES + 1] = {};
    try {
        CK(cudaSetDevice(plan->device));
        for (auto& e : ev) CK(cudaEventCreate(&e));
        EvalGuard g(plan, (cudaStream_t)stream);
        evaluate(plan, q, u, 1, parts, (cudaStream_t)stream, ev);
        CK(cudaEventSynchronize(ev[FFTPIM_N_STAGES]));
        for (int k = 0; k < FFTPIM_N_STAGES; ++k) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
            stage_ms[k] = ms;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        return FFTPIM_OK;
    } catch (const Fail& f) {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        return fail(f);
    }
}

int fftpim_plan_info(const FftpimPlan* plan, FftpimInfo* info) {
    if (!plan || !info) return fail(Fail{FFTPIM_VALUE, "null argument"});
    *info = plan->info;
    return FFTPIM_OK;
}

int fftpim_plan_export(const FftpimPlan* cplan, int32_t which, void* dst, int64_t bytes) {
    FftpimPlan* P = const_cast<FftpimPlan*>(cplan);
    if (!P || !dst) return fail(Fail{FFTPIM_VALUE, "null argument"});
    try {
        CK(cudaSetDevice(P->device));
        const int64_t M = P->M, N = P->N, npairs = P->info.n_pairs;
        auto need = [&](int64_t b) {
            if (bytes < b) throw Fail{FFTPIM_VALUE, "export buffer too small: need " + std::to_string(b) + " bytes"};
        };
        if (which == FFTPIM_FAR_KERNEL) {
            int64_t n = prod3(P->far_kdims);
            need(n * 16);
            CK(cudaMemcpy(dst, P->far_kernel, n * 16, cudaMemcpyDeviceToHost));
            return FFTPIM_OK;
        }
        if (which == FFTPIM_KERNEL_HAT) {
            need(P->n_fft * 16);
            CK(cudaMemcpy(dst, P->khat, P->n_fft * 16, cudaMemcpyDeviceToHost));
            double* d = (double*)dst;
            for (int64_t i = 0; i < 2 * P->n_fft; ++i) d[i] *= (double)P->n_fft;
            return FFTPIM_OK;
        }
        if (which >= FFTPIM_NEAR_SRC_START && which <= FFTPIM_FAR_OBS_W) {
            // stencils are held in sorted order; rows go back to the caller's order
            const bool far = which >= FFTPIM_FAR_SRC_START, obs = ((which - FFTPIM_NEAR_SRC_START) & 2) != 0;
            const bool wts = ((which - FFTPIM_NEAR_SRC_START) & 1) != 0;
            const int64_t n = obs ? M : N;
            const int Wd = (far ? P->prob.far_order : P->prob.near_order) + 1;
            const double* dw = far ? (obs ? P->obs_fw : P->src_fw) : (obs ? P->obs_w : P->src_w);
            const int* ds = far ? (obs ? P->obs_fstart : P->src_fstart) : (obs ? P->obs_start : P->src_start);
            if (!dw || !ds) throw Fail{FFTPIM_VALUE, "this plan does not hold the requested stencils"};
            if (P->sharded && obs) throw Fail{FFTPIM_VALUE, "observer stencils of a slab shard cover its own range only"};
            std::vector<int> perm(n);
            CK(cudaMemcpy(perm.data(), obs ? P->obs_perm : P->src_perm, sizeof(int) * n, cudaMemcpyDeviceToHost));
            if (wts) {
                need(n * 3 * Wd * 8);
                std::vector<double> h((size_t)n * 3 * Wd);
                CK(cudaMemcpy(h.data(), dw, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
                double* o = (double*)dst;
                for (int64_t i = 0; i < n; ++i)
                    std::copy(h.begin() + i * 3 * Wd, h.begin() + (i + 1) * 3 * Wd, o + (int64_t)perm[i] * 3 * Wd);
            } else {
                need(n * 3 * 4);
                std::vector<int> h((size_t)n * 3);
                CK(cudaMemcpy(h.data(), ds, sizeof(int) * h.size(), cudaMemcpyDeviceToHost));
                int* o = (int*)dst;
                for (int64_t i = 0; i < n; ++i)
                    for (int a = 0; a < 3; ++a) o[(int64_t)perm[i] * 3 + a] = h[i * 3 + a];
            }
            return FFTPIM_OK;
        }
        if (which < FFTPIM_PAIR_OBS || which > FFTPIM_PAIR_COEF) throw Fail{FFTPIM_VALUE, "unknown operand"};
        std::vector<int64_t> ptr(M + 1);
        std::vector<int> operm(M), sperm(N), psrc(npairs);
        CK(cudaMemcpy(ptr.data(), P->pair_ptr, sizeof(int64_t) * (M + 1), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(operm.data(), P->obs_perm, sizeof(int) * M, cudaMemcpyDeviceToHost));
        std::vector<int64_t> orank(M);
        for (int64_t i = 0; i < M; ++i) orank[operm[i]] = i;
        // reference order: by original observer index
        std::vector<int64_t> order;
        order.reserve(npairs);
        for (int64_t m = 0; m < M; ++m) {
            int64_t i = orank[m];
            for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) order.push_back(p);
        }
        if (which == FFTPIM_PAIR_OBS) {
            need(npairs * 4);
            int* o = (int*)dst;
            int64_t k = 0;
            for (int64_t m = 0; m < M; ++m) {
                int64_t i = orank[m];
                for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) o[k++] = (int)m;
            }
        } else if (which == FFTPIM_PAIR_SRC) {
            need(npairs * 4);
            if (P->pair_src) {
                CK(cudaMemcpy(psrc.data(), P->pair_src, sizeof(int) * npairs, cudaMemcpyDeviceToHost));
            } else {   // run-encoded plan that dropped its index array
                int* tmp = nullptr;
                CK(cudaMalloc(&tmp, sizeof(int) * (size_t)std::max<int64_t>(npairs, 1)));
                launch_run_decode(P->run_rec, P->run_bias, npairs, tmp, nullptr);
                cudaError_t e = cudaMemcpy(psrc.data(), tmp, sizeof(int) * npairs, cudaMemcpyDeviceToHost);
                cudaFree(tmp);
                CK(e);
            }
            CK(cudaMemcpy(sperm.data(), P->src_perm, sizeof(int) * N, cudaMemcpyDeviceToHost));
            int* o = (int*)dst;
            const int mask = P->sweep ? 0x3fffffff : -1;   // sweep plans pack the axis code in bits 30-31
            for (int64_t k = 0; k < npairs; ++k) o[k] = sperm[psrc[order[k]] & mask];
        } else if (which == FFTPIM_PAIR_CODE) {
            need(npairs * 3);
            std::vector<unsigned char> cid(npairs);
            if (!P->pair_codeid) throw Fail{FFTPIM_VALUE, "pair codes are not kept for plans with more than 2^31 pairs"};
            CK(cudaMemcpy(cid.data(), P->pair_codeid, npairs, cudaMemcpyDeviceToHost));
            signed char* o = (signed char*)dst;
            for (int64_t k = 0; k < npairs; ++k)
                for (int a = 0; a < 3; ++a) o[3 * k + a] = P->pg.code[cid[order[k]]][a];
        } else {
            need(npairs * 16);
            if (P->sweep) throw Fail{FFTPIM_VALUE, "sweep plans hold coefficient components, not coefficients"};
            double* o = (double*)dst;
            if (P->pair_coef_r) {
                std::vector<double> c(npairs);
                CK(cudaMemcpy(c.data(), P->pair_coef_r, sizeof(double) * npairs, cudaMemcpyDeviceToHost));
                for (int64_t k = 0; k < npairs; ++k) {
                    o[2 * k] = c[order[k]];
                    o[2 * k + 1] = 0.0;
                }
            } else {
                std::vector<cplx> c(npairs);
                CK(cudaMemcpy(c.data(), P->pair_coef, sizeof(cplx) * npairs, cudaMemcpyDeviceToHost));
                for (int64_t k = 0; k < npairs; ++k) {
                    o[2 * k] = c[order[k]].re;
                    o[2 * k + 1] = c[order[k]].im;
                }
            }
        }
        return FFTPIM_OK;
    } catch (const Fail& f) {
        return fail(f);
    }
}

int fftpim_plan_set_far_kernel(FftpimPlan* plan, const double* kernel, int64_t n_entries) {
    if (!plan || !kernel) return fail(Fail{FFTPIM_VALUE, "null argument"});
    try {
        if (n_entries != prod3(plan->far_kdims)) throw Fail{FFTPIM_KERNEL_CACHE, "far kernel table size mismatch"};
        CK(cudaSetDevice(plan->device));
        CK(cudaMemcpy(plan->far_kernel, kernel, n_entries * 16, cudaMemcpyHostToDevice));
        return FFTPIM_OK;
    } catch (const Fail& f) {
        return fail(f);
    }
}

void fftpim_plan_destroy(FftpimPlan* plan) {
    if (!plan) return;
    cudaSetDevice(plan->device);
    if (plan->build_stream) cudaStreamSynchronize(plan->build_stream);
    if (plan->fft_plan) cufftDestroy(plan->fft_plan);
    if (plan->graph_exec) cudaGraphExecDestroy(plan->graph_exec);
    if (plan->hgraph_exec) cudaGraphExecDestroy(plan->hgraph_exec);
    if (plan->pin_q) cudaFreeHost(plan->pin_q);
    if (plan->pin_u) cudaFreeHost(plan->pin_u);
    for (auto& e : plan->pin_ev)
        if (e) cudaEventDestroy(e);
    for (void* p : plan->allocations) cudaFree(p);
    for (auto st : plan->aux)
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    if (plan->ev_fork) cudaEventDestroy(plan->ev_fork);
    if (plan->ev_start) cudaEventDestroy(plan->ev_start);
    if (plan->ev_in) cudaEventDestroy(plan->ev_in);
    if (plan->ev_k1) cudaEventDestroy(plan->ev_k1);
    if (plan->ev_out) cudaEventDestroy(plan->ev_out);
    if (plan->ev_last) cudaEventDestroy(plan->ev_last);
    if (plan->gstream) cudaStreamDestroy(plan->gstream);
    for (auto e : plan->sw_ready) cudaEventDestroy(e);
    for (auto e : plan->ev_join)
        if (e) cudaEventDestroy(e);
    if (plan->build_stream) cudaStreamDestroy(plan->build_stream);
    delete plan;
}

const char* fftpim_last_error(void) { return g_last_error.c_str(); }

int64_t fftpim_launch_count(void) { return (int64_t)g_launches.load(); }

}  // extern "C"
