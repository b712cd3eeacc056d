// plan.cuh -- internal plan layout and the by-value parameter blocks the
// kernels receive.  See DESIGN.md "Data layout in HBM".
#pragma once
#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>
#include <cstdlib>

#include <mutex>
#include <string>
#include <vector>

#include "cmath.cuh"
#include "../../include/fftpim.h"

#define FFTPIM_MAX_IMAGES 125   // (2*i_d+1)^3 with i_d <= 2
#define FFTPIM_MAX_ORDER 6
#define FFTPIM_MAX_W (FFTPIM_MAX_ORDER + 1)

// One uniform grid + Lagrange stencil order (grids.py:25-56, 110-140).
struct StencilGeom {
    int n[3];          // grid planes per axis
    double origin[3];
    double h[3];       // spacing (0 on a single-plane axis)
    int order;
    int w[3];          // stencil width per axis: order+1, or 1 on single-plane axes
    int nc[3];         // number of distinct stencil starts per axis: n - w + 1
    double margin[3];  // allowed extrapolation beyond the hull
};

// Image list for G_near (pgf.py:114-123).
struct ImageSet {
    int count;
    double off[FFTPIM_MAX_IMAGES][3];
    double ph_re[FFTPIM_MAX_IMAGES];
    double ph_im[FFTPIM_MAX_IMAGES];
    double k0_re, k0_im;
    double sing_tol;  // near tables / direct terms (nearzone.py:213)
    double sep_tol;   // far kernel image subtraction (pgf.py:93-94)
};

// Correction-pair discovery geometry (nearzone.py:303-364).
struct PairGeom {
    int dims[3];
    double h[3];
    double inv_h[3];
    int nb[3];
    int jr[3];
    int ext[3];
    int max_pad;
    double r2_keep;
    double sing_tol;
    int same_points;
    int ncodes;                 // distinct image codes present (<= 27)
    signed char code[27][3];    // code vectors, index = code id
    double shift[27][3];        // code * L
    double phase_re[27], phase_im[27];   // exp(-j code.(kshift*L))
};

// Per-code window table of G_near(idx*h - c*L) (nearzone.py:439-451).
struct CodeTables {
    int64_t offset[27];
    int lo[27][3];
    int len[27][3];
};

// Device-side first-error record.
struct DevStatus {
    int code;           // FftpimStatus, 0 if none
    int where;          // kernel-specific detail
    long long a, b;     // indices for the message
    int kernel_terms;
    int pad_;
};

// One pruned column-FFT stage (fft_kernels.cu).
struct FftStage {
    const cplx* in;
    cplx* out;
    int L, lin, lout;           // transform length, nonzero inputs, kept outputs
    int64_t in_stride, out_stride;   // along the transform axis
    int nb0, nb1;               // columns: fast batch index (per block, B at a time) and grid.y
    int64_t in_s0, out_s0, in_s1, out_s1;
    int sign;                   // -1 forward, +1 inverse (ignored when spec is set)
    const cplx* spec;           // fused x stage: forward, multiply by spec, inverse
    int64_t spec_stride, spec_s0, spec_s1;
    // khat even along y / z (non-periodic axis, or periodic without phase
    // shift): the fused register stage reads column (ky, kz) at its folded
    // index, so only a quarter / half of the spectrum is touched and it stays
    // L2-resident (0 = no fold, else the axis length); spec_L2 = 2 n2
    int fold_y, fold_z, spec_L2;
    const cplx* tw;             // exp(-2 pi i t / L), t < L
    const cplx* twp;            // per-pass compact twiddles, pass order
    int ntwp;
    int nrad;
    int radix[24];
    int B;                      // columns per block
};

struct FftpimPlan {
    FftpimProblem prob;           // copy (pointers cleared)
    FftpimInfo info;
    int device;
    cudaStream_t build_stream;

    // geometry
    StencilGeom near_g, far_sg, far_og;
    ImageSet images;
    PairGeom pg;
    CodeTables tabs;
    int cdims[3];                 // circulant dims
    int64_t n_fft;                // prod(cdims)
    int64_t n_grid;               // prod(near dims)
    int64_t n_far;                // far nodes
    int far_kdims[3];             // far kernel table dims
    bool npsp;

    // points (sorted by near stencil cell)
    int64_t N, M;
    int* src_perm = nullptr;      // sorted -> original
    int* src_rank = nullptr;      // original -> sorted
    int* obs_perm = nullptr;
    int* cell_start = nullptr;    // (ncells+1) CSR of sorted sources by near stencil start
    double* src_w = nullptr;      // (N, 3, W) near axis weights, sorted order
    int* src_start = nullptr;     // (N, 3) near stencil starts, sorted order
    double* obs_w = nullptr;      // observers (aliases src_* if same_points)
    int* obs_start = nullptr;
    double* src_pos_s = nullptr;  // (N, 3) positions in sorted order (K1 line sweep computes stencils)
    bool k1_lines = false;        // K1 = line sweep (line_kernels.cu)
    double* src_rec = nullptr;    // (N, (3W+2)&~1) stencil records for the thread-independent line sweep
    double* obs_pos_s = nullptr;  // (M, 3) observer positions, sorted (aliases src_pos_s if same points)
    bool obs_pos_pass = false;    // observer pass computes its stencils from obs_pos_s
    bool obs_tile = false;        // ... and gathers the near grid from shared-memory tiles
    int* obs_cell_start = nullptr;   // observer cell CSR (aliases cell_start if same points)
    double* src_fw = nullptr;     // (N, 3, Wf) far source-grid weights
    int* src_fstart = nullptr;
    double* obs_fw = nullptr;     // far observer-grid weights
    int* obs_fstart = nullptr;

    // near FFT
    cplx* khat = nullptr;         // kernel_hat / M (numpy ifftn scaling folded in)
    cplx* work = nullptr;         // spectrum / inverse-FFT buffer (in place)
    cplx* pad_in = nullptr;       // zero-padded projection (corner written each eval)
    cufftHandle fft_plan = 0;
    cplx* q_sorted = nullptr;     // (N) charges permuted to sorted order
    double* q_re = nullptr;       // (N) their real parts (NPSP plans: K4 gathers 8 B when q is real)
    int* q_flag = nullptr;        // set by the permutation when some charge has a nonzero imaginary part
    cplx* k1_scratch = nullptr;   // tap-major K1 extended block tiles
    int* k1_cnt = nullptr;        // sliced-ELL K1 (eval_kernels.cu): entries per slot
    int* k1_row = nullptr;        // node of each slot
    int64_t* k1_off = nullptr;    // (slices + 1) entry offsets
    bool k1_orig = false;         // entries index the caller-order charges
    int* k1_idx = nullptr;
    int* k1_idx_sorted = nullptr;  // k1_orig plans: the same operator indexing q_sorted
    bool host_call = false;       // capturing the host entry's graph (upload inside)
    double* k1_wgt = nullptr;
    int64_t k1_slots = 0;

    // corrections (CSR over sorted observers)
    int64_t* pair_ptr = nullptr;  // (M+1)
    int* pair_src = nullptr;      // (P) sorted source index
    unsigned short* pair_off16 = nullptr;   // (P) 16-bit offsets from the 32-pair group base (K4)
    int* grp_base = nullptr;      // (P/32 + 8) group bases, -1: the group reads pair_src
    unsigned* run_rec = nullptr;  // (tiles, 96) run-encoded sources: tile records (corr_kernels.cu k_corr_runs)
    int* run_bias = nullptr;      // overflow biases; pair_src may be dropped once these exist
    unsigned long long* k4_counter = nullptr;   // tile queue shared by the overlapped K4 launches
    unsigned char* pair_codeid = nullptr;  // (P) code id (export only)
    cplx* pair_coef = nullptr;    // (P) complex coefficients (dynamic / static-shifted)
    double* pair_coef_r = nullptr;  // (P) real coefficients (NPSP)
    // pruned column-FFT pipeline (fft_kernels.cu); cuFFT full transforms otherwise
    bool custom_fft = false;
    cplx* qg = nullptr;           // (n0 n1 n2): K1 output, then the near potentials ug
    cplx* fbufA = nullptr;        // (n0 n1 2n2)
    cplx* fbufB = nullptr;        // (n0 2n1 2n2)
    cplx* twiddle[3] = {nullptr, nullptr, nullptr};
    cplx* twiddle_pass[3] = {nullptr, nullptr, nullptr};
    int n_twiddle_pass[3] = {0, 0, 0};
    bool stage_on[5] = {false, false, false, false, false};
    FftStage stage[5];
    int64_t n_tiles = 0;          // CORR_TILE-pair tiles of the correction stream
    int64_t n_segments = 0;       // (observer, tile) segments
    unsigned* head_bits = nullptr;
    int64_t* seg_base = nullptr;
    int64_t* seg_first = nullptr;
    cplx* seg_val = nullptr;

    // far
    cplx* far_kernel = nullptr;   // (2nf-1)^3
    cplx* far_qg = nullptr;       // projected far source grid
    cplx* far_partial = nullptr;  // per-block partial grids
    cplx* far_slots = nullptr;    // windowed far projection (line_kernels.cu): per-chunk windows
    int* far_win = nullptr;
    int far_chunk = 0, far_cap = 0;
    cplx* far_ug = nullptr;       // far observer-grid potentials
    cplx* obs_pre = nullptr;      // split observer pass: far + K4 fix-up (concurrent schedule)
    int far_blocks_seq = 0;            // far projection grid for sequential chains
    int far_blocks = 0;
    int far_warps = 0;

    // CUDA graph of the evaluation schedule, keyed by the caller's buffers
    bool use_graphs = true;
    bool capturing = false;
    cudaGraphExec_t graph_exec = nullptr;
    const double* g_q = nullptr;
    double* g_u = nullptr;
    int64_t g_batch = 0;
    int g_parts = 0;
    int kernels_per_eval = 0;
    // persistent device staging for fftpim_plan_evaluate_host
    double* h_q = nullptr;
    double* h_u = nullptr;
    int64_t h_batch = 0;
    cudaGraphExec_t hgraph_exec = nullptr;   // upload + evaluation + download, pinned buffers
    void* pin_q = nullptr;        // pinned staging for pageable caller buffers (host entry)
    void* pin_u = nullptr;
    size_t pin_bytes = 0;
    cudaEvent_t pin_ev[8] = {};
    const double* hg_q = nullptr;
    double* hg_u = nullptr;
    int64_t hg_batch = 0;
    int hg_parts = 0;
    int hkernels_per_eval = 0;

    // slab decomposition: shard `rank` of `world` owns near-grid
    // x-planes [X0, X1), the sorted observers/sources whose stencil starts there
    // [i0, i1), and FFT columns [C0, C1) for the x transforms
    int world = 1, rank = 0;
    bool sharded = false;           // built as a group shard (also for world == 1)
    int X0 = 0, X1 = 0, n0_loc = 0, halo = 0;
    int64_t i0 = 0, i1 = 0;
    int64_t C = 0, C0 = 0, C1 = 0;
    std::vector<int> plane_start;   // X_r for r = 0..world
    std::vector<int64_t> col_start; // C_r for r = 0..world
    cplx* a2a_send = nullptr;       // packed [peer][x_local][column]
    cplx* a2a_recv = nullptr;       // [x][own column]
    cplx* far_sum_tmp = nullptr;

    // concurrent evaluation schedule (near chain | K4 | far chain)
    cudaStream_t aux[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t ev_fork = nullptr;
    cudaEvent_t ev_start = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    cudaEvent_t ev_k1 = nullptr;                     // K4 gate (FFTPIM_K4_GATE)   // legacy-stream fence around graph replays
    cudaStream_t gstream = nullptr;                  // graph replay stream for legacy-stream callers
    cudaEvent_t ev_join[3] = {nullptr, nullptr, nullptr};

    // batched excitation sweep: E phase shifts differing only
    // along periodic axis sw_axis; one pair list with 2 i_d + 1 phase components
    // evaluations of one plan share its work buffers: a host mutex plus an
    // event from the previous evaluation's stream order them across callers
    std::mutex eval_mu;
    cudaEvent_t ev_last = nullptr;
    cudaStream_t last_stream = nullptr;
    bool has_last = false;
    bool sweep = false;
    bool near_only = false;            // i_d = 0: eval_near only (no far kernel)
    int sw_axis = 0, sw_E = 0, sw_ncomp = 0;
    std::vector<double> sw_k;          // (E, 2) kshift component along sw_axis
    cplx* sw_comp = nullptr;           // (ncomp, P) coefficient components
    std::vector<cudaEvent_t> sw_ready;   // host entry: excitation e's charges uploaded
    bool serial_sweep_required = getenv("FFTPIM_SWEEP_SERIAL") != nullptr;   // diagnostics: one stream
    cplx* sw_khat = nullptr;           // (E, n_fft) kernel_hat per excitation
    cplx* sw_far = nullptr;            // (E, nk) far kernel per excitation
    int bt_E = 0;                      // multi-RHS batches: right-hand sides per batched K4 pass
    cplx* bt_qt = nullptr;             // (N, bt_E) sorted charges, right-hand side fastest
    cplx* bt_corr = nullptr;           // (M, bt_E) batched K4 sums
    cplx* bt_omega = nullptr;          // (bt_E, 3) ones: unit phases for the one-component sweep kernel
    cplx* sw_omega = nullptr;          // (E, ncomp + 2) exp(-j m k_e L), m = -(i_d+1) .. i_d+1
    cplx* sw_qt = nullptr;             // (N, E) sorted charges, excitation fastest
    cplx* sw_corr = nullptr;           // (M, E) batched K4 sums, excitation fastest
    int64_t sw_batch_cap = 0;

    DevStatus* status = nullptr;
    int64_t device_bytes = 0;
    std::vector<void*> allocations;
};

// launch-count evidence (fftpim_launch_count)
void fftpim_count_launch(int n = 1);
