// kernels.h -- host-callable launch wrappers (plan build and evaluation).
#pragma once
#include "plan.cuh"

// Far-series parameters (pgf.py:166-462).
struct FarSeriesParams {
    int dim;
    int npsp;
    double L[3];
    double k0_re, k0_im;
    double ks_re[3], ks_im[3];
    double tol;        // series_tol
    double cutoff;     // ln(1/tol) + 8            pgf.py:56-58
    double sep;        // 1e-13 * max(Lmax, 1)     pgf.py:93-94
    double wood;       // 1e-8 * 2 pi / Lmax       pgf.py:88-90
    double zmin, zmax; // extrema over the whole point set (3D lattice lead, pgf.py:394-397)
    long long max_terms;
    int max_layers;
    int consecutive;   // layers in a row below tol that stop a point (TruncationPolicy.consecutive_small)
};

// ---- plan build (build_kernels.cu) ----
void launch_cell_keys(const double* pos, int64_t n, const StencilGeom& g, int* keys, DevStatus* st,
                      cudaStream_t s);
void launch_csr_from_sorted(const int* keys, int64_t n, int64_t ncells, int* start, cudaStream_t s);
void launch_stencils(const double* pos, const int* perm, int64_t n, const StencilGeom& g, double* w,
                     int* start, DevStatus* st, int where, cudaStream_t s);
void launch_rank(const int* perm, int64_t n, int* rank, cudaStream_t s);
void launch_embed_table(cplx* out, const int cdims[3], const int dims[3], const double h[3],
                        const ImageSet& im, cudaStream_t s);
void launch_count_coincident(const int dims[3], const double h[3], const ImageSet& im,
                             unsigned long long* cnt, cudaStream_t s);
void launch_scale(cplx* a, int64_t n, double f, cudaStream_t s);
void launch_wrap_flags(const double* pos, int64_t n, const int code[3], const double lo[3],
                       const double hi[3], unsigned char* flags, cudaStream_t s);
void launch_aug_keys(const double* pos, const int* aug_orig, const unsigned char* aug_code, int64_t A,
                     const PairGeom& pg, int* keys, cudaStream_t s);
void launch_fill_u8(unsigned char* p, int64_t n, unsigned char v, cudaStream_t s);
void launch_iota(int* p, int64_t n, cudaStream_t s);

struct PairArgs {
    const double* src_pos;      // original order AoS
    const double* obs_pos;
    const int* obs_perm;        // sorted obs -> original
    int64_t M;
    const int* box_start;
    const int* box_order;
    const int* aug_orig;
    const unsigned char* aug_code;
    const int* obs_start;       // sorted obs stencil starts (3 per point)
    const double* obs_w;
    const int* src_start;
    const double* src_w;
    const int* src_rank;
    int W;                      // weights stride per axis (order+1)
    int wdt[3];
    // count pass
    int64_t* counts;
    int* d0min;                 // (27*3)
    int* d0max;
    unsigned long long* tallies;   // [0] self, [1] wrapped
    // fill pass
    const int64_t* pair_ptr;
    const cplx* tables;
    int* pair_src;
    unsigned char* pair_codeid;
    cplx* coef;
    double* coef_r;
    DevStatus* st;
};
void launch_pairs_count(const PairGeom& pg, const PairArgs& a, cudaStream_t s);
void launch_pairs_fill(const PairGeom& pg, const ImageSet& im, const CodeTables& tabs, const PairArgs& a,
                       cudaStream_t s);
void launch_code_tables(const CodeTables& tabs, int ncodes, const PairGeom& pg, const ImageSet& im,
                        cplx* tables, int64_t total, cudaStream_t s);
void launch_far_series(const double* axes, const int kd[3], const FarSeriesParams& fp, const ImageSet& im,
                       const GLTable& gl, cplx* out, DevStatus* st, cudaStream_t s);

// ---- brute-force direct sums (direct_kernels.cu) ----
struct DirectArgs {
    const double* src;          // (N, 3) device
    const double* obs;          // (M, 3) device
    const cplx* q;              // (N,)
    int64_t N, m0, mc;          // this launch: observers [m0, m0 + mc), mc a multiple of 64 (or the tail)
    const double* zr;           // per 64-observer chunk: z extrema of its differences (3D lattice lead)
    int dim, npsp, far_only, free_space;
    double L[3];
    double floor_t;             // 1e-12 * max periodic L (oracle.py:31-32)
    cplx* vals;                 // (mc, N) G q per pair
    unsigned char* flags;       // (mc, N): 0 ok, 1 separation, 2 not converged
    int* chunk_sep;             // per chunk: separation failures
    long long* chunk_terms;     // per chunk: longest series
};
void launch_direct(const DirectArgs& a, const FarSeriesParams& fp, const ImageSet& im, const GLTable& gl,
                   cplx* u, DevStatus* st, cudaStream_t s);

// ---- evaluation (eval_kernels.cu) ----
struct EvalArgs {
    int64_t N, M;
    const cplx* q;              // caller order
    cplx* u;                    // caller order
    const int* src_perm;
    const int* obs_perm;
    cplx* q_sorted;
    double* q_re;               // NPSP: real parts of q_sorted (null: no real-charge path)
    int* q_flag;                // nonzero when this evaluation's charges are not all real
    // near
    StencilGeom g;
    int cdims[3];
    const int* cell_start;
    const double* src_w;
    const int* src_start;
    const double* obs_w;
    const int* obs_start;
    cplx* work;
    cplx* pad_in;               // zero-padded FFT input; only the n^3 corner is written
    cplx* k1_out;               // K1 target grid, indexed (((x-kx0)*go1 + y)*go2 + z)
    int go1, go2;
    int kx0, knx;               // K1 computes planes [kx0, kx0 + knx) (slab shards)
    cplx* k1_scratch;           // tap-major K1 block tiles (null: gather K1)
    const int* k1_cnt;          // sliced-ELL K1 (null: computed K1): entries per slot
    const int* k1_row;          // node of each slot
    const int64_t* k1_off;      // first entry of each 32-slot slice
    const int* k1_idx;          // source index per entry (into k1_q)
    const double* k1_wgt;       // weight product per entry
    const cplx* k1_q;           // charges K1 reads: q_sorted, or q itself (k1_orig)
    const double* k1_pos;       // K1 line sweep, staged (non-null selects it): sorted positions
    const double* k1_rec;       // K1 line sweep, independent threads (non-null selects it): stencil records
    const double* obs_pos;      // observer pass with in-kernel stencils (non-null selects it)
    const int* obs_cell_start;  // observer cell CSR (global sorted indices): grid-tile observer pass
    int64_t obs_i0;             // first observer of this plan (slab shard) in the global sorted order
    const cplx* interp_grid;    // near potentials on the grid, indexed (((x-gx0)*gi1 + y)*gi2 + z)
    int gi1, gi2;
    int gx0;
    const cplx* khat;
    int64_t n_fft;
    const int64_t* pair_ptr;
    const int* pair_src;
    const cplx* coef;
    const double* coef_r;
    int64_t n_pairs;
    const unsigned short* pair_off16;   // 16-bit source offsets per pair (non-null selects that K4)
    const int* grp_base;        // per 32-pair group: offset base, < 0 for int32 groups
    const unsigned* run_rec;    // run-encoded sources (non-null selects k_corr_runs): 96 words per tile
    const int* run_bias;        // biases past a tile record's 64 (source of a run's first pair - position)
    const unsigned* head_bits;  // bit p set where an observer's pair range starts
    const int64_t* seg_base;    // per CORR_TILE tile: global index of its first segment
    const int64_t* seg_first;   // per observer: global index of its first segment
    cplx* seg_val;              // (row, tile) segment sums
    int corr_blocks;            // K4 grid cap (0 = whole chip)
    unsigned long long* k4_counter;   // k_corr_runs: shared tile queue (null: static tile order)
    // far
    StencilGeom fs, fo;
    const double* src_fw;
    const int* src_fstart;
    const double* obs_fw;
    const int* obs_fstart;
    const cplx* far_kernel;
    cplx* far_partial;
    cplx* far_qg;
    cplx* far_ug;
    int far_blocks, far_warps;
    const cplx* far_q;          // sources projected onto the far grid (own range for shards)
    const double* far_pos;      // their sorted positions (non-null: windowed far projection)
    cplx* far_slots;            // windowed far projection: per-chunk windows
    int* far_win;
    int far_chunk, far_cap;     // points per warp chunk, shared-memory window entries per warp
    int64_t far_n;
    cplx* obs_pre;              // far + K4 fix-up per sorted observer (split observer pass)
    cplx* u_sorted;             // grid-tile observer pass: store near + far here in sorted order (no K4 term)
    const cplx* sw_corr;        // sweep: K4 sums (M, E) replace the segment fix-up
    int sw_E, sw_e;             // sw_e < 0: the observer pass leaves the K4 term out
    int parts;
};
void launch_permute_q(const EvalArgs& a, cudaStream_t s);
int64_t k1_scratch_elems(const StencilGeom& g, int knx);
void launch_near_project(const EvalArgs& a, cudaStream_t s);
void launch_k1_count(const EvalArgs& a, int* cnt_row, int* cnt_sorted, int* row_of, int64_t* slots,
                     cudaStream_t s);
void launch_k1_fill(const EvalArgs& a, const int* row_of, const int64_t* off, const int* remap, int* idx,
                    double* wgt, cudaStream_t s);
void launch_spectrum_mul(const EvalArgs& a, cudaStream_t s);
// ---- line-sweep K1 and sorted positions (line_kernels.cu)
bool launch_k1_lines(const EvalArgs& a, const double* pos, cudaStream_t s);
bool launch_k1_lines_g(const EvalArgs& a, const double* rec, cudaStream_t s);
int stencil_record_width(int W);
void launch_stencil_records(const double* w, const int* start, int64_t n, int W, double* rec, cudaStream_t s);
void launch_gather_pos(const double* pos, const int* perm, int64_t n, double* out, cudaStream_t s);
bool launch_observers_pos(const EvalArgs& a, const double* pos, cudaStream_t s, int mode);
bool launch_far_project_win(const EvalArgs& a, const double* pos, cplx* slots, int* win, cudaStream_t s);
int64_t far_win_max_chunks(int64_t n);
void far_win_setup(const StencilGeom& fs, const double* pos, int64_t n, int* win, int* chunk_out, int* cap_out,
                   cudaStream_t s);
int64_t launch_max_tile_count(const StencilGeom& g, const int* ocs, cudaStream_t s);
bool launch_observers_tile(const EvalArgs& a, const double* pos, const int* ocs, int64_t i0, cudaStream_t s,
                           int mode);
void launch_finish_corr(const EvalArgs& a, cudaStream_t s);   // u = u_sorted + K4 row sums
void launch_far_project(const EvalArgs& a, cudaStream_t s);
size_t far_project_smem(int nf, int warps, int order);
void launch_far_sum(const EvalArgs& a, cudaStream_t s);
void launch_axpy(cplx* acc, const cplx* x, int64_t n, cudaStream_t s);   // acc += x
void launch_observers(const EvalArgs& a, cudaStream_t s, int mode = 0);   // 0 fused, 1 pre, 2 post

// ---- pruned column-FFT stages (fft_kernels.cu)
size_t fft_stage_smem(const FftStage& st);
void launch_fft_stage(const FftStage& st, cudaStream_t s);

// ---- batched excitation sweep (sweep_kernels.cu)
struct SweepCodeAxis {
    int c[27];                  // code component along the sweep axis per code id
};
void launch_sweep_pack_src(int* pair_src, const unsigned char* codeid, const signed char* code_axis, int64_t P,
                           cudaStream_t s);
void launch_sweep_permute(const cplx* q, const int* perm, int64_t N, int E, const cplx* omega, int NS, int h,
                          cplx* qt3, cudaStream_t s);
void launch_corr_sweep(const int64_t* ptr, const int* pair_src, const cplx* comp, int ncomp, int64_t P,
                       const cplx* qt3, int64_t N, int E, const cplx* omega, cplx* corr, int64_t M, cudaStream_t s,
                       bool sorted_rows);
void launch_batch_permute(const cplx* q, const int* perm, int64_t N, int E, cplx* qt, cudaStream_t s);
void launch_sweep_add_corr(cplx* u, const cplx* corr, const int* obs_perm, int64_t M, int E, cudaStream_t s);

// ---- correction matvec (corr_kernels.cu)
#define CORR_TILE 256
void build_corr_metadata(const int64_t* ptr, int64_t M, int64_t P, int64_t T, unsigned* bits, int64_t* seg_first,
                         int64_t* seg_base, int64_t* spans_tmp, int64_t* n_segments, cudaStream_t s);
void launch_corr_tiles(const EvalArgs& a, cudaStream_t s);
bool sort_pair_rows(const int64_t* ptr, int64_t M, int* pair_src, cplx* const* carr, int ncarr, double* coef_r,
                    unsigned char* codeid, size_t budget, cudaStream_t s);
int64_t build_group_offsets(const int* src, int64_t P, int* base, unsigned short* off, cudaStream_t s);
int64_t build_run_records(const int* src, const unsigned* head, const int64_t* seg_base, int64_t P, int64_t T,
                          int64_t N, unsigned** rec_out, int** ovf_out, int64_t* bytes_out, cudaStream_t s);
#define CORR_QPAD 256   // zero charges kept past q_sorted[N) / q_re[N) (padding pairs of k_corr_runs)
void launch_run_decode(const unsigned* recs, const int* ovf, int64_t P, int* src, cudaStream_t s);
