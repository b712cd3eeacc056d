/*
 * fftpim.h -- C ABI of the B200-native FFT-PIM potential evaluation.
 *
 * Drop-in boundary for the reference's hot path (perisum 0.1.0, Python):
 *   build_plan(cfg, box, src, obs, params)   /root/reference/pkg/src/perisum/solver.py:35-45
 *   SolvePlan.evaluate(q) = eval_near+eval_far /root/reference/pkg/src/perisum/solver.py:24-25
 *   build_near_plan / eval_near               /root/reference/pkg/src/perisum/nearzone.py:194, 490
 *   build_far_plan / eval_far                 /root/reference/pkg/src/perisum/farzone.py:76, 150
 * Plain C types only: no torch, no CUDA types in the signatures (streams are
 * passed as void* = cudaStream_t).  All arithmetic is fp64 / complex128;
 * complex arrays are interleaved (re, im) doubles, exactly numpy complex128.
 *
 * Status codes map 1:1 onto the reference's exception classes
 * (/root/reference/pkg/src/perisum/errors.py:4-37):
 */
#ifndef FFTPIM_H
#define FFTPIM_H

#include <stdint.h>

#if defined(__GNUC__)
#define FFTPIM_API __attribute__((visibility("default")))
#else
#define FFTPIM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum FftpimStatus {
    FFTPIM_OK = 0,
    FFTPIM_VALIDATION = 1,      /* ValidationError      model.py:211-297            */
    FFTPIM_DOMAIN = 2,          /* DomainError          nearzone.py:410-416, pgf.py:143-147 */
    FFTPIM_WOOD_ANOMALY = 3,    /* WoodAnomalyError     pgf.py:239-240, 257-261, 271-275 */
    FFTPIM_NOT_CONVERGED = 4,   /* NotConvergedError    farzone.py:115-119, pgf.py:268-270 */
    FFTPIM_SEPARATION = 5,      /* SeparationError      pgf.py:227-229, 343-344     */
    FFTPIM_KERNEL_CACHE = 6,    /* KernelCacheError     farzone.py:186-212          */
    FFTPIM_CUDA = 7,            /* CUDA / cuFFT failure (no reference counterpart)  */
    FFTPIM_VALUE = 8            /* ValueError (length mismatch, bad grid)  nearzone.py:495-496 */
};

/* Regime codes follow the PIMF blob codes, farzone.py:29. */
enum FftpimRegime { FFTPIM_DYNAMIC = 1, FFTPIM_STATIC_SHIFTED = 2, FFTPIM_NPSP = 3 };

/* Evaluation parts: eval_near (nearzone.py:490) and eval_far (farzone.py:150). */
enum FftpimParts { FFTPIM_NEAR = 1, FFTPIM_FAR = 2, FFTPIM_ALL = 3 };

/* PeriodicityConfig (model.py:42-76) + TargetBox (model.py:80-88) +
 * SolverParams (model.py:166-190) + the point sets (model.py:99-126). */
typedef struct FftpimProblem {
    int32_t dim;                /* number of periodic axes: 1 (x), 2 (x,y), 3 (x,y,z) */
    int32_t regime;             /* FftpimRegime */
    double L[3];                /* lattice periods */
    double D[3];                /* target box extent */
    double k0[2];               /* complex wavenumber (re, im) */
    double kshift[3][2];        /* complex phase shift per axis */
    int32_t i_d;                /* near-image half width */
    int32_t near_order;
    int32_t near_grid[3];       /* resolved near grid; {0,0,0} = auto (model.py:146-162) */
    int32_t far_order;
    int32_t far_grid[3];
    double series_tol;
    int32_t er_range_boxes;
    int64_t n_src;
    int64_t n_obs;
    const double* src_pos;      /* (n_src, 3) row-major, HOST memory */
    const double* obs_pos;      /* (n_obs, 3) row-major, HOST memory; NULL = same as src */
    int32_t same_points;        /* 1: observers are the sources (nearzone.py:241-243) */
    int32_t device;             /* CUDA device ordinal */
    int32_t parts;              /* zones to build: FFTPIM_ALL (0 = ALL), FFTPIM_NEAR = build_near_plan
                                   (nearzone.py:194-273), FFTPIM_FAR = build_far_plan (farzone.py:76-131) */
    int32_t reserved_;
    const double* far_kernel;   /* HOST (2nf-1)^3 complex128 far-kernel table read from a PIMF blob, or
                                   NULL: tabulate it (farzone.py:103-123: a cache hit skips pgf_far_many) */
    int64_t far_kernel_terms;   /* the blob's kernel_terms (used with far_kernel) */
} FftpimProblem;

/* Summary read by the reference CLI (cli.py:232-236) and by the tests. */
typedef struct FftpimInfo {
    int32_t near_dims[3];
    int32_t fft_dims[3];        /* doubled (circulant) dims */
    int32_t far_dims[3];
    int32_t join_radius[3];
    int32_t jr_full;
    int32_t on_axis_offset;     /* 1 when the far source grid was moved off the axis (farzone.py:89-98) */
    int64_t n_src;
    int64_t n_obs;
    int64_t n_pairs;
    int64_t n_self_pairs;
    int64_t n_wrapped_pairs;
    int64_t coincident_kernel_terms;
    int64_t kernel_terms;       /* worst far-series length */
    int64_t device_bytes;       /* plan-owned device memory */
    double build_seconds;
    int32_t real_coefficients;  /* 1: correction coefficients stored as fp64 (NPSP) */
    int32_t k1_operator;        /* 1: projection held as the plan-time sliced-ELL operator */
    int32_t custom_fft;         /* 1: pruned column-FFT stages, 0: cuFFT full transforms */
    int64_t k1_slots;           /* sliced-ELL entries including padding */
    int32_t built_parts;        /* FFTPIM_NEAR | FFTPIM_FAR zones this plan can evaluate */
    int32_t reserved_;
    int64_t graph_captures;     /* evaluation graphs captured (caller buffers changed) */
    int64_t graph_instantiations;   /* of those, executables instantiated (the rest updated in place) */
    int64_t k4_wide_groups;     /* 32-pair groups whose source indices need 32 bits (-1: 16-bit offsets off) */
    int32_t pair_rows_source_order;   /* 1: each observer's pairs are stored (and exported) in source order,
                                         0: in the reference's discovery order (nearzone.py:374-478) */
    int32_t reserved2_;
    int64_t k4_runs;            /* runs of consecutive sources in the run-encoded pair stream, padding
                                   included (-1: K4 reads an int32 source index per pair) */
} FftpimInfo;

typedef struct FftpimPlan FftpimPlan;

/* Build a plan on `p->device`.  Replaces build_plan (solver.py:35-45), i.e.
 * build_near_plan (nearzone.py:194-273) + build_far_plan (farzone.py:76-131).
 * Validation (model.py:211-297) is the caller's job; geometry-dependent errors
 * (DomainError, WoodAnomaly, NotConverged, Separation) are returned here. */
FFTPIM_API int fftpim_plan_create(const FftpimProblem* p, FftpimPlan** out);

/* u = eval_near + eval_far for `batch` charge vectors.  q: (batch, n_src)
 * complex128 and u: (batch, n_obs) complex128, both DEVICE pointers aligned
 * to 16 bytes (FFTPIM_VALUE otherwise), stream ordered on `stream` (cudaStream_t; NULL = legacy default).  Replaces
 * SolvePlan.evaluate (solver.py:24-25); parts selects eval_near / eval_far. */
FFTPIM_API int fftpim_plan_evaluate(FftpimPlan* plan, const double* q, double* u, int64_t batch,
                         int32_t parts, void* stream);

/* Batched excitation sweep (C5).  E <= 64 excitations of one
 * geometry whose Floquet shifts differ only along the periodic axis `axis`:
 * excitation e uses p->kshift with component `axis` replaced by
 * kshift_axis[2e] + i kshift_axis[2e+1].  The plan stores the correction pairs
 * once with 2 i_d + 1 phase components (nearzone.py:405-457 is linear in the
 * image phases, pgf.py:114-123), plus kernel_hat and the far kernel per
 * excitation.  Equivalent to E plans built with fftpim_plan_create. */
FFTPIM_API int fftpim_sweep_create(const FftpimProblem* p, int32_t axis, int32_t n_exc, const double* kshift_axis,
                                   FftpimPlan** out);

/* u[e] = evaluate_e(q[e]) for all excitations: q (E, n_src) and u (E, n_obs)
 * complex128 DEVICE pointers (16-byte aligned), stream ordered. */
FFTPIM_API int fftpim_sweep_evaluate(FftpimPlan* plan, const double* q, double* u, void* stream);

/* Same with HOST q (E, n_src) / u (E, n_obs) (pinned or pageable), synchronous:
 * excitation e's upload overlaps the chains of the excitations before it, the
 * batched precorrection starts once every charge vector is resident, one
 * download at the end.  This is the call a reference-side binding makes for a
 * sweep (the reference evaluates each excitation with SolvePlan.evaluate,
 * solver.py:24-25). */
FFTPIM_API int fftpim_sweep_evaluate_host(FftpimPlan* plan, const double* q, double* u);

/* Device milliseconds: ms[0] the batched precorrection alone (with its
 * transposed permutation), ms[1] one whole sweep evaluation (the per-excitation
 * chains overlap the batched precorrection). */
FFTPIM_API int fftpim_sweep_profile(FftpimPlan* plan, const double* q, double* u, void* stream, double* ms);

/* axis and excitation count of a sweep plan (-1, 0 for ordinary plans). */
FFTPIM_API int fftpim_sweep_info(const FftpimPlan* plan, int32_t* axis, int32_t* n_exc);

/* Brute-force direct sums: the reference's accuracy oracle (oracle.py:62-123,
 * SURVEY.md 8f rank 4), one converged periodic-Green's-function series per
 * (observer, source) pair on the device.
 *   mode 0: eval_direct           u_m = sum_n G_p(r_m - r_n) q_n      (oracle.py:92-97)
 *   mode 1: eval_direct_farzone   G_p minus the |i| <= p->i_d images   (oracle.py:100-111)
 *   mode 2: eval_free_space       sum_n exp(-j k0 r) / (4 pi r) q_n   (oracle.py:114-123)
 * Uses p->dim, regime, L, k0, kshift, i_d (mode 1), n_src, n_obs, src_pos,
 * obs_pos (HOST, NULL = sources), device.  tol / max_terms / consecutive_small
 * are the TruncationPolicy (pgf.py:40-58).  q (n_src) and u (n_obs) are HOST
 * complex128.  Observers are taken in chunks of 64 like the reference: a chunk
 * with a pair violating the separation rule (oracle.py:35-59) keeps u = 0 and
 * reports its separation failures, otherwise its non-converged pairs are
 * reported.  failures: optional (max_failures, 3) int64 records
 * (observer, source, 1 = separation | 2 = not converged) in the reference's
 * order; rep->n_failures counts all of them.  Mode 2 returns FFTPIM_DOMAIN
 * when an observer coincides with a source (the reference's ZeroDivisionError). */
typedef struct FftpimDirectReport {
    int64_t worst_terms;        /* longest series over the evaluated chunks */
    int64_t n_failures;
    int64_t n_skipped_chunks;   /* chunks left at 0 by separation failures */
} FftpimDirectReport;
FFTPIM_API int fftpim_direct_evaluate(const FftpimProblem* p, int32_t mode, double tol, int64_t max_terms,
                                      int32_t consecutive_small, const double* q, double* u, int64_t* failures,
                                      int64_t max_failures, FftpimDirectReport* rep);

/* Same with HOST q/u (pinned or pageable): H2D copy, evaluate, D2H copy,
 * synchronous.  This is the call the reference's FFI binding makes. */
FFTPIM_API int fftpim_plan_evaluate_host(FftpimPlan* plan, const double* q, double* u, int64_t batch,
                              int32_t parts);

FFTPIM_API int fftpim_plan_info(const FftpimPlan* plan, FftpimInfo* info);

/* Operand export for parity tests (host destination, `bytes` capacity).
 * Pairs come out in the reference order (nearzone.py:465-478): sorted by
 * observer index, within an observer in discovery order; indices are the
 * caller's original point indices. */
enum FftpimOperand {
    FFTPIM_PAIR_OBS = 1,        /* int32 (P)            NearZonePlan.pair_obs  */
    FFTPIM_PAIR_SRC = 2,        /* int32 (P)            NearZonePlan.pair_src  */
    FFTPIM_PAIR_CODE = 3,       /* int8  (P,3)          NearZonePlan.pair_code */
    FFTPIM_PAIR_COEF = 4,       /* complex128 (P)       NearZonePlan.pair_coef */
    FFTPIM_FAR_KERNEL = 5,      /* complex128 (2n-1)^3  FarZonePlan.kernel     */
    FFTPIM_KERNEL_HAT = 6,      /* complex128 fft_dims  NearZonePlan.kernel_hat (numpy scaling) */
    /* Lagrange stencils (grids.py:110-140) in the caller's point order: starts int32 (n, 3),
     * weights float64 (n, 3, order + 1) (single-plane axes: weight 1 then zeros) */
    FFTPIM_NEAR_SRC_START = 7,  /* NearZonePlan.proj_op.axis_starts    */
    FFTPIM_NEAR_SRC_W = 8,      /* NearZonePlan.proj_op.axis_weights   */
    FFTPIM_NEAR_OBS_START = 9,  /* NearZonePlan.interp_op.axis_starts  */
    FFTPIM_NEAR_OBS_W = 10,     /* NearZonePlan.interp_op.axis_weights */
    FFTPIM_FAR_SRC_START = 11,  /* FarZonePlan.proj_op.axis_starts     */
    FFTPIM_FAR_SRC_W = 12,      /* FarZonePlan.proj_op.axis_weights    */
    FFTPIM_FAR_OBS_START = 13,  /* FarZonePlan.interp_op.axis_starts   */
    FFTPIM_FAR_OBS_W = 14       /* FarZonePlan.interp_op.axis_weights  */
};
FFTPIM_API int fftpim_plan_export(const FftpimPlan* plan, int32_t which, void* dst, int64_t bytes);

/* Replace the far kernel table (PIMF blob import, farzone.py:103-112). */
FFTPIM_API int fftpim_plan_set_far_kernel(FftpimPlan* plan, const double* kernel, int64_t n_entries);

FFTPIM_API void fftpim_plan_destroy(FftpimPlan* plan);

/* Thread-local message of the last non-OK status. */
FFTPIM_API const char* fftpim_last_error(void);

/* One evaluation (batch 1, device pointers) with CUDA events recorded on
 * `stream` between the stages; stage_ms[0..8] receives the device time of
 *   0 permute q  1 far projection  2 far grid sum  3 near projection
 *   4 forward FFT  5 spectrum multiply  6 inverse FFT  7 correction matvec  8 observer pass
 * (interpolation + precorrection + far interpolation).  Diagnostic only. */
#define FFTPIM_N_STAGES 9
FFTPIM_API int fftpim_plan_profile(FftpimPlan* plan, const double* q, double* u, int32_t parts,
                                   void* stream, double* stage_ms);

/* ---- multi-GPU slab decomposition (no reference counterpart:
 * the reference is single-process numpy).  The near grid is split into
 * `world` x-slabs; shard r owns those planes, the observers (= sources) whose
 * stencil starts there and their correction pairs, and 1/world of the FFT
 * columns for the x transforms (NCCL all-to-all transposes; far-grid
 * all-reduce; order-plane halo).  nccl_id != NULL: this process is shard `rank`
 * on p->device, all processes pass the same 128-byte id from
 * fftpim_nccl_unique_id.  nccl_id == NULL: all shards are emulated inside this
 * process on p->device (exchanges become device copies).  Observers must be the
 * sources; all three axes active. */
typedef struct FftpimGroup FftpimGroup;
FFTPIM_API int fftpim_nccl_unique_id(void* out, int64_t bytes);
FFTPIM_API int fftpim_group_create(const FftpimProblem* p, int32_t world, int32_t rank, const void* nccl_id,
                                   FftpimGroup** out);
/* q: all n_src amplitudes (device); u: n_obs outputs (device) -- each process
 * writes the observers its shard(s) own.  Stream ordered on `stream`. */
FFTPIM_API int fftpim_group_evaluate(FftpimGroup* g, const double* q, double* u, void* stream);
FFTPIM_API int fftpim_group_info(const FftpimGroup* g, int32_t shard, FftpimInfo* info);
FFTPIM_API void fftpim_group_destroy(FftpimGroup* g);

/* Number of kernel launches this library issued since load (evidence counter). */
FFTPIM_API int64_t fftpim_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FFTPIM_H */
