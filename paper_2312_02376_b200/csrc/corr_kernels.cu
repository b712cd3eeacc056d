// corr_kernels.cu -- the correction matvec (K4, nearzone.py:506-524) and the
// fused observer pass (K3 near interpolation grids.py:183-188 + K5c far
// interpolation farzone.py:159 + the K4 row fix-up).
//
// K4 streams the pair list flat, one warp per CORR_TILE (=256) consecutive
// pairs, independent of the row (observer) structure:
//   1. coalesced strided loads of the int32 source indices, the coefficients and
//      the tile's row-start bits (1 bit per pair, set where an observer's pairs
//      begin) -- all independent, one memory round trip;
//   2. the q gathers and products (second round trip, L2-resident q);
//   3. a shared-memory transpose to 8 consecutive pairs per lane, a lane-local
//      segmented sum and a 5-step warp segmented scan for the carries;
//   4. every (row, tile) segment total goes to seg_val[seg_base[tile] + k].
// The observer pass adds the <= 1 + P/M/256 segments of its row in order.
// No atomics, fixed orders: bitwise reproducible.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <climits>
#include <vector>

#include "geom.cuh"
#include "kernels.h"

static inline int nblk64(int64_t n, int t) { return (int)((n + t - 1) / t); }

__device__ __forceinline__ cplx wsum(cplx v) {
    for (int o = 16; o > 0; o >>= 1) {
        v.re += __shfl_xor_sync(0xffffffffu, v.re, o);
        v.im += __shfl_xor_sync(0xffffffffu, v.im, o);
    }
    return v;
}

// ------------------------------------------------------------- plan-build metadata
__global__ void k_head_bits(const int64_t* __restrict__ ptr, int64_t M, unsigned* bits) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    const int64_t p = ptr[i];
    if (p < ptr[i + 1]) atomicOr(bits + (p >> 5), 1u << (p & 31));
}

__global__ void k_row_spans(const int64_t* __restrict__ ptr, int64_t M, int64_t* spans) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > M) return;
    if (i == M) {
        spans[i] = 0;
        return;
    }
    const int64_t p0 = ptr[i], p1 = ptr[i + 1];
    spans[i] = p0 == p1 ? 0 : (p1 - 1) / CORR_TILE - p0 / CORR_TILE + 1;
}

// global index of the segment holding the first pair of tile t
__global__ void k_seg_base(const int64_t* __restrict__ ptr, const int64_t* __restrict__ seg_first, int64_t M,
                           int64_t T, int64_t* seg_base) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= T) return;
    const int64_t p = t * CORR_TILE;
    int64_t lo = 0, hi = M;   // last row with ptr[row] <= p (ptr[lo] <= p < ptr[hi])
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (ptr[mid] <= p) lo = mid; else hi = mid;
    }
    seg_base[t] = seg_first[lo] + (t - ptr[lo] / CORR_TILE);
}

void build_corr_metadata(const int64_t* ptr, int64_t M, int64_t P, int64_t T, unsigned* bits, int64_t* seg_first,
                         int64_t* seg_base, int64_t* spans_tmp, int64_t* n_segments, cudaStream_t s) {
    cudaMemsetAsync(bits, 0, sizeof(unsigned) * ((P + 31) / 32 + 8), s);
    if (M > 0) k_head_bits<<<nblk64(M, 256), 256, 0, s>>>(ptr, M, bits);
    k_row_spans<<<nblk64(M + 1, 256), 256, 0, s>>>(ptr, M, spans_tmp);
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, spans_tmp, seg_first, (int)(M + 1), s);
    void* tmp = nullptr;
    cudaMallocAsync(&tmp, bytes + 16, s);
    cub::DeviceScan::ExclusiveSum(tmp, bytes, spans_tmp, seg_first, (int)(M + 1), s);
    cudaFreeAsync(tmp, s);
    if (T > 0) k_seg_base<<<nblk64(T, 256), 256, 0, s>>>(ptr, seg_first, M, T, seg_base);
    cudaMemcpyAsync(n_segments, seg_first + M, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fftpim_count_launch(5);
}

// ------------------------------------------------------------- K4 warp tiles
// Tile = 8 groups of 32 consecutive pairs (pair e = 32k + lane), loaded
// coalesced.  Each lane keeps a running partial of the current (row, tile)
// segment; a group without a row start (the common case: ~221 pairs per row at
// C2, ~13k at C3) costs nothing beyond the FMAs.  A group containing row
// starts closes segments with one fixed-tree warp sum per start.
#ifndef CORR_WARPS
#define CORR_WARPS 8
#endif
#ifndef CORR_MINB
#define CORR_MINB 2
#endif
// one tile's streamed data: indices, coefficients, row-start word, segment base
struct CorrTile {
    int src[8];
    double cr[8], ci[8];
    unsigned word;
    int64_t sbase;
};

template <bool REAL>
__device__ __forceinline__ void corr_load(const EvalArgs& a, int64_t t, int lane, CorrTile& d) {
    const int64_t T0 = t * CORR_TILE;
    const int valid = (int)min((int64_t)CORR_TILE, a.n_pairs - T0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int e = 32 * k + lane;
        const bool ok = e < valid;
        d.src[k] = ok ? __ldcs(a.pair_src + T0 + e) : 0;
        if (REAL) {
            d.cr[k] = ok ? __ldcs(a.coef_r + T0 + e) : 0.0;
            d.ci[k] = 0.0;
        } else {
            const double2 c = ok ? __ldcs(reinterpret_cast<const double2*>(a.coef) + T0 + e) : make_double2(0.0, 0.0);
            d.cr[k] = c.x;
            d.ci[k] = c.y;
        }
    }
    // row-start words of the 8 groups: lane k < 8 loads word k, then broadcast per group
    d.word = lane < 8 ? a.head_bits[(T0 >> 5) + lane] : 0u;
    d.sbase = a.seg_base[t];
}

// segmented accumulation of one tile in pair order: every (row, tile) segment
// total goes to seg_val[sbase + k]
__device__ __forceinline__ void corr_reduce_tile(const EvalArgs& a, int lane, const double* cr, const double* ci,
                                                 const double* qr, const double* qi, unsigned myword, int64_t sbase) {
    double accr = 0.0, acci = 0.0;
    int seg = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const double pr = cr[k] * qr[k] - ci[k] * qi[k];
        const double pi = cr[k] * qi[k] + ci[k] * qr[k];
        unsigned f = __shfl_sync(0xffffffffu, myword, k);
        if (k == 0) f &= ~1u;   // a row starting at the tile start is segment 0 itself
        if (f == 0u) {
            accr += pr;
            acci += pi;
            continue;
        }
        // close the open segment with the lanes before the first start
        int s = __ffs(f) - 1;
        {
            double vr = accr + (lane < s ? pr : 0.0), vi = acci + (lane < s ? pi : 0.0);
            const cplx v = wsum(cplx{vr, vi});
            if (lane == 0) a.seg_val[sbase + seg] = v;
            ++seg;
        }
        f &= f - 1u;
        // segments wholly inside this group
        while (f) {
            const int s2 = __ffs(f) - 1;
            const bool in = lane >= s && lane < s2;
            const cplx v = wsum(cplx{in ? pr : 0.0, in ? pi : 0.0});
            if (lane == 0) a.seg_val[sbase + seg] = v;
            ++seg;
            s = s2;
            f &= f - 1u;
        }
        // the last start opens the new running segment
        accr = lane >= s ? pr : 0.0;
        acci = lane >= s ? pi : 0.0;
    }
    const cplx v = wsum(cplx{accr, acci});
    if (lane == 0) a.seg_val[sbase + seg] = v;
}

// NPSP plans with real charges: a three-stage software pipeline per warp --
// the stream of tile t + 2s, the 8-byte q gathers of tile t + s (its indices
// arrived one iteration earlier) and the reduction of tile t overlap, so the
// gather latency is hidden as well as the stream's.  Same operations in the
// same order as the generic path (imaginary parts exact zeros): identical bits.
struct RealTile {
    int src[8];
    double cr[8];
    unsigned word;
    int64_t sbase;
};

__device__ __forceinline__ void corr_load_real(const EvalArgs& a, int64_t t, int lane, RealTile& d) {
    const int64_t T0 = t * CORR_TILE;
    const int valid = (int)min((int64_t)CORR_TILE, a.n_pairs - T0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int e = 32 * k + lane;
        const bool ok = e < valid;
        d.src[k] = ok ? __ldcs(a.pair_src + T0 + e) : 0;
        d.cr[k] = ok ? __ldcs(a.coef_r + T0 + e) : 0.0;
    }
    d.word = lane < 8 ? a.head_bits[(T0 >> 5) + lane] : 0u;
    d.sbase = a.seg_base[t];
}

__device__ __forceinline__ void corr_tiles_realq(const EvalArgs& a, int64_t t, int64_t stride, int64_t T, int lane) {
    const double zero[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    RealTile c0, c1;
    double q0[8];
    if (t >= T) return;
    corr_load_real(a, t, lane, c0);
#pragma unroll
    for (int k = 0; k < 8; ++k) q0[k] = a.q_re[c0.src[k]];
    if (t + stride < T) corr_load_real(a, t + stride, lane, c1);
    for (; t < T; t += stride) {
        RealTile c2;
        if (t + 2 * stride < T) corr_load_real(a, t + 2 * stride, lane, c2);
        double q1[8];
        if (t + stride < T) {
#pragma unroll
            for (int k = 0; k < 8; ++k) q1[k] = a.q_re[c1.src[k]];
        }
        corr_reduce_tile(a, lane, c0.cr, zero, q0, zero, c0.word, c0.sbase);
        c0 = c1;
#pragma unroll
        for (int k = 0; k < 8; ++k) q0[k] = q1[k];
        c1 = c2;
    }
}

// CORR_PF: the next tile's stream loads are issued before this tile's gathers,
// so every warp keeps two tiles of pair data in flight
#ifndef CORR_PF
#define CORR_PF 1
#endif
#ifndef CORR_RQ_PIPE   // three-stage pipeline for real coefficients and real charges
#define CORR_RQ_PIPE 1
#endif
#ifndef CORR_PF_REAL
#define CORR_PF_REAL 1
#endif
// DEPTH: tiles of pair data in flight beyond the one being reduced (0: none)
template <bool REAL, int DEPTH>
__global__ void __launch_bounds__(32 * CORR_WARPS, CORR_MINB) k_corr_tiles(EvalArgs a) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t T = (a.n_pairs + CORR_TILE - 1) / CORR_TILE;
    const int64_t stride = (int64_t)gridDim.x * CORR_WARPS;
    int64_t t = (int64_t)blockIdx.x * CORR_WARPS + warp;
    const bool realq = REAL && a.q_re && *(volatile const int*)a.q_flag == 0;
#if CORR_RQ_PIPE
    if (REAL && realq) {
        corr_tiles_realq(a, t, stride, T, lane);
        return;
    }
#endif
    CorrTile cur, n1;
    if (DEPTH >= 1 && t < T) corr_load<REAL>(a, t, lane, cur);
    if (DEPTH >= 2 && t + stride < T) corr_load<REAL>(a, t + stride, lane, n1);
    for (; t < T; t += stride) {
        CorrTile nxt;
        if (DEPTH == 0) {
            corr_load<REAL>(a, t, lane, cur);
        } else if (t + DEPTH * stride < T) {
            corr_load<REAL>(a, t + DEPTH * stride, lane, nxt);
        }
        const int* src = cur.src;
        const double* cr = cur.cr;
        const double* ci = cur.ci;
        const unsigned myword = cur.word;
        const int64_t sbase = cur.sbase;
        // 2. gathers (all 8 in flight)
        double qr[8], qi[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
#ifdef CORR_NOGATHER   // diagnostic variant: stream-only cost of K4
            const cplx qv = a.q_sorted[(src[k] & 31) + lane];
#else
            cplx qv;
            if (realq) {
                qv.re = a.q_re[src[k]];
                qv.im = 0.0;
            } else {
                qv = a.q_sorted[src[k]];
            }
#endif
            qr[k] = qv.re;
            qi[k] = qv.im;
        }
        corr_reduce_tile(a, lane, cr, ci, qr, qi, myword, sbase);
        if (DEPTH == 1) {
            cur = nxt;
        } else if (DEPTH == 2) {
            cur = n1;
            n1 = nxt;
        }
    }
}

// ------------------------------------------------------------- K4, 16-bit indices
// The source index stream is 4 of the 20 (complex) or 12 (NPSP) bytes a pair
// costs.  Pairs are grouped by 32 (the K4 load groups); a group whose source
// indices span <= 65535 stores them as 16-bit offsets from a per-group int32
// base (grp_base >= 0), a wider group (observer-row or wrapped-copy transitions)
// is marked grp_base < 0 and reads the full int32 indices.  The group bases
// travel with the tile's row-start words one tile ahead of the stream, so the
// stream loads of a tile (16-bit offsets or int32 indices, coefficients) never
// wait on them.  Same pairs, same order, same arithmetic: the potentials are
// bit-identical to the int32 path.
struct CorrMeta {
    int gb;            // lane k < 8: base of the tile's group k (< 0: wide)
    unsigned word;     // lane k < 8: row-start bits of group k
    int64_t sbase;
};

__device__ __forceinline__ void corr_meta(const EvalArgs& a, int64_t t, int lane, CorrMeta& m) {
    const int64_t g0 = t * (CORR_TILE / 32);
    m.gb = lane < 8 ? __ldcs(a.grp_base + g0 + lane) : 0;
    m.word = lane < 8 ? a.head_bits[g0 + lane] : 0u;
    m.sbase = a.seg_base[t];
}

template <bool REAL>
__device__ __forceinline__ void corr_stream(const EvalArgs& a, int64_t t, int lane, const CorrMeta& m,
                                            CorrTile& d) {
    const int64_t T0 = t * CORR_TILE;
    const int valid = (int)min((int64_t)CORR_TILE, a.n_pairs - T0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int e = 32 * k + lane;
        const bool ok = e < valid;
        const int gb = __shfl_sync(0xffffffffu, m.gb, k);
        if (gb >= 0)
            d.src[k] = ok ? (int)__ldcs(a.pair_off16 + T0 + e) : 0;
        else
            d.src[k] = ok ? __ldcs(a.pair_src + T0 + e) : 0;
        if (REAL) {
            d.cr[k] = ok ? __ldcs(a.coef_r + T0 + e) : 0.0;
            d.ci[k] = 0.0;
        } else {
            const double2 c = ok ? __ldcs(reinterpret_cast<const double2*>(a.coef) + T0 + e) : make_double2(0.0, 0.0);
            d.cr[k] = c.x;
            d.ci[k] = c.y;
        }
    }
    d.word = m.word;
    d.sbase = m.sbase;
}

// 16-bit offsets -> sorted source indices (lane k < 8 of gbw holds group k's base)
__device__ __forceinline__ void corr_decode(int* src, int gbw) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int gb = __shfl_sync(0xffffffffu, gbw, k);
        if (gb >= 0) src[k] += gb;
    }
}

// NPSP real charges: the three-stage pipeline of corr_tiles_realq (stream of tile
// t + 2s, gathers of t + s, reduction of t) with the group bases one stage earlier
__device__ __forceinline__ void corr_stream_real(const EvalArgs& a, int64_t t, int lane, const CorrMeta& m,
                                                 RealTile& d) {
    const int64_t T0 = t * CORR_TILE;
    const int valid = (int)min((int64_t)CORR_TILE, a.n_pairs - T0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int e = 32 * k + lane;
        const bool ok = e < valid;
        const int gb = __shfl_sync(0xffffffffu, m.gb, k);
        if (gb >= 0)
            d.src[k] = ok ? (int)__ldcs(a.pair_off16 + T0 + e) : 0;
        else
            d.src[k] = ok ? __ldcs(a.pair_src + T0 + e) : 0;
        d.cr[k] = ok ? __ldcs(a.coef_r + T0 + e) : 0.0;
    }
    d.word = m.word;
    d.sbase = m.sbase;
}

__device__ __forceinline__ void corr_tiles_realq_c16(const EvalArgs& a, int64_t t, int64_t stride, int64_t T,
                                                     int lane) {
    const double zero[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    RealTile c0, c1;
    CorrMeta m0, m1, m2;
    double q0[8];
    int g1 = 0;
    corr_meta(a, t, lane, m0);
    corr_stream_real(a, t, lane, m0, c0);
    corr_decode(c0.src, m0.gb);
#pragma unroll
    for (int k = 0; k < 8; ++k) q0[k] = a.q_re[c0.src[k]];
    if (t + stride < T) {
        corr_meta(a, t + stride, lane, m1);
        corr_stream_real(a, t + stride, lane, m1, c1);
        g1 = m1.gb;
    }
    if (t + 2 * stride < T) corr_meta(a, t + 2 * stride, lane, m2);
    for (; t < T; t += stride) {
        CorrMeta m3;
        if (t + 3 * stride < T) corr_meta(a, t + 3 * stride, lane, m3);
        RealTile c2;
        int g2 = 0;
        if (t + 2 * stride < T) {
            corr_stream_real(a, t + 2 * stride, lane, m2, c2);
            g2 = m2.gb;
        }
        double q1[8];
        if (t + stride < T) {
            corr_decode(c1.src, g1);
#pragma unroll
            for (int k = 0; k < 8; ++k) q1[k] = a.q_re[c1.src[k]];
        }
        corr_reduce_tile(a, lane, c0.cr, zero, q0, zero, c0.word, c0.sbase);
        c0 = c1;
#pragma unroll
        for (int k = 0; k < 8; ++k) q0[k] = q1[k];
        c1 = c2;
        g1 = g2;
        m2 = m3;
    }
}

template <bool REAL>
__global__ void __launch_bounds__(32 * CORR_WARPS, CORR_MINB) k_corr_tiles_c16(EvalArgs a) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t T = (a.n_pairs + CORR_TILE - 1) / CORR_TILE;
    const int64_t stride = (int64_t)gridDim.x * CORR_WARPS;
    int64_t t = (int64_t)blockIdx.x * CORR_WARPS + warp;
    if (t >= T) return;
    const bool realq = REAL && a.q_re && *(volatile const int*)a.q_flag == 0;
    if (REAL && realq) {
        corr_tiles_realq_c16(a, t, stride, T, lane);
        return;
    }
    // pipeline: meta of tile t + 2s, stream of tile t + s, gathers + reduction of tile t
    CorrMeta m1, m2;
    CorrTile cur, nxt;
    int gcur, gnxt = 0;
    {
        CorrMeta m0;
        corr_meta(a, t, lane, m0);
        corr_stream<REAL>(a, t, lane, m0, cur);
        gcur = m0.gb;
    }
    if (t + stride < T) corr_meta(a, t + stride, lane, m1);
    for (; t < T; t += stride) {
        if (t + 2 * stride < T) corr_meta(a, t + 2 * stride, lane, m2);
        if (t + stride < T) {
            corr_stream<REAL>(a, t + stride, lane, m1, nxt);
            gnxt = m1.gb;
        }
        corr_decode(cur.src, gcur);
        double qr[8], qi[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            cplx qv;
            if (realq) {
                qv.re = a.q_re[cur.src[k]];
                qv.im = 0.0;
            } else {
                qv = a.q_sorted[cur.src[k]];
            }
            qr[k] = qv.re;
            qi[k] = qv.im;
        }
        corr_reduce_tile(a, lane, cur.cr, cur.ci, qr, qi, cur.word, cur.sbase);
        cur = nxt;
        gcur = gnxt;
        m1 = m2;
    }
}

// per 32-pair group: base = smallest source index if the group's indices span
// <= 65535 (16-bit offsets written), else -1 (the group keeps int32 indices)
__global__ void k_group_encode(const int* __restrict__ src, int64_t P, int64_t G, int* base, unsigned short* off,
                               unsigned long long* wide) {
    const int lane = threadIdx.x & 31;
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (g >= G) return;
    const int64_t p = g * 32 + lane;
    const int v = p < P ? src[p] : INT_MAX;
    int lo = v, hi = p < P ? v : INT_MIN;
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const bool narrow = (int64_t)hi - lo <= 65535;
    if (p < P) off[p] = narrow ? (unsigned short)(v - lo) : (unsigned short)0;
    if (lane == 0) {
        base[g] = narrow ? lo : -1;
        if (!narrow) atomicAdd(wide, 1ull);
    }
}

// base: (G + 8) ints (the last tile's lanes read up to 8 groups past the end)
int64_t build_group_offsets(const int* src, int64_t P, int* base, unsigned short* off, cudaStream_t s) {
    const int64_t G = (P + 31) / 32;
    unsigned long long* d = nullptr;
    cudaMallocAsync(&d, sizeof(unsigned long long), s);
    cudaMemsetAsync(d, 0, sizeof(unsigned long long), s);
    cudaMemsetAsync(base + G, 0, 8 * sizeof(int), s);
    if (G > 0) k_group_encode<<<nblk64(G * 32, 256), 256, 0, s>>>(src, P, G, base, off, d);
    unsigned long long h = 0;
    cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFreeAsync(d, s);
    fftpim_count_launch();
    return (int64_t)h;
}

// ------------------------------------------------------------- pair rows in source order
// K4 at C4 is bound by L1 wavefronts, and most of them are the q gathers: in the
// reference's pair order (box offsets db-major, nearzone.py:374-478) consecutive
// pairs of a row jump between the 4-8 stencil-cell rows a box straddles, so a
// warp's 32 gathers touch ~16 lines.  Sorting every row by source index makes
// consecutive lanes read consecutive charges (one or two lines per z run).  Same
// pair set, same coefficients; only the order of the row sum changes (~1e-16).
__global__ void k_chunk_offsets(const int64_t* __restrict__ ptr, int64_t r0, int64_t nseg, int* off, int* iota,
                                int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i <= nseg) off[i] = (int)(ptr[r0 + i] - ptr[r0]);
    if (i < n) iota[i] = (int)i;
}
template <typename T>
__global__ void k_permute_rows(const T* __restrict__ src, const int* __restrict__ perm, int64_t n, T* dst) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}

bool sort_pair_rows(const int64_t* ptr, int64_t M, int* pair_src, cplx* const* carr, int ncarr, double* coef_r,
                    unsigned char* codeid, size_t budget, cudaStream_t s) {
    std::vector<int64_t> hp(M + 1);
    if (cudaMemcpyAsync(hp.data(), ptr, sizeof(int64_t) * (M + 1), cudaMemcpyDeviceToHost, s) != cudaSuccess) return false;
    cudaStreamSynchronize(s);
    const int64_t P = hp[M];
    const size_t per = 4 + 4 + 4 + 16 + 1 + 16;   // keys out, iota, perm, coefficient and code copies, cub
    int64_t CH = std::min<int64_t>((int64_t)1 << 28, (int64_t)(budget / per));
    if (CH < (int64_t)1 << 20) return false;
    int *koff = nullptr, *iota = nullptr, *perm = nullptr, *kout = nullptr, *offs = nullptr;
    void* vtmp = nullptr;
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0;
    bool ok = true;
    auto fail = [&] { ok = false; };
    if (cudaMallocAsync(&iota, sizeof(int) * CH, s) || cudaMallocAsync(&perm, sizeof(int) * CH, s) ||
        cudaMallocAsync(&kout, sizeof(int) * CH, s) || cudaMallocAsync(&vtmp, sizeof(cplx) * CH, s))
        fail();
    (void)koff;
    int64_t r0 = 0;
    while (ok && r0 < M) {
        // rows [r0, r1) with at most CH pairs (a single longer row is left unsorted)
        int64_t r1 = r0 + 1;
        {
            int64_t lo = r0 + 1, hi = M;
            while (lo < hi) {   // largest r1 with hp[r1] - hp[r0] <= CH
                const int64_t mid = (lo + hi + 1) / 2;
                if (hp[mid] - hp[r0] <= CH) lo = mid; else hi = mid - 1;
            }
            r1 = lo;
        }
        const int64_t n = hp[r1] - hp[r0], nseg = r1 - r0;
        if (n > CH || nseg > ((int64_t)1 << 30)) {   // one row longer than a chunk: keep its order
            r0 = r1;
            continue;
        }
        if (n > 1) {
            if (cudaMallocAsync(&offs, sizeof(int) * (nseg + 1), s)) {
                fail();
                break;
            }
            k_chunk_offsets<<<nblk64(std::max(nseg + 1, n), 256), 256, 0, s>>>(ptr, r0, nseg, offs, iota, n);
            const int64_t p0 = hp[r0];
            size_t need = 0;
            cub::DeviceSegmentedSort::StableSortPairs(nullptr, need, pair_src + p0, kout, iota, perm, (int)n, (int)nseg,
                                                       offs, offs + 1, s);
            if (need > cub_bytes) {
                if (cub_tmp) cudaFreeAsync(cub_tmp, s);
                cub_tmp = nullptr;
                if (cudaMallocAsync(&cub_tmp, need, s)) {
                    fail();
                    break;
                }
                cub_bytes = need;
            }
            cub::DeviceSegmentedSort::StableSortPairs(cub_tmp, cub_bytes, pair_src + p0, kout, iota, perm, (int)n,
                                                       (int)nseg, offs, offs + 1, s);
            cudaMemcpyAsync(pair_src + p0, kout, sizeof(int) * n, cudaMemcpyDeviceToDevice, s);
            for (int c = 0; c < ncarr; ++c) {   // coefficients (or the sweep's phase components)
                cplx* coef = carr[c];
                k_permute_rows<cplx><<<nblk64(n, 256), 256, 0, s>>>(coef + p0, perm, n, (cplx*)vtmp);
                cudaMemcpyAsync(coef + p0, vtmp, sizeof(cplx) * n, cudaMemcpyDeviceToDevice, s);
            }
            if (coef_r) {
                k_permute_rows<double><<<nblk64(n, 256), 256, 0, s>>>(coef_r + p0, perm, n, (double*)vtmp);
                cudaMemcpyAsync(coef_r + p0, vtmp, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
            }
            if (codeid) {
                k_permute_rows<unsigned char><<<nblk64(n, 256), 256, 0, s>>>(codeid + p0, perm, n,
                                                                             (unsigned char*)vtmp);
                cudaMemcpyAsync(codeid + p0, vtmp, n, cudaMemcpyDeviceToDevice, s);
            }
            cudaFreeAsync(offs, s);
            offs = nullptr;
            fftpim_count_launch(3);
        }
        r0 = r1;
    }
    if (cub_tmp) cudaFreeAsync(cub_tmp, s);
    if (iota) cudaFreeAsync(iota, s);
    if (perm) cudaFreeAsync(perm, s);
    if (kout) cudaFreeAsync(kout, s);
    if (vtmp) cudaFreeAsync(vtmp, s);
    cudaStreamSynchronize(s);
    return ok && cudaGetLastError() == cudaSuccess;
}

// ------------------------------------------------------------- K4, run-encoded sources
// With rows in source order the source indices of consecutive pairs mostly
// count up by one (the sorted sources of one z run of stencil cells), so the
// int32 index per pair (4 of the 20 or 12 bytes a pair costs) is replaced by
//   * one more bit per pair (run starts: tile starts, row starts, breaks in the
//     index sequence) and
//   * one int32 per run: bias = source of the run's first pair - its position e
//     in the tile, so that src(e) = bias[rank(e)] + e, rank(e) = run starts at
//     positions <= e, minus one (a popcount prefix over the tile's 8 run words).
// Per tile the plan holds one 384-byte record: row-start words, run-start words,
// first segment, run count, and the tile's first RUNS_BIAS_CAP biases (later
// ones, rows in discovery order only, sit in an overflow array).
// The kernel streams with bulk asynchronous copies (cp.async.bulk -> shared
// memory, completion on an mbarrier) instead of per-thread loads: each warp owns
// a ring of RUNS_STAGES stage buffers (a tile's coefficients + its record), lane
// 0 issues the two copies of a tile RUNS_STAGES - 1 tiles ahead, and the
// in-flight stream lives in shared memory, not registers.  Same pairs, same
// order, same arithmetic as k_corr_tiles: bit-identical potentials.
#ifndef RUNS_WARPS
#define RUNS_WARPS 20
#endif
#ifndef RUNS_STAGES
#define RUNS_STAGES 2
#endif
#define RUNS_BIAS_CAP 64
#define RUNS_REC_WORDS 96   // 0-7 row-start words, 8-15 run-start words, 16-17 first segment,
                            // 18-19 first overflow bias, 20 runs, 21-22 run-count prefix of the 8
                            // groups (one byte each), 32-95 biases
#define RUNS_QPAD CORR_TILE // zero charges past q_sorted[N): the last tile's padding pairs read them

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!ok);
}
// global -> shared bulk copy (bytes a multiple of 16, both addresses 16-byte
// aligned), streamed through L2 with an evict-first policy
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

template <bool REAL>
struct RunsStage {
    static constexpr int coef_bytes = CORR_TILE * (REAL ? 8 : 16);
    static constexpr int bytes = coef_bytes + RUNS_REC_WORDS * 4;
};

// lane 0: start the two copies of tile t into one stage (the coefficient
// arrays are padded with zeros to whole tiles)
template <bool REAL>
__device__ __forceinline__ void runs_issue(const EvalArgs& a, int t, uint32_t stage, uint32_t bar, uint64_t pol) {
    mbar_expect_tx(bar, RunsStage<REAL>::bytes);
    if (REAL)
        bulk_g2s(stage, a.coef_r + (int64_t)t * CORR_TILE, RunsStage<REAL>::coef_bytes, bar, pol);
    else
        bulk_g2s(stage, a.coef + (int64_t)t * CORR_TILE, RunsStage<REAL>::coef_bytes, bar, pol);
    bulk_g2s(stage + RunsStage<REAL>::coef_bytes, a.run_rec + (int64_t)t * RUNS_REC_WORDS, RUNS_REC_WORDS * 4, bar, pol);
}

__device__ __forceinline__ int64_t meta_i64(unsigned m, int w) {
    const unsigned lo = __shfl_sync(0xffffffffu, m, w), hi = __shfl_sync(0xffffffffu, m, w + 1);
    return (int64_t)(((unsigned long long)hi << 32) | lo);
}

// Tile order of one warp.  Static: tiles warp, warp + stride, ... of a
// persistent grid.  Dynamic (a.k4_counter): chunks of RUNS_CHUNK consecutive
// tiles claimed from a global counter, one chunk ahead, so that launches sharing
// the counter (the main grid beside the near chain, a helper grid after it)
// and blocks that start late all drain one queue in stream order.
#define RUNS_CHUNK 8
struct TileQueue {
    int cur, end, step, T;
    unsigned next_raw;             // lane 0: the pre-claimed chunk
    unsigned* counter;             // null: static
    __device__ __forceinline__ void init(const EvalArgs& a, int T_, int warp, int warps, int lane) {
        T = T_;
        counter = reinterpret_cast<unsigned*>(a.k4_counter);
        next_raw = 0;
        if (counter) {
            unsigned c = 0;
            if (lane == 0) c = atomicAdd(counter, 1u);
            c = __shfl_sync(0xffffffffu, c, 0);
            cur = (int)min((unsigned)T, c * RUNS_CHUNK);
            end = min(cur + RUNS_CHUNK, T);
            if (lane == 0 && cur < T) next_raw = atomicAdd(counter, 1u);
            step = 1;
        } else {
            cur = blockIdx.x * warps + warp;
            step = gridDim.x * warps;
            end = T;
        }
    }
    // the next tile of this warp (>= T: none left)
    __device__ __forceinline__ int next(int lane) {
        if (cur < end) {
            const int t = cur;
            cur += step;
            return t;
        }
        if (!counter || cur >= T) return T;
        const unsigned c = __shfl_sync(0xffffffffu, next_raw, 0);
        cur = (int)min((unsigned)T, c * RUNS_CHUNK);
        end = min(cur + RUNS_CHUNK, T);
        if (cur >= T) return T;
        if (lane == 0) next_raw = atomicAdd(counter, 1u);
        return cur++;
    }
};

// segmented accumulation in pair order, one 32-pair group at a time (same
// operations and order as corr_reduce_tile)
struct SegAcc {
    double accr, acci;
    int seg;
    __device__ __forceinline__ void begin() {
        accr = acci = 0.0;
        seg = 0;
    }
    // f: row-start bits of the group (bit 0 of the tile's first group cleared by the caller)
    __device__ __forceinline__ void add(const EvalArgs& a, int lane, double pr, double pi, unsigned f, int64_t sbase) {
        if (f == 0u) {
            accr += pr;
            acci += pi;
            return;
        }
        int s = __ffs(f) - 1;
        {
            double vr = accr + (lane < s ? pr : 0.0), vi = acci + (lane < s ? pi : 0.0);
            const cplx v = wsum(cplx{vr, vi});
            if (lane == 0) a.seg_val[sbase + seg] = v;
            ++seg;
        }
        f &= f - 1u;
        while (f) {
            const int s2 = __ffs(f) - 1;
            const bool in = lane >= s && lane < s2;
            const cplx v = wsum(cplx{in ? pr : 0.0, in ? pi : 0.0});
            if (lane == 0) a.seg_val[sbase + seg] = v;
            ++seg;
            s = s2;
            f &= f - 1u;
        }
        accr = lane >= s ? pr : 0.0;
        acci = lane >= s ? pi : 0.0;
    }
    __device__ __forceinline__ void end(const EvalArgs& a, int lane, int64_t sbase) {
        const cplx v = wsum(cplx{accr, acci});
        if (lane == 0) a.seg_val[sbase + seg] = v;
    }
};

// one staged tile: sources from the record (rank of each pair among the run
// starts -> bias -> bias + e), gathers, products, segmented sums
template <bool REAL>
__device__ __forceinline__ void runs_tile(const EvalArgs& a, const unsigned char* st, int lane, unsigned le_mask,
                                          bool realq) {
    const uint4* rec4 = reinterpret_cast<const uint4*>(st + RunsStage<REAL>::coef_bytes);
    const int* sbias_m1 = reinterpret_cast<const int*>(rec4 + 8) - 1;
    const uint4 h0 = rec4[0], h1 = rec4[1], r0 = rec4[2], r1 = rec4[3], mt = rec4[4], mn = rec4[5];
    const unsigned hw[8] = {h0.x & ~1u, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
    const unsigned rw[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    const int64_t sbase = (int64_t)(((unsigned long long)mt.y << 32) | mt.x);
    const int nruns = (int)mn.x;
    int src[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const unsigned pk = k < 4 ? mn.y : mn.z;
        src[k] = (int)((pk >> (8 * (k & 3))) & 0xffu) + __popc(rw[k] & le_mask);   // rank + 1
    }
    if (nruns <= RUNS_BIAS_CAP) {
#pragma unroll
        for (int k = 0; k < 8; ++k) src[k] = sbias_m1[src[k]] + (32 * k + lane);
    } else {   // rows in discovery order: biases past the record
        const int64_t ob = (int64_t)(((unsigned long long)mt.w << 32) | mt.z);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int r = src[k] - 1;
            src[k] = (r < RUNS_BIAS_CAP ? sbias_m1[r + 1] : __ldg(a.run_bias + ob + (r - RUNS_BIAS_CAP))) +
                     (32 * k + lane);
        }
    }
    double qr[8], qi[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (realq) {
            qr[k] = a.q_re[src[k]];
            qi[k] = 0.0;
        } else {
            const cplx qv = a.q_sorted[src[k]];
            qr[k] = qv.re;
            qi[k] = qv.im;
        }
    }
    SegAcc acc;
    acc.begin();
    // most tiles lie inside one row (no row start past the tile's first pair):
    // straight-line sums, the same operations in the same order
    const bool one_row = ((hw[0] | hw[1] | hw[2] | hw[3]) | (hw[4] | hw[5] | hw[6] | hw[7])) == 0u;
    if (one_row) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double cr, ci;
            if (REAL) {
                cr = reinterpret_cast<const double*>(st)[32 * k + lane];
                ci = 0.0;
            } else {
                const double2 c = reinterpret_cast<const double2*>(st)[32 * k + lane];
                cr = c.x;
                ci = c.y;
            }
            acc.accr += cr * qr[k] - ci * qi[k];
            acc.acci += cr * qi[k] + ci * qr[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double cr, ci;
            if (REAL) {
                cr = reinterpret_cast<const double*>(st)[32 * k + lane];
                ci = 0.0;
            } else {
                const double2 c = reinterpret_cast<const double2*>(st)[32 * k + lane];
                cr = c.x;
                ci = c.y;
            }
            const double pr = cr * qr[k] - ci * qi[k];
            const double pi = cr * qi[k] + ci * qr[k];
            acc.add(a, lane, pr, pi, hw[k], sbase);
        }
    }
    acc.end(a, lane, sbase);
}

template <bool REAL>
__global__ void __launch_bounds__(32 * RUNS_WARPS, 1) k_corr_runs(EvalArgs a) {
    extern __shared__ __align__(128) unsigned char runs_smem[];
    constexpr int SS = RunsStage<REAL>::bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, warps = blockDim.x >> 5;
    const int T = (int)((a.n_pairs + CORR_TILE - 1) / CORR_TILE);
    TileQueue tq;
    tq.init(a, T, warp, warps, lane);
    const bool realq = REAL && a.q_re && *(volatile const int*)a.q_flag == 0;
    unsigned char* my = runs_smem + (size_t)warp * RUNS_STAGES * SS;
    const uint32_t stage0 = smem_addr(my);
    const uint32_t bar0 = smem_addr(runs_smem + (size_t)warps * RUNS_STAGES * SS) + warp * RUNS_STAGES * 8;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < RUNS_STAGES; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // the warp reduces its tiles in the order the queue hands them out, so it only
    // counts the tiles issued and not yet reduced
    int pending = 0;
#pragma unroll
    for (int j = 0; j < RUNS_STAGES; ++j) {
        const int tj = tq.next(lane);
        if (tj < T) {
            if (lane == 0) runs_issue<REAL>(a, tj, stage0 + j * SS, bar0 + 8 * j, pol);
            ++pending;
        }
    }
    uint32_t ph = 0;
    const unsigned le_mask = 0xffffffffu >> (31 - lane);
    while (pending > 0) {
#pragma unroll
        for (int s = 0; s < RUNS_STAGES; ++s) {   // static stage addresses
            if (pending == 0) break;
            mbar_wait(bar0 + 8 * s, ph);
            runs_tile<REAL>(a, my + s * SS, lane, le_mask, realq);
            // the stage is free again: refill it RUNS_STAGES tiles ahead
            __syncwarp();
            const int tn = tq.next(lane);
            --pending;
            if (tn < T) {
                if (lane == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    runs_issue<REAL>(a, tn, stage0 + s * SS, bar0 + 8 * s, pol);
                }
                ++pending;
            }
        }
        ph ^= 1u;
    }
}

// ---- the same run-encoded stream through per-thread loads: the coefficients
// and the tile record (3 coalesced words per lane: row/run words + rank prefixes,
// biases 0-31, biases 32-63) are loaded one tile ahead into registers and the
// biases are looked up with shuffles, so the whole L1 stays a cache for the q
// gathers (the bulk-copy kernel above gives most of it to its stage buffers).
template <bool REAL>
struct RlTile {
    double cr[8], ci[8];
    unsigned w0, b0, b1;
};

template <bool REAL>
__device__ __forceinline__ void rl_load(const EvalArgs& a, int t, int lane, RlTile<REAL>& d) {
    const int64_t T0 = (int64_t)t * CORR_TILE;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (REAL) {
            d.cr[k] = __ldcs(a.coef_r + T0 + 32 * k + lane);
            d.ci[k] = 0.0;
        } else {
            const double2 c = __ldcs(reinterpret_cast<const double2*>(a.coef) + T0 + 32 * k + lane);
            d.cr[k] = c.x;
            d.ci[k] = c.y;
        }
    }
    const unsigned* rec = a.run_rec + (int64_t)t * RUNS_REC_WORDS;
    d.w0 = __ldcs(rec + lane);
    d.b0 = __ldcs(rec + 32 + lane);
    d.b1 = __ldcs(rec + 64 + lane);
}

template <bool REAL>
__global__ void __launch_bounds__(32 * CORR_WARPS, CORR_MINB) k_corr_rl(EvalArgs a) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = (int)((a.n_pairs + CORR_TILE - 1) / CORR_TILE);
    TileQueue tq;
    tq.init(a, T, warp, CORR_WARPS, lane);
    const bool realq = REAL && a.q_re && *(volatile const int*)a.q_flag == 0;
    const unsigned le_mask = 0xffffffffu >> (31 - lane);
    RlTile<REAL> cur, nxt;
    int t = tq.next(lane);
    if (t >= T) return;
    rl_load<REAL>(a, t, lane, cur);
    for (;;) {
        const int tn = tq.next(lane);
        if (tn < T) rl_load<REAL>(a, tn, lane, nxt);
        const unsigned w0 = cur.w0;
        const int64_t sbase = meta_i64(w0, 16);
        const int nruns = (int)__shfl_sync(0xffffffffu, w0, 20);
        const unsigned pk0 = __shfl_sync(0xffffffffu, w0, 21), pk1 = __shfl_sync(0xffffffffu, w0, 22);
        int src[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const unsigned rw = __shfl_sync(0xffffffffu, w0, 8 + k);
            const unsigned pk = k < 4 ? pk0 : pk1;
            src[k] = (int)((pk >> (8 * (k & 3))) & 0xffu) + __popc(rw & le_mask) - 1;   // rank
        }
        if (nruns <= 32) {
#pragma unroll
            for (int k = 0; k < 8; ++k) src[k] = (int)__shfl_sync(0xffffffffu, cur.b0, src[k]) + (32 * k + lane);
        } else {
            const int64_t ob = meta_i64(w0, 18);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int r = src[k];
                const int v0 = (int)__shfl_sync(0xffffffffu, cur.b0, r & 31);
                const int v1 = (int)__shfl_sync(0xffffffffu, cur.b1, r & 31);
                int b = r < 32 ? v0 : v1;
                if (r >= RUNS_BIAS_CAP) b = __ldg(a.run_bias + ob + (r - RUNS_BIAS_CAP));
                src[k] = b + (32 * k + lane);
            }
        }
        double qr[8], qi[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (realq) {
                qr[k] = a.q_re[src[k]];
                qi[k] = 0.0;
            } else {
                const cplx qv = a.q_sorted[src[k]];
                qr[k] = qv.re;
                qi[k] = qv.im;
            }
        }
        corr_reduce_tile(a, lane, cur.cr, cur.ci, qr, qi, w0, sbase);
        if (tn >= T) break;
        cur = nxt;
    }
}

// ---- 16-bit source offsets on whole (zero-padded) tiles: the k_corr_tiles
// pipeline with a 2-byte offset per pair instead of the 4-byte index, no tail
// predicates, the 8 group bases of a tile riding in lanes 8-15 of the row-start
// word register, and the (rare) wide groups re-read as int32 after the stream
// loads, so the load phase has no branches.
template <bool REAL>
struct O16Tile {
    int off[8];
    double cr[8], ci[8];
    unsigned word;   // lanes 0-7: row-start words, lanes 8-15: group bases
    int64_t sbase;
};

template <bool REAL>
__device__ __forceinline__ void o16_load(const EvalArgs& a, int t, int lane, O16Tile<REAL>& d) {
    const int64_t T0 = (int64_t)t * CORR_TILE;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        d.off[k] = (int)__ldcs(a.pair_off16 + T0 + 32 * k + lane);
        if (REAL) {
            d.cr[k] = __ldcs(a.coef_r + T0 + 32 * k + lane);
            d.ci[k] = 0.0;
        } else {
            const double2 c = __ldcs(reinterpret_cast<const double2*>(a.coef) + T0 + 32 * k + lane);
            d.cr[k] = c.x;
            d.ci[k] = c.y;
        }
    }
    const int64_t g0 = (int64_t)t * (CORR_TILE / 32);
    d.word = lane < 8 ? a.head_bits[g0 + lane] : (lane < 16 ? (unsigned)__ldcs(a.grp_base + g0 + lane - 8) : 0u);
    d.sbase = a.seg_base[t];
}

template <bool REAL>
__global__ void __launch_bounds__(32 * CORR_WARPS, CORR_MINB) k_corr_o16(EvalArgs a) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int T = (int)((a.n_pairs + CORR_TILE - 1) / CORR_TILE);
    TileQueue tq;
    tq.init(a, T, warp, CORR_WARPS, lane);
    const bool realq = REAL && a.q_re && *(volatile const int*)a.q_flag == 0;
    O16Tile<REAL> cur, nxt;
    int t = tq.next(lane);
    if (t >= T) return;
    o16_load<REAL>(a, t, lane, cur);
    for (;;) {
        const int tn = tq.next(lane);
        if (tn < T) o16_load<REAL>(a, tn, lane, nxt);
        int src[8];
        bool wide = false;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int gb = (int)__shfl_sync(0xffffffffu, cur.word, 8 + k);
            src[k] = gb + cur.off[k];
            wide |= gb < 0;
        }
        if (wide) {   // uniform: some group of this tile keeps int32 indices
            const int64_t T0 = (int64_t)t * CORR_TILE;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int gb = (int)__shfl_sync(0xffffffffu, cur.word, 8 + k);
                if (gb < 0) src[k] = T0 + 32 * k + lane < a.n_pairs ? a.pair_src[T0 + 32 * k + lane] : 0;
            }
        }
        double qr[8], qi[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (realq) {
                qr[k] = a.q_re[src[k]];
                qi[k] = 0.0;
            } else {
                const cplx qv = a.q_sorted[src[k]];
                qr[k] = qv.re;
                qi[k] = qv.im;
            }
        }
        corr_reduce_tile(a, lane, cur.cr, cur.ci, qr, qi, cur.word, cur.sbase);
        if (tn >= T) break;
        cur = nxt;
        t = tn;
    }
}

size_t corr_runs_smem(bool real, int warps) {
    return (size_t)warps * RUNS_STAGES * (real ? RunsStage<true>::bytes : RunsStage<false>::bytes) +
           (size_t)warps * RUNS_STAGES * 8;
}

// ---- plan build of the run records
// run-start bits over the pair positions padded to whole tiles: tile starts, row
// starts, breaks in the source sequence, and the first padding position
__global__ void k_run_words(const int* __restrict__ src, const unsigned* __restrict__ head, int64_t P, int64_t Ppad,
                            unsigned* runw) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool f = false;
    if (p < P) f = (p % CORR_TILE) == 0 || ((head[p >> 5] >> (p & 31)) & 1u) || src[p] != src[p - 1] + 1;
    else if (p == P && p < Ppad) f = true;
    const unsigned w = __ballot_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && p < Ppad) runw[p >> 5] = w;
}
// runs past the record's RUNS_BIAS_CAP per tile
__global__ void k_tile_overflow(const unsigned* __restrict__ runw, int64_t T, int64_t* ovf) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t > T) return;
    int n = 0;
    if (t < T)
        for (int k = 0; k < 8; ++k) n += __popc(runw[t * 8 + k]);
    ovf[t] = max(0, n - RUNS_BIAS_CAP);
}
// one warp per tile: the record and the overflow biases.  Padding pairs (zero
// coefficients) read the zero charges q_sorted[N ..).
__global__ void k_run_fill(const int* __restrict__ src, const unsigned* __restrict__ head,
                           const unsigned* __restrict__ runw, const int64_t* __restrict__ seg_base,
                           const int64_t* __restrict__ ovf_base, int64_t P, int64_t T, int64_t N, unsigned* recs,
                           int* ovf, unsigned long long* total) {
    const int lane = threadIdx.x & 31;
    const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (t >= T) return;
    const int64_t T0 = t * CORR_TILE;
    const unsigned hw = lane < 8 ? head[(T0 >> 5) + lane] : 0u;
    const unsigned rw = lane < 8 ? runw[(T0 >> 5) + lane] : 0u;
    const unsigned long long ob = (unsigned long long)ovf_base[t], sb = (unsigned long long)seg_base[t];
    const int c = __popc(rw);
    int inc = c;   // inclusive prefix over lanes 0-7
    for (int d = 1; d < 8; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += v;
    }
    const int n = __shfl_sync(0xffffffffu, inc, 7);
    const unsigned ex = (unsigned)(inc - c);   // runs before group `lane`
    unsigned pk0 = 0u, pk1 = 0u;
    for (int k = 0; k < 4; ++k) {
        pk0 |= (__shfl_sync(0xffffffffu, ex, k) & 0xffu) << (8 * k);
        pk1 |= (__shfl_sync(0xffffffffu, ex, 4 + k) & 0xffu) << (8 * k);
    }
    const unsigned rws = __shfl_sync(0xffffffffu, rw, lane & 7);
    unsigned* rec = recs + t * RUNS_REC_WORDS;
    unsigned v = 0u;   // words 0-31: one per lane
    if (lane < 8) v = hw;
    else if (lane < 16) v = rws;
    else if (lane == 16) v = (unsigned)(sb & 0xffffffffull);
    else if (lane == 17) v = (unsigned)(sb >> 32);
    else if (lane == 18) v = (unsigned)(ob & 0xffffffffull);
    else if (lane == 19) v = (unsigned)(ob >> 32);
    else if (lane == 20) v = (unsigned)n;
    else if (lane == 21) v = pk0;
    else if (lane == 22) v = pk1;
    rec[lane] = v;
    rec[32 + lane] = 0u;
    rec[64 + lane] = 0u;
    __syncwarp();
    int pre = 0;
    for (int k = 0; k < 8; ++k) {
        const unsigned w = __shfl_sync(0xffffffffu, rw, k);
        const int e = 32 * k + lane;
        if ((w >> lane) & 1u) {
            const int r = pre + __popc(w & ((1u << lane) - 1u));
            const int b = (T0 + e < P ? src[T0 + e] : (int)N) - e;
            if (r < RUNS_BIAS_CAP) rec[32 + r] = (unsigned)b;
            else ovf[ob + (r - RUNS_BIAS_CAP)] = b;
        }
        pre += __popc(w);
    }
    if (lane == 0) atomicAdd(total, (unsigned long long)n);
}

// src <- bias[rank] + e (exports of plans that dropped their index array)
__global__ void k_run_decode(const unsigned* __restrict__ recs, const int* __restrict__ ovf, int64_t P, int* src) {
    const int lane = threadIdx.x & 31;
    const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t T = (P + CORR_TILE - 1) / CORR_TILE;
    if (t >= T) return;
    const unsigned* rec = recs + t * RUNS_REC_WORDS;
    const unsigned mw = rec[lane];
    const int64_t ob = meta_i64(mw, 18);
    const unsigned le_mask = 0xffffffffu >> (31 - lane);
    int pre = -1;
    for (int k = 0; k < 8; ++k) {
        const unsigned rw = __shfl_sync(0xffffffffu, mw, 8 + k);
        const int rank = pre + __popc(rw & le_mask);
        pre += __popc(rw);
        const int64_t p = t * CORR_TILE + 32 * k + lane;
        if (p < P)
            src[p] = (rank < RUNS_BIAS_CAP ? (int)rec[32 + rank] : ovf[ob + (rank - RUNS_BIAS_CAP)]) + 32 * k + lane;
    }
}

// Builds the run records of a pair list whose metadata (head bits, tile segment
// bases) exists.  *rec_out: (T, 96) words, *ovf_out: the overflow biases;
// returns the number of runs, or -1 when the arrays do not fit.
int64_t build_run_records(const int* src, const unsigned* head, const int64_t* seg_base, int64_t P, int64_t T,
                          int64_t N, unsigned** rec_out, int** ovf_out, int64_t* bytes_out, cudaStream_t s) {
    unsigned* runw = nullptr;
    int64_t* cnt = nullptr;
    int64_t* obase = nullptr;
    unsigned long long* dtot = nullptr;
    void* tmp = nullptr;
    *rec_out = nullptr;
    *ovf_out = nullptr;
    const int64_t Ppad = T * CORR_TILE;
    const int64_t W = Ppad / 32 + 8;
    int64_t total = -1;
    do {
        if (cudaMalloc(&runw, sizeof(unsigned) * W) || cudaMalloc(&cnt, sizeof(int64_t) * (T + 1)) ||
            cudaMalloc(&obase, sizeof(int64_t) * (T + 1)) || cudaMalloc(&dtot, sizeof(unsigned long long)))
            break;
        cudaMemsetAsync(runw, 0, sizeof(unsigned) * W, s);
        cudaMemsetAsync(dtot, 0, sizeof(unsigned long long), s);
        k_run_words<<<nblk64(Ppad, 256), 256, 0, s>>>(src, head, P, Ppad, runw);
        k_tile_overflow<<<nblk64(T + 1, 256), 256, 0, s>>>(runw, T, cnt);
        size_t bytes = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, obase, (int)(T + 1), s);
        if (cudaMalloc(&tmp, bytes + 16)) break;
        cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, obase, (int)(T + 1), s);
        int64_t h = 0;
        cudaMemcpyAsync(&h, obase + T, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) break;
        cudaFree(cnt);
        cnt = nullptr;
        cudaFree(tmp);
        tmp = nullptr;
        const size_t rec_bytes = sizeof(unsigned) * RUNS_REC_WORDS * (size_t)std::max<int64_t>(T, 1);
        const size_t ovf_bytes = sizeof(int) * (size_t)(h + 4);
        if (cudaMalloc(rec_out, rec_bytes) || cudaMalloc(ovf_out, ovf_bytes)) break;
        k_run_fill<<<nblk64(T * 32, 256), 256, 0, s>>>(src, head, runw, seg_base, obase, P, T, N, *rec_out,
                                                        *ovf_out, dtot);
        unsigned long long ht = 0;
        cudaMemcpyAsync(&ht, dtot, sizeof(ht), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) break;
        fftpim_count_launch(4);
        total = (int64_t)ht;
        *bytes_out = (int64_t)(rec_bytes + ovf_bytes);
    } while (0);
    if (runw) cudaFree(runw);
    if (cnt) cudaFree(cnt);
    if (obase) cudaFree(obase);
    if (dtot) cudaFree(dtot);
    if (tmp) cudaFree(tmp);
    if (total < 0) {
        cudaGetLastError();
        if (*rec_out) cudaFree(*rec_out);
        if (*ovf_out) cudaFree(*ovf_out);
        *rec_out = nullptr;
        *ovf_out = nullptr;
    }
    return total;
}

void launch_run_decode(const unsigned* recs, const int* ovf, int64_t P, int* src, cudaStream_t s) {
    const int64_t T = (P + CORR_TILE - 1) / CORR_TILE;
    if (T > 0) k_run_decode<<<nblk64(T * 32, 256), 256, 0, s>>>(recs, ovf, P, src);
    fftpim_count_launch();
}

void launch_corr_tiles(const EvalArgs& a, cudaStream_t s) {
    if (a.n_pairs == 0) return;
    const int64_t T = (a.n_pairs + CORR_TILE - 1) / CORR_TILE;
    // FFTPIM_K4_RUNS_KERNEL=bulk|ldg (read per launch: launches are captured into graphs)
    const char* erk = getenv("FFTPIM_K4_RUNS_KERNEL");
    const int rl_kind = erk && erk[0] == 'l' ? 1 : 0;
    if (a.run_rec && rl_kind == 1) {
        int64_t cap = 148 * CORR_MINB;
        if (a.corr_blocks > 0) cap = a.corr_blocks;
        if (a.corr_blocks < 0) cap = INT32_MAX;
        const int blocks = (int)std::min<int64_t>((T + CORR_WARPS - 1) / CORR_WARPS, cap);
        if (a.coef_r)
            k_corr_rl<true><<<blocks, 32 * CORR_WARPS, 0, s>>>(a);
        else
            k_corr_rl<false><<<blocks, 32 * CORR_WARPS, 0, s>>>(a);
        fftpim_count_launch();
        return;
    }
    if (a.run_rec) {
        // whole chip: one 16-warp block per SM.  Capped (a.corr_blocks counts 8-warp
        // blocks, the concurrent schedules): 8-warp blocks, so that other kernels
        // fit beside a resident block.  a.k4_counter selects the shared tile queue.
        const int warps = a.corr_blocks > 0 ? 8 : RUNS_WARPS;
        int64_t cap = 148;
        if (a.corr_blocks > 0) cap = a.corr_blocks;
        if (a.corr_blocks < 0) cap = INT32_MAX;
        const int blocks = (int)std::min<int64_t>((T + warps - 1) / warps, cap);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_corr_runs<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)corr_runs_smem(true, RUNS_WARPS));
            cudaFuncSetAttribute(k_corr_runs<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)corr_runs_smem(false, RUNS_WARPS));
            attr = true;
        }
        if (a.coef_r)
            k_corr_runs<true><<<blocks, 32 * warps, corr_runs_smem(true, warps), s>>>(a);
        else
            k_corr_runs<false><<<blocks, 32 * warps, corr_runs_smem(false, warps), s>>>(a);
        fftpim_count_launch();
        return;
    }
    // a.corr_blocks caps the grid (the concurrent schedule leaves SMs to the near chain)
    int64_t cap = 148 * CORR_MINB;
    if (a.corr_blocks > 0) cap = std::min<int64_t>(cap, a.corr_blocks);
    if (a.corr_blocks < 0) cap = INT32_MAX;   // one block per CORR_WARPS tiles (no grid-stride loop)
    const int blocks = (int)std::min<int64_t>((T + CORR_WARPS - 1) / CORR_WARPS, cap);
    if (a.pair_off16) {
        static const int o16_kind = [] {   // FFTPIM_K4_C16_KERNEL=old: the three-stage k_corr_tiles_c16
            const char* e = getenv("FFTPIM_K4_C16_KERNEL");
            return e && e[0] == 'o' ? 0 : 1;
        }();
        if (o16_kind == 1) {
            if (a.coef_r)
                k_corr_o16<true><<<blocks, 32 * CORR_WARPS, 0, s>>>(a);
            else
                k_corr_o16<false><<<blocks, 32 * CORR_WARPS, 0, s>>>(a);
        } else if (a.coef_r)
            k_corr_tiles_c16<true><<<blocks, 32 * CORR_WARPS, 0, s>>>(a);
        else
            k_corr_tiles_c16<false><<<blocks, 32 * CORR_WARPS, 0, s>>>(a);
        fftpim_count_launch();
        return;
    }
    // one tile in flight beyond the one being reduced (measured: deeper is not faster)
    if (a.coef_r)
        k_corr_tiles<true, CORR_PF_REAL><<<blocks, 32 * CORR_WARPS, 0, s>>>(a);
    else
        k_corr_tiles<false, CORR_PF><<<blocks, 32 * CORR_WARPS, 0, s>>>(a);
    fftpim_count_launch();
}

// ------------------------------------------------------------- K3 + K5c + fix-up
// LPO lanes per observer; lane sub takes the entries sub, sub + LPO, ...
// of the flattened (y, z) stencil plane for every x row, so a warp load reads
// each observer's consecutive z taps.  The far observer grid (<= 48 KB) is staged in
// shared memory.  The last lane fetches the observer's K4 segments, the lanes
// are reduced with a fixed xor tree and lane 0 stores.  Single-plane axes:
// weights past the first tap are zero and the indices are clamped, so those
// taps add exactly 0.
#ifndef OBS_SMALL_M
#define OBS_SMALL_M 16384
#endif
#ifndef OBS_MINB   // 4 resident blocks: measured faster than 1 (all gathers hoisted, 104 regs)
#define OBS_MINB 4
#endif
__device__ __forceinline__ cplx corr_of_row(const EvalArgs& a, int64_t i) {
    const int64_t p0 = a.pair_ptr[i], p1 = a.pair_ptr[i + 1];
    if (p0 == p1) return mk(0.0);
    const int64_t span = (p1 - 1) / CORR_TILE - p0 / CORR_TILE + 1;
    const cplx* sv = a.seg_val + a.seg_first[i];
    cplx s = sv[0];
    for (int64_t j = 1; j < span; ++j) s = s + sv[j];
    return s;
}

// MODE 0: near + far + K4 fix-up -> u.  MODE 1 (off the near chain, once the
// far chain and K4 are done): far + fix-up -> obs_pre.  MODE 2 (after the
// inverse FFT): near + obs_pre -> u.
template <int W, int WF, int MODE, int LPO>
__global__ void __launch_bounds__(256, OBS_MINB) k_observers(EvalArgs a) {
    extern __shared__ cplx sfar[];
    const int nfx = a.fo.n[0], nfy = a.fo.n[1], nfz = a.fo.n[2];
    if ((a.parts & FFTPIM_FAR) && MODE != 2) {
        for (int t = threadIdx.x; t < nfx * nfy * nfz; t += blockDim.x) sfar[t] = a.far_ug[t];
        __syncthreads();
    }
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t i = gt / LPO;
    const int sub = (int)(gt % LPO);
    const bool active = i < a.M;
    const int64_t ii = active ? i : a.M - 1;
    double ar = 0.0, ai = 0.0;
    if ((a.parts & FFTPIM_NEAR) && MODE != 2 && active && sub == LPO - 1 && a.sw_e >= 0) {
        // the observer's K4 segments, fetched by the last lane up front so the
        // dependent pointer chain overlaps the interpolation gathers
        const cplx c = a.sw_corr ? a.sw_corr[i * a.sw_E + a.sw_e] : corr_of_row(a, i);
        ar = c.re;
        ai = c.im;
    }
    if (MODE == 2 && active && sub == LPO - 1) {
        const cplx c = a.obs_pre[i];
        ar = c.re;
        ai = c.im;
    }
    if ((a.parts & FFTPIM_NEAR) && MODE != 1) {
        // lane sub takes the entries e = sub, sub + LPO, ... of the W x W
        // (y, z) stencil plane, for every x row, so one warp load reads each
        // observer's consecutive z taps and no lane idles on a partial row
        const double* w = a.obs_w + ii * 3 * W;
        const int* st = a.obs_start + 3 * ii;
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
    if ((a.parts & FFTPIM_FAR) && MODE != 2) {
        const double* w = a.obs_fw + ii * 3 * WF;
        const int* st = a.obs_fstart + 3 * ii;
        const int s0 = st[0], s1 = st[1], s2 = st[2];
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
    for (int o = 1; o < LPO; o <<= 1) {   // fixed xor tree over the observer's lanes
        ar += __shfl_xor_sync(0xffffffffu, ar, o);
        ai += __shfl_xor_sync(0xffffffffu, ai, o);
    }
    if (active && sub == 0) {
        if (MODE == 1)
            a.obs_pre[i] = cplx{ar, ai};
        else
            a.u[a.obs_perm[i]] = cplx{ar, ai};
    }
}

template <int W, int MODE, int LPO>
static void obs_dispatch_far(const EvalArgs& a, int blocks, size_t smem, cudaStream_t s) {
    switch (a.fo.order + 1) {
        case 2: k_observers<W, 2, MODE, LPO><<<blocks, 256, smem, s>>>(a); break;
        case 3: k_observers<W, 3, MODE, LPO><<<blocks, 256, smem, s>>>(a); break;
        case 4: k_observers<W, 4, MODE, LPO><<<blocks, 256, smem, s>>>(a); break;
        case 5: k_observers<W, 5, MODE, LPO><<<blocks, 256, smem, s>>>(a); break;
        case 6: k_observers<W, 6, MODE, LPO><<<blocks, 256, smem, s>>>(a); break;
        default: k_observers<W, 7, MODE, LPO><<<blocks, 256, smem, s>>>(a); break;
    }
}

// mode 0: the fused pass; 1: far + fix-up into obs_pre; 2: near + obs_pre
template <int LPO>
static void launch_observers_lpo(const EvalArgs& a, cudaStream_t s, int mode) {
    const int blocks = nblk64(a.M * LPO, 256);
    const size_t smem =
        ((a.parts & FFTPIM_FAR) && mode != 2) ? (size_t)a.fo.n[0] * a.fo.n[1] * a.fo.n[2] * sizeof(cplx) : 0;
    if (mode == 1) {
        obs_dispatch_far<2, 1, LPO>(a, blocks, smem, s);
    } else if (mode == 2) {
        switch (a.g.order + 1) {
            case 2: k_observers<2, 2, 2, LPO><<<blocks, 256, 0, s>>>(a); break;
            case 3: k_observers<3, 2, 2, LPO><<<blocks, 256, 0, s>>>(a); break;
            case 4: k_observers<4, 2, 2, LPO><<<blocks, 256, 0, s>>>(a); break;
            case 5: k_observers<5, 2, 2, LPO><<<blocks, 256, 0, s>>>(a); break;
            case 6: k_observers<6, 2, 2, LPO><<<blocks, 256, 0, s>>>(a); break;
            default: k_observers<7, 2, 2, LPO><<<blocks, 256, 0, s>>>(a); break;
        }
    } else {
        switch (a.g.order + 1) {
            case 2: obs_dispatch_far<2, 0, LPO>(a, blocks, smem, s); break;
            case 3: obs_dispatch_far<3, 0, LPO>(a, blocks, smem, s); break;
            case 4: obs_dispatch_far<4, 0, LPO>(a, blocks, smem, s); break;
            case 5: obs_dispatch_far<5, 0, LPO>(a, blocks, smem, s); break;
            case 6: obs_dispatch_far<6, 0, LPO>(a, blocks, smem, s); break;
            default: obs_dispatch_far<7, 0, LPO>(a, blocks, smem, s); break;
        }
    }
}

// lanes per observer: 4 for small observer sets (more threads in flight) and
// order >= 4, 2 otherwise (measured: C2 / C5 observer pass 10-30 % faster)
void launch_observers(const EvalArgs& a, cudaStream_t s, int mode) {
    if (a.M == 0) return;
    if (a.obs_pos && a.obs_cell_start && launch_observers_tile(a, a.obs_pos, a.obs_cell_start, a.obs_i0, s, mode))
        return;
    if (a.obs_pos && launch_observers_pos(a, a.obs_pos, s, mode)) return;
    // 5-tap (order 4) stencils: 13 entries per lane at 2 lanes spill under the
    // 64-register budget, so those keep 4 lanes
    if (a.M <= OBS_SMALL_M || a.g.order >= 4)
        launch_observers_lpo<4>(a, s, mode);
    else
        launch_observers_lpo<2>(a, s, mode);
    fftpim_count_launch();
}
