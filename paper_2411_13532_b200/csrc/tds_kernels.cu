// sm_100a kernels for the DistD2 batched tridiagonal solve.
//
// FAST PATH (k_fast): one CTA owns TL=16 lines (128-byte rows of the
// SZ-blocked layout) over the whole block of rows. The block is cut into C
// chunks of M rows; thread (chunk, lane) keeps its chunk of one line in
// registers for the whole solve:
//   1. load M+4 rows (2-row halos from the neighbour chunks / wrap / halo
//      buffers) -- all loads in flight before any use;
//   2. width-5 stencil fused with the Alg. 6 forward sweep, backward sweep
//      and closure (reference distributed.py:257-276) using the chunk's own
//      Alg. 5 tables -> decoupled rows d and the chunk's reduced rhs
//      (d[0], d[M-1]);
//   3. reduced system of all chunk boundary values: a precomputed dense map H
//      (host, plan.cpp) applied to the reduced rhs from shared memory -- exact
//      solve of the line (P=1) or the reference's rank-truncated DistD2
//      (emulated P>1 / per-rank pass B);
//   4. substitution (Alg. 7 at chunk level) in registers and one store.
// HBM traffic is the compulsory 8 B read + 8 B write per point.
//
// STAGED PATH: one thread per (line, rank block), the reference's own
// operation order with no FMA contraction (__dmul_rn/__dadd_rn), so results
// are bit-identical to the reference's NumPy code.
#include <cuda_runtime.h>

#include <cstdint>

#include "tds_device.cuh"
#include "tds_internal.h"

namespace tds {

__device__ __forceinline__ long long line_base(long long line, int rows, int sz) {
    return (line / sz) * (long long)rows * sz + (line % sz);
}
__device__ __forceinline__ long long halo_base(long long line, int sz) {
    return (line / sz) * 2LL * sz + (line % sz);
}

// ------------------------------------------------------------------ fast path

template <int M, int MODE, bool UNIFORM>
__global__ void __launch_bounds__(512) k_fast(const __grid_constant__ FastArgs p) {
    extern __shared__ double sY[];
    const int C = p.chunks;
    const int K = 2 * C;
    const int t = threadIdx.x;
    const int lane = t % TL;
    const int chunk = (t / TL) % C;
    const int tl = t / (TL * C);
    const long long line = ((long long)blockIdx.x * p.tiles_per_cta + tl) * TL + lane;
    const bool valid = line < p.lines;
    const long long lb = valid ? line_base(line, p.rows, p.sz) : 0;
    const long long hb = valid ? halo_base(line, p.sz) : 0;
    const double* __restrict__ ub = p.u + lb;
    const long long sz = p.sz;
    const int r0 = chunk * M;

    double v[M + 4];
#pragma unroll
    for (int i = 0; i < M + 4; ++i) {
        const int row = r0 - 2 + i;
        double x = 0.0;
        if (i < 2 || i >= M + 2) {
            if (row < 0) {
                if (p.edge_mode == EDGE_WRAP) {
                    if (valid) x = __ldg(ub + (row + p.rows) * sz);
                } else if (p.edge_mode == EDGE_HALO && p.halo_lo) {
                    if (valid) x = __ldg(p.halo_lo + hb + (row + 2) * sz);
                }
            } else if (row >= p.rows) {
                if (p.edge_mode == EDGE_WRAP) {
                    if (valid) x = __ldg(ub + (row - p.rows) * sz);
                } else if (p.edge_mode == EDGE_HALO && p.halo_hi) {
                    if (valid) x = __ldg(p.halo_hi + hb + (row - p.rows) * sz);
                }
            } else if (valid) {
                x = __ldg(ub + row * sz);
            }
        } else if (valid) {
            x = __ldg(ub + row * sz);
        }
        v[i] = x;
    }

    // table accessors
    const double* __restrict__ tb = p.tab + (size_t)r0 * NCOEF;
#define TAB(i, k) (UNIFORM ? 0.0 : __ldg(tb + (i) * NCOEF + (k)))

    // fused stencil + Alg. 6 sweeps (tds_device.cuh; shifted one-sided rows
    // of the first / last chunk included)
    double d[M];
    dev::chunk_sweeps_any<M, UNIFORM ? TAB_UNIFORM : TAB_GLOBAL>(p, tb, v, d, chunk);

    // reduced rhs of this chunk -> shared memory
    double* Y = sY + (size_t)tl * K * TL;
    double y0 = d[0], yL = d[M - 1];
    if (MODE == MODE_PASS_B) {
        if (chunk == 0 && valid) {
            const double d0 = p.d_first_in[line];
            y0 = p.has_prev ? (d0 - p.sa_first * p.prev_last[line]) / p.det_prev : d0;
        }
        if (chunk == C - 1 && valid) {
            const double dl = p.d_last_in[line];
            yL = p.has_next ? (dl - p.sc_last * p.next_first[line]) / p.det_next : dl;
        }
    }
    Y[(2 * chunk) * TL + lane] = y0;
    Y[(2 * chunk + 1) * TL + lane] = yL;
    __syncthreads();

    if (MODE == MODE_PASS_A) {
        if (!valid) return;
        if (chunk == 0) {
            double s = 0.0;
            for (int q = 0; q < K; ++q) s = fma(__ldg(p.g + q), Y[q * TL + lane], s);
            p.d_first_out[line] = s;
        }
        if (chunk == C - 1) {
            double s = 0.0;
            for (int q = 0; q < K; ++q) s = fma(__ldg(p.g + K + q), Y[q * TL + lane], s);
            p.d_last_out[line] = s;
        }
        return;
    }

    // chunk boundary values F (first row) and L (last row) of this chunk
    double F0 = 0.0, F1 = 0.0, L0 = 0.0, L1 = 0.0;
    const double2* __restrict__ hr = p.Hp + (size_t)chunk * K;
    int q = 0;
    for (; q + 1 < K; q += 2) {
        const double2 h0 = __ldg(hr + q);
        const double2 h1 = __ldg(hr + q + 1);
        const double ya = Y[q * TL + lane];
        const double yb = Y[(q + 1) * TL + lane];
        F0 = fma(h0.x, ya, F0);
        L0 = fma(h0.y, ya, L0);
        F1 = fma(h1.x, yb, F1);
        L1 = fma(h1.y, yb, L1);
    }
    const double F = F0 + F1, L = L0 + L1;

    if (!valid) return;
    double* __restrict__ ob = p.out + lb;
    __stcs(ob + (long long)r0 * sz, F);
#pragma unroll
    for (int i = 1; i < M - 1; ++i) {
        const double sa = UNIFORM ? p.ut.sa[i] : TAB(i, 8);
        const double sc = UNIFORM ? p.ut.sc[i] : TAB(i, 9);
        __stcs(ob + (long long)(r0 + i) * sz, fma(-sc, L, fma(-sa, F, d[i])));
    }
    __stcs(ob + (long long)(r0 + M - 1) * sz, L);
#undef TAB
}

template <int M, int MODE, bool UNI>
static int launch_fast_t(const FastArgs& a, long long tiles, cudaStream_t s) {
    const int threads = a.tiles_per_cta * a.chunks * TL;
    if (threads > 512)
        return set_err(TDS_ERR_UNSUPPORTED, "plans with more than 32 chunks need 8-line TMA tiles");
    const long long grid = (tiles + a.tiles_per_cta - 1) / a.tiles_per_cta;
    const size_t smem = (size_t)a.tiles_per_cta * 2 * a.chunks * TL * sizeof(double);
    if (grid <= 0) return TDS_OK;
    if (grid > 0x7fffffffLL) return set_err(TDS_ERR_INVALID, "too many lines for one launch");
    k_fast<M, MODE, UNI><<<(unsigned)grid, threads, smem, s>>>(a);
    return cuda_check(cudaGetLastError(), "k_fast launch");
}

int launch_fast(int M, int mode, bool uniform, const FastArgs& a, long long tiles,
                cudaStream_t s) {
    if (tma_eligible(M, a)) return launch_tma(M, mode, uniform, a, tiles, s);
    // k_fast has no per-chunk table switch: edge-special plans use the table path
    if (a.special_first || a.special_last) uniform = false;
#define DISPATCH_MODE(MM)                                                             \
    switch (mode) {                                                                   \
        case MODE_SOLVE:                                                              \
            return uniform ? launch_fast_t<MM, MODE_SOLVE, true>(a, tiles, s)         \
                           : launch_fast_t<MM, MODE_SOLVE, false>(a, tiles, s);       \
        case MODE_PASS_A:                                                             \
            return uniform ? launch_fast_t<MM, MODE_PASS_A, true>(a, tiles, s)        \
                           : launch_fast_t<MM, MODE_PASS_A, false>(a, tiles, s);      \
        default:                                                                      \
            return uniform ? launch_fast_t<MM, MODE_PASS_B, true>(a, tiles, s)        \
                           : launch_fast_t<MM, MODE_PASS_B, false>(a, tiles, s);      \
    }
    if (M == 32) { DISPATCH_MODE(32) }
    if (M == 16) { DISPATCH_MODE(16) }
#undef DISPATCH_MODE
    return set_err(TDS_ERR_UNSUPPORTED, "unsupported chunk size");
}

// ---------------------------------------------------------------- staged path
// Reference arithmetic: every product and sum rounded separately.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// distributed.py:205-208
__device__ __forceinline__ double stencil5(const double* c, double u0, double u1, double u2,
                                           double u3, double u4) {
    return add(add(add(add(mul(c[0], u0), mul(c[1], u1)), mul(c[2], u2)), mul(c[3], u3)),
               mul(c[4], u4));
}

// value of row `row` (relative to the array) of a line, with the edge rule
__device__ __forceinline__ double fetch(const StagedArgs& p, const double* __restrict__ ub, long long hb,
                                        int row) {
    const long long sz = p.sz;
    if (row >= 0 && row < p.rows) return ub[row * sz];
    if (p.edge_mode == EDGE_WRAP) return ub[(row < 0 ? row + p.rows : row - p.rows) * sz];
    if (p.edge_mode == EDGE_HALO) {
        if (row < 0) return p.halo_lo ? p.halo_lo[hb + (row + 2) * sz] : 0.0;
        return p.halo_hi ? p.halo_hi[hb + (row - p.rows) * sz] : 0.0;
    }
    return 0.0;
}

// window shift of block row `row` (one-sided closures, plan.cpp check_shift)
__device__ __forceinline__ int row_shift(const StagedArgs& p, int row) {
    if (!p.has_shift) return 0;
    if (row < 2) return p.sh[row];
    if (row >= p.rows - 2) return p.sh[4 - (p.rows - row)];
    return 0;
}

// stencil row with a shifted window: sum over u[row + o + s], o = -2..2, in
// the reference's left-to-right order (distributed.py:205-208)
__device__ __forceinline__ double stencil_shifted(const StagedArgs& p, const double* c,
                                                  const double* __restrict__ ub, long long hb, int row,
                                                  int s) {
    return stencil5(c, fetch(p, ub, hb, row - 2 + s), fetch(p, ub, hb, row - 1 + s),
                    fetch(p, ub, hb, row + s), fetch(p, ub, hb, row + 1 + s),
                    fetch(p, ub, hb, row + 2 + s));
}

// Alg. 6 decouple_fused per (line, block): distributed.py:257-276.
__global__ void k_staged_decouple(const StagedArgs p) {
    const long long line = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (line >= p.lines) return;
    const int off = p.boff[b], m = p.bsize[b];
    const long long sz = p.sz;
    const double* __restrict__ ub = p.u + line_base(line, p.rows, p.sz);
    double* __restrict__ ob = p.out + line_base(line, p.rows, p.sz);
    const long long hb = halo_base(line, p.sz);
    double u0 = fetch(p, ub, hb, off - 2), u1 = fetch(p, ub, hb, off - 1);
    double u2 = fetch(p, ub, hb, off), u3 = fetch(p, ub, hb, off + 1);
    double dprev = 0.0;
    #pragma unroll 8
    for (int j = 0; j < m; ++j) {
        const double u4 = fetch(p, ub, hb, off + j + 2);
        const int row = off + j;
        const int sh = row_shift(p, row);
        const double rhs = sh ? stencil_shifted(p, p.st + (size_t)row * 5, ub, hb, row, sh)
                              : stencil5(p.st + (size_t)row * 5, u0, u1, u2, u3, u4);
        double dj = (j < 2) ? mul(rhs, p.r[row]) : mul(sub(rhs, mul(p.r[row], dprev)), p.f[row]);
        ob[row * sz] = dj;
        dprev = dj;
        u0 = u1; u1 = u2; u2 = u3; u3 = u4;
    }
    double dn = dprev;   // d[m-1] (untouched by the backward sweep)
    double dl = dn;
    double dnext = ob[(long long)(off + m - 2) * sz];
    #pragma unroll 8
    for (int j = m - 3; j >= 1; --j) {
        const int row = off + j;
        const double dj = sub(ob[row * sz], mul(p.w[row], dnext));
        ob[row * sz] = dj;
        dnext = dj;
    }
    // dnext is now d[1]
    const double d0 = mul(sub(ob[(long long)off * sz], mul(p.w[off], dnext)), p.f[off]);
    ob[(long long)off * sz] = d0;
    p.d_first[(long long)b * p.lines + line] = d0;
    p.d_last[(long long)b * p.lines + line] = dl;
}

// 2x2 boundary pairs + Alg. 7 substitution per (line, block):
// distributed.py:279-305, 345-366. In place on the decoupled rows.
__global__ void k_staged_finish(const StagedArgs p) {
    const long long line = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (line >= p.lines) return;
    const int off = p.boff[b], m = p.bsize[b];
    const long long sz = p.sz;
    double* ob = p.out + line_base(line, p.rows, p.sz);
    const double* bc = p.bconst + (size_t)b * 6;
    const double sa_first = bc[0], sc_last = bc[1], det_prev = bc[2], det_next = bc[3];
    const bool hp = bc[4] != 0.0, hn = bc[5] != 0.0;
    const double d0 = p.d_first[(long long)b * p.lines + line];
    const double dl = p.d_last[(long long)b * p.lines + line];
    double us = d0, ue = dl;
    if (hp) {
        double prev_last;
        if (p.prev_last) prev_last = p.prev_last[line];
        else prev_last = p.d_last[(long long)((b - 1 + p.nb) % p.nb) * p.lines + line];
        us = dvd(sub(d0, mul(sa_first, prev_last)), det_prev);
    }
    if (hn) {
        double next_first;
        if (p.next_first) next_first = p.next_first[line];
        else next_first = p.d_first[(long long)((b + 1) % p.nb) * p.lines + line];
        ue = dvd(sub(dl, mul(sc_last, next_first)), det_next);
    }
    ob[(long long)off * sz] = us;
    #pragma unroll 8
    for (int j = 1; j < m - 1; ++j) {
        const int row = off + j;
        ob[row * sz] = sub(ob[row * sz], add(mul(p.sa[row], us), mul(p.sc[row], ue)));
    }
    ob[(long long)(off + m - 1) * sz] = ue;
}

// P=1: stencil + thomas_solve / periodic_thomas_solve (serial.py:26-90,
// distributed.py:380-396), one thread per line.
__global__ void k_thomas(const StagedArgs p) {
    const long long line = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= p.lines) return;
    const int n = p.rows;
    const long long sz = p.sz;
    // u and out never alias (the ABI requires distinct buffers): the row
    // loads can run ahead of the stores
    const double* __restrict__ ub = p.u + line_base(line, p.rows, p.sz);
    double* __restrict__ ob = p.out + line_base(line, p.rows, p.sz);
    const long long hb = halo_base(line, p.sz);
    double u0 = fetch(p, ub, hb, -2), u1 = fetch(p, ub, hb, -1);
    double u2 = fetch(p, ub, hb, 0), u3 = fetch(p, ub, hb, 1);
    double dprev = 0.0;
    #pragma unroll 8
    for (int j = 0; j < n; ++j) {
        const double u4 = fetch(p, ub, hb, j + 2);
        const int sh = row_shift(p, j);
        const double rhs = sh ? stencil_shifted(p, p.st + (size_t)j * 5, ub, hb, j, sh)
                              : stencil5(p.st + (size_t)j * 5, u0, u1, u2, u3, u4);
        const double dj = (j == 0) ? dvd(rhs, p.th_b0)
                                   : mul(sub(rhs, mul(p.th_a[j], dprev)), p.th_w[j]);
        ob[j * sz] = dj;
        dprev = dj;
        u0 = u1; u1 = u2; u2 = u3; u3 = u4;
    }
    double dnext = dprev;
    #pragma unroll 8
    for (int j = n - 2; j >= 0; --j) {
        const double dj = sub(ob[j * sz], mul(p.th_cp[j], dnext));
        ob[j * sz] = dj;
        dnext = dj;
    }
    if (p.periodic) {
        const double y0 = dnext, yl = ob[(long long)(n - 1) * sz];
        const double fac = dvd(add(y0, mul(p.th_qlast, yl)), p.th_den);
        #pragma unroll 8
        for (int j = 0; j < n; ++j) ob[j * sz] = sub(ob[j * sz], mul(fac, p.th_z[j]));
    }
}

static dim3 staged_grid(long long lines, int nb, int threads) {
    return dim3((unsigned)((lines + threads - 1) / threads), (unsigned)nb);
}

int launch_staged_decouple(const StagedArgs& a, cudaStream_t s) {
    if (a.lines == 0) return TDS_OK;
    k_staged_decouple<<<staged_grid(a.lines, a.nb, 128), 128, 0, s>>>(a);
    return cuda_check(cudaGetLastError(), "k_staged_decouple launch");
}
int launch_staged_finish(const StagedArgs& a, cudaStream_t s) {
    if (a.lines == 0) return TDS_OK;
    k_staged_finish<<<staged_grid(a.lines, a.nb, 128), 128, 0, s>>>(a);
    return cuda_check(cudaGetLastError(), "k_staged_finish launch");
}
int launch_thomas(const StagedArgs& a, cudaStream_t s) {
    if (a.lines == 0) return TDS_OK;
    k_thomas<<<staged_grid(a.lines, 1, 128), 128, 0, s>>>(a);
    return cuda_check(cudaGetLastError(), "k_thomas launch");
}

// ------------------------------------------------------------- small kernels

// rows {0,1} -> first2 and {m-2,m-1} -> last2, (G,2,sz) each (ROUND 1 payload,
// transport.py:156-159)
__global__ void k_halo_rows(const double* __restrict__ u, double* __restrict__ first2,
                            double* __restrict__ last2, long long lines, int rows, int sz) {
    const long long line = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= lines) return;
    const double* ub = u + line_base(line, rows, sz);
    const long long hb = halo_base(line, sz);
    first2[hb] = ub[0];
    first2[hb + sz] = ub[(long long)sz];
    last2[hb] = ub[(long long)(rows - 2) * sz];
    last2[hb + sz] = ub[(long long)(rows - 1) * sz];
}

int launch_halo_rows(const double* u, double* first2, double* last2, long long lines, int rows,
                     int sz, cudaStream_t s) {
    if (lines == 0) return TDS_OK;
    k_halo_rows<<<(unsigned)((lines + 255) / 256), 256, 0, s>>>(u, first2, last2, lines, rows, sz);
    return cuda_check(cudaGetLastError(), "k_halo_rows launch");
}

// position-major phase kernels (reference phase functions)
struct Shift4 {
    int s[4];   // window shifts of rows 0, 1, m-2, m-1
};

__global__ void k_decouple_pm(const double* __restrict__ ue, const double* __restrict__ st,
                              const Shift4 sh4, const double* __restrict__ w,
                              const double* __restrict__ f, const double* __restrict__ r,
                              double* __restrict__ d, int m, long long lanes) {
    const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= lanes) return;
    double u0 = ue[l], u1 = ue[lanes + l], u2 = ue[2 * lanes + l], u3 = ue[3 * lanes + l];
    double dprev = 0.0;
    for (int j = 0; j < m; ++j) {
        const double u4 = ue[(long long)(j + 4) * lanes + l];
        const int sh = j < 2 ? sh4.s[j] : (j >= m - 2 ? sh4.s[4 - (m - j)] : 0);
        // shifted window: u_ext rows j + sh .. j + sh + 4 (ue row = position + 2)
        const double rhs =
            sh ? stencil5(st + (size_t)j * 5, ue[(long long)(j + sh) * lanes + l],
                          ue[(long long)(j + sh + 1) * lanes + l],
                          ue[(long long)(j + sh + 2) * lanes + l],
                          ue[(long long)(j + sh + 3) * lanes + l],
                          ue[(long long)(j + sh + 4) * lanes + l])
               : stencil5(st + (size_t)j * 5, u0, u1, u2, u3, u4);
        const double dj = (j < 2) ? mul(rhs, r[j]) : mul(sub(rhs, mul(r[j], dprev)), f[j]);
        d[(long long)j * lanes + l] = dj;
        dprev = dj;
        u0 = u1; u1 = u2; u2 = u3; u3 = u4;
    }
    double dnext = d[(long long)(m - 2) * lanes + l];
    for (int j = m - 3; j >= 1; --j) {
        const double dj = sub(d[(long long)j * lanes + l], mul(w[j], dnext));
        d[(long long)j * lanes + l] = dj;
        dnext = dj;
    }
    d[l] = mul(sub(d[l], mul(w[0], dnext)), f[0]);
}

__global__ void k_substitute_pm(const double* __restrict__ d, const double* __restrict__ sa,
                                const double* __restrict__ sc, const double* __restrict__ us,
                                const double* __restrict__ ue, double* __restrict__ out, int m,
                                long long lanes) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)m * lanes) return;
    const int j = (int)(idx / lanes);
    const long long l = idx % lanes;
    double v;
    if (j == 0) v = us[l];
    else if (j == m - 1) v = ue[l];
    else v = sub(d[idx], add(mul(sa[j], us[l]), mul(sc[j], ue[l])));
    out[idx] = v;
}

__global__ void k_pair(const double* __restrict__ dl, const double* __restrict__ df, double sc,
                       double sa, double det, double* __restrict__ ul, double* __restrict__ uf,
                       long long lanes) {
    const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= lanes) return;
    const double a = dl[l], b = df[l];
    ul[l] = dvd(sub(a, mul(sc, b)), det);
    uf[l] = dvd(sub(b, mul(sa, a)), det);
}

int launch_decouple_pm(const double* u_ext, const double* st, const int* sh4, const double* w,
                       const double* f, const double* r, double* d, int m, long long lanes,
                       cudaStream_t s) {
    if (lanes == 0) return TDS_OK;
    Shift4 sh{{sh4[0], sh4[1], sh4[2], sh4[3]}};
    k_decouple_pm<<<(unsigned)((lanes + 127) / 128), 128, 0, s>>>(u_ext, st, sh, w, f, r, d, m,
                                                                  lanes);
    return cuda_check(cudaGetLastError(), "k_decouple_pm launch");
}
int launch_substitute_pm(const double* d, const double* sa, const double* sc, const double* us,
                         const double* ue, double* out, int m, long long lanes, cudaStream_t s) {
    long long total = (long long)m * lanes;
    if (total == 0) return TDS_OK;
    k_substitute_pm<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(d, sa, sc, us, ue, out, m, lanes);
    return cuda_check(cudaGetLastError(), "k_substitute_pm launch");
}
int launch_pair(const double* dl, const double* df, double sc, double sa, double det, double* ul,
                double* uf, long long lanes, cudaStream_t s) {
    if (lanes == 0) return TDS_OK;
    k_pair<<<(unsigned)((lanes + 255) / 256), 256, 0, s>>>(dl, df, sc, sa, det, ul, uf, lanes);
    return cuda_check(cudaGetLastError(), "k_pair launch");
}

// Cartesian (nx,ny,nz) C-order <-> SZ-blocked field (layout.py:82-141).
// One thread per field element: field writes (reads) are coalesced. Ghost
// lines (transverse index >= lines, layout.py:130-133) are zero.
__global__ void k_pack(const double* __restrict__ src, double* __restrict__ dst, int nx, int ny,
                       int nz, int sz, int dir, long long groups, bool to_field) {
    const int n = dir == 0 ? nx : (dir == 1 ? ny : nz);
    const long long total = groups * sz * n;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const long long lines = (long long)nx * ny * nz / n;
    const long long lane = idx % sz;
    const long long pos = (idx / sz) % n;
    const long long grp = idx / ((long long)sz * n);
    const long long tt = grp * sz + lane;   // transverse index
    if (tt >= lines) {
        if (to_field) dst[idx] = 0.0;
        return;
    }
    long long i, j, k;
    if (dir == 0) { i = pos; j = tt % ny; k = tt / ny; }
    else if (dir == 1) { j = pos; i = tt % nx; k = tt / nx; }
    else { k = pos; i = tt % nx; j = tt / nx; }
    const long long c = (i * ny + j) * nz + k;
    if (to_field) dst[idx] = src[c];
    else dst[c] = src[idx];
}

// Tiled variant: every direction's permutation is a 2-D transpose between the
// Cartesian fastest axis k and the field's fastest axis, the LANE axis (j for
// x lines, i for y and z lines), at fixed third index o (i for x, j for y and
// z). A 32 x 32 shared-memory tile makes both the Cartesian reads (runs of k)
// and the field writes (runs of lanes) coalesced. blockIdx = (k tile, lane
// tile, o); block = 32 x 8 threads.
__device__ __forceinline__ long long field_index(int i, int j, int k, int nx, int ny, int nz,
                                                 int sz, int lsz, int dir) {
    // transverse index < 2^31 for every supported field (lines x sz fits int)
    unsigned t, pos, n;
    if (dir == 0) { t = (unsigned)j + (unsigned)ny * (unsigned)k; pos = i; n = nx; }
    else if (dir == 1) { t = (unsigned)i + (unsigned)nx * (unsigned)k; pos = j; n = ny; }
    else { t = (unsigned)i + (unsigned)nx * (unsigned)j; pos = k; n = nz; }
    unsigned g, l;
    if (lsz >= 0) { g = t >> lsz; l = t & ((1u << lsz) - 1u); }
    else { g = t / (unsigned)sz; l = t - g * (unsigned)sz; }
    return ((long long)g * n + pos) * sz + l;
}

__global__ void k_pack_tiled(const double* __restrict__ src, double* __restrict__ dst, int nx,
                             int ny, int nz, int sz, int lsz, int dir, bool to_field) {
    __shared__ double tile[32][33];
    const int k0 = blockIdx.x * 32;
    const int a0 = blockIdx.y * 32;
    const int o = blockIdx.z;
    const int na = dir == 0 ? ny : nx;     // extent of the lane axis
    const int tx = threadIdx.x, ty = threadIdx.y;
    auto ijk = [&](int a, int k, int& i, int& j) {
        if (dir == 0) { i = o; j = a; }
        else { i = a; j = o; }
        (void)k;
    };
    if (to_field) {
#pragma unroll
        for (int r = ty; r < 32; r += 8) {       // read runs of k: coalesced
            const int a = a0 + r, k = k0 + tx;
            if (a < na && k < nz) {
                int i, j;
                ijk(a, k, i, j);
                tile[r][tx] = __ldcs(src + ((long long)i * ny + j) * nz + k);
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = ty; r < 32; r += 8) {       // write runs of lanes: coalesced
            const int a = a0 + tx, k = k0 + r;
            if (a < na && k < nz) {
                int i, j;
                ijk(a, k, i, j);
                __stcs(dst + field_index(i, j, k, nx, ny, nz, sz, lsz, dir), tile[tx][r]);
            }
        }
    } else {
#pragma unroll
        for (int r = ty; r < 32; r += 8) {       // read runs of lanes
            const int a = a0 + tx, k = k0 + r;
            if (a < na && k < nz) {
                int i, j;
                ijk(a, k, i, j);
                tile[tx][r] = __ldcs(src + field_index(i, j, k, nx, ny, nz, sz, lsz, dir));
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = ty; r < 32; r += 8) {       // write runs of k
            const int a = a0 + r, k = k0 + tx;
            if (a < na && k < nz) {
                int i, j;
                ijk(a, k, i, j);
                __stcs(dst + ((long long)i * ny + j) * nz + k, tile[r][tx]);
            }
        }
    }
}

int launch_pack(const double* src, double* dst, int nx, int ny, int nz, int sz, int dir,
                long long groups, bool to_field, cudaStream_t s) {
    const int n = dir == 0 ? nx : (dir == 1 ? ny : nz);
    long long total = groups * sz * n;
    if (total == 0) return TDS_OK;
    const long long lines = (long long)nx * ny * nz / n;
    const bool tiled = getenv("TDS_PACK_SIMPLE") == nullptr;
    if (tiled) {
        if (to_field && groups * sz > lines) {   // ghost lines are zero
            int rc = cuda_check(cudaMemsetAsync(dst, 0, (size_t)total * sizeof(double), s),
                                "cudaMemsetAsync(ghost lines)");
            if (rc) return rc;
        }
        const int na = dir == 0 ? ny : nx;
        const int no = dir == 0 ? nx : ny;
        dim3 grid((nz + 31) / 32, (na + 31) / 32, no);
        int lsz = -1;
        if ((sz & (sz - 1)) == 0) {
            lsz = 0;
            while ((1 << lsz) < sz) ++lsz;
        }
        k_pack_tiled<<<grid, dim3(32, 8), 0, s>>>(src, dst, nx, ny, nz, sz, lsz, dir, to_field);
        return cuda_check(cudaGetLastError(), "k_pack_tiled launch");
    }
    k_pack<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(src, dst, nx, ny, nz, sz, dir, groups,
                                                          to_field);
    return cuda_check(cudaGetLastError(), "k_pack launch");
}

}  // namespace tds
