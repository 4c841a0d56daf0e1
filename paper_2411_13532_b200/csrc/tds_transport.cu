// Momentum-transport right-hand side building blocks (sm_100a), the consumer
// of the DistD2 path in the reference (momentum.py:102-169):
//
//   k_transport   one (component i, direction j) contribution
//                   -1/2 (u_j d(u_i)/dx_j + d(u_j u_i)/dx_j) + nu d2(u_i)/dx_j2
//                 in ONE pass: each thread reads its chunk of u_i and u_j,
//                 runs the three compact solves of that chunk (d/dx of u_i,
//                 d/dx of u_j u_i, d2/dx2 of u_i; fused stencil + Alg. 6
//                 sweeps, exact reduced map, substitution) and writes -- or
//                 accumulates -- the contribution. 24 B/point (16 on the
//                 diagonal i = j) instead of three solves + products.
//   k_reorder     field -> field re-layout between directions, optionally
//                 accumulating (reorder / accumulate of momentum.py:129-139)
//                 in one pass through a 32 x 32 shared-memory tile.
//   k_transport_combine   elementwise combine for the rank-emulated path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "tds_device.cuh"
#include "tds_tma.h"

namespace tds {

using namespace dev;

struct TransportArgs {
    const double* ui;
    const double* uj;
    double* out;
    const double2* H1;     // reduced map of the d/dx operator
    const double2* H2;     // reduced map of the d2/dx2 operator
    long long lines;
    int rows, sz, chunks, tiles_per_cta;
    int accumulate;
    int has_nu;
    double nu;
    UniformTable t1, t2;   // chunk tables of the two periodic operators
    const double2* Hb1;    // banded reduced maps (plan.cpp upload_H)
    const double2* Hb2;
    const int* bq1;
    const int* bq2;
    int nb1, nb2;
    int geom;              // GEOM_LINES, GEOM_XZ / GEOM_XY: z / y lines of an x-layout box
    int nx, ny, nz;        // GEOM_XY / GEOM_XZ: the (nx, ny, nz) block (rows = ny / nz)
};

// Tile geometry of k_transport_tma: GEOM_LINES reads / writes the field in
// its own (groups, rows, sz) layout; GEOM_XZ reads the z lines of a cubic
// x-layout box in place (4-D tensor map: lanes, x, y-group, z) and ADDS the
// contribution into an x-layout accumulator -- the z direction of the
// transport RHS without re-layout passes. GEOM_XY does the same for the y
// lines (sz = 32): a tile is 16 y lines (consecutive x at one z), loaded as
// two 16-lane halves with the 128-byte TMA swizzle so that the 16 lines of
// a warp read distinct banks; the window is read 16 bytes (two rows) at a
// time.
enum { GEOM_LINES = 0, GEOM_XZ = 1, GEOM_XY = 2 };

namespace {

template <int M>
__device__ __forceinline__ void load_window(const double* ub, long long sz, int r0, int rows,
                                            bool valid, double (&v)[M + 4]) {
#pragma unroll
    for (int i = 0; i < M + 4; ++i) {
        int row = r0 - 2 + i;
        if (row < 0) row += rows;
        else if (row >= rows) row -= rows;
        v[i] = valid ? __ldg(ub + row * sz) : 0.0;
    }
}

template <int M>
__device__ __forceinline__ void load_window_prod(const double* ua, const double* ub, long long sz,
                                                 int r0, int rows, bool valid,
                                                 double (&v)[M + 4]) {
#pragma unroll
    for (int i = 0; i < M + 4; ++i) {
        int row = r0 - 2 + i;
        if (row < 0) row += rows;
        else if (row >= rows) row -= rows;
        v[i] = valid ? __ldg(ua + row * sz) * __ldg(ub + row * sz) : 0.0;
    }
}

// fused stencil + Alg. 6 with a kernel-parameter table
template <int M>
__device__ __forceinline__ void sweeps(const UniformTable& T, const double (&v)[M + 4],
                                       double (&d)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double rhs = T.st[0] * v[i];
        rhs = fma(T.st[1], v[i + 1], rhs);
        rhs = fma(T.st[2], v[i + 2], rhs);
        rhs = fma(T.st[3], v[i + 3], rhs);
        rhs = fma(T.st[4], v[i + 4], rhs);
        if (i < 2) d[i] = rhs * T.r[i];
        else d[i] = fma(-T.r[i], d[i - 1], rhs) * T.f[i];
    }
#pragma unroll
    for (int i = M - 3; i >= 1; --i) d[i] = fma(-T.w[i], d[i + 1], d[i]);
    d[0] = fma(-T.w[0], d[1], d[0]) * T.f[0];
}

__device__ __forceinline__ void bounds(const double2* __restrict__ hr, const double* Y, int K,
                                       int lane, double& F, double& L) {
    double F0 = 0.0, F1 = 0.0, L0 = 0.0, L1 = 0.0;
    for (int q = 0; q + 1 < K; q += 2) {
        const double2 h0 = __ldg(hr + q), h1 = __ldg(hr + q + 1);
        const double ya = Y[q * TL + lane], yb = Y[(q + 1) * TL + lane];
        F0 = fma(h0.x, ya, F0);
        L0 = fma(h0.y, ya, L0);
        F1 = fma(h1.x, yb, F1);
        L1 = fma(h1.y, yb, L1);
    }
    F = F0 + F1;
    L = L0 + L1;
}

}  // namespace

template <int M>
__global__ void __launch_bounds__(512) k_transport(const __grid_constant__ TransportArgs p) {
    extern __shared__ double sY[];                     // [3][tpc][K][TL]
    const int C = p.chunks, K = 2 * C;
    const int t = threadIdx.x;
    const int lane = t % TL;
    const int chunk = (t / TL) % C;
    const int tl = t / (TL * C);
    const long long line = ((long long)blockIdx.x * p.tiles_per_cta + tl) * TL + lane;
    const bool valid = line < p.lines;
    const long long sz = p.sz;
    const long long lb = valid ? line_base(line, p.rows, p.sz) : 0;
    const double* ui = p.ui + lb;
    const double* uj = p.uj + lb;
    double* ob = p.out + lb + (long long)(chunk * M) * sz;
    const int r0 = chunk * M;
    const size_t ybuf = (size_t)p.tiles_per_cta * K * TL;
    double* Y = sY + (size_t)tl * K * TL;

    // The running contribution lives in `out` (this thread's own rows, kept
    // in L2 between the three solves), not in registers: each solve needs
    // the full single-solve register budget.
    double v[M + 4], d[M];
    double F, L;

    // (A) d(u_i)/dx_j  ->  out = u_j * du_i
    load_window<M>(ui, sz, r0, p.rows, valid, v);
    sweeps<M>(p.t1, v, d);
    Y[(2 * chunk) * TL + lane] = d[0];
    Y[(2 * chunk + 1) * TL + lane] = d[M - 1];
    __syncthreads();
    bounds(p.H1 + (size_t)chunk * K, Y, K, lane, F, L);
    if (valid) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const double x = i == 0 ? F : (i == M - 1 ? L : fma(-p.t1.sc[i], L, fma(-p.t1.sa[i], F, d[i])));
            ob[(long long)i * sz] = __ldg(uj + (long long)(r0 + i) * sz) * x;
        }
    }

    // (B) d(u_j u_i)/dx_j  ->  out = -1/2 (out + dprod)
    load_window_prod<M>(uj, ui, sz, r0, p.rows, valid, v);
    sweeps<M>(p.t1, v, d);
    Y += ybuf;
    Y[(2 * chunk) * TL + lane] = d[0];
    Y[(2 * chunk + 1) * TL + lane] = d[M - 1];
    __syncthreads();
    bounds(p.H1 + (size_t)chunk * K, Y, K, lane, F, L);
    const bool last = !p.has_nu;
    if (valid) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const double x = i == 0 ? F : (i == M - 1 ? L : fma(-p.t1.sc[i], L, fma(-p.t1.sa[i], F, d[i])));
            const double val = -0.5 * (ob[(long long)i * sz] + x);
            if (last) __stcs(ob + (long long)i * sz, val);
            else ob[(long long)i * sz] = val;
        }
    }

    // (C) out += nu d2(u_i)/dx_j2
    if (p.has_nu) {
        load_window<M>(ui, sz, r0, p.rows, valid, v);
        sweeps<M>(p.t2, v, d);
        Y += ybuf;
        Y[(2 * chunk) * TL + lane] = d[0];
        Y[(2 * chunk + 1) * TL + lane] = d[M - 1];
        __syncthreads();
        bounds(p.H2 + (size_t)chunk * K, Y, K, lane, F, L);
        if (valid) {
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const double x = i == 0 ? F : (i == M - 1 ? L : fma(-p.t2.sc[i], L, fma(-p.t2.sa[i], F, d[i])));
                __stcs(ob + (long long)i * sz, fma(p.nu, x, ob[(long long)i * sz]));
            }
        }
    }
}

int launch_transport(const TransportArgs& a, cudaStream_t s) {
    const int threads = a.tiles_per_cta * a.chunks * TL;
    if (threads > 512) return set_err(TDS_ERR_UNSUPPORTED, "fused transport: n > 1024");
    if (a.accumulate) return set_err(TDS_ERR_UNSUPPORTED, "fused transport writes, never accumulates");
    const long long tiles = (a.lines + TL - 1) / TL;
    const long long grid = (tiles + a.tiles_per_cta - 1) / a.tiles_per_cta;
    if (grid <= 0) return TDS_OK;
    const size_t smem = (size_t)3 * a.tiles_per_cta * 2 * a.chunks * TL * sizeof(double);
    k_transport<32><<<(unsigned)grid, threads, smem, s>>>(a);
    return cuda_check(cudaGetLastError(), "k_transport launch");
}

// ------------------------------------------------ TMA-staged k_transport
//
// k_transport_tma<M, TLT>: persistent CTAs; the u_i and u_j tiles of TLT
// lines arrive by TMA (3-D tensor maps, one mbarrier) and ALL three solves
// read them from shared memory, so HBM sees u_i and u_j once and `out`
// once (24 B/pt, 16 on the diagonal). 16-row chunks keep the running
// contribution in registers (acc[16] + d[16]); every solve streams its
// stencil window straight out of shared memory, and the next item's TMA is
// issued as soon as the last solve's sweeps have read the tiles.
struct TransportTmaArgs {
    TransportArgs p;
    CUtensorMap map_i, map_j;
    int boxr;
    long long items;
};

namespace {

template <int M, typename Src>
__device__ __forceinline__ void sweeps_src(const UniformTable& T, Src v, double (&d)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double rhs = T.st[0] * v(i);
        rhs = fma(T.st[1], v(i + 1), rhs);
        rhs = fma(T.st[2], v(i + 2), rhs);
        rhs = fma(T.st[3], v(i + 3), rhs);
        rhs = fma(T.st[4], v(i + 4), rhs);
        if (i < 2) d[i] = rhs * T.r[i];
        else d[i] = fma(-T.r[i], d[i - 1], rhs) * T.f[i];
    }
#pragma unroll
    for (int i = M - 3; i >= 1; --i) d[i] = fma(-T.w[i], d[i + 1], d[i]);
    d[0] = fma(-T.w[0], d[1], d[0]) * T.f[0];
}

// Two solves of the SAME window (d/dx and d2/dx2 of u_i) in one pass: every
// window value is read once for both stencils and both forward / backward
// sweeps interleave (independent recurrences: twice the ILP per thread).
template <int M, typename Src>
__device__ __forceinline__ void sweeps2_src(const UniformTable& T1, const UniformTable& T2, Src v,
                                            double (&d1)[M], double (&d2)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const double v0 = v(i), v1 = v(i + 1), v2 = v(i + 2), v3 = v(i + 3), v4 = v(i + 4);
        double a = T1.st[0] * v0, b = T2.st[0] * v0;
        a = fma(T1.st[1], v1, a);
        b = fma(T2.st[1], v1, b);
        a = fma(T1.st[2], v2, a);
        b = fma(T2.st[2], v2, b);
        a = fma(T1.st[3], v3, a);
        b = fma(T2.st[3], v3, b);
        a = fma(T1.st[4], v4, a);
        b = fma(T2.st[4], v4, b);
        if (i < 2) {
            d1[i] = a * T1.r[i];
            d2[i] = b * T2.r[i];
        } else {
            d1[i] = fma(-T1.r[i], d1[i - 1], a) * T1.f[i];
            d2[i] = fma(-T2.r[i], d2[i - 1], b) * T2.f[i];
        }
    }
#pragma unroll
    for (int i = M - 3; i >= 1; --i) {
        d1[i] = fma(-T1.w[i], d1[i + 1], d1[i]);
        d2[i] = fma(-T2.w[i], d2[i + 1], d2[i]);
    }
    d1[0] = fma(-T1.w[0], d1[1], d1[0]) * T1.f[0];
    d2[0] = fma(-T2.w[0], d2[1], d2[0]) * T2.f[0];
}

__device__ __forceinline__ double subst(const UniformTable& T, int i, int M, double F, double L,
                                        double di) {
    return i == 0 ? F : (i == M - 1 ? L : fma(-T.sc[i], L, fma(-T.sa[i], F, di)));
}

}  // namespace

template <int M, int TLT, int GEOM, int SZC>
__global__ void __launch_bounds__(512, 1) k_transport_tma(const __grid_constant__ TransportTmaArgs A) {
    const TransportArgs& p = A.p;
    extern __shared__ __align__(1024) unsigned char smem[];
    const int C = p.chunks, K = 2 * C, rows = p.rows, tpc = p.tiles_per_cta;
    const int t = threadIdx.x;
    const int lane = t % TLT;
    const int chunk = (t / TLT) % C;
    const int tl = t / (TLT * C);
    const long long sz = SZC ? SZC : p.sz;
    const int r0 = chunk * M;
    const size_t tile_elems = (size_t)rows * TLT;
    double* ti = reinterpret_cast<double*>(smem);
    double* tj = ti + (size_t)tpc * tile_elems;
    double* sY = tj + (size_t)tpc * tile_elems;          // [3][tpc][K][TLT]
    const size_t ybuf = (size_t)tpc * K * TLT;
    // coefficient tables in shared memory: read per use inside the item
    // loop (a kernel-parameter table would be hoisted out of the persistent
    // loop into registers and spill)
    UniformTable* sT = reinterpret_cast<UniformTable*>(sY + 3 * ybuf);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sT + 2);
    const bool diag = p.ui == p.uj;
    {
        const double* src1 = reinterpret_cast<const double*>(&p.t1);
        const double* src2 = reinterpret_cast<const double*>(&p.t2);
        double* dst = reinterpret_cast<double*>(sT);
        constexpr int W = sizeof(UniformTable) / sizeof(double);
        for (int k = t; k < 2 * W; k += blockDim.x) dst[k] = k < W ? src1[k] : src2[k - W];
    }
    const UniformTable& T1 = sT[0];
    const UniformTable& T2 = sT[1];
    const int bq1 = __ldg(p.bq1 + chunk), bq2 = __ldg(p.bq2 + chunk);

    auto issue = [&](long long item) {
        uint32_t bytes = 0;
        for (int j = 0; j < tpc; ++j)
            if ((item * tpc + j) * TLT < p.lines)
                bytes += (uint32_t)((diag ? 1 : 2) * tile_elems * sizeof(double));
        mbar_expect_tx(bar, bytes);
        for (int j = 0; j < tpc; ++j) {
            const long long first = (item * tpc + j) * TLT;
            if (first >= p.lines) break;
            if (GEOM == GEOM_XY) {
                // tile = x-block + (n/TLT) * z; halves of 16 lanes, all y-groups
                const long long tile = first / TLT;
                const int nxb = p.nx / TLT;
                const int x0 = (int)(tile % nxb) * TLT, z = (int)(tile / nxb);
                const size_t half = tile_elems / 2;
                for (int h = 0; h < 2; ++h) {
                    tma_load_4d(ti + j * tile_elems + h * half, &A.map_i, bar, h * 16, x0, 0, z);
                    if (!diag)
                        tma_load_4d(tj + j * tile_elems + h * half, &A.map_j, bar, h * 16, x0, 0,
                                    z);
                }
                continue;
            }
            if (GEOM == GEOM_XZ) {
                // line = lane-block + sz * (y-group + (n/sz) * x): z line (x, y)
                const long long tile = first / TLT;
                const int nlb = p.sz / TLT, ngj = p.ny / p.sz;
                const int l0 = (int)(tile % nlb) * TLT;
                const int gj = (int)((tile / nlb) % ngj);
                const int x = (int)(tile / ((long long)nlb * ngj));
                for (int b = 0; b * A.boxr < rows; ++b) {
                    tma_load_4d(ti + j * tile_elems + (size_t)b * A.boxr * TLT, &A.map_i, bar, l0,
                                x, gj, b * A.boxr);
                    if (!diag)
                        tma_load_4d(tj + j * tile_elems + (size_t)b * A.boxr * TLT, &A.map_j,
                                    bar, l0, x, gj, b * A.boxr);
                }
                continue;
            }
            const int g = (int)(first / p.sz), l0 = (int)(first % p.sz);
            for (int b = 0; b * A.boxr < rows; ++b) {
                tma_load_3d(ti + j * tile_elems + (size_t)b * A.boxr * TLT, &A.map_i, bar, l0,
                            b * A.boxr, g);
                if (!diag)
                    tma_load_3d(tj + j * tile_elems + (size_t)b * A.boxr * TLT, &A.map_j, bar,
                                l0, b * A.boxr, g);
            }
        }
    };

    if (t == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    long long item = blockIdx.x;
    if (t == 0 && item < A.items) issue(item);
    uint32_t phase = 0;
    const double* Ti = ti + tl * tile_elems;
    const double* Tj = (diag ? ti : tj) + tl * tile_elems;
    // stencil window of row r0 - 2 + i: rows r0 .. r0+M-1 at immediate
    // offsets from `base`, the 2 + 2 periodic halo rows at wrapped offsets
    // GEOM_XY: row y of line `lane` in the swizzled [half][y-group][line][16]
    // tile: 16-byte unit (y & 15) / 2 of the 128-byte row (group, line) sits at
    // unit ^ (line & 7)
    const int xy_half = rows * TLT / 2;
    auto xy_off = [&](int y) {
        return ((y >> 4) & 1) * xy_half + (((y >> 5) * TLT + lane) << 4) +
               ((((y & 15) >> 1) ^ (lane & 7)) << 1) + (y & 1);
    };
    const int base = GEOM == GEOM_XY ? xy_off(r0) - ((lane & 7) << 1) : r0 * TLT + lane;
    const int lo = GEOM == GEOM_XY ? 0 : (chunk == 0 ? rows - 2 : r0 - 2) * TLT + lane;
    const int hi = GEOM == GEOM_XY ? 0 : (chunk == C - 1 ? 0 : r0 + M) * TLT + lane;
    const int ylo = chunk == 0 ? rows - 2 : r0 - 2, yhi = chunk == C - 1 ? 0 : r0 + M;
    const int xh0 = GEOM == GEOM_XY ? xy_off(ylo) : 0, xh1 = GEOM == GEOM_XY ? xy_off(ylo + 1) : 0;
    const int xh2 = GEOM == GEOM_XY ? xy_off(yhi) : 0, xh3 = GEOM == GEOM_XY ? xy_off(yhi + 1) : 0;
    auto wrap = [&](int i) {
        if (GEOM == GEOM_XY) {
            if (i < 2) return i == 0 ? xh0 : xh1;
            if (i >= M + 2) return i == M + 2 ? xh2 : xh3;
            const int l = i - 2;   // row r0 + l, r0 % 16 == 0
            return base + ((((l >> 1) ^ (lane & 7))) << 1) + (l & 1);
        }
        return i < 2 ? lo + i * TLT : (i >= M + 2 ? hi + (i - M - 2) * TLT : base + (i - 2) * TLT);
    };
    double* Y0 = sY + (size_t)tl * K * TLT;
    // every thread has read its last tile value: hand the buffers to the
    // next item's TMA (it overlaps the reduced solve, substitution, stores)
    auto release = [&](long long nxt) {
        __syncthreads();
        if (t == 0 && nxt < A.items) {
            fence_proxy_async();
            issue(nxt);
        }
    };

    for (; item < A.items; item += gridDim.x) {
        const long long line = (item * tpc + tl) * TLT + lane;
        const bool valid = line < p.lines;
        const long long nxt = item + gridDim.x;
        while (!mbar_try_wait(bar, phase)) {
        }
        phase ^= 1u;
        double acc[M], d[M];
        double F, L;

        // Pass 1 -- the two solves of u_i: (A) d(u_i)/dx_j and (C) d2(u_i)/dx_j2
        // from one read of the window, one barrier for both reduced systems:
        //   acc = -1/2 u_j du_i + nu d2u_i
        if (p.has_nu) {
            double d2[M];
            sweeps2_src<M>(T1, T2, [&](int i) { return Ti[wrap(i)]; }, d, d2);
            double* YA = Y0;
            double* YC = Y0 + 2 * ybuf;
            YA[(2 * chunk) * TLT + lane] = d[0];
            YA[(2 * chunk + 1) * TLT + lane] = d[M - 1];
            YC[(2 * chunk) * TLT + lane] = d2[0];
            YC[(2 * chunk + 1) * TLT + lane] = d2[M - 1];
            __syncthreads();
            double F2, L2;
            band_bounds<TLT>(p.Hb1 + (size_t)chunk * p.nb1, bq1, p.nb1, YA, K, lane, F, L);
            band_bounds<TLT>(p.Hb2 + (size_t)chunk * p.nb2, bq2, p.nb2, YC, K, lane, F2, L2);
#pragma unroll
            for (int i = 0; i < M; ++i)
                acc[i] = fma(-0.5 * Tj[wrap(i + 2)], subst(T1, i, M, F, L, d[i]),
                             p.nu * subst(T2, i, M, F2, L2, d2[i]));
        } else {
            sweeps_src<M>(T1, [&](int i) { return Ti[wrap(i)]; }, d);
            double* YA = Y0;
            YA[(2 * chunk) * TLT + lane] = d[0];
            YA[(2 * chunk + 1) * TLT + lane] = d[M - 1];
            __syncthreads();
            band_bounds<TLT>(p.Hb1 + (size_t)chunk * p.nb1, bq1, p.nb1, YA, K, lane, F, L);
#pragma unroll
            for (int i = 0; i < M; ++i)
                acc[i] = -0.5 * Tj[wrap(i + 2)] * subst(T1, i, M, F, L, d[i]);
        }

        // Pass 2 -- (B) d(u_j u_i)/dx_j: acc -= 1/2 dprod. Its sweeps are the
        // last reads of the tiles: hand them to the next item's TMA.
        sweeps_src<M>(T1, [&](int i) { const int o = wrap(i); return Tj[o] * Ti[o]; }, d);
        release(nxt);
        {
            double* YB = Y0 + ybuf;
            YB[(2 * chunk) * TLT + lane] = d[0];
            YB[(2 * chunk + 1) * TLT + lane] = d[M - 1];
            __syncthreads();
            band_bounds<TLT>(p.Hb1 + (size_t)chunk * p.nb1, bq1, p.nb1, YB, K, lane, F, L);
        }
#pragma unroll
        for (int i = 0; i < M; ++i) acc[i] = fma(-0.5, subst(T1, i, M, F, L, d[i]), acc[i]);
        if (valid && GEOM == GEOM_XY) {
            // x-layout address of (x, y, z): ((y/sz + z n/sz) n + x) sz + y % sz
            const long long tile = line / TLT;
            const int nxb = p.nx / TLT;
            const long long x = (tile % nxb) * TLT + lane, z = tile / nxb;
            double2* ob = reinterpret_cast<double2*>(
                p.out + (((long long)(r0 >> 5) + z * (p.ny / p.sz)) * p.nx + x) * sz + (r0 & 31));
#pragma unroll
            for (int i = 0; i < M / 2; ++i) {
                double2 o = ob[i];
                o.x += acc[2 * i];
                o.y += acc[2 * i + 1];
                ob[i] = o;
            }
        } else if (valid && GEOM == GEOM_XZ) {
            // x-layout address of (x, y, z): ((y-group + z n/sz) n + x) sz + lane
            const long long tile = line / TLT;
            const int nlb = p.sz / TLT, ngj = p.ny / p.sz;
            const long long x = tile / ((long long)nlb * ngj);
            const long long gj = (tile / nlb) % ngj;
            const long long rs = (long long)p.nx * p.ny;        // z stride: nx ny
            double* ob = p.out + (gj * p.nx + x) * sz + (tile % nlb) * TLT + lane + r0 * rs;
#pragma unroll
            for (int i = 0; i < M; ++i) ob[i * rs] = ob[i * rs] + acc[i];
        } else if (valid) {
            double* ob = p.out + line_base_t<SZC>(line, rows, p.sz) + (long long)r0 * sz;
#pragma unroll
            for (int i = 0; i < M; ++i) __stcs(ob + (long long)i * sz, acc[i]);
        }
    }
}

// 4-D view of an x-layout (nx, ny, nz) block (G = ny nz/sz, nx, sz):
// (lane, x, y-group, z) with group = y-group + z * ny/sz; box TLT lanes x
// 1 x 1 x boxr z-rows.
int encode_xz_map(const double* u, int nx, int ny, int nz, int sz, int M, int tl,
                  CUtensorMap* map, int* boxr) {
    *boxr = box_rows(nz, M);
    cuuint64_t dims[4] = {(cuuint64_t)sz, (cuuint64_t)nx, (cuuint64_t)(ny / sz), (cuuint64_t)nz};
    cuuint64_t strides[3] = {(cuuint64_t)sz * 8, (cuuint64_t)nx * sz * 8,
                             (cuuint64_t)nx * (cuuint64_t)ny * 8};
    cuuint32_t box[4] = {(cuuint32_t)tl, 1, 1, (cuuint32_t)*boxr};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult cr = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(u),
                              dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return set_err(TDS_ERR_CUDA, "cuTensorMapEncodeTiled (xz) failed");
    return TDS_OK;
}

namespace {

// The same 4-D view, box 16 lanes x TLT x-positions x all y-groups x 1 z,
// 128-byte swizzle (GEOM_XY tiles).
int encode_xy_map(const double* u, int nx, int ny, int nz, int sz, int tl, CUtensorMap* map) {
    cuuint64_t dims[4] = {(cuuint64_t)sz, (cuuint64_t)nx, (cuuint64_t)(ny / sz), (cuuint64_t)nz};
    cuuint64_t strides[3] = {(cuuint64_t)sz * 8, (cuuint64_t)nx * sz * 8,
                             (cuuint64_t)nx * (cuuint64_t)ny * 8};
    cuuint32_t box[4] = {16, (cuuint32_t)tl, (cuuint32_t)(ny / sz), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult cr = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(u),
                              dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return set_err(TDS_ERR_CUDA, "cuTensorMapEncodeTiled (xy) failed");
    return TDS_OK;
}

template <int M, int TLT, int GEOM, int SZC = 0>
int launch_transport_tma_t(const TransportArgs& a, cudaStream_t s) {
    TransportTmaArgs A;
    A.p = a;
    const int per_tile = a.chunks * TLT;
    A.p.tiles_per_cta = per_tile >= 256 ? 1 : 256 / per_tile;
    const long long tiles = (a.lines + TLT - 1) / TLT;
    A.items = (tiles + A.p.tiles_per_cta - 1) / A.p.tiles_per_cta;
    if (A.items <= 0) return TDS_OK;
    FastArgs fi{}, fj{};
    fi.u = a.ui;
    fj.u = a.uj;
    fi.rows = fj.rows = a.rows;
    fi.sz = fj.sz = a.sz;
    fi.lines = fj.lines = a.lines;
    int rc;
    if (GEOM == GEOM_XY) {
        if ((rc = encode_xy_map(a.ui, a.nx, a.ny, a.nz, a.sz, TLT, &A.map_i))) return rc;
        if ((rc = encode_xy_map(a.uj, a.nx, a.ny, a.nz, a.sz, TLT, &A.map_j))) return rc;
        A.boxr = a.rows;
    } else if (GEOM == GEOM_XZ) {
        if ((rc = encode_xz_map(a.ui, a.nx, a.ny, a.nz, a.sz, M, TLT, &A.map_i, &A.boxr)))
            return rc;
        if ((rc = encode_xz_map(a.uj, a.nx, a.ny, a.nz, a.sz, M, TLT, &A.map_j, &A.boxr)))
            return rc;
    } else {
        if ((rc = encode_field_map(fi, M, TLT, &A.map_i, &A.boxr))) return rc;
        if ((rc = encode_field_map(fj, M, TLT, &A.map_j, &A.boxr))) return rc;
    }
    const int threads = A.p.tiles_per_cta * per_tile;
    const size_t smem = (size_t)A.p.tiles_per_cta *
                            (2 * (size_t)a.rows * TLT + 3 * (size_t)2 * a.chunks * TLT) *
                            sizeof(double) + 2 * sizeof(UniformTable) + 16;
    const void* fn = reinterpret_cast<const void*>(k_transport_tma<M, TLT, GEOM, SZC>);
    if ((rc = ensure_smem(fn, smem, "cudaFuncSetAttribute(k_transport_tma)"))) return rc;
    const long long grid = persistent_grid(fn, threads, smem, A.items, 0);
    if (grid < 1) return set_err(TDS_ERR_UNSUPPORTED, "k_transport_tma does not fit on an SM");
    k_transport_tma<M, TLT, GEOM, SZC><<<(unsigned)grid, threads, smem, s>>>(A);
    return cuda_check(cudaGetLastError(), "k_transport_tma launch");
}

}  // namespace

// TMA transport eligibility: 16-row chunks, tiles of 8 / 16 lines that fit.
static int transport_tma_tl(const TransportArgs& a) {
    if (const char* e = getenv("TDS_TRANSPORT_TMA"))
        if (e[0] == '0') return 0;
    if (reinterpret_cast<uintptr_t>(a.ui) % 16 || reinterpret_cast<uintptr_t>(a.uj) % 16 ||
        reinterpret_cast<uintptr_t>(a.out) % 16)
        return 0;
    if (box_rows(a.rows, 16) == 0) return 0;
    int pref = 16;
    if (const char* e = getenv("TDS_TRANSPORT_TL")) pref = atoi(e) == 8 ? 8 : 16;
    for (int tl : {pref, 24 - pref}) {
        if (a.sz % tl) continue;
        const int per_tile = a.chunks * tl;
        if (per_tile > 512) continue;
        const int tpc = per_tile >= 256 ? 1 : 256 / per_tile;
        const size_t smem =
            (size_t)tpc * (2 * (size_t)a.rows * tl + 6 * (size_t)a.chunks * tl) * 8 +
            2 * sizeof(UniformTable) + 16;
        if (smem <= 200 * 1024) return tl;
    }
    return 0;
}

int launch_transport_tma(const TransportArgs& a, cudaStream_t s) {
    const int tl = transport_tma_tl(a);
    if (a.geom == GEOM_XY) {
        // 8- or 16-line tiles: the swizzle row of (y-group, line) is line & 7
        if (a.sz != 32 || a.ny % 32 || (tl != 16 && tl != 8) || a.nx % tl)
            return set_err(TDS_ERR_UNSUPPORTED, "xy transport: sz = 32, 32 | ny, tile | nx");
        if (tl == 16) return launch_transport_tma_t<16, 16, GEOM_XY>(a, s);
        return launch_transport_tma_t<16, 8, GEOM_XY>(a, s);
    }
    if (a.geom == GEOM_XZ) {
        if (a.ny % a.sz) return set_err(TDS_ERR_UNSUPPORTED, "xz transport: sz must divide ny");
        if (tl == 16) return launch_transport_tma_t<16, 16, GEOM_XZ>(a, s);
        if (tl == 8) return launch_transport_tma_t<16, 8, GEOM_XZ>(a, s);
    } else {
        if (tl == 16 && a.sz == 32 && !(getenv("TDS_SZC") && getenv("TDS_SZC")[0] == '0'))
            return launch_transport_tma_t<16, 16, GEOM_LINES, 32>(a, s);
        if (tl == 16) return launch_transport_tma_t<16, 16, GEOM_LINES>(a, s);
        if (tl == 8) return launch_transport_tma_t<16, 8, GEOM_LINES>(a, s);
    }
    return set_err(TDS_ERR_UNSUPPORTED, "fused transport: shape not TMA-tileable");
}

// ------------------------------------------- one direction, all components
//
// k_transport_dir<TLT, GEOM, SZC>: the three contributions of ONE direction
// j (components i = 0, 1, 2) in one pass. Per item the u_0, u_1, u_2 tiles of
// TLT lines arrive by TMA, each on its own mbarrier, and feed the nine
// compact solves of the item. HBM sees every velocity component once per
// direction (instead of 5 tile reads for 3 per-term launches) and every
// output once: 48 B/pt for the x pass (3 reads + 3 writes), 72 B/pt for the
// in-place y / z passes (3 reads + 3 read-modify-writes).
//
// A component phase is the two passes of k_transport_tma: d/dx and d2/dx2
// of u_i from one read of the window (one barrier for both reduced
// systems), then d/dx of u_j u_i. Components run in the order a, b, j (j =
// the advecting one, read by every phase). The x pass re-arms a tile right
// after the phase's last read of it (its second barrier). The y / z passes
// stage the phase's contribution in the freed tile, in its load layout, and
// add it into the accumulator by TMA reduce-add; tiles a and b are re-armed
// at the next phase's first barrier (once the TMA engine has read them), u_j
// at once (the next item needs it early). 16-line tiles: one CTA of 512
// threads and 3 x 64 KB of tiles per SM at n = 512.
//
// Instruction diet (the kernel is issue / latency bound, not HBM bound):
// per-row coefficients of both operators sit in shared memory as 16-byte
// pairs (DirRow, one LDS.128 per pair); the periodic P = 1 reduced map is
// block-circulant, so every chunk's band row is the same nb values -- they
// travel in the kernel-parameter bank and, with the band lengths as
// template constants (NB1 / NB2), enter the bounds as uniform-register DFMA
// operands; the x / y passes take the stencil weights the same way.
constexpr int NBC_MAX = 24;

struct TransportDirArgs {
    TransportArgs p;          // geometry, tables and reduced maps (ui/uj/out unused)
    const double* u[3];
    double* out[3];
    CUtensorMap map[3];
    CUtensorMap omap[3];      // the outputs (y / z passes: TMA reduce-add targets)
    int boxr;
    int jdir;                 // solve direction = the advecting component
    long long items;
    int nbc1, nbc2;           // circulant band length and first column of chunk 0
    int q01, q02;
    int ydup;                 // Y entries duplicated past K (>= both band lengths, even)
    double2 hc1[NBC_MAX], hc2[NBC_MAX];
    // dynamic item schedule (null: round-robin): ctr[0] hands out items past
    // the grid's first, ctr[1] counts CTAs out (a slot of the d/dx plan's ring)
    unsigned long long* ctr;
};

namespace {

// (F, L) of a chunk from a circulant band row held in the parameter bank:
// the same terms and association as band_bounds (even columns into F0 / L0,
// odd into F1 / L1). Yb = this chunk's first band column in the extended Y
// buffer (K entries plus a copy of the first NBC_MAX: no wrap), so every
// read is an immediate offset from one address.
template <int TLT, int NB = 0>
__device__ __forceinline__ void circ_bounds(const double2 (&h)[NBC_MAX], int nb,
                                            const double* Yb, double& F, double& L) {
    double F0 = 0.0, F1 = 0.0, L0 = 0.0, L1 = 0.0;
    // NB > 0: the band length known at compile time (no per-column
    // predicates: the band row can stay constant-bank operands)
#pragma unroll
    for (int j = 0; j < (NB ? NB : NBC_MAX); ++j) {
        if (NB || j < nb) {
            const double y = Yb[j * TLT];
            if (j & 1) {
                F1 = fma(h[j].x, y, F1);
                L1 = fma(h[j].y, y, L1);
            } else {
                F0 = fma(h[j].x, y, F0);
                L0 = fma(h[j].y, y, L0);
            }
        }
    }
    F = F0 + F1;
    L = L0 + L1;
}

}  // namespace

template <int TLT, int GEOM, int SZC, int NB1, int NB2>
__global__ void __launch_bounds__(512) k_transport_dir(const __grid_constant__ TransportDirArgs A) {
    constexpr int M = 16;
    constexpr bool ACC = GEOM != GEOM_LINES;   // x pass writes, y / z passes add
    // staged output (TMA reduce-add) in the y / z passes. The x pass keeps
    // per-thread streaming stores: staging it for TMA stores measured 2.47
    // vs 2.27 ms at 512^3 (the extra barrier and the delayed tile reload).
    constexpr bool STAGE = ACC;
    const TransportArgs& p = A.p;
    extern __shared__ __align__(1024) unsigned char smem[];
    const int C = p.chunks, K = 2 * C, rows = p.rows, tpc = p.tiles_per_cta;
    const int t = threadIdx.x;
    const int lane = t % TLT;
    const int chunk = (t / TLT) % C;
    const int tl = t / (TLT * C);
    const long long sz = SZC ? SZC : p.sz;
    const int r0 = chunk * M;
    const size_t tile_elems = (size_t)rows * TLT;
    const size_t field_elems = (size_t)tpc * tile_elems;
    double* tiles = reinterpret_cast<double*>(smem);            // [3][tpc][rows][TLT]
    const int KE = K + A.ydup;                                   // extended Y: no wrap
    double* sY = tiles + 3 * field_elems;                        // [3][tpc][KE][TLT]
    const size_t ybuf = (size_t)tpc * KE * TLT;
    DirRow* sR = reinterpret_cast<DirRow*>(sY + 3 * ybuf);       // [M]
    double* sst = reinterpret_cast<double*>(sR + M);             // stencils [2][5] (+ pad)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sst + 12);       // one per component tile
    for (int i = t; i < M; i += blockDim.x) {
        DirRow r;
        r.rf1 = make_double2(p.t1.r[i], p.t1.f[i]);
        r.rf2 = make_double2(p.t2.r[i], p.t2.f[i]);
        r.w12 = make_double2(p.t1.w[i], p.t2.w[i]);
        r.s1 = make_double2(p.t1.sa[i], p.t1.sc[i]);
        r.s2 = make_double2(p.t2.sa[i], p.t2.sc[i]);
        sR[i] = r;
    }
    if (t < 10) sst[t] = t < 5 ? p.t1.st[t] : p.t2.st[t - 5];
    // (a kernel-parameter copy of the table is hoisted into registers and
    // spills: measured 10.6 vs 9.87 ms for the 512^3 RHS)
    const DirRow (&RT)[16] = *reinterpret_cast<const DirRow(*)[16]>(sR);
    // stencil weights: kernel-parameter bank (uniform-register operands;
    // measured x 1.88 -> 1.75, y 2.14 -> 1.93 ms at 512^3) except in the z
    // pass, where they cost registers and spills (2.08 -> 2.35 ms)
    const double* st1 = GEOM == GEOM_XZ ? sst : p.t1.st;
    const double* st2 = GEOM == GEOM_XZ ? sst + 5 : p.t2.st;
    // circulant band: chunk k's window starts at (q0 + 2k) mod K
    const int q1 = (A.q01 + 2 * chunk) % K, q2 = (A.q02 + 2 * chunk) % K;
    const bool dup = 2 * chunk < A.ydup;   // this chunk's Y entries also go to K + 2k
    const int jd = A.jdir;
    const int ca = jd == 0 ? 1 : 0, cb = jd == 2 ? 1 : 2;

    auto issue = [&](int c, long long item) {
        uint32_t bytes = 0;
        for (int q = 0; q < tpc; ++q)
            if ((item * tpc + q) * TLT < p.lines)
                bytes += (uint32_t)(tile_elems * sizeof(double));
        mbar_expect_tx(bar + c, bytes);
        double* dst0 = tiles + c * field_elems;
        const CUtensorMap* map = &A.map[c];
        for (int q = 0; q < tpc; ++q) {
            const long long first = (item * tpc + q) * TLT;
            if (first >= p.lines) break;
            double* dst = dst0 + q * tile_elems;
            if (GEOM == GEOM_XY) {
                const long long tile = first / TLT;
                const int nxb = p.nx / TLT;
                const int x0 = (int)(tile % nxb) * TLT, z = (int)(tile / nxb);
                const size_t half = tile_elems / 2;
                for (int h = 0; h < 2; ++h) tma_load_4d(dst + h * half, map, bar + c, h * 16, x0, 0, z);
            } else if (GEOM == GEOM_XZ) {
                const long long tile = first / TLT;
                const int nlb = p.sz / TLT, ngj = p.ny / p.sz;
                const int l0 = (int)(tile % nlb) * TLT;
                const int gj = (int)((tile / nlb) % ngj);
                const int x = (int)(tile / ((long long)nlb * ngj));
                for (int b = 0; b * A.boxr < rows; ++b)
                    tma_load_4d(dst + (size_t)b * A.boxr * TLT, map, bar + c, l0, x, gj, b * A.boxr);
            } else {
                const int g = (int)(first / p.sz), l0 = (int)(first % p.sz);
                for (int b = 0; b * A.boxr < rows; ++b)
                    tma_load_3d(dst + (size_t)b * A.boxr * TLT, map, bar + c, l0, b * A.boxr, g);
            }
        }
    };

    // staged output of the y / z passes: add tile c -- holding the item's
    // contribution in the layout its load used -- into out[c] with the TMA
    // engine: the inverse of issue(c, item)
    auto reduce_out = [&](int c, long long item) {
        const double* src0 = tiles + c * field_elems;
        const CUtensorMap* map = &A.omap[c];
        for (int q = 0; q < tpc; ++q) {
            const long long first = (item * tpc + q) * TLT;
            if (first >= p.lines) break;
            const double* src = src0 + q * tile_elems;
            if (GEOM == GEOM_XY) {
                const long long tile = first / TLT;
                const int nxb = p.nx / TLT;
                const int x0 = (int)(tile % nxb) * TLT, z = (int)(tile / nxb);
                const size_t half = tile_elems / 2;
                for (int h = 0; h < 2; ++h) tma_reduce_add_4d(map, src + h * half, h * 16, x0, 0, z);
            } else if (GEOM == GEOM_XZ) {
                const long long tile = first / TLT;
                const int nlb = p.sz / TLT, ngj = p.ny / p.sz;
                const int l0 = (int)(tile % nlb) * TLT;
                const int gj = (int)((tile / nlb) % ngj);
                const int x = (int)(tile / ((long long)nlb * ngj));
                for (int b = 0; b * A.boxr < rows; ++b)
                    tma_reduce_add_4d(map, src + (size_t)b * A.boxr * TLT, l0, x, gj, b * A.boxr);
            }
        }
        bulk_commit();
    };

    if (t == 0) {
        for (int c = 0; c < 3; ++c) mbar_init(bar + c, 1);
        fence_mbar_init();
    }
    __syncthreads();
    long long item = blockIdx.x;
    if (t == 0 && item < A.items) {
        issue(ca, item);
        issue(jd, item);
        issue(cb, item);
    }
    uint32_t phases = 0;   // bit c: parity of the next completion of tile c
    int pend = -1;         // thread 0: staged tile whose reload waits for its TMA read

    // window offsets (the same in every tile): see k_transport_tma
    const int xy_half = rows * TLT / 2;
    auto xy_off = [&](int y) {
        return ((y >> 4) & 1) * xy_half + (((y >> 5) * TLT + lane) << 4) +
               ((((y & 15) >> 1) ^ (lane & 7)) << 1) + (y & 1);
    };
    const int base = GEOM == GEOM_XY ? xy_off(r0) - ((lane & 7) << 1) : r0 * TLT + lane;
    const int lo = GEOM == GEOM_XY ? 0 : (chunk == 0 ? rows - 2 : r0 - 2) * TLT + lane;
    const int hi = GEOM == GEOM_XY ? 0 : (chunk == C - 1 ? 0 : r0 + M) * TLT + lane;
    const int ylo = chunk == 0 ? rows - 2 : r0 - 2, yhi = chunk == C - 1 ? 0 : r0 + M;
    const int xh0 = GEOM == GEOM_XY ? xy_off(ylo) : 0, xh1 = GEOM == GEOM_XY ? xy_off(ylo + 1) : 0;
    const int xh2 = GEOM == GEOM_XY ? xy_off(yhi) : 0, xh3 = GEOM == GEOM_XY ? xy_off(yhi + 1) : 0;
    auto wrap = [&](int i) {
        if (GEOM == GEOM_XY) {
            if (i < 2) return i == 0 ? xh0 : xh1;
            if (i >= M + 2) return i == M + 2 ? xh2 : xh3;
            const int l = i - 2;
            return base + ((((l >> 1) ^ (lane & 7))) << 1) + (l & 1);
        }
        return i < 2 ? lo + i * TLT : (i >= M + 2 ? hi + (i - M - 2) * TLT : base + (i - 2) * TLT);
    };
    // window row i of a tile; the y-line tiles (GEOM_XY) hold rows 2k, 2k+1
    // of a line in one 16-byte unit: read it whole (LDS.128, the two calls of
    // a pair are one load), 4 wavefronts per warp instead of 4 per 8 bytes
    auto rd = [&](const double* T, int i) -> double {
        if (GEOM == GEOM_XY) {
            const double2 q = *reinterpret_cast<const double2*>(T + wrap(i & ~1));
            return (i & 1) ? q.y : q.x;
        }
        return T[wrap(i)];
    };
    double* Y0 = sY + (size_t)tl * KE * TLT;
    double* YA = Y0;
    double* YB = Y0 + ybuf;
    double* YC = Y0 + 2 * ybuf;
    auto post = [&](double* Y, double first, double last) {
        Y[(2 * chunk) * TLT + lane] = first;
        Y[(2 * chunk + 1) * TLT + lane] = last;
        if (dup) {
            Y[(K + 2 * chunk) * TLT + lane] = first;
            Y[(K + 2 * chunk + 1) * TLT + lane] = last;
        }
    };
    const int yo1 = q1 * TLT + lane, yo2 = q2 * TLT + lane;
    auto wait_tile = [&](int c) {
        const uint32_t ph = (phases >> c) & 1u;
        while (!mbar_try_wait(bar + c, ph)) {
        }
        phases ^= 1u << c;
    };

    // items past the first: round-robin, or (A.ctr) handed out in order of
    // request. Thread 0 claims the next item at the top of an item (its
    // tiles are issued from the first phase on) and everyone reads it after
    // the item's barriers; s_next[it & 1] is rewritten two items later.
    // The y pass keeps the round-robin schedule: the schedule's extra live
    // state spills there (y 1.96 -> 2.21 ms at 512^3).
    constexpr bool DYN = GEOM != GEOM_XY;
    __shared__ long long s_next[2];
    for (int it = 0; item < A.items; item = DYN ? s_next[it & 1] : item + gridDim.x, ++it) {
        const long long line = (item * tpc + tl) * TLT + lane;
        const bool valid = line < p.lines;
        if (DYN && t == 0)
            s_next[it & 1] = A.ctr ? (long long)gridDim.x + (long long)atomicAdd(A.ctr, 1ULL)
                                   : item + gridDim.x;
        // thread 0 reads the next item back where it issues its tiles (a
        // shared load, not a register live across the item)
        auto next_item = [&]() -> long long { return DYN ? s_next[it & 1] : item + gridDim.x; };
        // this thread's output rows (component offset added per phase)
        long long orow = 0, ostride = sz;
        if (GEOM == GEOM_XY) {
            const long long tile = line / TLT;
            const int nxb = p.nx / TLT;
            const long long x = (tile % nxb) * TLT + lane, z = tile / nxb;
            orow = (((long long)(r0 >> 5) + z * (p.ny / p.sz)) * p.nx + x) * sz + (r0 & 31);
            ostride = 1;
        } else if (GEOM == GEOM_XZ) {
            const long long tile = line / TLT;
            const int nlb = p.sz / TLT, ngj = p.ny / p.sz;
            const long long x = tile / ((long long)nlb * ngj);
            const long long gj = (tile / nlb) % ngj;
            ostride = (long long)p.nx * p.ny;
            orow = (gj * p.nx + x) * sz + (tile % nlb) * TLT + lane + r0 * ostride;
        } else {
            orow = valid ? line_base_t<SZC>(line, rows, p.sz) + (long long)r0 * sz : 0;
        }
        const double* Tj = tiles + jd * field_elems + tl * tile_elems;
#pragma unroll 1
        for (int s = 0; s < 3; ++s) {
            const int c = s == 0 ? ca : (s == 1 ? cb : jd);
            const double* Tc = tiles + c * field_elems + tl * tile_elems;
            double* ob = A.out[c] + orow;
            if (c != jd) wait_tile(c);   // u_j: waited for once per item, below
            double acc[M], d[M];
            double F, L;

            // pass 1: d(u_c) and d2(u_c) from one read of the window
            if (p.has_nu) {
                double d2[M];
                dsweeps2<M>(RT, st1, st2, [&](int i) { return rd(Tc, i); }, d, d2);
                post(YA, d[0], d[M - 1]);
                post(YC, d2[0], d2[M - 1]);
                __syncthreads();
                if (STAGE && t == 0 && pend >= 0) {
                    bulk_wait_read<0>();
                    issue(pend, next_item());
                    pend = -1;
                }
                if (s == 0) wait_tile(jd);
                double F2, L2;
                circ_bounds<TLT, NB1>(A.hc1, A.nbc1, YA + yo1, F, L);
                circ_bounds<TLT, NB2>(A.hc2, A.nbc2, YC + yo2, F2, L2);
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const DirRow& R = RT[i];
                    acc[i] = fma(-0.5 * rd(Tj, i + 2), subst2(R.s1, i, M, F, L, d[i]),
                                 p.nu * subst2(R.s2, i, M, F2, L2, d2[i]));
                }
            } else {
                dsweeps1<M>(RT, st1, [&](int i) { return rd(Tc, i); }, d);
                post(YA, d[0], d[M - 1]);
                __syncthreads();
                if (STAGE && t == 0 && pend >= 0) {
                    bulk_wait_read<0>();
                    issue(pend, next_item());
                    pend = -1;
                }
                if (s == 0) wait_tile(jd);
                circ_bounds<TLT, NB1>(A.hc1, A.nbc1, YA + yo1, F, L);
#pragma unroll
                for (int i = 0; i < M; ++i)
                    acc[i] = -0.5 * rd(Tj, i + 2) * subst2(RT[i].s1, i, M, F, L, d[i]);
            }

            // pass 2: d(u_j u_c); its sweeps are the phase's last tile reads
            dsweeps1<M>(RT, st1, [&](int i) { return rd(Tj, i) * rd(Tc, i); }, d);
            post(YB, d[0], d[M - 1]);
            __syncthreads();
            if (!STAGE && t == 0 && next_item() < A.items) {
                fence_proxy_async();
                issue(c, next_item());
            }
            circ_bounds<TLT, NB1>(A.hc1, A.nbc1, YB + yo1, F, L);
#pragma unroll
            for (int i = 0; i < M; ++i) acc[i] = fma(-0.5, subst2(RT[i].s1, i, M, F, L, d[i]), acc[i]);
            if (!STAGE) {
                if (valid) {
#pragma unroll
                    for (int i = 0; i < M; ++i) __stcs(ob + i * ostride, acc[i]);
                }
            } else {
                // the contribution goes into tile c (free since the barrier)
                // in its load layout, and the TMA engine adds it into out[c]
                // in L2: no accumulator reads by the SM, and the per-thread
                // 128-byte rows of a y line never go through the LSU
                double* Tw = tiles + c * field_elems + tl * tile_elems;
                if (GEOM == GEOM_XY) {
#pragma unroll
                    for (int u = 0; u < M / 2; ++u)
                        *reinterpret_cast<double2*>(Tw + wrap(2 * u + 2)) =
                            make_double2(acc[2 * u], acc[2 * u + 1]);
                } else {
#pragma unroll
                    for (int i = 0; i < M; ++i) Tw[wrap(i + 2)] = acc[i];
                }
                fence_proxy_async();
                __syncthreads();
                if (t == 0) {
                    reduce_out(c, item);
                    if (next_item() < A.items) {
                        if (s == 2) {
                            // u_j is needed early in the next item: re-arm
                            // as soon as the TMA engine has read the tile
                            bulk_wait_read<0>();
                            issue(c, next_item());
                        } else {
                            pend = c;          // at the next phase's barrier
                        }
                    }
                }
            }
        }
    }
    if (STAGE && t == 0) bulk_wait_all();   // the last stores / reduces complete before exit
    if (A.ctr && t == 0) {
        // every CTA has taken its last item once all have come here: the
        // last one out resets the slot for the next launch that uses it
        __threadfence();
        if (atomicAdd(A.ctr + 1, 1ULL) == gridDim.x - 1) {
            A.ctr[0] = 0;
            A.ctr[1] = 0;
            __threadfence();
        }
    }
}

namespace {

template <int TLT, int GEOM, int SZC, int NB1, int NB2>
int launch_transport_dir_nb(const TransportDirArgs& a0, cudaStream_t s) {
    TransportDirArgs A = a0;
    const TransportArgs& a = A.p;
    const int per_tile = a.chunks * TLT;
    A.p.tiles_per_cta = per_tile >= 256 ? 1 : 256 / per_tile;
    const long long tiles = (a.lines + TLT - 1) / TLT;
    A.items = (tiles + A.p.tiles_per_cta - 1) / A.p.tiles_per_cta;
    if (A.items <= 0) return TDS_OK;
    int rc;
    for (int c = 0; c < 3; ++c) {
        if (GEOM == GEOM_XY) {
            if ((rc = encode_xy_map(A.u[c], a.nx, a.ny, a.nz, a.sz, TLT, &A.map[c]))) return rc;
            if ((rc = encode_xy_map(A.out[c], a.nx, a.ny, a.nz, a.sz, TLT, &A.omap[c]))) return rc;
            A.boxr = a.rows;
        } else if (GEOM == GEOM_XZ) {
            if ((rc = encode_xz_map(A.u[c], a.nx, a.ny, a.nz, a.sz, 16, TLT, &A.map[c], &A.boxr)))
                return rc;
            if ((rc = encode_xz_map(A.out[c], a.nx, a.ny, a.nz, a.sz, 16, TLT, &A.omap[c],
                                    &A.boxr)))
                return rc;
        } else {
            FastArgs f{};
            f.u = A.u[c];
            f.rows = a.rows;
            f.sz = a.sz;
            f.lines = a.lines;
            if ((rc = encode_field_map(f, 16, TLT, &A.map[c], &A.boxr))) return rc;
        }
    }
    const int threads = A.p.tiles_per_cta * per_tile;
    const size_t smem = (size_t)A.p.tiles_per_cta *
                            (3 * (size_t)a.rows * TLT + 3 * (size_t)(2 * a.chunks + A.ydup) * TLT) *
                            sizeof(double) + 16 * sizeof(DirRow) + 12 * sizeof(double) +
                        3 * sizeof(uint64_t);
    const void* fn = reinterpret_cast<const void*>(k_transport_dir<TLT, GEOM, SZC, NB1, NB2>);
    if ((rc = ensure_smem(fn, smem, "cudaFuncSetAttribute(k_transport_dir)"))) return rc;
    const long long grid = persistent_grid(fn, threads, smem, A.items, 0);
    if (grid < 1) return set_err(TDS_ERR_UNSUPPORTED, "k_transport_dir does not fit on an SM");
    k_transport_dir<TLT, GEOM, SZC, NB1, NB2><<<(unsigned)grid, threads, smem, s>>>(A);
    return cuda_check(cudaGetLastError(), "k_transport_dir launch");
}

// the band lengths of the 6th-order d/dx and d2/dx2 operators with 16-row
// chunks (16 / 8 columns at 2^-70) as compile-time constants; others (or
// nu = 0, TDS_TRANSPORT_DIR_NB=0) take the predicated runtime loop
template <int TLT, int GEOM, int SZC = 0>
int launch_transport_dir_t(const TransportDirArgs& a, cudaStream_t s) {
    const char* e = getenv("TDS_TRANSPORT_DIR_NB");
    if (!(e && e[0] == '0') && a.nbc1 == 16 && a.nbc2 == 8 && a.p.has_nu)
        return launch_transport_dir_nb<TLT, GEOM, SZC, 16, 8>(a, s);
    return launch_transport_dir_nb<TLT, GEOM, SZC, 0, 0>(a, s);
}

// tile width of k_transport_dir: 16 lines (one CTA of 512 threads per SM at
// n = 512; measured 9.87 vs 10.05 ms for the 512^3 RHS against 8-line tiles
// at two CTAs per SM, whose four chunks per warp read the same banks) unless
// TDS_TRANSPORT_DIR_TL=8; 0 if no width fits
int transport_dir_tl(const TransportArgs& a, int ydup, const double* const* u, double* const* out) {
    for (int c = 0; c < 3; ++c)
        if (reinterpret_cast<uintptr_t>(u[c]) % 16 || reinterpret_cast<uintptr_t>(out[c]) % 16)
            return 0;
    if (box_rows(a.rows, 16) == 0) return 0;
    int pref = 16;
    if (const char* e = getenv("TDS_TRANSPORT_DIR_TL")) pref = atoi(e) == 8 ? 8 : 16;
    for (int tl : {pref, 24 - pref}) {
        if (a.sz % tl) continue;
        const int per_tile = a.chunks * tl;
        if (per_tile > 512) continue;
        const int tpc = per_tile >= 256 ? 1 : 256 / per_tile;
        const size_t smem =
            (size_t)tpc * (3 * (size_t)a.rows * tl + 3 * (size_t)(2 * a.chunks + ydup) * tl) * 8 +
            16 * sizeof(DirRow) + 96 + 24;
        if (smem <= 227 * 1024) return tl;
    }
    return 0;
}

}  // namespace

int transport_direction_from_plans(const tds_plan* d1, const tds_plan* d2, const double* const* u,
                                   double* const* out, double nu, int nx, int ny, int nz, int sz,
                                   int dir, cudaStream_t s) {
    TransportDirArgs A{};
    TransportArgs& a = A.p;
    a.geom = dir == 0 ? GEOM_LINES : (dir == 1 ? GEOM_XY : GEOM_XZ);
    a.nx = nx;
    a.ny = ny;
    a.nz = nz;
    a.rows = d1->block_rows;
    a.sz = sz;
    a.chunks = d1->C;
    a.lines = dir == 0 ? (long long)ny * nz : (dir == 1 ? (long long)nx * nz : (long long)nx * ny);
    a.accumulate = dir != 0;
    a.has_nu = d2 ? 1 : 0;
    a.nu = nu;
    a.t1 = d1->ut;
    a.t2 = d2 ? d2->ut : d1->ut;
    a.H1 = d1->d_Hp;
    a.H2 = d2 ? d2->d_Hp : d1->d_Hp;
    a.Hb1 = d1->d_Hb;
    a.Hb2 = d2 ? d2->d_Hb : d1->d_Hb;
    a.bq1 = d1->d_bq0;
    a.bq2 = d2 ? d2->d_bq0 : d1->d_bq0;
    a.nb1 = d1->band_n;
    a.nb2 = d2 ? d2->band_n : d1->band_n;
    for (int c = 0; c < 3; ++c) {
        A.u[c] = u[c];
        A.out[c] = out[c];
    }
    A.jdir = dir;
    // dynamic item schedule, x and z passes (knob TDS_DYN=0 /
    // TDS_TRANSPORT_DYN=0: round-robin)
    if (dir != 1 && d1->d_ctr && !(getenv("TDS_DYN") && getenv("TDS_DYN")[0] == '0') &&
        !(getenv("TDS_TRANSPORT_DYN") && getenv("TDS_TRANSPORT_DYN")[0] == '0')) {
        const unsigned slot = __atomic_fetch_add(&d1->ctr_next, 1u, __ATOMIC_RELAXED);
        A.ctr = d1->d_ctr + 2 * (slot % CTR_SLOTS);
    }
    if (!d1->band_circ || d1->band_n > NBC_MAX || (d2 && (!d2->band_circ || d2->band_n > NBC_MAX)))
        return set_err(TDS_ERR_UNSUPPORTED, "direction transport: reduced map not circulant");
    A.nbc1 = d1->band_n;
    A.q01 = d1->band_q0;
    for (int j = 0; j < d1->band_n; ++j) A.hc1[j] = d1->band_row[j];
    const tds_plan* e2 = d2 ? d2 : d1;
    A.nbc2 = e2->band_n;
    A.q02 = e2->band_q0;
    for (int j = 0; j < e2->band_n; ++j) A.hc2[j] = e2->band_row[j];
    if (getenv("TDS_DEBUG_BAND"))
        fprintf(stderr, "k_transport_dir: rows %d band %d / %d (q0 %d / %d)\n", a.rows, A.nbc1,
                A.nbc2, A.q01, A.q02);
    A.ydup = std::max(A.nbc1, A.nbc2);
    A.ydup += A.ydup & 1;
    if (A.ydup > 2 * a.chunks) return set_err(TDS_ERR_UNSUPPORTED, "direction transport: band > K");
    const int tl = transport_dir_tl(a, A.ydup, u, out);
    if (a.geom == GEOM_XY) {
        if (sz != 32 || ny % 32 || (tl != 16 && tl != 8) || nx % tl)
            return set_err(TDS_ERR_UNSUPPORTED, "xy transport: sz = 32, 32 | ny, tile | nx");
        if (tl == 16) return launch_transport_dir_t<16, GEOM_XY>(A, s);
        return launch_transport_dir_t<8, GEOM_XY>(A, s);
    }
    if (a.geom == GEOM_XZ) {
        if (ny % sz) return set_err(TDS_ERR_UNSUPPORTED, "xz transport: sz must divide ny");
        if (tl == 16) return launch_transport_dir_t<16, GEOM_XZ>(A, s);
        if (tl == 8) return launch_transport_dir_t<8, GEOM_XZ>(A, s);
        return set_err(TDS_ERR_UNSUPPORTED, "direction transport: shape not TMA-tileable");
    }
    if (tl == 16 && sz == 32) return launch_transport_dir_t<16, GEOM_LINES, 32>(A, s);
    if (tl == 8 && sz == 32) return launch_transport_dir_t<8, GEOM_LINES, 32>(A, s);
    if (tl == 16) return launch_transport_dir_t<16, GEOM_LINES>(A, s);
    if (tl == 8) return launch_transport_dir_t<8, GEOM_LINES>(A, s);
    return set_err(TDS_ERR_UNSUPPORTED, "direction transport: shape not TMA-tileable");
}

// ----------------------------------------------------------- re-layout

__device__ __forceinline__ long long fidx(int i, int j, int k, int nx, int ny, int nz, int sz,
                                          int lsz, int dir) {
    unsigned t, pos, n;
    if (dir == 0) { t = (unsigned)j + (unsigned)ny * (unsigned)k; pos = i; n = nx; }
    else if (dir == 1) { t = (unsigned)i + (unsigned)nx * (unsigned)k; pos = j; n = ny; }
    else { t = (unsigned)i + (unsigned)nx * (unsigned)j; pos = k; n = nz; }
    unsigned g, l;
    if (lsz >= 0) { g = t >> lsz; l = t & ((1u << lsz) - 1u); }
    else { g = t / (unsigned)sz; l = t - g * (unsigned)sz; }
    return ((long long)g * n + pos) * sz + l;
}

// (nx, ny, nz) field in `src_dir` layout -> `dst_dir` layout (dst = or +=).
// The fastest field axis is j for x layouts and i for y / z layouts, so a
// 32 x 32 (i, j) tile at fixed k serves every pair of directions. KB
// k-slices per block keep KB tiles of loads in flight per thread.
template <int KB>
__global__ void __launch_bounds__(256) k_reorder(const double* __restrict__ src,
                                                 double* __restrict__ dst, int nx, int ny,
                                                 int nz, int sz, int lsz, int src_dir,
                                                 int dst_dir, int accumulate) {
    __shared__ double tile[KB][32][33];               // [kk][jj][ii]
    const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32, k0 = blockIdx.z * KB;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const bool src_fast_i = src_dir != 0, dst_fast_i = dst_dir != 0;
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
        const int k = k0 + kk;
#pragma unroll
        for (int r = ty; r < 32; r += 8) {
            const int ii = src_fast_i ? tx : r, jj = src_fast_i ? r : tx;
            const int i = i0 + ii, j = j0 + jj;
            if (i < nx && j < ny && k < nz)
                tile[kk][jj][ii] = __ldcs(src + fidx(i, j, k, nx, ny, nz, sz, lsz, src_dir));
        }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
        const int k = k0 + kk;
#pragma unroll
        for (int r = ty; r < 32; r += 8) {
            const int ii = dst_fast_i ? tx : r, jj = dst_fast_i ? r : tx;
            const int i = i0 + ii, j = j0 + jj;
            if (i < nx && j < ny && k < nz) {
                double* o = dst + fidx(i, j, k, nx, ny, nz, sz, lsz, dst_dir);
                const double v = tile[kk][jj][ii];
                if (accumulate) *o = *o + v;
                else __stcs(o, v);
            }
        }
    }
}

int launch_reorder(const double* src, double* dst, int nx, int ny, int nz, int sz, int src_dir,
                   int dst_dir, int accumulate, cudaStream_t s) {
    int lsz = -1;
    if ((sz & (sz - 1)) == 0) {
        lsz = 0;
        while ((1 << lsz) < sz) ++lsz;
    }
    int kb = 1;   // measured: 2 / 4 k-slices per block are no faster
    if (const char* e = getenv("TDS_REORDER_KB")) kb = atoi(e);
    const dim3 blk(32, 8);
    if (kb == 4) {
        k_reorder<4><<<dim3((nx + 31) / 32, (ny + 31) / 32, (nz + 3) / 4), blk, 0, s>>>(
            src, dst, nx, ny, nz, sz, lsz, src_dir, dst_dir, accumulate);
    } else if (kb == 2) {
        k_reorder<2><<<dim3((nx + 31) / 32, (ny + 31) / 32, (nz + 1) / 2), blk, 0, s>>>(
            src, dst, nx, ny, nz, sz, lsz, src_dir, dst_dir, accumulate);
    } else {
        k_reorder<1><<<dim3((nx + 31) / 32, (ny + 31) / 32, nz), blk, 0, s>>>(
            src, dst, nx, ny, nz, sz, lsz, src_dir, dst_dir, accumulate);
    }
    return cuda_check(cudaGetLastError(), "k_reorder launch");
}

// out (=|+=) -1/2 (uj * du + dp) + nu * d2u   (rank-emulated transport path)
__global__ void k_transport_combine(const double* __restrict__ uj, const double* __restrict__ du,
                                    const double* __restrict__ dp, const double* __restrict__ d2u,
                                    double nu, double* __restrict__ out, long long count,
                                    int accumulate) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= count) return;
    double v = -0.5 * fma(uj[idx], du[idx], dp[idx]);
    if (d2u) v = fma(nu, d2u[idx], v);
    out[idx] = accumulate ? out[idx] + v : v;
}

// out = a + w * b (the Euler update of the transport demo) or, with
// w = NaN, out = a * b (the u_j u_i product of the 3-solve fallback path)
__global__ void k_axpy_mul(const double* __restrict__ a, const double* __restrict__ b, double w,
                           int mul, double* __restrict__ out, long long count) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    out[i] = mul ? a[i] * b[i] : fma(w, b[i], a[i]);
}

int launch_axpy_mul(const double* a, const double* b, double w, int mul, double* out,
                    long long count, cudaStream_t s) {
    if (count == 0) return TDS_OK;
    k_axpy_mul<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(a, b, w, mul, out, count);
    return cuda_check(cudaGetLastError(), "k_axpy_mul launch");
}

int launch_transport_combine(const double* uj, const double* du, const double* dp,
                             const double* d2u, double nu, double* out, long long count,
                             int accumulate, cudaStream_t s) {
    if (count == 0) return TDS_OK;
    k_transport_combine<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(uj, du, dp, d2u, nu, out,
                                                                       count, accumulate);
    return cuda_check(cudaGetLastError(), "k_transport_combine launch");
}

}  // namespace tds

namespace tds {

int transport_launch_from_plans(const tds_plan* d1, const tds_plan* d2, const double* ui,
                                const double* uj, double* out, double nu, int accumulate,
                                long long lines, int sz, cudaStream_t s, int geom, int nx, int ny,
                                int nz) {
    TransportArgs a;
    a.geom = geom;
    a.nx = nx;
    a.ny = ny;
    a.nz = nz;
    a.ui = ui;
    a.uj = uj;
    a.out = out;
    a.H1 = d1->d_Hp;
    a.H2 = d2 ? d2->d_Hp : d1->d_Hp;
    a.lines = lines;
    a.rows = d1->block_rows;
    a.sz = sz;
    a.chunks = d1->C;
    const int per_tile = d1->C * TL;
    a.tiles_per_cta = per_tile >= 256 ? 1 : 256 / per_tile;
    a.accumulate = accumulate;
    a.has_nu = d2 ? 1 : 0;
    a.nu = nu;
    a.t1 = d1->ut;
    a.t2 = d2 ? d2->ut : d1->ut;
    a.Hb1 = d1->d_Hb;
    a.Hb2 = d2 ? d2->d_Hb : d1->d_Hb;
    a.bq1 = d1->d_bq0;
    a.bq2 = d2 ? d2->d_bq0 : d1->d_bq0;
    a.nb1 = d1->band_n;
    a.nb2 = d2 ? d2->band_n : d1->band_n;
    if (d1->M == 16) {
        if (accumulate != (geom != GEOM_LINES))
            return set_err(TDS_ERR_UNSUPPORTED, "fused transport: lines layout writes, xz adds");
        return launch_transport_tma(a, s);
    }
    if (geom != GEOM_LINES) return set_err(TDS_ERR_UNSUPPORTED, "xz transport needs 16-row chunks");
    return launch_transport(a, s);
}

}  // namespace tds
