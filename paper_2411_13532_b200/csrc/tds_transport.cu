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

#include <cstdint>

#include "tds_device.cuh"

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
};

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
// 32 x 32 (i, j) tile at fixed k serves every pair of directions.
__global__ void k_reorder(const double* __restrict__ src, double* __restrict__ dst, int nx,
                          int ny, int nz, int sz, int lsz, int src_dir, int dst_dir,
                          int accumulate) {
    __shared__ double tile[32][33];                   // [jj][ii]
    const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32, k = blockIdx.z;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const bool src_fast_i = src_dir != 0, dst_fast_i = dst_dir != 0;
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
        const int ii = src_fast_i ? tx : r, jj = src_fast_i ? r : tx;
        const int i = i0 + ii, j = j0 + jj;
        if (i < nx && j < ny)
            tile[jj][ii] = __ldcs(src + fidx(i, j, k, nx, ny, nz, sz, lsz, src_dir));
    }
    __syncthreads();
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
        const int ii = dst_fast_i ? tx : r, jj = dst_fast_i ? r : tx;
        const int i = i0 + ii, j = j0 + jj;
        if (i < nx && j < ny) {
            double* o = dst + fidx(i, j, k, nx, ny, nz, sz, lsz, dst_dir);
            const double v = tile[jj][ii];
            if (accumulate) *o = *o + v;
            else __stcs(o, v);
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
    dim3 grid((nx + 31) / 32, (ny + 31) / 32, nz);
    k_reorder<<<grid, dim3(32, 8), 0, s>>>(src, dst, nx, ny, nz, sz, lsz, src_dir, dst_dir,
                                           accumulate);
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
                                long long lines, int sz, cudaStream_t s) {
    TransportArgs a;
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
    return launch_transport(a, s);
}

}  // namespace tds
