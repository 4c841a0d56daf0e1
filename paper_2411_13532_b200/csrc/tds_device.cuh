// Device-side building blocks shared by the fast kernels (k_tma, k_dd):
// PTX wrappers (mbarrier, TMA, sys-scope acquire/release) and the per-chunk
// arithmetic of the fused DistD2 solve.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "tds_internal.h"

namespace tds {
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar))
        : "memory");
}
// bulk async copy shared -> global (TMA engine, no tensor map): `bytes` a
// multiple of 16, both addresses 16-byte aligned; tracked per issuing thread
// in bulk groups
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// wait until at most N of this thread's bulk groups still read shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// TMA reduce-add of a shared-memory box into global memory (the box and
// layout of the tensor map; fp64 add is done in L2), tracked in bulk groups
__device__ __forceinline__ void tma_reduce_add_4d(const CUtensorMap* map, const void* src, int c0,
                                                  int c1, int c2, int c3) {
    asm volatile(
        "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group"
        " [%0, {%2, %3, %4, %5}], [%1];" ::"l"(reinterpret_cast<uint64_t>(map)),
        "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
// L2 prefetch of `bytes` (multiple of 16, 16-byte aligned) by the TMA engine
__device__ __forceinline__ void bulk_prefetch_l2(const void* gsrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gsrc), "r"(bytes) : "memory");
}
// system-scope flag protocol for NVLink peer memory
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ long long line_base(long long line, int rows, int sz) {
    return (line / sz) * (long long)rows * sz + (line % sz);
}
__device__ __forceinline__ long long halo_base(long long line, int sz) {
    return (line / sz) * 2LL * sz + (line % sz);
}
// compile-time lane width (SZC = 32, the benchmark layout) or runtime (0):
// with SZC the line decomposition is shifts and every row address of a
// line is an immediate offset from one base pointer
template <int SZC>
__device__ __forceinline__ long long line_base_t(long long line, int rows, int sz) {
    if (SZC) return (line / SZC) * (long long)rows * SZC + (line % SZC);
    return line_base(line, rows, sz);
}
template <int SZC>
__device__ __forceinline__ long long halo_base_t(long long line, int sz) {
    if (SZC) return (line / SZC) * 2LL * SZC + (line % SZC);
    return halo_base(line, sz);
}

// Window value v[i + o + s] of chunk row i for a stencil window shifted by s
// (one-sided closures; plan.cpp check_shift): s in 1..2 only on rows 0, 1 of
// a line start, s in -2..-1 only on its last two rows. i and o are
// compile-time after unrolling, so every candidate is a register.
template <int M>
__device__ __forceinline__ double wv(const double (&v)[M + 4], int i, int o, int s) {
    if (i < 2) return s == 2 ? v[i + o + 2] : (s == 1 ? v[i + o + 1] : v[i + o]);
    if (i >= M - 2) return s == -2 ? v[i + o - 2] : (s == -1 ? v[i + o - 1] : v[i + o]);
    return v[i + o];
}

// shifts of chunk rows 0, 1, M-2, M-1 (non-zero only in the block's first /
// last chunk). Plain scalars picked by the compile-time row index (a struct
// with an accessor was demoted to local memory: an LDL at the head of the
// edge warps' sweep chain, -11% for the whole kernel).
struct RowShift {
    int f0, f1, b0, b1;
};
#define TDS_ROW_SHIFT(rs, i, M) \
    ((i) == 0 ? (rs).f0 : ((i) == 1 ? (rs).f1 : ((i) == (M) - 2 ? (rs).b0 : ((i) == (M) - 1 ? (rs).b1 : 0))))

// Fused width-5 stencil + Alg. 6 (reference distributed.py:257-276) on one
// chunk of M rows held in registers: v = rows r0-2 .. r0+M+1, d = decoupled.
template <int M, bool UNIFORM, bool SHIFT = false>
__device__ __forceinline__ void chunk_sweeps(const FastArgs& p, const double* __restrict__ tb,
                                             const double (&v)[M + 4], double (&d)[M],
                                             RowShift rs = RowShift{0, 0, 0, 0}) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double s0, s1, s2, s3, s4, f, r;
        if (UNIFORM) {
            s0 = p.ut.st[0]; s1 = p.ut.st[1]; s2 = p.ut.st[2]; s3 = p.ut.st[3]; s4 = p.ut.st[4];
            f = p.ut.f[i]; r = p.ut.r[i];
        } else {
            // tb: the per-row table in global or (k_tma) shared memory. The
            // empty asm ties row i's loads to d[i - 2]: without it the
            // compiler issues all 32 rows' loads up front and spills.
            const double* tr = tb + i * NCOEF;
            if (i >= 2) asm volatile("" : "+l"(tr) : "d"(d[i - 2]));
            const double2 c01 = *reinterpret_cast<const double2*>(tr);
            const double2 c23 = *reinterpret_cast<const double2*>(tr + 2);
            const double2 c4f = *reinterpret_cast<const double2*>(tr + 4);
            s0 = c01.x; s1 = c01.y; s2 = c23.x; s3 = c23.y; s4 = c4f.x; f = c4f.y;
            r = tr[6];
        }
        const int sh = SHIFT ? TDS_ROW_SHIFT(rs, i, M) : 0;
        double rhs = s0 * wv<M>(v, i, 0, sh);
        rhs = fma(s1, wv<M>(v, i, 1, sh), rhs);
        rhs = fma(s2, wv<M>(v, i, 2, sh), rhs);
        rhs = fma(s3, wv<M>(v, i, 3, sh), rhs);
        rhs = fma(s4, wv<M>(v, i, 4, sh), rhs);
        if (i < 2) d[i] = rhs * r;
        else d[i] = fma(-r, d[i - 1], rhs) * f;
    }
#pragma unroll
    for (int i = M - 3; i >= 1; --i) {
        double w;
        if (UNIFORM) {
            w = p.ut.w[i];
        } else {
            const double* tr = tb + i * NCOEF + 7;
            if (i + 3 < M) asm volatile("" : "+l"(tr) : "d"(d[i + 3]));
            w = *tr;
        }
        d[i] = fma(-w, d[i + 1], d[i]);
    }
    const double w0 = UNIFORM ? p.ut.w[0] : tb[7];
    const double f0 = UNIFORM ? p.ut.f[0] : tb[5];
    d[0] = fma(-w0, d[1], d[0]) * f0;
}

// Chunk boundary values (F, L) = rows 2k, 2k+1 of H applied to the reduced
// rhs Y (K entries, stride TLT in shared memory). If pins are given, Y[0] and
// Y[K-1] are replaced by pin0 / pin1 (the rank's u_start / u_end).
template <int TLT>
__device__ __forceinline__ void chunk_bounds(const double2* __restrict__ hr, const double* Y,
                                             int K, int lane, const double* pin0,
                                             const double* pin1, double& F, double& L) {
    double F0 = 0.0, F1 = 0.0, L0 = 0.0, L1 = 0.0;
    int q0 = 0, q1 = K;
    if (pin0) {
        const double2 h = __ldg(hr);
        const double2 hl = __ldg(hr + K - 1);
        const double a = pin0[lane], b = pin1[lane];
        F0 = fma(h.x, a, 0.0);
        L0 = fma(h.y, a, 0.0);
        F1 = fma(hl.x, b, 0.0);
        L1 = fma(hl.y, b, 0.0);
        q0 = 1;
        q1 = K - 1;
    }
    int q = q0;
    for (; q + 1 < q1; q += 2) {
        const double2 h0 = __ldg(hr + q);
        const double2 h1 = __ldg(hr + q + 1);
        const double ya = Y[q * TLT + lane];
        const double yb = Y[(q + 1) * TLT + lane];
        F0 = fma(h0.x, ya, F0);
        L0 = fma(h0.y, ya, L0);
        F1 = fma(h1.x, yb, F1);
        L1 = fma(h1.y, yb, L1);
    }
    if (q < q1) {
        const double2 h0 = __ldg(hr + q);
        const double ya = Y[q * TLT + lane];
        F0 = fma(h0.x, ya, F0);
        L0 = fma(h0.y, ya, L0);
    }
    F = F0 + F1;
    L = L0 + L1;
}

// (F, L) of a chunk from the banded reduced map: nb columns starting at q0
// (cyclic), Y in shared memory with stride TLT
template <int TLT>
__device__ __forceinline__ void band_bounds(const double2* __restrict__ hb, int q0, int nb,
                                            const double* Y, int K, int lane, double& F,
                                            double& L) {
    double F0 = 0.0, F1 = 0.0, L0 = 0.0, L1 = 0.0;
    int q = q0, j = 0;
    for (; j + 1 < nb; j += 2) {
        const double2 h0 = __ldg(hb + j), h1 = __ldg(hb + j + 1);
        const int qb = q + 1 == K ? 0 : q + 1;
        const double ya = Y[q * TLT + lane], yb = Y[qb * TLT + lane];
        F0 = fma(h0.x, ya, F0);
        L0 = fma(h0.y, ya, L0);
        F1 = fma(h1.x, yb, F1);
        L1 = fma(h1.y, yb, L1);
        q = qb + 1 == K ? 0 : qb + 1;
    }
    if (j < nb) {
        const double2 h0 = __ldg(hb + j);
        const double ya = Y[q * TLT + lane];
        F0 = fma(h0.x, ya, F0);
        L0 = fma(h0.y, ya, L0);
    }
    F = F0 + F1;
    L = L0 + L1;
}

// The same with the rank pins' columns (q = 0 and q = K-1 of a per-rank map)
// left out: they are applied separately once u_start / u_end are known.
template <int TLT>
__device__ __forceinline__ void band_bounds_nopins(const double2* __restrict__ hb, int q0, int nb,
                                                   const double* Y, int K, int lane, double& F,
                                                   double& L) {
    double F0 = 0.0, F1 = 0.0, L0 = 0.0, L1 = 0.0;
    int q = q0, j = 0;
    for (; j + 1 < nb; j += 2) {
        const double2 h0 = __ldg(hb + j), h1 = __ldg(hb + j + 1);
        const int qb = q + 1 == K ? 0 : q + 1;
        const double ya = (q == 0 || q == K - 1) ? 0.0 : Y[q * TLT + lane];
        const double yb = (qb == 0 || qb == K - 1) ? 0.0 : Y[qb * TLT + lane];
        F0 = fma(h0.x, ya, F0);
        L0 = fma(h0.y, ya, L0);
        F1 = fma(h1.x, yb, F1);
        L1 = fma(h1.y, yb, L1);
        q = qb + 1 == K ? 0 : qb + 1;
    }
    if (j < nb) {
        const double2 h0 = __ldg(hb + j);
        const double ya = (q == 0 || q == K - 1) ? 0.0 : Y[q * TLT + lane];
        F0 = fma(h0.x, ya, F0);
        L0 = fma(h0.y, ya, L0);
    }
    F = F0 + F1;
    L = L0 + L1;
}

// The rank's Alg. 6 boundary row r (0: d[0] = g0 . Y, 1: d[m-1] = g1 . Y)
// over its significant terms only (plan.cpp upload_H: g_n0 leading / g_n1
// trailing entries above 2^-70 of the largest).
template <int TLT>
__device__ __forceinline__ double gdot(const FastArgs& p, int r, const double* Y, int K,
                                       int lane) {
    const double* g = p.g + r * K;
    const int q0 = r == 0 ? 0 : K - p.g_n1, q1 = r == 0 ? p.g_n0 : K;
    double a = 0.0, b = 0.0;
    int q = q0;
    for (; q + 1 < q1; q += 2) {
        a = fma(__ldg(g + q), Y[q * TLT + lane], a);
        b = fma(__ldg(g + q + 1), Y[(q + 1) * TLT + lane], b);
    }
    if (q < q1) a = fma(__ldg(g + q), Y[q * TLT + lane], a);
    return a + b;
}

// Alg. 7 at chunk level + one streaming store per row.
template <int M, bool UNIFORM>
__device__ __forceinline__ void chunk_store(const FastArgs& p, const double* __restrict__ tb,
                                            double* __restrict__ ob, long long sz, int r0,
                                            const double (&d)[M], double F, double L,
                                            bool stream) {
    if (stream) {
        __stcs(ob + (long long)r0 * sz, F);
#pragma unroll
        for (int i = 1; i < M - 1; ++i) {
            const double sa = UNIFORM ? p.ut.sa[i] : tb[i * NCOEF + 8];
            const double sc = UNIFORM ? p.ut.sc[i] : tb[i * NCOEF + 9];
            __stcs(ob + (long long)(r0 + i) * sz, fma(-sc, L, fma(-sa, F, d[i])));
        }
        __stcs(ob + (long long)(r0 + M - 1) * sz, L);
    } else {
        ob[(long long)r0 * sz] = F;
#pragma unroll
        for (int i = 1; i < M - 1; ++i) {
            const double sa = UNIFORM ? p.ut.sa[i] : tb[i * NCOEF + 8];
            const double sc = UNIFORM ? p.ut.sc[i] : tb[i * NCOEF + 9];
            ob[(long long)(r0 + i) * sz] = fma(-sc, L, fma(-sa, F, d[i]));
        }
        ob[(long long)(r0 + M - 1) * sz] = L;
    }
}

// Sweeps / store of a special (edge) chunk of a uniform plan: per-row
// coefficients from an EdgeTable in kernel-parameter space, so they stay
// constant-bank operands like the uniform table (no global loads to hoist).
// Sweeps of a special (edge) chunk of a uniform plan: per-row coefficients
// from an EdgeTable in kernel-parameter space (constant-bank operands, no
// loads to hoist). Rows 0, 1, M-2, M-1 use the table's 7-tap rows, which
// carry any window shift (one-sided closures) as plain coefficients.
template <int M>
__device__ __forceinline__ void edge_sweeps(const EdgeTable& T, const double (&v)[M + 4],
                                            double (&d)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const double* c = T.c[i];
        double rhs;
        if (i < 2 || i >= M - 2) {
            const int q = i < 2 ? i : i - (M - 4);      // 0, 1 | 2, 3
            const int b = i < 2 ? i : i - 2;            // first window row
            const double* x = T.x7[q];
            rhs = x[0] * v[b];
#pragma unroll
            for (int j = 1; j < 7; ++j) rhs = fma(x[j], v[b + j], rhs);
        } else {
            rhs = c[0] * v[i];
            rhs = fma(c[1], v[i + 1], rhs);
            rhs = fma(c[2], v[i + 2], rhs);
            rhs = fma(c[3], v[i + 3], rhs);
            rhs = fma(c[4], v[i + 4], rhs);
        }
        if (i < 2) d[i] = rhs * c[6];
        else d[i] = fma(-c[6], d[i - 1], rhs) * c[5];
    }
#pragma unroll
    for (int i = M - 3; i >= 1; --i) d[i] = fma(-T.c[i][7], d[i + 1], d[i]);
    d[0] = fma(-T.c[0][7], d[1], d[0]) * T.c[0][5];
}

template <int M>
__device__ __forceinline__ void edge_store(const EdgeTable& T, double* __restrict__ ob,
                                           long long sz, int r0, const double (&d)[M], double F,
                                           double L, bool stream) {
    if (stream) {
        __stcs(ob + (long long)r0 * sz, F);
#pragma unroll
        for (int i = 1; i < M - 1; ++i)
            __stcs(ob + (long long)(r0 + i) * sz, fma(-T.c[i][9], L, fma(-T.c[i][8], F, d[i])));
        __stcs(ob + (long long)(r0 + M - 1) * sz, L);
    } else {
        ob[(long long)r0 * sz] = F;
#pragma unroll
        for (int i = 1; i < M - 1; ++i)
            ob[(long long)(r0 + i) * sz] = fma(-T.c[i][9], L, fma(-T.c[i][8], F, d[i]));
        ob[(long long)(r0 + M - 1) * sz] = L;
    }
}

// Chunk sweeps of a (possibly edge-special) chunk. Measured at 512^3: a
// select-based shifted window on the edge warps (the barrier-critical path
// of every item) cost open d2/dx2 ~11%; the 7-tap edge rows cost nothing.
template <int M, int TAB>
__device__ __forceinline__ void chunk_sweeps_any(const FastArgs& p, const double* __restrict__ tb,
                                                 const double (&v)[M + 4], double (&d)[M],
                                                 int chunk) {
    // only the block's first / last chunk can hold shifted rows; the plan
    // (plan.cpp fast_tables) keeps them out of TAB_UNIFORM tables and inside
    // the special chunks of TAB_EDGES ones, so only TAB_GLOBAL needs the
    // select-based copy
    if constexpr (TAB == TAB_GLOBAL) {
        if (p.has_shift && (chunk == 0 || chunk == p.chunks - 1)) {
            RowShift rs{0, 0, 0, 0};
            if (chunk == 0) {
                rs.f0 = p.sh[0];
                rs.f1 = p.sh[1];
            }
            if (chunk == p.chunks - 1) {
                rs.b0 = p.sh[2];
                rs.b1 = p.sh[3];
            }
            chunk_sweeps<M, false, true>(p, tb, v, d, rs);
            return;
        }
    }
    // TAB_EDGES: the special (edge) chunks carry their shifts in the 7-tap
    // rows of their EdgeTable; other chunks with shifted rows (uncommon
    // table layouts) take the select-based copy
    if (TAB == TAB_EDGES && p.special_first && chunk == 0)
        edge_sweeps<M>(p.e_first, v, d);
    else if (TAB == TAB_EDGES && p.special_last && chunk == p.chunks - 1)
        edge_sweeps<M>(p.e_last, v, d);
    else chunk_sweeps<M, TAB != TAB_GLOBAL, false>(p, tb, v, d);
}

template <int M, int TAB>
__device__ __forceinline__ void chunk_store_any(const FastArgs& p, const double* __restrict__ tb,
                                                double* __restrict__ ob, long long sz, int r0,
                                                const double (&d)[M], double F, double L,
                                                bool stream, int chunk) {
    if (TAB == TAB_EDGES && p.special_first && chunk == 0)
        edge_store<M>(p.e_first, ob, sz, r0, d, F, L, stream);
    else if (TAB == TAB_EDGES && p.special_last && chunk == p.chunks - 1)
        edge_store<M>(p.e_last, ob, sz, r0, d, F, L, stream);
    else chunk_store<M, TAB != TAB_GLOBAL>(p, tb, ob, sz, r0, d, F, L, stream);
}


// per-row coefficients of the d/dx (1) and d2/dx2 (2) chunk tables
struct DirRow {
    double2 rf1, rf2;         // (r, f)
    double2 w12;              // (w1, w2)
    double2 s1, s2;           // (sa, sc)
};

// two solves of one window (tables 1 and 2) / one solve (table 1), the
// arithmetic of sweeps2_src / sweeps_src with the DirRow table
template <int M, typename Src>
__device__ __forceinline__ void dsweeps2(const DirRow (&R)[16], const double* st1,
                                         const double* st2, Src v, double (&d1)[M],
                                         double (&d2)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const double v0 = v(i), v1 = v(i + 1), v2 = v(i + 2), v3 = v(i + 3), v4 = v(i + 4);
        double a = st1[0] * v0, b = st2[0] * v0;
        a = fma(st1[1], v1, a);
        b = fma(st2[1], v1, b);
        a = fma(st1[2], v2, a);
        b = fma(st2[2], v2, b);
        a = fma(st1[3], v3, a);
        b = fma(st2[3], v3, b);
        a = fma(st1[4], v4, a);
        b = fma(st2[4], v4, b);
        const double2 rf1 = R[i].rf1, rf2 = R[i].rf2;
        if (i < 2) {
            d1[i] = a * rf1.x;
            d2[i] = b * rf2.x;
        } else {
            d1[i] = fma(-rf1.x, d1[i - 1], a) * rf1.y;
            d2[i] = fma(-rf2.x, d2[i - 1], b) * rf2.y;
        }
    }
#pragma unroll
    for (int i = M - 3; i >= 1; --i) {
        const double2 w = R[i].w12;
        d1[i] = fma(-w.x, d1[i + 1], d1[i]);
        d2[i] = fma(-w.y, d2[i + 1], d2[i]);
    }
    const double2 w = R[0].w12;
    d1[0] = fma(-w.x, d1[1], d1[0]) * R[0].rf1.y;
    d2[0] = fma(-w.y, d2[1], d2[0]) * R[0].rf2.y;
}

template <int M, typename Src>
__device__ __forceinline__ void dsweeps1(const DirRow (&R)[16], const double* st, Src v,
                                         double (&d)[M]) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        double rhs = st[0] * v(i);
        rhs = fma(st[1], v(i + 1), rhs);
        rhs = fma(st[2], v(i + 2), rhs);
        rhs = fma(st[3], v(i + 3), rhs);
        rhs = fma(st[4], v(i + 4), rhs);
        const double2 rf = R[i].rf1;
        if (i < 2) d[i] = rhs * rf.x;
        else d[i] = fma(-rf.x, d[i - 1], rhs) * rf.y;
    }
#pragma unroll
    for (int i = M - 3; i >= 1; --i) d[i] = fma(-R[i].w12.x, d[i + 1], d[i]);
    d[0] = fma(-R[0].w12.x, d[1], d[0]) * R[0].rf1.y;
}

__device__ __forceinline__ double subst2(double2 s, int i, int M, double F, double L, double di) {
    return i == 0 ? F : (i == M - 1 ? L : fma(-s.y, L, fma(-s.x, F, di)));
}

}  // namespace dev
}  // namespace tds
