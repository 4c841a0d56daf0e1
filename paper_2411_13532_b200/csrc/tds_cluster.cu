// Long lines (more chunks than one CTA holds) on the 16 B/point path:
// k_tmc splits each line across the Q CTAs of a THREAD-BLOCK CLUSTER.
//
// A work item is TLT lines. CTA q of the cluster owns rows [q R, (q+1) R) of
// them (R = rows / Q, Cl = R / M chunks): its rows arrive by TMA exactly as in
// k_tma, every thread runs the fused stencil + Alg. 6 sweeps of its chunk in
// registers and writes the chunk's reduced rhs (d[0], d[M-1]) to shared
// memory. One cluster barrier later every CTA reads the reduced rhs entries
// its chunks' rows of the banded reduced map H need -- most are its own, the
// ones near its row-range ends live in the neighbouring CTAs and are read
// through DISTRIBUTED SHARED MEMORY (ld.shared::cluster) -- and finishes the
// substitution and the single store. HBM traffic stays the compulsory 8 B read
// + 8 B write per point; the only extra reads are the 2-row stencil halos at
// the CTA row-range ends (L2 hits: the neighbour CTA loads those rows).
//
// Reference semantics: the whole-line operator of run_distd2
// (distributed.py:380-449) -- P=1 (periodic) Thomas or the rank-truncated
// DistD2, both folded into H by the plan (plan.cpp) as for k_tma.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "tds_device.cuh"
#include "tds_tma.h"

namespace tds {

using namespace dev;

namespace {

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared variable in CTA `rank`
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ double ld_cluster(uint32_t addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ long long ld_cluster_s64(uint32_t addr) {
    long long v;
    asm volatile("ld.shared::cluster.s64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
    return v;
}

struct TmcArgs {
    TmaArgs t;
    int Q;          // CTAs per cluster (line split)
    int R;          // rows per CTA
    int Cl;         // chunks per CTA
};

}  // namespace

template <int M, int TAB, int TLT, int SZC>
__global__ void __launch_bounds__(512, 1) k_tmc(const __grid_constant__ TmcArgs A) {
    const FastArgs& p = A.t.f;
    extern __shared__ __align__(1024) unsigned char smem[];
    const int Q = A.Q, R = A.R, Cl = A.Cl;
    const int C = p.chunks;                 // chunks of the whole line
    const int K = 2 * C;
    const int rows = p.rows;
    const uint32_t q = cluster_rank();
    const int t = threadIdx.x;
    const int lane = t % TLT;
    const int lchunk = t / TLT;             // chunk within this CTA
    const int chunk = (int)q * Cl + lchunk; // chunk of the line
    const long long sz = SZC ? SZC : p.sz;
    const int r0 = chunk * M;               // first row (line coordinates)
    const int lr0 = lchunk * M;             // first row (tile coordinates)
    double* tile = reinterpret_cast<double*>(smem);
    const size_t tile_elems = (size_t)R * TLT;
    double* sY = tile + tile_elems;         // [2][2 Cl][TLT]
    const size_t ybuf = (size_t)2 * Cl * TLT;
    // TAB_GLOBAL: this CTA's rows of the per-row table, staged once
    double* stab = sY + 2 * ybuf;
    uint64_t* bar = reinterpret_cast<uint64_t*>(stab + (TAB == TAB_GLOBAL ? (size_t)R * NCOEF : 0));
    if (TAB == TAB_GLOBAL)
        for (int k = t; k < R * NCOEF; k += blockDim.x)
            stab[k] = __ldg(p.tab + (size_t)q * R * NCOEF + k);
    const double* __restrict__ tb =
        TAB == TAB_GLOBAL ? stab + (size_t)lr0 * NCOEF : p.tab + (size_t)r0 * NCOEF;
    const long long nclusters = gridDim.x / Q;

    auto issue = [&](long long item) {
        mbar_expect_tx(bar, (uint32_t)(tile_elems * sizeof(double)));
        const long long first = item * TLT;
        const int g = (int)(first / p.sz), l0 = (int)(first % p.sz);
        for (int b = 0; b * A.t.boxr < R; ++b)
            tma_load_3d(tile + (size_t)b * A.t.boxr * TLT, &A.t.map, bar, l0,
                        (int)q * R + b * A.t.boxr, g);
    };

    // item schedule: round-robin over the clusters, or (p.ctr) handed out in
    // order of request by the cluster's CTA 0, which claims two items ahead
    // into s_q[k % 3] (the cluster's k-th item); the other CTAs read it
    // through distributed shared memory after the iteration's cluster
    // barrier, so every CTA of a cluster loads the same item
    __shared__ long long s_q[3];
    const bool leader = q == 0;
    const uint32_t q_addr = map_rank(smem_u32(s_q), 0);
    auto claim = [&](long long prev) -> long long {
        return p.ctr ? (long long)nclusters + (long long)atomicAdd(p.ctr, 1ULL) : prev + nclusters;
    };
    if (t == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        if (leader) s_q[1] = claim(blockIdx.x / Q);
    }
    __syncthreads();
    cluster_sync();
    long long item = blockIdx.x / Q;
    if (t == 0 && item < p.items) issue(item);
    uint32_t phase = 0;

    for (int it = 0; item < p.items; ++it) {
        const long long nxt = ld_cluster_s64(q_addr + 8 * ((it + 1) % 3));
        const long long line = item * TLT + lane;
        const bool valid = line < p.lines;
        const long long lb = valid ? line_base_t<SZC>(line, rows, p.sz) : 0;
        // stencil halos at this CTA's row-range ends: the neighbour CTA's
        // rows (or the periodic wrap / open zeros at the line ends), from
        // global memory -- loads in flight across the TMA wait
        double h0 = 0.0, h1 = 0.0, h2 = 0.0, h3 = 0.0;
        if (valid && lchunk == 0) {
            const int ra = r0 - 2;
            if (ra >= 0) {
                h0 = __ldg(p.u + lb + (long long)ra * sz);
                h1 = __ldg(p.u + lb + (long long)(ra + 1) * sz);
            } else if (p.edge_mode == EDGE_WRAP) {
                h0 = __ldg(p.u + lb + (long long)(rows - 2) * sz);
                h1 = __ldg(p.u + lb + (long long)(rows - 1) * sz);
            }
        }
        if (valid && lchunk == Cl - 1) {
            const int rb = r0 + M;
            if (rb < rows) {
                h2 = __ldg(p.u + lb + (long long)rb * sz);
                h3 = __ldg(p.u + lb + (long long)(rb + 1) * sz);
            } else if (p.edge_mode == EDGE_WRAP) {
                h2 = __ldg(p.u + lb);
                h3 = __ldg(p.u + lb + sz);
            }
        }
        while (!mbar_try_wait(bar, phase)) {
        }
        phase ^= 1u;
        double v[M + 4];
#pragma unroll
        for (int i = 0; i < M + 4; ++i) {
            double x;
            if (i < 2) x = lchunk == 0 ? (i == 0 ? h0 : h1) : tile[(lr0 - 2 + i) * TLT + lane];
            else if (i >= M + 2)
                x = lchunk == Cl - 1 ? (i == M + 2 ? h2 : h3) : tile[(lr0 - 2 + i) * TLT + lane];
            else x = tile[(lr0 - 2 + i) * TLT + lane];
            v[i] = x;
        }
        __syncthreads();   // tile consumed: prefetch the next item
        if (t == 0) {
            if (nxt < p.items) {
                fence_proxy_async();
                issue(nxt);
            }
            // the item after next, visible to the cluster after its barrier
            if (leader) s_q[(it + 2) % 3] = nxt >= p.items ? p.items : claim(nxt);
        }

        double d[M];
        chunk_sweeps_any<M, TAB>(p, tb, v, d, chunk);
        double* Y = sY + (it & 1) * ybuf;
        Y[(2 * lchunk) * TLT + lane] = d[0];
        Y[(2 * lchunk + 1) * TLT + lane] = d[M - 1];
        // the reduced rhs of the whole line is now spread over the cluster;
        // double-buffered by iteration, so one barrier per item suffices
        // (a CTA re-writes this buffer only after the NEXT barrier, which
        // every reader passes after its reads). (Measured: splitting it into
        // arrive / own-columns / wait / remote-columns is 3% slower.)
        cluster_sync();

        // banded reduced map: nb columns starting at bq0 (cyclic over K);
        // column c = 2 k + e lives in CTA k / Cl
        const double2* __restrict__ hb = p.Hb + (size_t)chunk * p.nb;
        const uint32_t ybase = smem_u32(Y) + lane * 8;
        double F0 = 0.0, F1 = 0.0, L0 = 0.0, L1 = 0.0;
        int c = __ldg(p.bq0 + chunk);
        for (int j = 0; j < p.nb; ++j) {
            const int k = c >> 1;
            const uint32_t owner = (uint32_t)(k / Cl);
            const int lc = c - 2 * (int)owner * Cl;
            const double y = ld_cluster(map_rank(ybase + (uint32_t)(lc * TLT * 8), owner));
            const double2 h = __ldg(hb + j);
            if (j & 1) {
                F1 = fma(h.x, y, F1);
                L1 = fma(h.y, y, L1);
            } else {
                F0 = fma(h.x, y, F0);
                L0 = fma(h.y, y, L0);
            }
            c = c + 1 == K ? 0 : c + 1;
        }
        if (valid)
            chunk_store_any<M, TAB>(p, tb, p.out + lb, sz, r0, d, F0 + F1, L0 + L1,
                                    A.t.store_cs != 0, chunk);
        item = nxt;
    }
    cluster_sync();   // no CTA leaves while a neighbour may still read its Y / s_q
    if (p.ctr && t == 0) {
        // the last CTA out resets the counter slot for its next launch
        __threadfence();
        if (atomicAdd(p.ctr + 1, 1ULL) == gridDim.x - 1) {
            p.ctr[0] = 0;
            p.ctr[1] = 0;
            __threadfence();
        }
    }
}

namespace {

template <int M, int TAB, int TLT, int SZC>
int launch_tmc_t(const FastArgs& a, int Q, cudaStream_t s) {
    TmcArgs A;
    std::memset(&A, 0, sizeof(A));
    A.t.f = a;
    // dynamic item schedule only for 2-CTA clusters: measured n = 2048 4773 ->
    // 5119 GB/s; with 4 / 8 CTAs the DSMEM read per item cost what the
    // balance gained (4602 -> 4606, 4065 -> 4003)
    if (Q > 2) A.t.f.ctr = nullptr;
    A.Q = Q;
    A.R = a.rows / Q;
    A.Cl = a.chunks / Q;
    A.t.f.tiles_per_cta = 1;
    A.t.f.items = (a.lines + TLT - 1) / TLT;
    if (A.t.f.items <= 0) return TDS_OK;
    A.t.store_cs = store_policy();
    // the tensor map's boxes tile one CTA's row range (rows / Q, chunk-aligned)
    int rc;
    A.t.boxr = box_rows(A.R, M);
    if (A.t.boxr == 0) return set_err(TDS_ERR_UNSUPPORTED, "cluster rows not boxable");
    {
        const long long groups = a.lines / a.sz;
        cuuint64_t dims[3] = {(cuuint64_t)a.sz, (cuuint64_t)a.rows, (cuuint64_t)groups};
        cuuint64_t strides[2] = {(cuuint64_t)a.sz * 8, (cuuint64_t)a.rows * a.sz * 8};
        cuuint32_t box[3] = {(cuuint32_t)TLT, (cuuint32_t)A.t.boxr, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult cr = encode_fn()(&A.t.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                                  const_cast<double*>(a.u), dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  TLT >= 16 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                            : CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return set_err(TDS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    }
    const int threads = A.Cl * TLT;
    const size_t smem = (size_t)A.R * TLT * 8 + (size_t)2 * 2 * A.Cl * TLT * 8 +
                         (TAB == TAB_GLOBAL ? (size_t)A.R * NCOEF * 8 : 0) + 16;
    const void* fn = reinterpret_cast<const void*>(k_tmc<M, TAB, TLT, SZC>);
    if ((rc = ensure_smem(fn, smem, "cudaFuncSetAttribute(k_tmc)"))) return rc;
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = Q;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (Q > 8 &&
        (rc = cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                         "cudaFuncSetAttribute(k_tmc, non-portable cluster)")))
        return rc;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.gridDim = dim3(Q);
    int clusters = 0;
    rc = cuda_check(cudaOccupancyMaxActiveClusters(&clusters, fn, &cfg),
                    "cudaOccupancyMaxActiveClusters(k_tmc)");
    if (rc) return rc;
    if (clusters < 1) return set_err(TDS_ERR_UNSUPPORTED, "k_tmc cluster does not fit");
    long long nc = clusters;
    if (nc > A.t.f.items) nc = A.t.f.items;
    cfg.gridDim = dim3((unsigned)(nc * Q));
    rc = cuda_check(cudaLaunchKernelEx(&cfg, k_tmc<M, TAB, TLT, SZC>, A), "k_tmc launch");
    return rc;
}

// cluster shape for a line of `chunks` chunks: (lines per tile, CTAs per
// cluster), 0 if none fits (<= 8 CTAs, <= 512 threads, <= ~200 KB smem)
void tmc_shape(const FastArgs& a, int M, bool table, int* tl, int* q) {
    // candidates: TLT lines per tile (32 needs the sz = 32 compile-time
    // width), Q CTAs per cluster (<= 16; > 8 is the non-portable size),
    // Cl = chunks / Q >= 2 chunks and <= 512 threads per CTA. Default: 16-line
    // tiles (then 32, 8) and the SMALLEST cluster that fits, i.e. the longest
    // row range per CTA -- measured at n = 2048 / 4096 / 8192: 16-line tiles
    // of 1024 rows (Q = 2 / 4 / 8) 4858 / 4720 / 4200 GB/s; 32-line tiles of
    // 512 rows 4695 / 4191 / 3897 (Q = 8 / 8 / 16); 16-line tiles of 512 rows
    // 4815 / 4480 / 3822; 8-line tiles <= 4636. Knobs: TDS_TMC_TL, TDS_TMC_Q.
    int want_tl = 0, want_q = 0;
    if (const char* e = getenv("TDS_TMC_TL")) want_tl = atoi(e);
    if (const char* e = getenv("TDS_TMC_Q")) want_q = atoi(e);
    size_t best = ~(size_t)0;
    *tl = 0;
    *q = 0;
    for (int TLT : {32, 16, 8}) {
        if (a.sz % TLT || (TLT == 32 && a.sz != 32)) continue;
        if (want_tl && TLT != want_tl) continue;
        for (int Q = 2; Q <= 16; Q *= 2) {
            if (want_q && Q != want_q) continue;
            if (a.chunks % Q) continue;
            const int Cl = a.chunks / Q;
            if (Cl * TLT > 512 || Cl < 2) continue;
            const size_t sm = (size_t)Cl * M * TLT * 8 + (size_t)4 * Cl * TLT * 8 +
                              (table ? (size_t)Cl * M * NCOEF * 8 : 0) + 16;
            if (sm > 200 * 1024 || box_rows(Cl * M, M) == 0) continue;
            const size_t score = (size_t)(TLT == 16 ? 0 : TLT == 32 ? 1 : 2) * 100 + Q;
            if (score < best) {
                best = score;
                *tl = TLT;
                *q = Q;
            }
        }
    }
}

}  // namespace

bool tmc_eligible(int M, bool uniform, const FastArgs& a) {
    if (const char* e = getenv("TDS_TMA"))
        if (e[0] == '0') return false;
    if (!a.Hb || a.nb <= 0) return false;
    if (reinterpret_cast<uintptr_t>(a.u) % 16 != 0 || encode_fn() == nullptr) return false;
    int tl, q;
    tmc_shape(a, M, !uniform, &tl, &q);   // TAB_GLOBAL also stages its per-row table
    return tl != 0;
}

int launch_tmc(int M, bool uniform, const FastArgs& a, cudaStream_t s) {
    int tl, q;
    tmc_shape(a, M, !uniform, &tl, &q);
    if (!tl) return set_err(TDS_ERR_UNSUPPORTED, "no cluster shape for this line");
    const int tab = !uniform ? TAB_GLOBAL
                    : (a.special_first || a.special_last) ? TAB_EDGES : TAB_UNIFORM;
#define TMC_TAB(MM, TLT, SZC)                                                           \
    return tab == TAB_UNIFORM ? launch_tmc_t<MM, TAB_UNIFORM, TLT, SZC>(a, q, s)        \
           : tab == TAB_EDGES ? launch_tmc_t<MM, TAB_EDGES, TLT, SZC>(a, q, s)          \
                              : launch_tmc_t<MM, TAB_GLOBAL, TLT, SZC>(a, q, s);
    if (M == 32) {
        if (tl == 32) { TMC_TAB(32, 32, 32) }
        if (tl == 16) { TMC_TAB(32, 16, 0) }
        TMC_TAB(32, 8, 0)
    }
    if (M == 16) {
        if (tl == 32) { TMC_TAB(16, 32, 32) }
        if (tl == 16) { TMC_TAB(16, 16, 0) }
        TMC_TAB(16, 8, 0)
    }
#undef TMC_TAB
    return set_err(TDS_ERR_UNSUPPORTED, "unsupported chunk size");
}

}  // namespace tds
