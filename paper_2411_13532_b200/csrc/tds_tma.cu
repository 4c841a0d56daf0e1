// TMA-staged persistent variant of the fast DistD2 kernel (sm_100a).
//
// Same arithmetic as k_fast (tds_kernels.cu) -- fused stencil + Alg. 6
// sweeps per chunk in registers, dense reduced map H over the chunk boundary
// values, Alg. 7 substitution, one store -- but the input tile reaches the
// CTA through the Tensor Memory Accelerator:
//   * a 3-D tensor map views the field as (groups, rows, sz) fp64; one box
//     is TLT lanes (TLT x 8 bytes) x up to 256 rows, so a tile of TLT lines
//     is one to a few cp.async.bulk.tensor loads completing on an mbarrier;
//   * the CTA is persistent (resident CTAs x SMs) and issues the NEXT item's
//     TMA as soon as every thread has copied the current tile from shared
//     memory into registers, so HBM reads stay in flight through the sweeps,
//     the reduced solve, the substitution and the stores of this item --
//     without spending registers on the prefetch.
// TLT (lines per tile) is 16 (128-byte row segments, 256-thread CTAs) or 8
// (64-byte segments, 128-thread CTAs: twice the independent items per SM).
// Eligible when sz % TLT == 0, the field is 16-byte aligned and a tile fits
// in shared memory.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "tds_device.cuh"
#include "tds_tma.h"

namespace tds {

using namespace dev;

// Output row i of a chunk after the Alg. 7 substitution (the value
// chunk_store_any writes), for the staged bulk-store path.
template <int M, int TAB>
__device__ __forceinline__ double chunk_row(const FastArgs& p, const double* __restrict__ tb,
                                            const double (&d)[M], double F, double L, int i,
                                            int chunk) {
    if (i == 0) return F;
    if (i == M - 1) return L;
    double sa, sc;
    if (TAB == TAB_EDGES && p.special_first && chunk == 0) {
        sa = p.e_first.c[i][8];
        sc = p.e_first.c[i][9];
    } else if (TAB == TAB_EDGES && p.special_last && chunk == p.chunks - 1) {
        sa = p.e_last.c[i][8];
        sc = p.e_last.c[i][9];
    } else if (TAB != TAB_GLOBAL) {
        sa = p.ut.sa[i];
        sc = p.ut.sc[i];
    } else {
        sa = tb[i * NCOEF + 8];
        sc = tb[i * NCOEF + 9];
    }
    return fma(-sc, L, fma(-sa, F, d[i]));
}

// BST (bulk stores; 32-line tiles of an sz = 32 field, where a chunk's M rows
// of its 32 lines are one contiguous M x 256-byte block): each warp writes
// its chunk 8 rows at a time into one of two 2 KiB shared-memory staging
// buffers, and one lane hands each 2 KiB to the TMA engine
// (cp.async.bulk shared -> global), instead of 32 warp-wide STG per thread.
template <int M, int MODE, int TAB, int TLT, int SZC, int BST = 0>
__global__ void __launch_bounds__(512) k_tma(const __grid_constant__ TmaArgs A) {
    constexpr bool UNIFORM = TAB != TAB_GLOBAL;
    const FastArgs& p = A.f;
    extern __shared__ __align__(1024) unsigned char smem[];
    const int C = p.chunks;
    const int K = 2 * C;
    const int rows = p.rows;
    const int tpc = p.tiles_per_cta;
    const int t = threadIdx.x;
    const int lane = t % TLT;
    const int chunk = (t / TLT) % C;
    const int tl = t / (TLT * C);
    const long long sz = SZC ? SZC : p.sz;
    const int r0 = chunk * M;
    double* tiles = reinterpret_cast<double*>(smem);
    const size_t tile_elems = (size_t)rows * TLT;
    double* sY = tiles + (size_t)tpc * tile_elems;
    const size_t ybuf = (size_t)tpc * K * TLT;
    // TAB_GLOBAL: the block's per-row table (shared by every line) is staged
    // in shared memory once per CTA when it fits
    double* stab = sY + 2 * ybuf;
    double* sStage = stab + (TAB == TAB_GLOBAL && A.tab_smem ? (size_t)rows * NCOEF : 0);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sStage + (BST ? (size_t)blockDim.x * 16 : 0));
    if (TAB == TAB_GLOBAL && A.tab_smem)
        for (int k = t; k < rows * NCOEF; k += blockDim.x) stab[k] = __ldg(p.tab + k);
    const double* __restrict__ tb =
        (TAB == TAB_GLOBAL && A.tab_smem ? stab : p.tab) + (size_t)r0 * NCOEF;

    auto issue = [&](long long item) {
        uint32_t bytes = 0;
        for (int j = 0; j < tpc; ++j)
            if ((item * tpc + j) * TLT < p.lines) bytes += (uint32_t)(tile_elems * sizeof(double));
        mbar_expect_tx(bar, bytes);
        for (int j = 0; j < tpc; ++j) {
            const long long first = (item * tpc + j) * TLT;
            if (first >= p.lines) break;
            const int g = (int)(first / p.sz), l0 = (int)(first % p.sz);
            for (int b = 0; b * A.boxr < rows; ++b)
                tma_load_3d(tiles + j * tile_elems + (size_t)b * A.boxr * TLT, &A.map, bar, l0,
                            b * A.boxr, g);
        }
    };

    __shared__ long long s_next[2];   // next item (dynamic schedule), by iteration parity
    if (t == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    long long item = blockIdx.x;
    if (t == 0 && item < p.items) issue(item);
    uint32_t phase = 0;

    // items past the first: round-robin, or (p.ctr) handed out in order of
    // request -- thread 0 takes the next when it issues its TMA, everyone
    // reads it after the iteration's second barrier
    for (int it = 0; item < p.items; item = s_next[it & 1], ++it) {
        const long long line = (item * tpc + tl) * TLT + lane;
        const bool valid = line < p.lines;

        while (!mbar_try_wait(bar, phase)) {
        }
        phase ^= 1u;
        // tile rows (+ 2-row halos) -> registers
        const double* tile = tiles + tl * tile_elems;
        double v[M + 4];
        const long long hb = valid ? halo_base_t<SZC>(line, p.sz) : 0;
#pragma unroll
        for (int i = 0; i < M + 4; ++i) {
            const int row = r0 - 2 + i;
            double x = 0.0;
            if (i < 2 || i >= M + 2) {
                if (row < 0) {
                    if (p.edge_mode == EDGE_WRAP) x = tile[(row + rows) * TLT + lane];
                    else if (p.edge_mode == EDGE_HALO && p.halo_lo && valid)
                        x = __ldg(p.halo_lo + hb + (row + 2) * sz);
                } else if (row >= rows) {
                    if (p.edge_mode == EDGE_WRAP) x = tile[(row - rows) * TLT + lane];
                    else if (p.edge_mode == EDGE_HALO && p.halo_hi && valid)
                        x = __ldg(p.halo_hi + hb + (row - rows) * sz);
                } else {
                    x = tile[row * TLT + lane];
                }
            } else {
                x = tile[row * TLT + lane];
            }
            v[i] = x;
        }
        __syncthreads();   // every thread holds its rows: the tile buffer is free
        if (t == 0) {
            const long long nxt =
                p.ctr ? (long long)gridDim.x + (long long)atomicAdd(p.ctr, 1ULL) : item + gridDim.x;
            s_next[it & 1] = nxt;
            if (nxt < p.items) {
                fence_proxy_async();
                issue(nxt);
            }
        }

        double d[M];
        chunk_sweeps_any<M, TAB>(p, tb, v, d, chunk);

        double* Y = sY + (it & 1) * ybuf + (size_t)tl * K * TLT;
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
        Y[(2 * chunk) * TLT + lane] = y0;
        Y[(2 * chunk + 1) * TLT + lane] = yL;
        __syncthreads();

        if (MODE == MODE_PASS_A) {
            if (valid && chunk == 0) p.d_first_out[line] = gdot<TLT>(p, 0, Y, K, lane);
            if (valid && chunk == C - 1) p.d_last_out[line] = gdot<TLT>(p, 1, Y, K, lane);
            continue;
        }

        double F, L;
        // banded reduced map (plan.cpp upload_H: every entry above 2^-70 of the
        // chunk's largest); TDS_BAND=0 -> the full K-term row
        if (A.band)
            band_bounds<TLT>(p.Hb + (size_t)chunk * p.nb, __ldg(p.bq0 + chunk), p.nb, Y, K, lane,
                             F, L);
        else
            chunk_bounds<TLT>(p.Hp + (size_t)chunk * K, Y, K, lane, nullptr, nullptr, F, L);
        if constexpr (BST != 0) {
            static_assert(TLT == 32 && SZC == 32 && M % 8 == 0, "bulk stores: sz = 32 tiles");
            // every line of a tile is valid (lines = groups x 32)
            double* stg = sStage + (size_t)(t >> 5) * 512;
            double* gout = p.out + (line >> 5) * (long long)rows * 32 + (long long)r0 * 32;
#pragma unroll
            for (int s8 = 0; s8 < M / 8; ++s8) {
                double* buf = stg + (s8 & 1) * 256;
                if (lane == 0) bulk_wait_read<1>();      // this buffer's last copy has read it
                __syncwarp();
#pragma unroll
                for (int r = 0; r < 8; ++r)
                    buf[r * 32 + lane] = chunk_row<M, TAB>(p, tb, d, F, L, s8 * 8 + r, chunk);
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    bulk_store(gout + s8 * 256, buf, 8 * 32 * sizeof(double));
                    bulk_commit();
                }
            }
        } else if (valid) {
            chunk_store_any<M, TAB>(p, tb, p.out + line_base_t<SZC>(line, p.rows, p.sz), sz, r0, d, F,
                                    L, A.store_cs != 0, chunk);
        }
    }
    if constexpr (BST != 0)
        if (lane == 0) bulk_wait_all();                // staging reads done before exit
    if (p.ctr && t == 0) {
        // every CTA has taken its last item once all have come here: the last
        // one out resets the slot for the next launch that uses it
        __threadfence();
        if (atomicAdd(p.ctr + 1, 1ULL) == gridDim.x - 1) {
            p.ctr[0] = 0;
            p.ctr[1] = 0;
            __threadfence();
        }
    }
}

namespace {

template <int M, int MODE, int UNI, int TLT, int SZC = 0, int BST = 0>
int launch_tma_t(const FastArgs& a, TileCfg cfg, cudaStream_t s) {
    TmaArgs A;
    A.f = a;
    A.f.tiles_per_cta = cfg.tpc;
    const long long tiles = (a.lines + TLT - 1) / TLT;
    A.f.items = (tiles + cfg.tpc - 1) / cfg.tpc;
    if (A.f.items <= 0) return TDS_OK;
    int rc = encode_field_map(a, M, TLT, &A.map, &A.boxr);
    if (rc) return rc;
    A.store_cs = store_policy();
    A.band = a.Hb && a.nb > 0 && !(getenv("TDS_BAND") && getenv("TDS_BAND")[0] == '0');
    const int threads = cfg.tpc * a.chunks * TLT;
    size_t smem = tma_smem(a, cfg);
    const size_t tab_bytes = (size_t)a.rows * NCOEF * sizeof(double);
    A.tab_smem = UNI == TAB_GLOBAL && smem + tab_bytes <= 227 * 1024 &&
                 !(getenv("TDS_TAB_SMEM") && getenv("TDS_TAB_SMEM")[0] == '0');
    if (A.tab_smem) smem += tab_bytes;
    if (BST) smem += (size_t)threads * 16 * sizeof(double);   // 2 x 8 rows per warp
    const void* fn = reinterpret_cast<const void*>(k_tma<M, MODE, UNI, TLT, SZC, BST>);
    if ((rc = ensure_smem(fn, smem, "cudaFuncSetAttribute(k_tma)"))) return rc;
    const long long grid = persistent_grid(fn, threads, smem, A.f.items, 0);
    if (grid < 1) return set_err(TDS_ERR_UNSUPPORTED, "k_tma does not fit on an SM");
    k_tma<M, MODE, UNI, TLT, SZC, BST><<<(unsigned)grid, threads, smem, s>>>(A);
    return cuda_check(cudaGetLastError(), "k_tma launch");
}

template <int M, int MODE, int UNI>
int launch_tma_m(const FastArgs& a, cudaStream_t s) {
    const TileCfg cfg = tile_cfg(a);
    // 32-line tiles (1 CTA of 512 threads per SM): one chunk per warp, so a
    // special edge chunk never diverges from a uniform neighbour, 256-byte row
    // segments, and (with the compile-time lane width and the banded map)
    // fewer instructions. Measured at 512^3, 1000 steps under the power cap:
    // 5812 / 5823 GB/s vs 5523 / 5532 for 16-line tiles. Knob TDS_TMA_TL32=0.
    const char* e32 = getenv("TDS_TMA_TL32");
    const bool want32 = e32 ? e32[0] == '1' : true;
    if (want32 && MODE == MODE_SOLVE && a.sz % 32 == 0 && a.chunks * 32 <= 512 &&
        (size_t)a.rows * 32 * 8 + 4 * a.chunks * 32 * 8 <= 200 * 1024)
    {
        // compile-time lane width: 5147 vs 4980 GB/s for open d/dx at 512^3
        // (the compile-time width is only right for sz == 32 itself)
        if (a.sz != 32 || (getenv("TDS_SZC_TMA") && getenv("TDS_SZC_TMA")[0] == '0'))
            return launch_tma_t<M, MODE, UNI, 32>(a, TileCfg{32, 1}, s);
        // bulk (TMA-engine) stores through shared-memory staging: A/B knob
        // TDS_BULK_ST=1 (needs an sz = 32 field, 16-byte aligned output)
        const char* eb = getenv("TDS_BULK_ST");
        const bool bulk = eb && eb[0] == '1' && a.sz == 32 &&
                          reinterpret_cast<uintptr_t>(a.out) % 16 == 0 &&
                          (size_t)a.rows * 32 * 8 + 4 * a.chunks * 32 * 8 +
                                  (size_t)a.chunks * 32 * 16 * 8 <= 220 * 1024;
        if constexpr (MODE == MODE_SOLVE)
            if (bulk) return launch_tma_t<M, MODE, UNI, 32, 32, 1>(a, TileCfg{32, 1}, s);
        return launch_tma_t<M, MODE, UNI, 32, 32>(a, TileCfg{32, 1}, s);
    }
    if (cfg.tl == 8) return launch_tma_t<M, MODE, UNI, 8>(a, cfg, s);
    // compile-time lane width (sz = 32): a win for k_dd / k_dd2 (+9% at
    // m = 512 in loopback) and 32-line tiles, but measured slower for 16-line
    // uniform tiles (5516 vs 5863 GB/s at 512^3): runtime width unless
    // TDS_SZC_TMA=1
    if constexpr (M == 32 && MODE == MODE_SOLVE)
        if (a.sz == 32 && getenv("TDS_SZC_TMA") && getenv("TDS_SZC_TMA")[0] == '1')
            return launch_tma_t<M, MODE, UNI, 16, 32>(a, cfg, s);
    return launch_tma_t<M, MODE, UNI, 16>(a, cfg, s);
}

}  // namespace

int ensure_smem(const void* fn, size_t smem, const char* what) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cuda_check(cudaGetLastError(), what);
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = done[{fn, dev}];
    if (smem <= cur) return TDS_OK;
    int rc = cuda_check(
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), what);
    if (!rc) cur = smem;
    return rc;
}

long long persistent_grid(const void* fn, int threads, size_t smem, long long items,
                          int max_ctas) {
    int dev = 0, sms = 0, nb = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem);
    if (nb < 1) return 0;
    long long grid = (long long)nb * sms;
    if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
    if (max_ctas < 0) grid = grid / -(long long)max_ctas > 0 ? grid / -(long long)max_ctas : 1;
    if (grid > items) grid = items;
    return grid;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

TileCfg tile_cfg(const FastArgs& a) {
    int tl = 16;
    if (const char* e = getenv("TDS_TL")) tl = atoi(e) == 8 ? 8 : 16;
    if (a.sz % tl != 0) tl = (a.sz % 8 == 0) ? 8 : 0;
    if (tl && a.chunks * tl > 512) tl = (a.chunks * 8 <= 512 && a.sz % 8 == 0) ? 8 : 0;
    TileCfg c{tl, 1};
    if (tl) {
        const int per_tile = a.chunks * tl;
        const int target = tl == 8 ? 128 : 256;
        c.tpc = per_tile >= target ? 1 : target / per_tile;
    }
    return c;
}

size_t tma_smem(const FastArgs& a, TileCfg c) {
    return (size_t)c.tpc * a.rows * c.tl * sizeof(double) +
           (size_t)2 * c.tpc * 2 * a.chunks * c.tl * sizeof(double) + 16;
}

int box_rows(int rows, int M) {
    int C = rows / M, best = 0;
    for (int d = 1; d <= C; ++d)
        if (C % d == 0 && d * M <= 256) best = d * M;
    return best;
}

int store_policy() {
    int cs = 1;   // measured: +2% over write-back stores on B200
    if (const char* e = getenv("TDS_STCS")) cs = e[0] != '0';
    return cs;
}

int encode_field_map(const FastArgs& a, int M, int tl, CUtensorMap* map, int* boxr) {
    *boxr = box_rows(a.rows, M);
    CUtensorMapL2promotion prom =
        tl >= 16 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    if (const char* e = getenv("TDS_L2PROMO")) {
        if (e[0] == '0') prom = CU_TENSOR_MAP_L2_PROMOTION_NONE;
        else if (e[0] == '1') prom = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
        else if (e[0] == '2') prom = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }
    const long long groups = a.lines / a.sz;
    cuuint64_t dims[3] = {(cuuint64_t)a.sz, (cuuint64_t)a.rows, (cuuint64_t)groups};
    cuuint64_t strides[2] = {(cuuint64_t)a.sz * 8, (cuuint64_t)a.rows * a.sz * 8};
    cuuint32_t box[3] = {(cuuint32_t)tl, (cuuint32_t)*boxr, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(a.u),
                              dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, prom,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return set_err(TDS_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return TDS_OK;
}

bool tma_eligible(int M, const FastArgs& a) {
    if (const char* e = getenv("TDS_TMA"))
        if (e[0] == '0') return false;
    const TileCfg c = tile_cfg(a);
    if (c.tl == 0) return false;
    if (reinterpret_cast<uintptr_t>(a.u) % 16 != 0) return false;
    if (box_rows(a.rows, M) == 0) return false;
    if (tma_smem(a, c) > 200 * 1024) return false;
    return encode_fn() != nullptr;
}

int launch_tma(int M, int mode, bool uniform, const FastArgs& a, long long /*tiles*/,
               cudaStream_t s) {
    const int tab = !uniform ? TAB_GLOBAL
                    : (a.special_first || a.special_last) ? TAB_EDGES : TAB_UNIFORM;
#define DISPATCH_TAB(MM, MO)                                                            \
    return tab == TAB_UNIFORM ? launch_tma_m<MM, MO, TAB_UNIFORM>(a, s)                 \
           : tab == TAB_EDGES ? launch_tma_m<MM, MO, TAB_EDGES>(a, s)                   \
                              : launch_tma_m<MM, MO, TAB_GLOBAL>(a, s);
#define DISPATCH_MODE(MM)                                                               \
    switch (mode) {                                                                     \
        case MODE_SOLVE: DISPATCH_TAB(MM, MODE_SOLVE)                                   \
        case MODE_PASS_A: DISPATCH_TAB(MM, MODE_PASS_A)                                 \
        default: DISPATCH_TAB(MM, MODE_PASS_B)                                          \
    }
    if (M == 32) { DISPATCH_MODE(32) }
    if (M == 16) { DISPATCH_MODE(16) }
#undef DISPATCH_MODE
#undef DISPATCH_TAB
    return set_err(TDS_ERR_UNSUPPORTED, "unsupported chunk size");
}

}  // namespace tds
