// Fused single-pass DistD2 for one rank per GPU (sm_100a): the whole
// per-rank solve of distributed.py:327-366 -- both neighbour rounds included
// -- in ONE kernel launch, 16 B/point of HBM traffic.
//
// Each rank owns a MAILBOX in its HBM that its neighbours map through CUDA
// IPC (NVLink peer memory). Per tile of TLT lines:
//   ROUND 1 (halo, transport.py:142-171): the rank stores its first two rows
//     into prev's mailbox and its last two rows into next's, one item AHEAD
//     of use;
//   decoupling: TMA tile -> registers, Alg. 6 sweeps (as k_tma);
//   ROUND 2 (boundary rows, transport.py:174-191): g0.Y / g1.Y are the
//     rank's d[0], d[m-1]; they go to prev / next the same way, and the 2x2
//     pairs (distributed.py:279-293) give u_start / u_end in-kernel;
//   substitution with the pinned reduced map, one streaming store.
// Messages are fence-free (sentinel-armed slots, see Mail). Deadlock
// freedom: every rank runs the same persistent schedule (same grid, same
// item order); in every iteration a CTA posts before it waits, and what it
// waits for is posted by the same CTA index of the neighbour in the same or
// an earlier iteration. Every wait has a device-side timeout that records an
// error word instead of hanging the GPU.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "tds_device.cuh"
#include "tds_tma.h"

namespace tds {

using namespace dev;

struct DDArgs {
    TmaArgs t;
    double* mail;          // own mailbox
    double* mail_prev;     // prev rank's mailbox (peer mapping), null on an open edge
    double* mail_next;     // next rank's mailbox
    unsigned long long epoch;
    unsigned long long timeout_ns;
    int max_ctas;          // host-side grid cap (0: resident capacity)
    int query;             // host-side: return the grid instead of launching
};

// Mailbox layout (8-byte words), L = lines. Two parity halves (epoch & 1)
// of 6L value slots each, then three STATUS words (not sentinel slots;
// tds_mailbox_init zeroes them): the error word and the cumulative counts of
// halo / boundary words this rank has posted to its neighbours (the measured
// message accounting of transport.py:45-48,71-80):
//   D_FROM_PREV [L]  prev's d[m-1] per line      D_FROM_NEXT [L]  next's d[0]
//   H_LO [2L]  prev's last two rows (G,2,sz)     H_HI [2L]  next's first two rows
// A slot holds either the SENTINEL bit pattern (all ones: the byte-uniform
// fill of cudaMemset(0xFF)) or a value. Writers canonicalise NaNs, so no
// value equals the sentinel; readers poll their own slot and re-arm it. The
// next write to the same slot is two epochs later, i.e. in a kernel that
// starts after this one has finished -- no fences and no flags are needed.
struct Mail {
    long long L;
    __host__ __device__ long long half(unsigned long long epoch) const {
        return (long long)(epoch & 1ULL) * 6 * L;
    }
    __host__ __device__ long long d_from_prev() const { return 0; }
    __host__ __device__ long long d_from_next() const { return L; }
    __host__ __device__ long long h_lo() const { return 2 * L; }
    __host__ __device__ long long h_hi() const { return 4 * L; }
    __host__ __device__ long long err() const { return 12 * L; }
    __host__ __device__ long long words() const { return 12 * L + 3; }
};

constexpr unsigned long long SENTINEL = ~0ULL;
constexpr unsigned long long ERR_TIMEOUT = 1ULL;
constexpr int STATUS_WORDS = 3;   // error, halo words posted, boundary words posted

namespace {

__device__ __forceinline__ double canon(double x) {
    return isnan(x) ? __longlong_as_double(0x7FF8000000000000LL) : x;
}
// post a value into a neighbour's mailbox slot (NVLink peer store)
__device__ __forceinline__ void post(double* slot, double x) {
    asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(slot), "d"(canon(x)) : "memory");
}
__device__ __forceinline__ unsigned long long ld_sys_u64(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// wait for a neighbour's value in my mailbox slot, consume it, re-arm the slot
// (v: the slot's value if already loaded, else SENTINEL)
#ifdef TDS_WAIT_PROF
// debug builds (TDS_NVCC_EXTRA=-DTDS_WAIT_PROF, tools/wait_prof.py): ns spent
// in take_v per call site (0: halo rows, 1: boundary rows), summed over threads
__device__ unsigned long long g_wait_ns[2];
__device__ unsigned long long g_wait_n[2];
#endif
template <class Args>
__device__ double take_v(double* slot, unsigned long long v, const Args& A,
                         unsigned long long* err, int site = 1) {
    if (v == SENTINEL) v = ld_sys_u64(slot);
#ifdef TDS_WAIT_PROF
    const unsigned long long tp0 = globaltimer();
    atomicAdd(&g_wait_n[site], 1ULL);
#else
    (void)site;
#endif
    if (v == SENTINEL) {
        const unsigned long long t0 = globaltimer();
        unsigned ns = 32;
        for (;;) {
            __nanosleep(ns);
            if (ns < 256) ns *= 2;
            v = ld_sys_u64(slot);
            if (v != SENTINEL) break;
            if (*reinterpret_cast<volatile unsigned long long*>(err) == ERR_TIMEOUT ||
                globaltimer() - t0 > A.timeout_ns) {
                atomicExch(err, ERR_TIMEOUT);
                // poison: a timed-out solve must not look like a result
                return __longlong_as_double(0x7FF8000000000000LL);
            }
        }
    }
    *reinterpret_cast<unsigned long long*>(slot) = SENTINEL;
#ifdef TDS_WAIT_PROF
    atomicAdd(&g_wait_ns[site], globaltimer() - tp0);
#endif
    return __longlong_as_double((long long)v);
}
template <class Args>
__device__ __forceinline__ double take(double* slot, const Args& A, unsigned long long* err) {
    return take_v(slot, SENTINEL, A, err);
}
// Message accounting (status words err + 1 / err + 2: halo / boundary-row
// words this rank posted). At kernel exit every thread adds the words its
// role posts per item times the valid items it processed -- the posts are
// unconditional, so this is exactly what the kernel stored, and the hot
// loop carries no counter (a live per-store counter cost k_dd2 7% at
// m = 512: it sits at the 128-register cap). One atomic per warp.
__device__ __forceinline__ unsigned valid_items(long long items, long long lines, int tpc, int tl,
                                                int TLT, int lane) {
    unsigned n = 0;
    for (long long it = blockIdx.x; it < items; it += gridDim.x)
        n += ((it * tpc + tl) * TLT + lane < lines) ? 1u : 0u;
    return n;
}
__device__ __forceinline__ void flush_counts(unsigned long long* err, unsigned halo_words,
                                             unsigned bnd_words) {
    const unsigned mask = __activemask();
    const unsigned a = __reduce_add_sync(mask, halo_words), b = __reduce_add_sync(mask, bnd_words);
    if ((threadIdx.x & 31) == __ffs(mask) - 1) {
        if (a) atomicAdd(err + 1, (unsigned long long)a);
        if (b) atomicAdd(err + 2, (unsigned long long)b);
    }
}

}  // namespace

template <int M, int TAB, int TLT, int SZC>
__global__ void __launch_bounds__(512) k_dd(const __grid_constant__ DDArgs A) {
    constexpr bool UNIFORM = TAB != TAB_GLOBAL;
    const FastArgs& p = A.t.f;
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
    const Mail mb{p.lines};
    const long long par = mb.half(A.epoch);
    unsigned long long* err = reinterpret_cast<unsigned long long*>(A.mail + mb.err());
    double* tiles = reinterpret_cast<double*>(smem);
    const size_t tile_elems = (size_t)rows * TLT;
    double* sY = tiles + (size_t)tpc * tile_elems;
    const size_t ybuf = (size_t)tpc * K * TLT;
    double* sP = sY + 2 * ybuf;                        // pins: [tpc][2][TLT]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sP + (size_t)tpc * 2 * TLT);
    const double* __restrict__ tb = p.tab + (size_t)r0 * NCOEF;
    const bool first_chunk = chunk == 0, last_chunk = chunk == C - 1;

    auto issue = [&](long long item) {
        uint32_t bytes = 0;
        for (int j = 0; j < tpc; ++j)
            if ((item * tpc + j) * TLT < p.lines) bytes += (uint32_t)(tile_elems * sizeof(double));
        mbar_expect_tx(bar, bytes);
        for (int j = 0; j < tpc; ++j) {
            const long long first = (item * tpc + j) * TLT;
            if (first >= p.lines) break;
            const int g = (int)(first / p.sz), l0 = (int)(first % p.sz);
            for (int b = 0; b * A.t.boxr < rows; ++b)
                tma_load_3d(tiles + j * tile_elems + (size_t)b * A.t.boxr * TLT, &A.t.map, bar,
                            l0, b * A.t.boxr, g);
        }
    };
    // ROUND 1 for `item`: my first two rows -> prev's high halo, my last two
    // rows -> next's low halo (read straight from my block in HBM)
    auto publish_halo = [&](long long item) {
        const long long ln = (item * tpc + tl) * TLT + lane;
        if (ln >= p.lines) return;
        const double* ub = p.u + line_base_t<SZC>(ln, rows, p.sz);
        const long long hb = halo_base_t<SZC>(ln, p.sz);
        if (first_chunk && A.mail_prev) {
            const double a0 = __ldg(ub), a1 = __ldg(ub + sz);
            post(A.mail_prev + par + mb.h_hi() + hb, a0);
            post(A.mail_prev + par + mb.h_hi() + hb + sz, a1);
        }
        if (last_chunk && A.mail_next) {
            const double a0 = __ldg(ub + (long long)(rows - 2) * sz);
            const double a1 = __ldg(ub + (long long)(rows - 1) * sz);
            post(A.mail_next + par + mb.h_lo() + hb, a0);
            post(A.mail_next + par + mb.h_lo() + hb + sz, a1);
        }
    };

    // item schedule: round-robin, or (p.ctr) handed out by a per-plan
    // counter in increasing order (the SMs stream HBM at different rates).
    // Thread 0 claims two items ahead (the halo rows of the next item are
    // posted at the top of an iteration); s_q[k % 3] = the CTA's k-th item.
    // Deadlock freedom with independent counters per rank: the smallest
    // item claimed but not finished on either rank always progresses -- its
    // partner on the other rank is claimed (counters are monotonic) and, as
    // every CTA posts before it waits, already posted.
    __shared__ long long s_q[3];
    if (t == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        s_q[1] = p.ctr ? (long long)gridDim.x + (long long)atomicAdd(p.ctr, 1ULL)
                       : (long long)blockIdx.x + gridDim.x;
    }
    __syncthreads();
    long long item = blockIdx.x;
    unsigned nvalid = 0;     // items with a valid line for this thread (message accounting)
    if (item < p.items) {
        if (t == 0) issue(item);
        publish_halo(item);
    }
    uint32_t phase = 0;

    for (int it = 0; item < p.items; item = s_q[(it + 1) % 3], ++it) {
        const long long line = (item * tpc + tl) * TLT + lane;
        const bool valid = line < p.lines;
        nvalid += valid ? 1u : 0u;
        const long long nxt = s_q[(it + 1) % 3];
        // halo slots of this item: loads in flight across the TMA wait (the
        // next item's halo posts come later, during ROUND 2)
        const long long hb = valid ? halo_base_t<SZC>(line, p.sz) : 0;
        double* hlo = (valid && first_chunk && A.mail_prev) ? A.mail + par + mb.h_lo() + hb : nullptr;
        double* hhi = (valid && last_chunk && A.mail_next) ? A.mail + par + mb.h_hi() + hb : nullptr;
        unsigned long long a0 = SENTINEL, a1 = SENTINEL, b0 = SENTINEL, b1 = SENTINEL;
        if (hlo) {
            a0 = ld_sys_u64(hlo);
            a1 = ld_sys_u64(hlo + sz);
        }
        if (hhi) {
            b0 = ld_sys_u64(hhi);
            b1 = ld_sys_u64(hhi + sz);
        }

        while (!mbar_try_wait(bar, phase)) {
        }
        phase ^= 1u;
        const double* tl_tile = tiles + tl * tile_elems;
        double v[M + 4];
        // halos of the rank block come from the neighbours' ROUND-1 posts
        double h0 = 0.0, h1 = 0.0, h2 = 0.0, h3 = 0.0;
        if (hlo) {
            h0 = take_v(hlo, a0, A, err, 0);
            h1 = take_v(hlo + sz, a1, A, err, 0);
        }
        if (hhi) {
            h2 = take_v(hhi, b0, A, err, 0);
            h3 = take_v(hhi + sz, b1, A, err, 0);
        }
#pragma unroll
        for (int i = 0; i < M + 4; ++i) {
            // only the 2 + 2 outer window rows can leave the block (first /
            // last chunk): the interior rows are plain tile reads
            const int row = r0 - 2 + i;
            double x;
            if (i < 2) x = first_chunk ? (i == 0 ? h0 : h1) : tl_tile[row * TLT + lane];
            else if (i >= M + 2) x = last_chunk ? (i == M + 2 ? h2 : h3) : tl_tile[row * TLT + lane];
            else x = tl_tile[row * TLT + lane];
            v[i] = x;
        }
        __syncthreads();   // tile buffer free
        if (t == 0) {
            if (nxt < p.items) {
                fence_proxy_async();
                issue(nxt);
            }
            // the item after next (read at the top of the next iteration,
            // after this iteration's second barrier)
            s_q[(it + 2) % 3] = nxt >= p.items ? p.items
                                : p.ctr ? (long long)gridDim.x + (long long)atomicAdd(p.ctr, 1ULL)
                                        : nxt + gridDim.x;
        }

        double d[M];
        chunk_sweeps_any<M, TAB>(p, tb, v, d, chunk);

        double* Y = sY + (it & 1) * ybuf + (size_t)tl * K * TLT;
        Y[(2 * chunk) * TLT + lane] = d[0];
        Y[(2 * chunk + 1) * TLT + lane] = d[M - 1];
        __syncthreads();

        // ROUND 2 posts first (the rank's decoupled boundary rows), then the
        // pin-independent part of the reduced map while they travel, then
        // the neighbours' rows -> 2x2 pairs -> pins
        double g0y = 0.0, g1y = 0.0;
        if (valid && (first_chunk || last_chunk)) {
            g0y = first_chunk ? gdot<TLT>(p, 0, Y, K, lane) : 0.0;
            g1y = last_chunk ? gdot<TLT>(p, 1, Y, K, lane) : 0.0;
            if (first_chunk && A.mail_prev) {
                post(A.mail_prev + par + mb.d_from_next() + line, g0y);
            }
            if (last_chunk && A.mail_next) {
                post(A.mail_next + par + mb.d_from_prev() + line, g1y);
            }
        }
        // ROUND 1 of the next item while the boundary rows travel: the HBM
        // reads of its halo rows overlap the neighbour round trip (half an
        // item ahead of use; deadlock-free as above: a post depends only on
        // earlier items and on same-item posts that precede their waits)
        if (nxt < p.items) publish_halo(nxt);
        double F, L;
        if (A.t.band)   // banded reduced map, pin columns excluded (TDS_BAND=0: full row)
            band_bounds_nopins<TLT>(p.Hb + (size_t)chunk * p.nb, __ldg(p.bq0 + chunk), p.nb, Y,
                                    K, lane, F, L);
        else
            chunk_bounds<TLT>(p.Hp + (size_t)chunk * K + 1, Y + TLT, K - 2, lane, nullptr,
                              nullptr, F, L);
        double* P = sP + (size_t)tl * 2 * TLT;
        if (valid && (first_chunk || last_chunk)) {
            if (first_chunk) {
                double us = g0y;
                if (p.has_prev) {
                    const double prev_last = take(A.mail + par + mb.d_from_prev() + line, A, err);
                    us = (g0y - p.sa_first * prev_last) / p.det_prev;
                }
                P[lane] = us;
            }
            if (last_chunk) {
                double ue = g1y;
                if (p.has_next) {
                    const double next_first = take(A.mail + par + mb.d_from_next() + line, A, err);
                    ue = (g1y - p.sc_last * next_first) / p.det_next;
                }
                P[TLT + lane] = ue;
            }
        }
        __syncthreads();

        {
            const double2 h0 = __ldg(p.Hp + (size_t)chunk * K);
            const double2 hl = __ldg(p.Hp + (size_t)chunk * K + K - 1);
            const double us = P[lane], ue = P[TLT + lane];
            F = fma(h0.x, us, fma(hl.x, ue, F));
            L = fma(h0.y, us, fma(hl.y, ue, L));
        }
        if (valid)
            chunk_store_any<M, TAB>(p, tb, p.out + line_base_t<SZC>(line, rows, p.sz), sz, r0, d, F, L,
                                        A.t.store_cs != 0, chunk);
    }
    {
        const unsigned n = nvalid;
        const unsigned per = (first_chunk && A.mail_prev ? 1u : 0u) + (last_chunk && A.mail_next ? 1u : 0u);
        flush_counts(err, 2 * per * n, per * n);   // 2 halo rows + 1 boundary row per edge
    }
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

// ---------------------------------------------------------------------------
// k_dd2: the fused per-rank kernel with DEFERRED EDGES. The plan guarantees
// (plan.cpp, dd_defer) that chunks outside the first / last warp of a tile
// depend on the rank pins u_start / u_end by less than 2^-70: those chunks
// store their final rows in the same iteration, without waiting for the
// neighbour. The two edge warps of a tile post ROUND 2 for item t, stash
// their chunks (F', L', d rows, g.Y) in shared memory, and finish item t-1
// -- whose neighbour values arrived an iteration ago -- so the NVLink round
// trip is off the critical path.
template <int M, int TAB, int TLT, int SZC>
__global__ void __launch_bounds__(512) k_dd2(const __grid_constant__ DDArgs A) {
    constexpr bool UNIFORM = TAB != TAB_GLOBAL;
    const FastArgs& p = A.t.f;
    extern __shared__ __align__(1024) unsigned char smem[];
    constexpr int CW = 32 / TLT;                       // chunks per warp
    // edge region: the first / last ECH chunks of a tile (plan.cpp dd_defer:
    // 2 chunks for 16- and 32-line tiles, 4 for 8-line tiles), EW warps per
    // side, NE stash slots per tile
    constexpr int ECH = TLT == 8 ? 4 : 2;
    constexpr int EW = ECH / CW;
    constexpr int NE = 2 * EW;
    const int C = p.chunks;
    const int K = 2 * C;
    const int rows = p.rows;
    const int tpc = p.tiles_per_cta;
    const int t = threadIdx.x;
    const int wl = t & 31;
    const int lane = t % TLT;
    const int chunk = (t / TLT) % C;
    const int tl = t / (TLT * C);
    const int wc0 = chunk - (wl / TLT);                // first chunk of my warp
    const bool first_chunk = chunk == 0, last_chunk = chunk == C - 1;
    const bool has_first = wc0 < ECH, has_last = wc0 + CW - 1 >= C - ECH;
    const bool edge_warp = has_first || has_last;
    // helper roles of interior warps: form and post g0.Y / g1.Y (gy_role 0 /
    // 1), post the halo rows. 8- / 16-line tiles (>= 4 warps per tile): warp 1
    // holds both g.Y roles (one per chunk), warp 2 both halo roles. 32-line
    // tiles (one chunk per warp, >= 2 EW + 4 warps): one warp per role after
    // the first-side edge warps.
    const int NW = C * TLT / 32;
    const int wt = (t >> 5) % NW;
    const int role = wl / TLT;
    // without enough warps there are no helpers: the first / last chunk
    // threads post their own halos and ROUND 2
    const bool helpers = CW == 1 ? NW >= 2 * EW + 4 : NW >= 4;
    const int gy_role = !helpers || edge_warp ? -1
                        : CW == 1 ? (wt == EW ? 0 : (wt == EW + 1 ? 1 : -1))
                                  : (wt == 1 && role < 2 ? role : -1);
    const bool halo_lo_poster =
        helpers ? (CW == 1 ? wt == EW + 2 : (wt == 2 && role == 0)) : first_chunk;
    const bool halo_hi_poster =
        helpers ? (CW == 1 ? wt == EW + 3 : (wt == 2 && role == 1)) : last_chunk;
    const long long sz = SZC ? SZC : p.sz;
    const int r0 = chunk * M;
    const Mail mb{p.lines};
    const long long par = mb.half(A.epoch);
    unsigned long long* err = reinterpret_cast<unsigned long long*>(A.mail + mb.err());
    double* tiles = reinterpret_cast<double*>(smem);
    const size_t tile_elems = (size_t)rows * TLT;
    double* sY = tiles + (size_t)tpc * tile_elems;
    const size_t ybuf = (size_t)tpc * K * TLT;
    double* sS = sY + 2 * ybuf;                        // stash: [tpc][NE][M+1][32]
    double* sGY = sS + (size_t)tpc * NE * (M + 1) * 32; // rank d[0], d[m-1]: [2][tpc][2][TLT]
    double* sPin = sGY + (size_t)2 * tpc * 2 * TLT;    // pins (32-line tiles): [tpc][2][TLT]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sPin + (CW == 1 ? (size_t)tpc * 2 * TLT : 0));
    const int es = CW == 1 ? (has_first ? wt : EW + wt - (NW - EW)) : (has_first ? 0 : 1);
    double* stash = sS + ((size_t)(NE * tl + es) * (M + 1)) * 32 + wl;
    const double* __restrict__ tb = p.tab + (size_t)r0 * NCOEF;

    auto issue = [&](long long item) {
        uint32_t bytes = 0;
        for (int j = 0; j < tpc; ++j)
            if ((item * tpc + j) * TLT < p.lines) bytes += (uint32_t)(tile_elems * sizeof(double));
        mbar_expect_tx(bar, bytes);
        for (int j = 0; j < tpc; ++j) {
            const long long first = (item * tpc + j) * TLT;
            if (first >= p.lines) break;
            const int g = (int)(first / p.sz), l0 = (int)(first % p.sz);
            for (int b = 0; b * A.t.boxr < rows; ++b)
                tma_load_3d(tiles + j * tile_elems + (size_t)b * A.t.boxr * TLT, &A.t.map, bar,
                            l0, b * A.t.boxr, g);
        }
    };
    auto publish_halo = [&](long long item) {
        if (!halo_lo_poster && !halo_hi_poster) return;
        const long long ln = (item * tpc + tl) * TLT + lane;
        if (ln >= p.lines) return;
        const double* ub = p.u + line_base_t<SZC>(ln, rows, p.sz);
        const long long hb = halo_base_t<SZC>(ln, p.sz);
        if (halo_lo_poster && A.mail_prev) {
            const double a0 = __ldg(ub), a1 = __ldg(ub + sz);
            post(A.mail_prev + par + mb.h_hi() + hb, a0);
            post(A.mail_prev + par + mb.h_hi() + hb + sz, a1);
        }
        if (halo_hi_poster && A.mail_next) {
            const double a0 = __ldg(ub + (long long)(rows - 2) * sz);
            const double a1 = __ldg(ub + (long long)(rows - 1) * sz);
            post(A.mail_next + par + mb.h_lo() + hb, a0);
            post(A.mail_next + par + mb.h_lo() + hb + sz, a1);
        }
    };
    auto edge_finish = [&](const EdgeTable& T, double* ob, double F, double L) {
        __stcs(ob + (long long)r0 * sz, F);
#pragma unroll
        for (int i = 1; i < M - 1; ++i)
            __stcs(ob + (long long)(r0 + i) * sz,
                   fma(-T.c[i][9], L, fma(-T.c[i][8], F, stash[i * 32])));
        __stcs(ob + (long long)(r0 + M - 1) * sz, L);
    };
    // finish the stashed item `fi` (edge warps only; warp-synchronous)
    // the neighbour's row slot finish() takes for item fi (edge threads)
    auto pin_slot = [&](long long fi) -> double* {
        const long long fl = (fi * tpc + tl) * TLT + lane;
        return A.mail + par + (first_chunk ? mb.d_from_prev() : mb.d_from_next()) + fl;
    };
    // pv: the slot's value if loaded early (at the top of the iteration, so
    // the L2 round trip overlaps the tile wait), else SENTINEL
    auto finish = [&](long long fi, int fslot, unsigned long long pv) {
        const double* GY = sGY + ((size_t)fslot * tpc + tl) * 2 * TLT;
        const long long fl = (fi * tpc + tl) * TLT + lane;
        const bool fv = fl < p.lines;
        double us = 0.0, ue = 0.0;
        if (first_chunk) {
            us = GY[lane];
            if (fv && p.has_prev) {
                const double prev_last = take_v(pin_slot(fi), pv, A, err);
                us = (us - p.sa_first * prev_last) / p.det_prev;
            }
        }
        if (last_chunk) {
            ue = GY[TLT + lane];
            if (fv && p.has_next) {
                const double next_first = take_v(pin_slot(fi), pv, A, err);
                ue = (ue - p.sc_last * next_first) / p.det_next;
            }
        }
        if (CW == 1) {
            // 32-line tiles: the pins reach the other edge warp of each side
            // through shared memory (named barrier of the edge warps)
            double* PP = sPin + (size_t)tl * 2 * TLT;
            if (first_chunk) PP[lane] = us;
            if (last_chunk) PP[TLT + lane] = ue;
            asm volatile("bar.sync 1, %0;" ::"r"(tpc * NE * 32) : "memory");
            us = PP[lane];
            ue = PP[TLT + lane];
        } else {
            // broadcast the pins of each line to every chunk of this warp
            us = __shfl_sync(0xffffffffu, us, lane);
            ue = __shfl_sync(0xffffffffu, ue, (C - 1 - wc0) * TLT + lane);
        }
        const double2 h0 = __ldg(p.Hp + (size_t)chunk * K);
        const double2 hl = __ldg(p.Hp + (size_t)chunk * K + K - 1);
        double F = stash[0], L = stash[(M - 1) * 32];
        if (has_first) {
            F = fma(h0.x, us, F);
            L = fma(h0.y, us, L);
        }
        if (has_last) {
            F = fma(hl.x, ue, F);
            L = fma(hl.y, ue, L);
        }
        if (!fv) return;
        double* ob = p.out + line_base_t<SZC>(fl, rows, p.sz);
        if (TAB == TAB_EDGES && p.special_first && first_chunk) {
            edge_finish(p.e_first, ob, F, L);
            return;
        }
        if (TAB == TAB_EDGES && p.special_last && last_chunk) {
            edge_finish(p.e_last, ob, F, L);
            return;
        }
        __stcs(ob + (long long)r0 * sz, F);
#pragma unroll
        for (int i = 1; i < M - 1; ++i) {
            const double sa = UNIFORM ? p.ut.sa[i] : __ldg(tb + i * NCOEF + 8);
            const double sc = UNIFORM ? p.ut.sc[i] : __ldg(tb + i * NCOEF + 9);
            __stcs(ob + (long long)(r0 + i) * sz, fma(-sc, L, fma(-sa, F, stash[i * 32])));
        }
        __stcs(ob + (long long)(r0 + M - 1) * sz, L);
    };

    // item schedule: round-robin, or (p.ctr) handed out by a per-plan
    // counter in increasing order (the SMs stream HBM at different rates).
    // Thread 0 claims two items ahead (the halo rows of the next item are
    // posted at the top of an iteration); s_q[k % 3] = the CTA's k-th item.
    // Deadlock freedom with independent counters per rank: the smallest
    // item claimed but not finished on either rank always progresses -- its
    // partner on the other rank is claimed (counters are monotonic) and, as
    // every CTA posts before it waits, already posted.
    __shared__ long long s_q[3];
    if (t == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        s_q[1] = p.ctr ? (long long)gridDim.x + (long long)atomicAdd(p.ctr, 1ULL)
                       : (long long)blockIdx.x + gridDim.x;
    }
    __syncthreads();
    long long item = blockIdx.x;
    unsigned nvalid = 0;     // items with a valid line for this thread (message accounting)
    if (item < p.items) {
        if (t == 0) issue(item);
        publish_halo(item);
    }
    uint32_t phase = 0;
    long long prev_item = -1;

    int it = 0;
    for (; item < p.items; item = s_q[(it + 1) % 3], ++it) {
        const long long line = (item * tpc + tl) * TLT + lane;
        const bool valid = line < p.lines;
        nvalid += valid ? 1u : 0u;
        const long long nxt = s_q[(it + 1) % 3];
        if (nxt < p.items) publish_halo(nxt);          // one item ahead
        // (posting after the mailbox loads, as k_dd does, measured slower
        // here: 0.896 vs 0.908 per rank at m = 512 on 2 GPUs)
        const long long hb = valid ? halo_base_t<SZC>(line, p.sz) : 0;
        double* hlo = (valid && first_chunk && A.mail_prev) ? A.mail + par + mb.h_lo() + hb : nullptr;
        double* hhi = (valid && last_chunk && A.mail_next) ? A.mail + par + mb.h_hi() + hb : nullptr;
        unsigned long long a0 = SENTINEL, a1 = SENTINEL, b0 = SENTINEL, b1 = SENTINEL;
        if (hlo) {
            a0 = ld_sys_u64(hlo);
            a1 = ld_sys_u64(hlo + sz);
        }
        if (hhi) {
            b0 = ld_sys_u64(hhi);
            b1 = ld_sys_u64(hhi + sz);
        }
        unsigned long long pin_pre = SENTINEL;
        if (prev_item >= 0 && ((first_chunk && p.has_prev) || (last_chunk && p.has_next)) &&
            (prev_item * tpc + tl) * TLT + lane < p.lines)
            pin_pre = ld_sys_u64(pin_slot(prev_item));

        while (!mbar_try_wait(bar, phase)) {
        }
        phase ^= 1u;
        const double* tl_tile = tiles + tl * tile_elems;
        double v[M + 4];
        double h0 = 0.0, h1 = 0.0, h2 = 0.0, h3 = 0.0;
        if (hlo) {
            h0 = take_v(hlo, a0, A, err, 0);
            h1 = take_v(hlo + sz, a1, A, err, 0);
        }
        if (hhi) {
            h2 = take_v(hhi, b0, A, err, 0);
            h3 = take_v(hhi + sz, b1, A, err, 0);
        }
#pragma unroll
        for (int i = 0; i < M + 4; ++i) {
            // only the 2 + 2 outer window rows can leave the block (first /
            // last chunk): the interior rows are plain tile reads
            const int row = r0 - 2 + i;
            double x;
            if (i < 2) x = first_chunk ? (i == 0 ? h0 : h1) : tl_tile[row * TLT + lane];
            else if (i >= M + 2) x = last_chunk ? (i == M + 2 ? h2 : h3) : tl_tile[row * TLT + lane];
            else x = tl_tile[row * TLT + lane];
            v[i] = x;
        }
        __syncthreads();   // tile buffer free
        if (t == 0) {
            if (nxt < p.items) {
                fence_proxy_async();
                issue(nxt);
            }
            // the item after next (read at the top of the next iteration,
            // after this iteration's second barrier)
            s_q[(it + 2) % 3] = nxt >= p.items ? p.items
                                : p.ctr ? (long long)gridDim.x + (long long)atomicAdd(p.ctr, 1ULL)
                                        : nxt + gridDim.x;
        }

        double d[M];
        chunk_sweeps_any<M, TAB>(p, tb, v, d, chunk);

        double* Y = sY + (it & 1) * ybuf + (size_t)tl * K * TLT;
        Y[(2 * chunk) * TLT + lane] = d[0];
        Y[(2 * chunk + 1) * TLT + lane] = d[M - 1];
        __syncthreads();

        // ROUND 2 posts of this item first (helper warp): the rank's d[0] /
        // d[m-1], on their way while the chunk boundary values are formed
        if (gy_role >= 0 && valid) {
            const double gy = gdot<TLT>(p, gy_role, Y, K, lane);
            if (gy_role == 0 && A.mail_prev) {
                post(A.mail_prev + par + mb.d_from_next() + line, gy);
            }
            if (gy_role == 1 && A.mail_next) {
                post(A.mail_next + par + mb.d_from_prev() + line, gy);
            }
            sGY[(((size_t)(it & 1) * tpc + tl) * 2 + gy_role) * TLT + lane] = gy;
        }
        // chunk boundary values without the rank pins
        double F, L;
        if (A.t.band)   // banded reduced map, pin columns excluded (TDS_BAND=0: full row)
            band_bounds_nopins<TLT>(p.Hb + (size_t)chunk * p.nb, __ldg(p.bq0 + chunk), p.nb, Y,
                                    K, lane, F, L);
        else
            chunk_bounds<TLT>(p.Hp + (size_t)chunk * K + 1, Y + TLT, K - 2, lane, nullptr,
                              nullptr, F, L);
        if (!edge_warp) {
            if (valid)
                chunk_store<M, UNIFORM>(p, tb, p.out + line_base_t<SZC>(line, rows, p.sz), sz, r0, d, F,
                                        L, true);   // interior warps: never a special chunk
        } else {
            if (!helpers && valid && (first_chunk || last_chunk)) {
                for (int r = 0; r < 2; ++r) {
                    if ((r == 0 && !first_chunk) || (r == 1 && !last_chunk)) continue;
                    const double gy = gdot<TLT>(p, r, Y, K, lane);
                    if (r == 0 && A.mail_prev) {
                        post(A.mail_prev + par + mb.d_from_next() + line, gy);
                            }
                    if (r == 1 && A.mail_next) {
                        post(A.mail_next + par + mb.d_from_prev() + line, gy);
                            }
                    sGY[(((size_t)(it & 1) * tpc + tl) * 2 + r) * TLT + lane] = gy;
                }
            }
            if (prev_item >= 0) finish(prev_item, (it & 1) ^ 1, pin_pre);
            __syncwarp();
            stash[0] = F;
#pragma unroll
            for (int i = 1; i < M - 1; ++i) stash[i * 32] = d[i];
            stash[(M - 1) * 32] = L;
            __syncwarp();
        }
        prev_item = item;
    }
    if (prev_item >= 0) {
        __syncthreads();   // the helper warp's g.Y of the last item
        if (edge_warp) finish(prev_item, (it - 1) & 1, SENTINEL);
    }
    {
        const unsigned n = nvalid;
        const unsigned h = (halo_lo_poster && A.mail_prev ? 2u : 0u) +
                           (halo_hi_poster && A.mail_next ? 2u : 0u);
        unsigned b = 0;
        if (helpers) {
            if (gy_role == 0 && A.mail_prev) b = 1;
            if (gy_role == 1 && A.mail_next) b = 1;
        } else {
            b = (first_chunk && A.mail_prev ? 1u : 0u) + (last_chunk && A.mail_next ? 1u : 0u);
        }
        flush_counts(err, h * n, b * n);
    }
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

// The fused per-rank kernels wait on other CTAs of the neighbour ranks, so
// every CTA of the persistent grid must be resident at once: launch them
// cooperatively -- the driver then guarantees co-residency of the grid or
// fails the launch (cudaErrorCooperativeLaunchTooLarge) instead of letting
// an unscheduled CTA deadlock its partners. TDS_COOP=0: plain launch.
template <class Args>
int launch_resident(const void* fn, long long grid, int threads, size_t smem, cudaStream_t s,
                    const Args& A, const char* what) {
    if (const char* e = getenv("TDS_COOP"))
        if (e[0] == '0') {
            void* args[1] = {const_cast<Args*>(&A)};
            return cuda_check(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(threads), args, smem, s),
                              what);
        }
    void* args[1] = {const_cast<Args*>(&A)};
    return cuda_check(
        cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(threads), args, smem, s), what);
}

size_t dd_smem(const FastArgs& a, TileCfg c) {
    return tma_smem(a, c) + (size_t)c.tpc * 2 * c.tl * 8;
}

template <int M, int UNI, int TLT, int SZC = 0>
int launch_dd_t(const DDArgs& A0, TileCfg cfg, cudaStream_t s) {
    DDArgs A = A0;
    FastArgs& a = A.t.f;
    // k_dd waits for an item's neighbour rows in the same iteration: it
    // keeps the round-robin schedule, under which a CTA and its partner on
    // the neighbour rank reach an item together (a dynamic schedule measured
    // 13.6 vs 21.1 TB/s on 4 GPUs; k_dd2's one-iteration deferral absorbs
    // the skew and gains from it)
    a.ctr = nullptr;
    a.tiles_per_cta = cfg.tpc;
    const long long tiles = (a.lines + TLT - 1) / TLT;
    a.items = (tiles + cfg.tpc - 1) / cfg.tpc;
    if (a.items <= 0) return TDS_OK;
    int rc = encode_field_map(a, M, TLT, &A.t.map, &A.t.boxr);
    if (rc) return rc;
    A.t.store_cs = store_policy();
    const int threads = cfg.tpc * a.chunks * TLT;
    const size_t smem = dd_smem(a, cfg);
    const void* fns[3] = {reinterpret_cast<const void*>(k_dd<M, TAB_GLOBAL, TLT, SZC>),
                          reinterpret_cast<const void*>(k_dd<M, TAB_UNIFORM, TLT, SZC>),
                          reinterpret_cast<const void*>(k_dd<M, TAB_EDGES, TLT, SZC>)};
    // at most the resident capacity (every CTA co-resident: no wait on an
    // unscheduled CTA), capped by max_ctas when several ranks share a device.
    // IDENTICAL on every rank: the minimum over the coefficient-table
    // variants, since neighbouring ranks may run different ones (edge ranks
    // of an open operator hold special chunks)
    // (max_ctas > 0: a grid the ranks agreed on, tds_fused_grid)
    long long grid = a.items;
    for (const void* f : fns) {
        if ((rc = ensure_smem(f, smem, "cudaFuncSetAttribute(k_dd)"))) return rc;
        if ((A.max_ctas > 0 || A.query) && f != fns[UNI]) continue;   // own variant
        grid = std::min(grid, persistent_grid(f, threads, smem, a.items, A.max_ctas));
    }
    if (A.query) return (int)std::min<long long>(grid, 1 << 30);
    if (grid < 1) return set_err(TDS_ERR_UNSUPPORTED, "k_dd does not fit on an SM");
    return launch_resident(reinterpret_cast<const void*>(k_dd<M, UNI, TLT, SZC>), grid, threads,
                           smem, s, A, "k_dd launch");
}

size_t dd2_smem(const FastArgs& a, TileCfg c, int M) {
    const int ne = c.tl == 32 ? 4 : 2;   // stash slots per tile (k_dd2 NE)
    return tma_smem(a, c) + (size_t)c.tpc * ne * (M + 1) * 32 * 8 +
           (size_t)4 * c.tpc * c.tl * 8 + (c.tl == 32 ? (size_t)2 * c.tpc * c.tl * 8 : 0);
}

template <int M, int UNI, int TLT, int SZC = 0>
int launch_dd2_t(const DDArgs& A0, TileCfg cfg, cudaStream_t s) {
    DDArgs A = A0;
    FastArgs& a = A.t.f;
    // keep >= 2 CTAs per SM: fewer tiles per CTA if the stash does not fit
    while (cfg.tpc > 1 && dd2_smem(a, cfg, M) > 110 * 1024) cfg.tpc /= 2;
    a.tiles_per_cta = cfg.tpc;
    const long long tiles = (a.lines + TLT - 1) / TLT;
    a.items = (tiles + cfg.tpc - 1) / cfg.tpc;
    if (a.items <= 0) return TDS_OK;
    int rc = encode_field_map(a, M, TLT, &A.t.map, &A.t.boxr);
    if (rc) return rc;
    const int threads = cfg.tpc * a.chunks * TLT;
    const size_t smem = dd2_smem(a, cfg, M);
    const void* fns[3] = {reinterpret_cast<const void*>(k_dd2<M, TAB_GLOBAL, TLT, SZC>),
                          reinterpret_cast<const void*>(k_dd2<M, TAB_UNIFORM, TLT, SZC>),
                          reinterpret_cast<const void*>(k_dd2<M, TAB_EDGES, TLT, SZC>)};
    long long grid = a.items;    // identical on every rank (see launch_dd_t)
    for (const void* f : fns) {
        if ((rc = ensure_smem(f, smem, "cudaFuncSetAttribute(k_dd2)"))) return rc;
        if ((A.max_ctas > 0 || A.query) && f != fns[UNI]) continue;   // own variant
        grid = std::min(grid, persistent_grid(f, threads, smem, a.items, A.max_ctas));
    }
    if (A.query) return (int)std::min<long long>(grid, 1 << 30);
    if (grid < 1) return set_err(TDS_ERR_UNSUPPORTED, "k_dd2 does not fit on an SM");
    return launch_resident(reinterpret_cast<const void*>(k_dd2<M, UNI, TLT, SZC>), grid, threads,
                           smem, s, A, "k_dd2 launch");
}

bool defer_policy() {
    if (const char* e = getenv("TDS_DEFER")) return e[0] != '0';
    return true;
}

template <int M, int UNI>
int launch_dd_m(const DDArgs& A, cudaStream_t s) {
    TileCfg cfg = tile_cfg(A.t.f);
    if (const char* e = getenv("TDS_DD_TPC")) cfg.tpc = std::max(1, atoi(e));
    // deferral pays only if some warps are interior (chunks > 2 warps' worth)
    const int cw = 32 / (cfg.tl ? cfg.tl : 16);
    const char* ev = getenv("TDS_DEFER");
    const bool force = ev && ev[0] == '2';
    const bool defer = defer_policy() && (force || A.t.f.chunks > 2 * cw) &&
                       (cfg.tl == 8 ? A.t.f.dd_defer8 : A.t.f.dd_defer16);
    if (cfg.tl == 8)
        return defer ? launch_dd2_t<M, UNI, 8>(A, cfg, s) : launch_dd_t<M, UNI, 8>(A, cfg, s);
    if constexpr (M == 32) {
        // k_dd2 with 32-line tiles (one chunk per warp; two edge warps and
        // four helper warps per tile, so >= 8 chunks: m >= 256) at two CTAs
        // per SM. Same choice on every rank (plan and sz only). Knob
        // TDS_DD2_TL32=0.
        const int C = A.t.f.chunks;
        if (defer && A.t.f.sz == 32 && C >= 8 && C * 32 <= 512 &&
            !(getenv("TDS_DD2_TL32") && getenv("TDS_DD2_TL32")[0] == '0') &&
            !(getenv("TDS_SZC") && getenv("TDS_SZC")[0] == '0')) {
            const int per_tile = C * 32;
            const TileCfg c32{32, per_tile >= 256 ? 1 : 256 / per_tile};
            if (dd2_smem(A.t.f, c32, M) <= 113 * 1024) return launch_dd2_t<M, UNI, 32, 32>(A, c32, s);
        }
    }
    if constexpr (M == 32) {
        // k_dd with 32-line tiles (one chunk per warp) when no deferral
        // applies and the block has more than 4 chunks. Same choice on every
        // rank: it depends on the plan and sz only. Knob TDS_DD_TL32=0.
        const bool tl32 = !defer && A.t.f.sz == 32 && A.t.f.chunks * 32 <= 512 &&
                          A.t.f.chunks > 4 &&
                          !(getenv("TDS_DD_TL32") && getenv("TDS_DD_TL32")[0] == '0') &&
                          !(getenv("TDS_SZC") && getenv("TDS_SZC")[0] == '0');
        if (tl32) {
            const int per_tile = A.t.f.chunks * 32;
            TileCfg c32{32, per_tile >= 256 ? 1 : 256 / per_tile};
            // TDS_DD_TPC: tiles per CTA (fewer, smaller CTAs keep more items
            // in flight per SM against the neighbour round trip)
            if (const char* e = getenv("TDS_DD_TPC")) c32.tpc = std::max(1, atoi(e));
            if (dd_smem(A.t.f, c32) <= 200 * 1024) return launch_dd_t<M, UNI, 32, 32>(A, c32, s);
        }
    }
    // k_dd on a short block (<= 4 chunks, m = 128 at N = 8: every chunk waits
    // for the neighbours' rows in its own iteration): one 16-line tile per
    // CTA, so 8 small CTAs per SM keep items in flight across the round
    // trip. Measured at m = 128 on 4 GPUs (512^3): per-rank 0.694 vs 0.619
    // for two 32-line tiles per CTA.
    if (!defer && A.t.f.chunks <= 4 && !getenv("TDS_DD_TPC")) cfg.tpc = 1;
    if constexpr (M == 32)
        if (A.t.f.sz == 32 && !(getenv("TDS_SZC") && getenv("TDS_SZC")[0] == '0'))
            return defer ? launch_dd2_t<M, UNI, 16, 32>(A, cfg, s)
                         : launch_dd_t<M, UNI, 16, 32>(A, cfg, s);
    return defer ? launch_dd2_t<M, UNI, 16>(A, cfg, s) : launch_dd_t<M, UNI, 16>(A, cfg, s);
}

}  // namespace

long long dd_mail_words(long long lines) { return Mail{lines}.words(); }

bool dd_eligible(int M, const FastArgs& a) {
    if (const char* e = getenv("TDS_FUSED"))
        if (e[0] == '0') return false;
    if (!tma_eligible(M, a)) return false;
    return dd_smem(a, tile_cfg(a)) <= 200 * 1024;
}

int launch_dd(int M, bool uniform, const FastArgs& a, double* mail, double* mail_prev,
              double* mail_next, unsigned long long epoch, int max_ctas, cudaStream_t s,
              bool query) {
    DDArgs A;
    std::memset(&A, 0, sizeof(A));
    A.max_ctas = max_ctas;
    A.query = query ? 1 : 0;
    A.t.f = a;
    A.mail = mail;
    A.mail_prev = mail_prev;
    A.mail_next = mail_next;
    A.epoch = epoch;
    A.timeout_ns = 10ULL * 1000 * 1000 * 1000;   // 10 s: a stall records an error
    A.t.band = a.Hb && a.nb > 0 && !(getenv("TDS_BAND") && getenv("TDS_BAND")[0] == '0');
    if (const char* e = getenv("TDS_FUSED_TIMEOUT_MS"))
        A.timeout_ns = (unsigned long long)atoll(e) * 1000000ULL;
    const int tab = !uniform ? TAB_GLOBAL
                    : (a.special_first || a.special_last) ? TAB_EDGES : TAB_UNIFORM;
#define DISPATCH_TAB(MM)                                                                \
    return tab == TAB_UNIFORM ? launch_dd_m<MM, TAB_UNIFORM>(A, s)                      \
           : tab == TAB_EDGES ? launch_dd_m<MM, TAB_EDGES>(A, s)                        \
                              : launch_dd_m<MM, TAB_GLOBAL>(A, s);
    if (M == 32) { DISPATCH_TAB(32) }
    if (M == 16) { DISPATCH_TAB(16) }
#undef DISPATCH_TAB
    return set_err(TDS_ERR_UNSUPPORTED, "unsupported chunk size");
}

// ===========================================================================
// k_dd_transport: one (i, j) term of the transport RHS along a direction
// that is split over the ranks (SlabTransport's z terms), as ONE kernel per
// rank: -1/2 (u_j d(u_i) + d(u_j u_i)) + nu d2(u_i) with the three compact
// solves of every chunk fused as in k_transport_tma (16-row chunks, running
// contribution in registers, u_i / u_j tiles by TMA read from shared memory)
// and each solve's two neighbour rounds done in-kernel as in k_dd: ROUND 1
// posts the first / last two rows of u_i and u_j one item ahead, ROUND 2
// posts each solve's g.Y and takes the neighbour's (2x2 pair -> pins). The
// reference's per-term pipeline (momentum.py:102-126 with run_distd2 over
// rank_count ranks) is three DistD2 solves + products; here the HBM traffic
// is u_i, u_j read once and the term written once (24 B/point).
//
// Mailbox (TrMail, 8-byte sentinel slots, two parity halves, 14 L used of 30):
//   DP(s) [L], s = 0..2   prev's d[m-1] of solve s
//   DN(s) [L]             next's d[0] of solve s
//   HLO_I, HLO_J [2L]     prev's last two rows of u_i, u_j
//   HHI_I, HHI_J [2L]     next's first two rows of u_i, u_j
// Deadlock freedom as k_dd: identical persistent schedule on every rank,
// posts before waits, waits only on the same CTA index of a neighbour.
// (The halves are 30 L apart and the status words sit at 60 L: the layout
// shared with k_dd_transport_dir, TdMail, so one mailbox serves both.)
struct TrMail {
    long long L;
    __host__ __device__ long long half(unsigned long long epoch) const {
        return (long long)(epoch & 1ULL) * 30 * L;
    }
    __host__ __device__ long long dp(int s) const { return s * L; }
    __host__ __device__ long long dn(int s) const { return (3 + s) * L; }
    __host__ __device__ long long hlo_i() const { return 6 * L; }
    __host__ __device__ long long hlo_j() const { return 8 * L; }
    __host__ __device__ long long hhi_i() const { return 10 * L; }
    __host__ __device__ long long hhi_j() const { return 12 * L; }
    __host__ __device__ long long err() const { return 60 * L; }
    __host__ __device__ long long words() const { return 60 * L + 3; }   // + status words
};

struct TrDDArgs {
    FastArgs f1, f2;           // rank plans: d/dx (f1), d2/dx2 (f2); Hp = pinned map
    CUtensorMap map_i, map_j;
    int boxr;
    const double* ui;
    const double* uj;
    double* out;
    double nu;
    int has_nu;
    long long lines;
    int rows, sz, chunks, tpc;
    long long items;
    int band;
    double* mail;
    double* mail_prev;
    double* mail_next;
    unsigned long long epoch;
    unsigned long long timeout_ns;
    int max_ctas;
    // in-place mode (XZ): the z lines of an x-layout (nx, ny, rows) slab,
    // the term added into `out` (x layout) by TMA reduce-add
    int nx, ny;
    CUtensorMap omap;
};

namespace {

template <int M, typename Src>
__device__ __forceinline__ void tr_sweeps(const UniformTable& T, Src v, double (&d)[M]) {
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

__device__ __forceinline__ double tr_subst(const UniformTable& T, int i, int M, double F,
                                           double L, double di) {
    return i == 0 ? F : (i == M - 1 ? L : fma(-T.sc[i], L, fma(-T.sa[i], F, di)));
}

}  // namespace

template <int TLT, int SZC, int XZ>
__global__ void __launch_bounds__(512, 1) k_dd_transport(const __grid_constant__ TrDDArgs A) {
    constexpr int M = 16;
    extern __shared__ __align__(1024) unsigned char smem[];
    const int C = A.chunks, K = 2 * C, rows = A.rows, tpc = A.tpc;
    const int t = threadIdx.x;
    const int lane = t % TLT;
    const int chunk = (t / TLT) % C;
    const int tl = t / (TLT * C);
    const long long sz = SZC ? SZC : A.sz;
    const int r0 = chunk * M;
    const TrMail mb{A.lines};
    const long long par = mb.half(A.epoch);
    unsigned long long* err = reinterpret_cast<unsigned long long*>(A.mail + mb.err());
    const size_t tile_elems = (size_t)rows * TLT;
    double* ti = reinterpret_cast<double*>(smem);
    double* tj = ti + (size_t)tpc * tile_elems;
    double* sY = tj + (size_t)tpc * tile_elems;           // [3][tpc][K][TLT]
    const size_t ybuf = (size_t)tpc * K * TLT;
    double* sP = sY + 3 * ybuf;                           // [3][tpc][2][TLT]
    UniformTable* sT = reinterpret_cast<UniformTable*>(sP + (size_t)3 * tpc * 2 * TLT);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sT + 2);
    const bool first_chunk = chunk == 0, last_chunk = chunk == C - 1;
    {
        const double* s1 = reinterpret_cast<const double*>(&A.f1.ut);
        const double* s2 = reinterpret_cast<const double*>(&A.f2.ut);
        double* dst = reinterpret_cast<double*>(sT);
        constexpr int W = sizeof(UniformTable) / sizeof(double);
        for (int k = t; k < 2 * W; k += blockDim.x) dst[k] = k < W ? s1[k] : s2[k - W];
    }
    const UniformTable& T1 = sT[0];
    const UniformTable& T2 = sT[1];

    // XZ: tile = TLT lanes of y-group gj at x (lane blocks fastest), z rows
    // at stride nx ny; a line's rows start at xz_base(line)
    const int nlb = XZ ? A.sz / TLT : 1, ngj = XZ ? A.ny / A.sz : 1;
    const long long rstride = XZ ? (long long)A.nx * A.ny : sz;
    auto xz_tile = [&](long long tile, int& l0, int& x, int& gj) {
        l0 = (int)(tile % nlb) * TLT;
        gj = (int)((tile / nlb) % ngj);
        x = (int)(tile / ((long long)nlb * ngj));
    };
    auto row0 = [&](long long ln) -> long long {
        if (XZ) {
            int l0, x, gj;
            xz_tile(ln / TLT, l0, x, gj);
            return ((long long)gj * A.nx + x) * sz + l0 + ln % TLT;
        }
        return line_base_t<SZC>(ln, rows, A.sz);
    };
    auto issue = [&](long long item) {
        uint32_t bytes = 0;
        for (int j = 0; j < tpc; ++j)
            if ((item * tpc + j) * TLT < A.lines)
                bytes += (uint32_t)(2 * tile_elems * sizeof(double));
        mbar_expect_tx(bar, bytes);
        for (int j = 0; j < tpc; ++j) {
            const long long first = (item * tpc + j) * TLT;
            if (first >= A.lines) break;
            if (XZ) {
                int l0, x, gj;
                xz_tile(first / TLT, l0, x, gj);
                for (int b = 0; b * A.boxr < rows; ++b) {
                    tma_load_4d(ti + j * tile_elems + (size_t)b * A.boxr * TLT, &A.map_i, bar, l0,
                                x, gj, b * A.boxr);
                    tma_load_4d(tj + j * tile_elems + (size_t)b * A.boxr * TLT, &A.map_j, bar, l0,
                                x, gj, b * A.boxr);
                }
                continue;
            }
            const int g = (int)(first / A.sz), l0 = (int)(first % A.sz);
            for (int b = 0; b * A.boxr < rows; ++b) {
                tma_load_3d(ti + j * tile_elems + (size_t)b * A.boxr * TLT, &A.map_i, bar, l0,
                            b * A.boxr, g);
                tma_load_3d(tj + j * tile_elems + (size_t)b * A.boxr * TLT, &A.map_j, bar, l0,
                            b * A.boxr, g);
            }
        }
    };
    // XZ: add the staged term (tile i, load layout) into out by TMA
    auto reduce_out = [&](long long item) {
        for (int j = 0; j < tpc; ++j) {
            const long long first = (item * tpc + j) * TLT;
            if (first >= A.lines) break;
            int l0, x, gj;
            xz_tile(first / TLT, l0, x, gj);
            for (int b = 0; b * A.boxr < rows; ++b)
                tma_reduce_add_4d(&A.omap, ti + j * tile_elems + (size_t)b * A.boxr * TLT, l0, x,
                                  gj, b * A.boxr);
        }
        bulk_commit();
    };
    // ROUND 1 of `item`: first two rows of u_i, u_j -> prev, last two -> next
    auto publish_halo = [&](long long item) {
        if (!first_chunk && !last_chunk) return;
        const long long ln = (item * tpc + tl) * TLT + lane;
        if (ln >= A.lines) return;
        const long long lb = row0(ln);
        const double* bi = A.ui + lb;
        const double* bj = A.uj + lb;
        const long long hb = halo_base_t<SZC>(ln, A.sz);
        if (first_chunk && A.mail_prev) {
            double* m = A.mail_prev + par;
            post(m + mb.hhi_i() + hb, __ldg(bi));
            post(m + mb.hhi_i() + hb + sz, __ldg(bi + rstride));
            post(m + mb.hhi_j() + hb, __ldg(bj));
            post(m + mb.hhi_j() + hb + sz, __ldg(bj + rstride));
        }
        if (last_chunk && A.mail_next) {
            double* m = A.mail_next + par;
            const long long a = (long long)(rows - 2) * rstride, b = (long long)(rows - 1) * rstride;
            post(m + mb.hlo_i() + hb, __ldg(bi + a));
            post(m + mb.hlo_i() + hb + sz, __ldg(bi + b));
            post(m + mb.hlo_j() + hb, __ldg(bj + a));
            post(m + mb.hlo_j() + hb + sz, __ldg(bj + b));
        }
    };
    auto release = [&](long long nxt) {
        __syncthreads();
        if (t == 0 && nxt < A.items) {
            fence_proxy_async();
            issue(nxt);
        }
    };

    if (t == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    long long item = blockIdx.x;
    if (item < A.items) {
        if (t == 0) issue(item);
        publish_halo(item);
    }
    uint32_t phase = 0;
    const double* Ti = ti + tl * tile_elems;
    const double* Tj = tj + tl * tile_elems;
    const int base = (r0 - 2) * TLT + lane;

    for (; item < A.items; item += gridDim.x) {
        const long long line = (item * tpc + tl) * TLT + lane;
        const bool valid = line < A.lines;
        const long long nxt = item + gridDim.x;
        if (nxt < A.items) publish_halo(nxt);            // one item ahead
        const long long hb = valid ? halo_base_t<SZC>(line, A.sz) : 0;
        const bool hlo = valid && first_chunk && A.mail_prev;
        const bool hhi = valid && last_chunk && A.mail_next;
        // halo slots of this item: the four loads in flight together, across
        // the TMA wait (a serial take() each would put four L2 round trips
        // on the edge threads' critical path)
        double* hs = A.mail + par + (hlo ? mb.hlo_i() : mb.hhi_i()) + hb;
        double* hsj = A.mail + par + (hlo ? mb.hlo_j() : mb.hhi_j()) + hb;
        unsigned long long s0 = SENTINEL, s1 = SENTINEL, s2 = SENTINEL, s3 = SENTINEL;
        if (hlo || hhi) {
            s0 = ld_sys_u64(hs);
            s1 = ld_sys_u64(hs + sz);
            s2 = ld_sys_u64(hsj);
            s3 = ld_sys_u64(hsj + sz);
        }
        while (!mbar_try_wait(bar, phase)) {
        }
        phase ^= 1u;
        // rank-edge halos of u_i and u_j (ROUND 1 of this item)
        double hi0 = 0.0, hi1 = 0.0, hi2 = 0.0, hi3 = 0.0;
        double hj0 = 0.0, hj1 = 0.0, hj2 = 0.0, hj3 = 0.0;
        if (hlo || hhi) {
            const double a0 = take_v(hs, s0, A, err), a1 = take_v(hs + sz, s1, A, err);
            const double b0 = take_v(hsj, s2, A, err), b1 = take_v(hsj + sz, s3, A, err);
            if (hlo) { hi0 = a0; hi1 = a1; hj0 = b0; hj1 = b1; }
            else { hi2 = a0; hi3 = a1; hj2 = b0; hj3 = b1; }
        }
        // window row i (= block row r0 - 2 + i) of u_i / u_j
        auto wi = [&](int i) {
            if (i < 2 && first_chunk) return i == 0 ? hi0 : hi1;
            if (i >= M + 2 && last_chunk) return i == M + 2 ? hi2 : hi3;
            return Ti[base + i * TLT];
        };
        auto wj = [&](int i) {
            if (i < 2 && first_chunk) return i == 0 ? hj0 : hj1;
            if (i >= M + 2 && last_chunk) return i == M + 2 ? hj2 : hj3;
            return Tj[base + i * TLT];
        };
        double acc[M], d[M];
        double F, L;
        // Each solve: Y, ROUND 2 posts, and the pin-free chunk boundary values
        // (F, L); the pins of all three solves are taken once at the end of
        // the item and applied as a correction (x is affine in the pins:
        // x_i += dx_i(dF, dL) with dF = h0.x us + hl.x ue, dL = h0.y us +
        // hl.y ue), so the three neighbour round trips overlap the item.
        auto post_bounds = [&](int s, const FastArgs& p) {
            double* Y = sY + (size_t)s * ybuf + (size_t)tl * K * TLT;
            Y[(2 * chunk) * TLT + lane] = d[0];
            Y[(2 * chunk + 1) * TLT + lane] = d[M - 1];
            __syncthreads();
            double* P = sP + ((size_t)s * tpc + tl) * 2 * TLT;
            if (valid && (first_chunk || last_chunk)) {
                // own rows now (g0.Y / g1.Y); the pair solve comes at the end
                if (first_chunk) {
                    const double g0y = gdot<TLT>(p, 0, Y, K, lane);
                    if (A.mail_prev) {
                        post(A.mail_prev + par + mb.dn(s) + line, g0y);
                            }
                    P[lane] = g0y;
                }
                if (last_chunk) {
                    const double g1y = gdot<TLT>(p, 1, Y, K, lane);
                    if (A.mail_next) {
                        post(A.mail_next + par + mb.dp(s) + line, g1y);
                            }
                    P[TLT + lane] = g1y;
                }
            }
            if (A.band)
                band_bounds_nopins<TLT>(p.Hb + (size_t)chunk * p.nb, __ldg(p.bq0 + chunk), p.nb,
                                        Y, K, lane, F, L);
            else
                chunk_bounds<TLT>(p.Hp + (size_t)chunk * K + 1, Y + TLT, K - 2, lane, nullptr,
                                  nullptr, F, L);
        };
        // the neighbours' rows of solve s -> 2x2 pairs -> pins in P (edge threads)
        auto take_pins = [&](int s, const FastArgs& p, unsigned long long v) {
            double* P = sP + ((size_t)s * tpc + tl) * 2 * TLT;
            if (!valid) return;
            if (first_chunk && p.has_prev) {
                const double prev_last = take_v(A.mail + par + mb.dp(s) + line, v, A, err);
                P[lane] = (P[lane] - p.sa_first * prev_last) / p.det_prev;
            }
            if (last_chunk && p.has_next) {
                const double next_first = take_v(A.mail + par + mb.dn(s) + line, v, A, err);
                P[TLT + lane] = (P[TLT + lane] - p.sc_last * next_first) / p.det_next;
            }
        };
        // the pin slot this thread reads for solve s (edge threads), loaded early
        auto pin_slot = [&](int s) -> double* {
            return A.mail + par + (first_chunk ? mb.dp(s) : mb.dn(s)) + line;
        };
        // pin correction of solve s, scaled by w (and by u_j for solve A)
        auto correct = [&](int s, const FastArgs& p, const UniformTable& T, double w, bool by_uj) {
            const double* P = sP + ((size_t)s * tpc + tl) * 2 * TLT;
            const double2 h0 = __ldg(p.Hp + (size_t)chunk * K);
            const double2 hl = __ldg(p.Hp + (size_t)chunk * K + K - 1);
            const double us = P[lane], ue = P[TLT + lane];
            const double dF = fma(h0.x, us, hl.x * ue), dL = fma(h0.y, us, hl.y * ue);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                double dx = i == 0 ? dF : (i == M - 1 ? dL : -fma(T.sc[i], dL, T.sa[i] * dF));
                if (by_uj) dx *= Tj[base + (i + 2) * TLT];
                acc[i] = fma(w, dx, acc[i]);
            }
        };

        // (A) d(u_i) -> acc = u_j * du_i   (pin-free part)
        tr_sweeps<M>(T1, wi, d);
        post_bounds(0, A.f1);
#pragma unroll
        for (int i = 0; i < M; ++i) acc[i] = Tj[base + (i + 2) * TLT] * tr_subst(T1, i, M, F, L, d[i]);
        // (B) d(u_j u_i) -> acc = -1/2 (acc + dprod)
        tr_sweeps<M>(T1, [&](int i) { return wj(i) * wi(i); }, d);
        post_bounds(1, A.f1);
#pragma unroll
        for (int i = 0; i < M; ++i) acc[i] = -0.5 * (acc[i] + tr_subst(T1, i, M, F, L, d[i]));
        // (C) acc += nu d2(u_i)
        if (A.has_nu) {
            tr_sweeps<M>(T2, wi, d);
            post_bounds(2, A.f2);
#pragma unroll
            for (int i = 0; i < M; ++i) acc[i] = fma(A.nu, tr_subst(T2, i, M, F, L, d[i]), acc[i]);
        }
        // the three solves' pins (one wait point: the slot loads in flight
        // together) and their corrections
        unsigned long long v0 = SENTINEL, v1 = SENTINEL, v2 = SENTINEL;
        if (valid && ((first_chunk && A.f1.has_prev) || (last_chunk && A.f1.has_next))) {
            v0 = ld_sys_u64(pin_slot(0));
            v1 = ld_sys_u64(pin_slot(1));
            if (A.has_nu) v2 = ld_sys_u64(pin_slot(2));
        }
        take_pins(0, A.f1, v0);
        take_pins(1, A.f1, v1);
        if (A.has_nu) take_pins(2, A.f2, v2);
        __syncthreads();
        correct(0, A.f1, T1, -0.5, true);
        correct(1, A.f1, T1, -0.5, false);
        if (A.has_nu) correct(2, A.f2, T2, A.nu, false);
        if (XZ) {
            // the term goes into tile i (its last reader was the sweeps,
            // before the pin barrier) and is added into out by the TMA
            // engine; the tiles are re-armed once it has read them
            double* Tw = ti + tl * tile_elems;
#pragma unroll
            for (int i = 0; i < M; ++i) Tw[base + (i + 2) * TLT] = acc[i];
            fence_proxy_async();
            __syncthreads();
            if (t == 0) {
                reduce_out(item);
                if (nxt < A.items) {
                    bulk_wait_read<0>();
                    issue(nxt);
                }
            }
        } else {
            release(nxt);         // tiles consumed (u_j rows of the A correction)
            if (valid) {
                double* ob = A.out + line_base_t<SZC>(line, rows, A.sz) + (long long)r0 * sz;
#pragma unroll
                for (int i = 0; i < M; ++i) __stcs(ob + (long long)i * sz, acc[i]);
            }
        }
    }
    if (XZ && t == 0) bulk_wait_all();   // the last reduces complete before exit
    {
        const unsigned n = valid_items(A.items, A.lines, tpc, tl, TLT, lane);
        const unsigned per = (first_chunk && A.mail_prev ? 1u : 0u) + (last_chunk && A.mail_next ? 1u : 0u);
        // u_i and u_j halos (4 rows) + one boundary row per solve
        flush_counts(err, 4 * per * n, (A.has_nu ? 3u : 2u) * per * n);
    }
}

namespace {

template <int TLT, int SZC, int XZ = 0>
int launch_dd_transport_t(const TrDDArgs& A0, cudaStream_t s) {
    TrDDArgs A = A0;
    const int per_tile = A.chunks * TLT;
    A.tpc = per_tile >= 256 ? 1 : 256 / per_tile;
    const long long tiles = (A.lines + TLT - 1) / TLT;
    A.items = (tiles + A.tpc - 1) / A.tpc;
    if (A.items <= 0) return TDS_OK;
    FastArgs fi{}, fj{};
    fi.u = A.ui;
    fj.u = A.uj;
    fi.rows = fj.rows = A.rows;
    fi.sz = fj.sz = A.sz;
    fi.lines = fj.lines = A.lines;
    int rc;
    if (XZ) {
        if ((rc = encode_xz_map(A.ui, A.nx, A.ny, A.rows, A.sz, 16, TLT, &A.map_i, &A.boxr)) ||
            (rc = encode_xz_map(A.uj, A.nx, A.ny, A.rows, A.sz, 16, TLT, &A.map_j, &A.boxr)) ||
            (rc = encode_xz_map(A.out, A.nx, A.ny, A.rows, A.sz, 16, TLT, &A.omap, &A.boxr)))
            return rc;
    } else {
        if ((rc = encode_field_map(fi, 16, TLT, &A.map_i, &A.boxr))) return rc;
        if ((rc = encode_field_map(fj, 16, TLT, &A.map_j, &A.boxr))) return rc;
    }
    const int threads = A.tpc * per_tile;
    const size_t smem = (size_t)A.tpc *
                            (2 * (size_t)A.rows * TLT + 3 * (size_t)2 * A.chunks * TLT +
                             3 * 2 * TLT) * sizeof(double) +
                        2 * sizeof(UniformTable) + 16;
    const void* fn = reinterpret_cast<const void*>(k_dd_transport<TLT, SZC, XZ>);
    if ((rc = ensure_smem(fn, smem, "cudaFuncSetAttribute(k_dd_transport)"))) return rc;
    // co-resident, identical on every rank (max_ctas: ranks sharing a device)
    const long long grid = persistent_grid(fn, threads, smem, A.items, A.max_ctas);
    if (grid < 1) return set_err(TDS_ERR_UNSUPPORTED, "k_dd_transport does not fit on an SM");
    return launch_resident(fn, grid, threads, smem, s, A, "k_dd_transport launch");
}

}  // namespace

long long dd_transport_mail_words(long long lines) { return TrMail{lines}.words(); }
long long dd_transport_err_word(long long lines) { return TrMail{lines}.err(); }

int launch_dd_transport(const FastArgs& f1, const FastArgs& f2, const double* ui,
                        const double* uj, double* out, double nu, long long lines, int sz,
                        double* mail, double* mail_prev, double* mail_next,
                        unsigned long long epoch, int max_ctas, cudaStream_t s, int nx, int ny) {
    TrDDArgs A;
    std::memset(&A, 0, sizeof(A));
    A.nx = nx;
    A.ny = ny;
    A.max_ctas = max_ctas;
    A.f1 = f1;
    A.f2 = f2;
    A.ui = ui;
    A.uj = uj;
    A.out = out;
    A.nu = nu;
    A.has_nu = nu != 0.0;
    A.lines = lines;
    A.rows = f1.rows;
    A.sz = sz;
    A.chunks = f1.chunks;
    A.band = f1.Hb && f1.nb > 0 && (!A.has_nu || (f2.Hb && f2.nb > 0)) &&
             !(getenv("TDS_BAND") && getenv("TDS_BAND")[0] == '0');
    A.mail = mail;
    A.mail_prev = mail_prev;
    A.mail_next = mail_next;
    A.epoch = epoch;
    A.timeout_ns = 10ULL * 1000 * 1000 * 1000;
    if (const char* e = getenv("TDS_FUSED_TIMEOUT_MS"))
        A.timeout_ns = (unsigned long long)atoll(e) * 1000000ULL;
    int tl = 16;
    if (const char* e = getenv("TDS_TRANSPORT_TL")) tl = atoi(e) == 8 ? 8 : 16;
    if (nx > 0) {
        // in place from the x layout (the z lines of a slab), added into out
        if (ny % sz || reinterpret_cast<uintptr_t>(out) % 16)
            return set_err(TDS_ERR_UNSUPPORTED, "in-place distributed transport: sz | ny");
        if (tl == 16 && sz % 16 == 0 && A.chunks * 16 <= 512)
            return launch_dd_transport_t<16, 0, 1>(A, s);
        if (sz % 8 == 0 && A.chunks * 8 <= 512) return launch_dd_transport_t<8, 0, 1>(A, s);
        return set_err(TDS_ERR_UNSUPPORTED, "in-place distributed transport: tile");
    }
    if (tl == 16 && sz % 16 == 0 && A.chunks * 16 <= 512) {
        if (sz == 32) return launch_dd_transport_t<16, 32>(A, s);
        return launch_dd_transport_t<16, 0>(A, s);
    }
    if (sz % 8 == 0 && A.chunks * 8 <= 512) {
        if (sz == 32) return launch_dd_transport_t<8, 32>(A, s);
        return launch_dd_transport_t<8, 0>(A, s);
    }
    return set_err(TDS_ERR_UNSUPPORTED, "fused distributed transport: sz % 8, tile <= 512 threads");
}


// ===========================================================================
// k_dd_transport_dir: the three z contributions (components i = 0, 1, 2) of
// a rank's z-slab in ONE kernel per rank -- k_transport_dir's schedule with
// k_dd_transport's neighbour rounds. The slab stays in the x layout: u_0..u_2
// tiles (TLT lanes x m z-rows) arrive by TMA through 4-D tensor maps, each
// on its own mbarrier, into tiles with two spare rows at each end that the
// rank-edge threads fill from the neighbours' halo posts; every phase's
// result is staged in its freed tile and added into the accumulator by TMA
// reduce-add. HBM: u_0..u_2 read once, three accumulators read-modify-
// written in L2: 72 B/pt, against 96 for three k_dd_transport launches and
// 192 for the reorder pipeline.
//
// Per item: ROUND 1 posts the first / last two rows of u_0..u_2 one item
// ahead. Per component phase (order a, b, j as k_transport_dir): pass 1
// (d/dx and d2/dx2 of u_c, one window read), pass 2 (d/dx of u_j u_c); after
// each pass's barrier the rank-edge threads post that pass's g0.Y / g1.Y
// (ROUND 2) and every chunk forms its pin-free (F, L). At the end of the
// phase the edge threads take the neighbours' three rows (posted a pass or
// more earlier), form the 2x2 pins, and every chunk applies the affine pin
// correction before staging. Deadlock freedom as k_dd: identical persistent
// schedules, posts before waits, waits only on the same CTA index of a
// neighbour in the same or an earlier iteration.
//
// Mailbox (TdMail, sentinel slots, two parity halves of 30 L; the layout of
// TrMail's status words):
//   DP(s), DN(s) [L] s = 3 c + k (k: 0 d/dx, 1 d2/dx2, 2 d/dx of u_j u_c)
//   HLO(c), HHI(c) [2L]   prev's last / next's first two rows of u_c
struct TdMail {
    long long L;
    __host__ __device__ long long half(unsigned long long epoch) const {
        return (long long)(epoch & 1ULL) * 30 * L;
    }
    __host__ __device__ long long dp(int s) const { return s * L; }
    __host__ __device__ long long dn(int s) const { return (9 + s) * L; }
    __host__ __device__ long long hlo(int c) const { return (18 + 2 * c) * L; }
    __host__ __device__ long long hhi(int c) const { return (24 + 2 * c) * L; }
    __host__ __device__ long long err() const { return 60 * L; }
    __host__ __device__ long long words() const { return 60 * L + 3; }
};

struct TdArgs {
    FastArgs f1, f2;           // rank plans: d/dx (f1), d2/dx2 (f2)
    CUtensorMap map[3], omap[3];
    const double* u[3];
    double* out[3];
    int boxr;
    double nu;
    int has_nu;
    long long lines;
    int rows, sz, chunks, tpc, nx, ny;
    long long items;
    double* mail;
    double* mail_prev;
    double* mail_next;
    unsigned long long epoch;
    unsigned long long timeout_ns;
    int max_ctas;
};

template <int TLT>
__global__ void __launch_bounds__(512, 1) k_dd_transport_dir(const __grid_constant__ TdArgs A) {
    constexpr int M = 16;
    extern __shared__ __align__(1024) unsigned char smem[];
    const int C = A.chunks, K = 2 * C, rows = A.rows, tpc = A.tpc;
    const int t = threadIdx.x;
    const int lane = t % TLT;
    const int chunk = (t / TLT) % C;
    const int tl = t / (TLT * C);
    const long long sz = A.sz;
    const int r0 = chunk * M;
    const TdMail mb{A.lines};
    const long long par = mb.half(A.epoch);
    unsigned long long* err = reinterpret_cast<unsigned long long*>(A.mail + mb.err());
    const bool first_chunk = chunk == 0, last_chunk = chunk == C - 1;
    // tiles with two spare rows at each end: [3][tpc][rows + 4][TLT]
    const size_t tile_elems = (size_t)(rows + 4) * TLT;
    const size_t field_elems = (size_t)tpc * tile_elems;
    double* tiles = reinterpret_cast<double*>(smem);
    double* sY = tiles + 3 * field_elems;                        // [3][tpc][K][TLT]
    const size_t ybuf = (size_t)tpc * K * TLT;
    double* sP = sY + 3 * ybuf;                                  // [3][tpc][2][TLT]
    DirRow* sR = reinterpret_cast<DirRow*>(sP + (size_t)3 * tpc * 2 * TLT);
    double* sst = reinterpret_cast<double*>(sR + M);             // stencils [2][5] (+ pad)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sst + 12);
    const FastArgs& p1 = A.f1;
    const FastArgs& p2 = A.f2;
    for (int i = t; i < M; i += blockDim.x) {
        DirRow r;
        r.rf1 = make_double2(p1.ut.r[i], p1.ut.f[i]);
        r.rf2 = make_double2(p2.ut.r[i], p2.ut.f[i]);
        r.w12 = make_double2(p1.ut.w[i], p2.ut.w[i]);
        r.s1 = make_double2(p1.ut.sa[i], p1.ut.sc[i]);
        r.s2 = make_double2(p2.ut.sa[i], p2.ut.sc[i]);
        sR[i] = r;
    }
    if (t < 10) sst[t] = t < 5 ? p1.ut.st[t] : p2.ut.st[t - 5];
    const DirRow (&RT)[16] = *reinterpret_cast<const DirRow(*)[16]>(sR);
    const double* st1 = sst;
    const double* st2 = sst + 5;
    const int jd = 2;                              // the slab's split direction: z
    const int ca = 0, cb = 1;
    const int nlb = A.sz / TLT, ngj = A.ny / A.sz;
    const long long rs = (long long)A.nx * A.ny;   // z-row stride
    auto xz_tile = [&](long long tile, int& l0, int& x, int& gj) {
        l0 = (int)(tile % nlb) * TLT;
        gj = (int)((tile / nlb) % ngj);
        x = (int)(tile / ((long long)nlb * ngj));
    };
    auto row0 = [&](long long ln) -> long long {
        int l0, x, gj;
        xz_tile(ln / TLT, l0, x, gj);
        return ((long long)gj * A.nx + x) * sz + l0 + ln % TLT;
    };
    auto issue = [&](int c, long long item) {
        uint32_t bytes = 0;
        for (int q = 0; q < tpc; ++q)
            if ((item * tpc + q) * TLT < A.lines) bytes += (uint32_t)((size_t)rows * TLT * 8);
        mbar_expect_tx(bar + c, bytes);
        for (int q = 0; q < tpc; ++q) {
            const long long first = (item * tpc + q) * TLT;
            if (first >= A.lines) break;
            int l0, x, gj;
            xz_tile(first / TLT, l0, x, gj);
            double* dst = tiles + c * field_elems + q * tile_elems + 2 * TLT;
            for (int b = 0; b * A.boxr < rows; ++b)
                tma_load_4d(dst + (size_t)b * A.boxr * TLT, &A.map[c], bar + c, l0, x, gj,
                            b * A.boxr);
        }
    };
    auto reduce_out = [&](int c, long long item) {
        for (int q = 0; q < tpc; ++q) {
            const long long first = (item * tpc + q) * TLT;
            if (first >= A.lines) break;
            int l0, x, gj;
            xz_tile(first / TLT, l0, x, gj);
            const double* src = tiles + c * field_elems + q * tile_elems + 2 * TLT;
            for (int b = 0; b * A.boxr < rows; ++b)
                tma_reduce_add_4d(&A.omap[c], src + (size_t)b * A.boxr * TLT, l0, x, gj,
                                  b * A.boxr);
        }
        bulk_commit();
    };
    // ROUND 1 of `item`: first two rows of u_0..u_2 -> prev, last two -> next
    auto publish_halo = [&](long long item) {
        if (!first_chunk && !last_chunk) return;
        const long long ln = (item * tpc + tl) * TLT + lane;
        if (ln >= A.lines) return;
        const long long o = row0(ln);
        const long long hb = halo_base(ln, A.sz);
        for (int c = 0; c < 3; ++c) {
            const double* b = A.u[c] + o;
            if (first_chunk && A.mail_prev) {
                double* m = A.mail_prev + par + mb.hhi(c) + hb;
                post(m, __ldg(b));
                post(m + sz, __ldg(b + rs));
            }
            if (last_chunk && A.mail_next) {
                double* m = A.mail_next + par + mb.hlo(c) + hb;
                post(m, __ldg(b + (long long)(rows - 2) * rs));
                post(m + sz, __ldg(b + (long long)(rows - 1) * rs));
            }
        }
    };

    if (t == 0) {
        for (int c = 0; c < 3; ++c) mbar_init(bar + c, 1);
        fence_mbar_init();
    }
    __syncthreads();
    long long item = blockIdx.x;
    if (item < A.items) {
        if (t == 0) {
            issue(ca, item);
            issue(jd, item);
            issue(cb, item);
        }
        publish_halo(item);
    }
    uint32_t phases = 0;
    int pend = -1;
    auto wait_tile = [&](int c) {
        const uint32_t ph = (phases >> c) & 1u;
        while (!mbar_try_wait(bar + c, ph)) {
        }
        phases ^= 1u << c;
    };
    // window row i of the chunk (block row r0 - 2 + i) in an extended tile
    const int wbase = r0 * TLT + lane;
    double* Y0 = sY + (size_t)tl * K * TLT;
    double* YA = Y0;
    double* YB = Y0 + ybuf;
    double* YC = Y0 + 2 * ybuf;
    double* P = sP + (size_t)tl * 2 * TLT;        // + k * tpc * 2 * TLT: solve k of the phase
    const size_t pstride = (size_t)tpc * 2 * TLT;
    const int bq1 = __ldg(p1.bq0 + chunk), bq2 = __ldg(p2.bq0 + chunk);

    for (; item < A.items; item += gridDim.x) {
        const long long line = (item * tpc + tl) * TLT + lane;
        const bool valid = line < A.lines;
        const long long nxt = item + gridDim.x;
        if (nxt < A.items) publish_halo(nxt);                 // one item ahead
        const bool hlo = valid && first_chunk && A.mail_prev;
        const bool hhi = valid && last_chunk && A.mail_next;
        const long long hb = valid ? halo_base(line, A.sz) : 0;
        // rank-edge halos of this item -> the spare rows of the three tiles
        // (only this thread reads them back: no barrier)
        if (hlo || hhi) {
            unsigned long long v[6];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double* hs = A.mail + par + (hlo ? mb.hlo(c) : mb.hhi(c)) + hb;
                v[2 * c] = ld_sys_u64(hs);
                v[2 * c + 1] = ld_sys_u64(hs + sz);
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double* hs = A.mail + par + (hlo ? mb.hlo(c) : mb.hhi(c)) + hb;
                const double a0 = take_v(hs, v[2 * c], A, err);
                const double a1 = take_v(hs + sz, v[2 * c + 1], A, err);
                double* T = tiles + c * field_elems + tl * tile_elems;
                const int o = hlo ? lane : (rows + 2) * TLT + lane;
                T[o] = a0;
                T[o + TLT] = a1;
            }
        }
        const double* Tj = tiles + jd * field_elems + tl * tile_elems;
#pragma unroll 1
        for (int s = 0; s < 3; ++s) {
            const int c = s == 0 ? ca : (s == 1 ? cb : jd);
            double* Tc = tiles + c * field_elems + tl * tile_elems;
            if (c != jd) wait_tile(c);
            double acc[M], d[M];
            double F, L, F2, L2;
            // ROUND 2 of solve k after its barrier: own boundary rows (g.Y)
            // to the neighbours, kept in P for the pair solve
            auto round2 = [&](int k, const FastArgs& p, const double* Y) {
                if (!valid || (!first_chunk && !last_chunk)) return;
                const int sid = 3 * c + k;
                double* Pk = P + k * pstride;
                if (first_chunk) {
                    const double g0y = gdot<TLT>(p, 0, Y, K, lane);
                    if (A.mail_prev) post(A.mail_prev + par + mb.dn(sid) + line, g0y);
                    Pk[lane] = g0y;
                }
                if (last_chunk) {
                    const double g1y = gdot<TLT>(p, 1, Y, K, lane);
                    if (A.mail_next) post(A.mail_next + par + mb.dp(sid) + line, g1y);
                    Pk[TLT + lane] = g1y;
                }
            };

            // pass 1: d(u_c) and d2(u_c) from one read of the window
            if (A.has_nu) {
                double d2[M];
                dsweeps2<M>(RT, st1, st2, [&](int i) { return Tc[wbase + i * TLT]; }, d, d2);
                YA[(2 * chunk) * TLT + lane] = d[0];
                YA[(2 * chunk + 1) * TLT + lane] = d[M - 1];
                YC[(2 * chunk) * TLT + lane] = d2[0];
                YC[(2 * chunk + 1) * TLT + lane] = d2[M - 1];
                __syncthreads();
                if (t == 0 && pend >= 0) {
                    bulk_wait_read<0>();
                    issue(pend, nxt);
                    pend = -1;
                }
                if (s == 0) wait_tile(jd);
                round2(0, p1, YA);
                round2(1, p2, YC);
                band_bounds_nopins<TLT>(p1.Hb + (size_t)chunk * p1.nb, bq1, p1.nb, YA, K, lane, F,
                                        L);
                band_bounds_nopins<TLT>(p2.Hb + (size_t)chunk * p2.nb, bq2, p2.nb, YC, K, lane, F2,
                                        L2);
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const DirRow& R = RT[i];
                    acc[i] = fma(-0.5 * Tj[wbase + (i + 2) * TLT], subst2(R.s1, i, M, F, L, d[i]),
                                 A.nu * subst2(R.s2, i, M, F2, L2, d2[i]));
                }
            } else {
                dsweeps1<M>(RT, st1, [&](int i) { return Tc[wbase + i * TLT]; }, d);
                YA[(2 * chunk) * TLT + lane] = d[0];
                YA[(2 * chunk + 1) * TLT + lane] = d[M - 1];
                __syncthreads();
                if (t == 0 && pend >= 0) {
                    bulk_wait_read<0>();
                    issue(pend, nxt);
                    pend = -1;
                }
                if (s == 0) wait_tile(jd);
                round2(0, p1, YA);
                band_bounds_nopins<TLT>(p1.Hb + (size_t)chunk * p1.nb, bq1, p1.nb, YA, K, lane, F,
                                        L);
#pragma unroll
                for (int i = 0; i < M; ++i)
                    acc[i] = -0.5 * Tj[wbase + (i + 2) * TLT] * subst2(RT[i].s1, i, M, F, L, d[i]);
            }
            // pass 2: d(u_j u_c)
            dsweeps1<M>(RT, st1,
                        [&](int i) { return Tj[wbase + i * TLT] * Tc[wbase + i * TLT]; }, d);
            YB[(2 * chunk) * TLT + lane] = d[0];
            YB[(2 * chunk + 1) * TLT + lane] = d[M - 1];
            __syncthreads();
            round2(2, p1, YB);
            band_bounds_nopins<TLT>(p1.Hb + (size_t)chunk * p1.nb, bq1, p1.nb, YB, K, lane, F, L);
#pragma unroll
            for (int i = 0; i < M; ++i) acc[i] = fma(-0.5, subst2(RT[i].s1, i, M, F, L, d[i]), acc[i]);

            // the neighbours' rows of the phase's solves -> 2x2 pairs -> pins
            if (valid && ((first_chunk && p1.has_prev) || (last_chunk && p1.has_next))) {
                const int nk = A.has_nu ? 3 : 2;
                unsigned long long v[3] = {SENTINEL, SENTINEL, SENTINEL};
                double* slot[3];
                for (int k = 0; k < 3; ++k) {
                    const int kk = k == 1 ? 2 : (k == 2 ? 1 : 0);   // A, B, C
                    const int sid = 3 * c + kk;
                    slot[k] = A.mail + par + (first_chunk ? mb.dp(sid) : mb.dn(sid)) + line;
                    if (k < nk) v[k] = ld_sys_u64(slot[k]);
                }
                for (int k = 0; k < nk; ++k) {
                    const int kk = k == 1 ? 2 : (k == 2 ? 1 : 0);
                    const FastArgs& p = kk == 1 ? p2 : p1;
                    double* Pk = P + kk * pstride;
                    const double nb_row = take_v(slot[k], v[k], A, err);
                    if (first_chunk) Pk[lane] = (Pk[lane] - p.sa_first * nb_row) / p.det_prev;
                    else Pk[TLT + lane] = (Pk[TLT + lane] - p.sc_last * nb_row) / p.det_next;
                }
            }
            __syncthreads();
            // affine pin corrections: x += dx(dF, dL), dF = h0.x us + hl.x ue
            auto correct = [&](int k, const FastArgs& p, double w, bool by_uj, bool second) {
                const double* Pk = P + k * pstride;
                const double2 h0 = __ldg(p.Hp + (size_t)chunk * K);
                const double2 hl = __ldg(p.Hp + (size_t)chunk * K + K - 1);
                const double us = Pk[lane], ue = Pk[TLT + lane];
                const double dF = fma(h0.x, us, hl.x * ue), dL = fma(h0.y, us, hl.y * ue);
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const double2 sc = second ? RT[i].s2 : RT[i].s1;
                    double dx = i == 0 ? dF : (i == M - 1 ? dL : -fma(sc.y, dL, sc.x * dF));
                    if (by_uj) dx *= Tj[wbase + (i + 2) * TLT];
                    acc[i] = fma(w, dx, acc[i]);
                }
            };
            correct(0, p1, -0.5, true, false);
            correct(2, p1, -0.5, false, false);
            if (A.has_nu) correct(1, p2, A.nu, false, true);
            // stage in tile c (every read of it is done: own rows only) and
            // add into out[c] with the TMA engine
#pragma unroll
            for (int i = 0; i < M; ++i) Tc[wbase + (i + 2) * TLT] = acc[i];
            fence_proxy_async();
            __syncthreads();
            if (t == 0) {
                reduce_out(c, item);
                if (nxt < A.items) {
                    if (s == 2) {
                        bulk_wait_read<0>();
                        issue(c, nxt);
                    } else {
                        pend = c;
                    }
                }
            }
        }
    }
    if (t == 0) bulk_wait_all();
    {
        const unsigned n = valid_items(A.items, A.lines, tpc, tl, TLT, lane);
        const unsigned per = (first_chunk && A.mail_prev ? 1u : 0u) + (last_chunk && A.mail_next ? 1u : 0u);
        // halos: 2 rows of 3 fields; boundary rows: one per solve (9 or 6)
        flush_counts(err, 6 * per * n, (A.has_nu ? 9u : 6u) * per * n);
    }
}

namespace {

template <int TLT>
int launch_dd_transport_dir_t(const TdArgs& A0, cudaStream_t s) {
    TdArgs A = A0;
    const int per_tile = A.chunks * TLT;
    A.tpc = per_tile >= 256 ? 1 : 256 / per_tile;
    const long long tiles = (A.lines + TLT - 1) / TLT;
    A.items = (tiles + A.tpc - 1) / A.tpc;
    if (A.items <= 0) return TDS_OK;
    int rc;
    for (int c = 0; c < 3; ++c)
        if ((rc = encode_xz_map(A.u[c], A.nx, A.ny, A.rows, A.sz, 16, TLT, &A.map[c], &A.boxr)) ||
            (rc = encode_xz_map(A.out[c], A.nx, A.ny, A.rows, A.sz, 16, TLT, &A.omap[c],
                                &A.boxr)))
            return rc;
    const int threads = A.tpc * per_tile;
    const size_t smem = (size_t)A.tpc *
                            (3 * (size_t)(A.rows + 4) * TLT + 3 * (size_t)2 * A.chunks * TLT +
                             3 * 2 * TLT) * sizeof(double) +
                        16 * sizeof(DirRow) + 12 * sizeof(double) + 3 * sizeof(uint64_t);
    const void* fn = reinterpret_cast<const void*>(k_dd_transport_dir<TLT>);
    if ((rc = ensure_smem(fn, smem, "cudaFuncSetAttribute(k_dd_transport_dir)"))) return rc;
    const long long grid = persistent_grid(fn, threads, smem, A.items, A.max_ctas);
    if (grid < 1) return set_err(TDS_ERR_UNSUPPORTED, "k_dd_transport_dir does not fit on an SM");
    return launch_resident(fn, grid, threads, smem, s, A, "k_dd_transport_dir launch");
}

}  // namespace

int launch_dd_transport_dir(const FastArgs& f1, const FastArgs& f2, const double* const* u,
                            double* const* out, double nu, int nx, int ny, int m, int sz,
                            double* mail, double* mail_prev, double* mail_next,
                            unsigned long long epoch, int max_ctas, cudaStream_t s) {
    TdArgs A;
    std::memset(&A, 0, sizeof(A));
    A.f1 = f1;
    A.f2 = f2;
    for (int c = 0; c < 3; ++c) {
        A.u[c] = u[c];
        A.out[c] = out[c];
        if (reinterpret_cast<uintptr_t>(u[c]) % 16 || reinterpret_cast<uintptr_t>(out[c]) % 16)
            return set_err(TDS_ERR_UNSUPPORTED, "direction distributed transport: alignment");
    }
    A.nu = nu;
    A.has_nu = nu != 0.0;
    A.lines = (long long)nx * ny;
    A.rows = m;
    A.sz = sz;
    A.chunks = f1.chunks;
    A.nx = nx;
    A.ny = ny;
    A.max_ctas = max_ctas;
    A.mail = mail;
    A.mail_prev = mail_prev;
    A.mail_next = mail_next;
    A.epoch = epoch;
    A.timeout_ns = 10ULL * 1000 * 1000 * 1000;
    if (const char* e = getenv("TDS_FUSED_TIMEOUT_MS"))
        A.timeout_ns = (unsigned long long)atoll(e) * 1000000ULL;
    if (ny % sz || !f1.Hb || f1.nb <= 0 || (A.has_nu && (!f2.Hb || f2.nb <= 0)))
        return set_err(TDS_ERR_UNSUPPORTED, "direction distributed transport: shape / band");
    int tl = 16;
    if (const char* e = getenv("TDS_TRANSPORT_TL")) tl = atoi(e) == 8 ? 8 : 16;
    const size_t need16 = (size_t)3 * (m + 4) * 16 * 8;
    if (tl == 16 && sz % 16 == 0 && A.chunks * 16 <= 512 && need16 <= 200 * 1024)
        return launch_dd_transport_dir_t<16>(A, s);
    if (sz % 8 == 0 && A.chunks * 8 <= 512 && (size_t)3 * (m + 4) * 8 * 8 <= 200 * 1024)
        return launch_dd_transport_dir_t<8>(A, s);
    return set_err(TDS_ERR_UNSUPPORTED, "direction distributed transport: tile");
}

#ifdef TDS_WAIT_PROF
// debug builds only (not in the C ABI header): [halo ns, boundary ns, halo
// takes, boundary takes] since the last call, then reset
extern "C" int tds_debug_wait_stats(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_wait_ns, 2 * sizeof(unsigned long long));
    cudaMemcpyFromSymbol(out + 2, g_wait_n, 2 * sizeof(unsigned long long));
    const unsigned long long z[2] = {0, 0};
    cudaMemcpyToSymbol(g_wait_ns, z, sizeof(z));
    cudaMemcpyToSymbol(g_wait_n, z, sizeof(z));
    return 0;
}
#endif
}  // namespace tds
