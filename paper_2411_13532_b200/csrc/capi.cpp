// C-ABI entry points (include/tds_b200.h): argument checking and dispatch of
// the plan to the fast or staged kernels. No allocation on the solve path
// except the phase-level calls that take host coefficient arrays.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "tds_internal.h"
#include "tds_tma.h"

using tds::set_err;

namespace {

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

int check_field(const tds_plan* p, long long groups, int sz) {
    if (!p) return set_err(TDS_ERR_INVALID, "null plan");
    if (groups < 0 || sz < 1) return set_err(TDS_ERR_INVALID, "bad field shape");
    return TDS_OK;
}

tds::FastArgs fast_args(const tds_plan* p, long long lines, int sz) {
    tds::FastArgs a;
    std::memset(&a, 0, sizeof(a));
    a.tab = p->d_tab;
    a.Hp = p->d_Hp;
    a.Hb = p->d_Hb;
    a.bq0 = p->d_bq0;
    a.nb = p->band_n;
    a.g_n0 = p->g_n0 ? p->g_n0 : 2 * p->C;
    a.g_n1 = p->g_n1 ? p->g_n1 : 2 * p->C;
    a.g = p->d_g;
    a.lines = lines;
    a.rows = p->block_rows;
    a.sz = sz;
    a.chunks = p->C;
    int per_tile = p->C * tds::TL;
    a.tiles_per_cta = per_tile >= 256 ? 1 : 256 / per_tile;
    a.has_prev = p->has_prev;
    a.has_next = p->has_next;
    a.sa_first = p->sa_first;
    a.sc_last = p->sc_last;
    a.prev_sc_last = p->prev_sc_last;
    a.next_sa_first = p->next_sa_first;
    a.det_prev = p->det_prev;
    a.det_next = p->det_next;
    a.ut = p->ut;
    a.special_first = p->special_first;
    a.e_first = p->e_first;
    a.e_last = p->e_last;
    a.special_last = p->special_last;
    a.dd_defer16 = p->dd_defer[0];
    a.dd_defer8 = p->dd_defer[1];
    for (int i = 0; i < 4; ++i) a.sh[i] = p->sh[i];
    a.has_shift = p->sh[0] | p->sh[1] | p->sh[2] | p->sh[3];
    return a;
}

long long tiles_of(long long lines) { return (lines + tds::TL - 1) / tds::TL; }

tds::StagedArgs staged_args(const tds_plan* p, long long lines, int sz) {
    tds::StagedArgs a;
    std::memset(&a, 0, sizeof(a));
    a.st = p->d_st;
    a.w = p->d_w;
    a.f = p->d_f;
    a.r = p->d_r;
    a.sa = p->d_sa;
    a.sc = p->d_sc;
    a.boff = p->d_boff;
    a.bsize = p->d_bsize;
    a.bconst = p->d_bconst;
    a.lines = lines;
    a.rows = p->block_rows;
    a.sz = sz;
    a.nb = p->nb;
    a.th_a = p->d_tha;
    a.th_w = p->d_thw;
    a.th_cp = p->d_thcp;
    a.th_z = p->d_thz;
    a.th_b0 = p->th_b0;
    a.th_qlast = p->th_qlast;
    a.th_den = p->th_den;
    a.periodic = p->periodic;
    for (int i = 0; i < 4; ++i) a.sh[i] = p->sh[i];
    a.has_shift = p->sh[0] | p->sh[1] | p->sh[2] | p->sh[3];
    return a;
}

// scratch for the staged path's boundary rows, stream-ordered
int scratch_alloc(double** ptr, size_t count, cudaStream_t s) {
    return tds::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(ptr),
                                           (count ? count : 1) * sizeof(double), s),
                           "cudaMallocAsync");
}

}  // namespace

extern "C" int tds_solve(const tds_plan* p, const double* u, double* out, long long groups,
                         int sz, void* stream) {
    int rc = check_field(p, groups, sz);
    if (rc) return rc;
    if (p->rank >= 0 && p->P > 1)
        return set_err(TDS_ERR_INVALID, "tds_solve needs a whole-operator plan (rank = -1)");
    if (!u || !out) return set_err(TDS_ERR_INVALID, "null field pointer");
    const long long lines = groups * sz;
    if (p->path == TDS_PATH_FAST) {
        tds::FastArgs a = fast_args(p, lines, sz);
        a.u = u;
        a.out = out;
        a.edge_mode = p->periodic ? tds::EDGE_WRAP : tds::EDGE_ZERO;
        // dynamic item schedule (SMs stream HBM at different rates: a static
        // round-robin leaves the fastest idle for the slowest). Knob
        // TDS_DYN=0: static.
        if (p->d_ctr && !(getenv("TDS_DYN") && getenv("TDS_DYN")[0] == '0')) {
            const unsigned slot = __atomic_fetch_add(&p->ctr_next, 1u, __ATOMIC_RELAXED);
            a.ctr = p->d_ctr + 2 * (slot % tds::CTR_SLOTS);
        }
        if (p->C <= tds::MAX_CHUNKS)
            return tds::launch_fast(p->M, tds::MODE_SOLVE, p->uniform, a, tiles_of(lines),
                                    S(stream));
        // a line longer than one CTA holds: split over a thread-block cluster
        // (k_tmc), else the plan's staged tables
        if (tds::tmc_eligible(p->M, p->uniform, a)) return tds::launch_tmc(p->M, p->uniform, a, S(stream));
        if (!p->has_staged) return set_err(TDS_ERR_UNSUPPORTED, "no kernel for this line length");
    }
    tds::StagedArgs a = staged_args(p, lines, sz);
    a.u = u;
    a.out = out;
    a.edge_mode = p->periodic ? tds::EDGE_WRAP : tds::EDGE_ZERO;
    if (p->P == 1) return tds::launch_thomas(a, S(stream));
    double* rows = nullptr;
    if ((rc = scratch_alloc(&rows, size_t(2) * p->nb * lines, S(stream)))) return rc;
    a.d_first = rows;
    a.d_last = rows + size_t(p->nb) * lines;
    rc = tds::launch_staged_decouple(a, S(stream));
    if (!rc) rc = tds::launch_staged_finish(a, S(stream));
    cudaFreeAsync(rows, S(stream));
    return rc;
}

extern "C" int tds_halo_rows(const tds_plan* p, const double* u, double* first2, double* last2,
                             long long groups, int sz, void* stream) {
    int rc = check_field(p, groups, sz);
    if (rc) return rc;
    return tds::launch_halo_rows(u, first2, last2, groups * sz, p->block_rows, sz, S(stream));
}

extern "C" int tds_boundary_rows(const tds_plan* p, const double* u, const double* halo_lo,
                                 const double* halo_hi, double* d_first, double* d_last,
                                 double* scratch, long long groups, int sz, void* stream) {
    int rc = check_field(p, groups, sz);
    if (rc) return rc;
    if (p->rank < 0 || p->P < 2) return set_err(TDS_ERR_INVALID, "per-rank plan required");
    const long long lines = groups * sz;
    if (p->path == TDS_PATH_FAST) {
        tds::FastArgs a = fast_args(p, lines, sz);
        a.u = u;
        a.halo_lo = halo_lo;
        a.halo_hi = halo_hi;
        a.edge_mode = tds::EDGE_HALO;
        a.d_first_out = d_first;
        a.d_last_out = d_last;
        return tds::launch_fast(p->M, tds::MODE_PASS_A, p->uniform, a, tiles_of(lines), S(stream));
    }
    if (!scratch) return set_err(TDS_ERR_INVALID, "staged path needs the scratch block");
    tds::StagedArgs a = staged_args(p, lines, sz);
    a.u = u;
    a.out = scratch;
    a.halo_lo = halo_lo;
    a.halo_hi = halo_hi;
    a.edge_mode = tds::EDGE_HALO;
    a.d_first = d_first;
    a.d_last = d_last;
    return tds::launch_staged_decouple(a, S(stream));
}

extern "C" int tds_finish(const tds_plan* p, const double* u, const double* halo_lo,
                          const double* halo_hi, const double* d_first, const double* d_last,
                          const double* prev_last, const double* next_first, double* out,
                          long long groups, int sz, void* stream) {
    int rc = check_field(p, groups, sz);
    if (rc) return rc;
    if (p->rank < 0 || p->P < 2) return set_err(TDS_ERR_INVALID, "per-rank plan required");
    if ((p->has_prev && !prev_last) || (p->has_next && !next_first))
        return set_err(TDS_ERR_INVALID, "missing neighbour boundary rows");
    const long long lines = groups * sz;
    if (p->path == TDS_PATH_FAST) {
        tds::FastArgs a = fast_args(p, lines, sz);
        a.u = u;
        a.out = out;
        a.halo_lo = halo_lo;
        a.halo_hi = halo_hi;
        a.edge_mode = tds::EDGE_HALO;
        a.d_first_in = d_first;
        a.d_last_in = d_last;
        a.prev_last = prev_last;
        a.next_first = next_first;
        return tds::launch_fast(p->M, tds::MODE_PASS_B, p->uniform, a, tiles_of(lines), S(stream));
    }
    tds::StagedArgs a = staged_args(p, lines, sz);
    a.out = out;
    a.d_first = const_cast<double*>(d_first);
    a.d_last = const_cast<double*>(d_last);
    a.prev_last = prev_last;
    a.next_first = next_first;
    return tds::launch_staged_finish(a, S(stream));
}

// ------------------------------------------------------------ phase kernels


extern "C" int tds_decouple_fused(const double* u_ext, const double* stencil,
                                  const int* shift4, const double* w, const double* f,
                                  const double* r, double* d, int m, long long lanes,
                                  void* stream) {
    if (m < 4) return set_err(TDS_ERR_INVALID, "local block needs at least 4 rows");
    if (lanes > 0 && (!u_ext || !stencil || !w || !f || !r || !d))
        return set_err(TDS_ERR_INVALID, "null argument");
    int sh[4] = {0, 0, 0, 0};
    if (shift4) {
        for (int i = 0; i < 4; ++i) sh[i] = shift4[i];
        if (sh[0] < 0 || sh[0] > 2 || sh[1] < 0 || sh[1] > 2 || sh[2] > 0 || sh[2] < -2 ||
            sh[3] > 0 || sh[3] < -2 || (m < 8 && (sh[0] | sh[1] | sh[2] | sh[3])))
            return set_err(TDS_ERR_INVALID, "bad stencil shifts");
    }
    return tds::launch_decouple_pm(u_ext, stencil, sh, w, f, r, d, m, lanes, S(stream));
}

extern "C" int tds_substitute(const double* d, const double* s_a, const double* s_c,
                              const double* u_start, const double* u_end, double* out, int m,
                              long long lanes, void* stream) {
    if (m < 4) return set_err(TDS_ERR_INVALID, "local block needs at least 4 rows");
    if (lanes > 0 && (!d || !s_a || !s_c || !u_start || !u_end || !out))
        return set_err(TDS_ERR_INVALID, "null argument");
    return tds::launch_substitute_pm(d, s_a, s_c, u_start, u_end, out, m, lanes, S(stream));
}

extern "C" int tds_boundary_pair(const double* d_last, const double* d_first, double s_c_last,
                                 double s_a_first, double* u_last, double* u_first,
                                 long long lanes, void* stream) {
    double det = 1.0 - s_c_last * s_a_first;
    if (!(det >= tds::PAIR_DET_FLOOR || det <= -tds::PAIR_DET_FLOOR)) {
        char msg[64];
        std::snprintf(msg, sizeof(msg), "boundary determinant %.3e", det);
        return set_err(TDS_ERR_SINGULAR_PAIR, msg);
    }
    return tds::launch_pair(d_last, d_first, s_c_last, s_a_first, det, u_last, u_first, lanes,
                            S(stream));
}

namespace tds {
int thomas_plan(const double* lower, const double* diag, const double* upper, int periodic, int n,
                double pivot_floor, const tds_plan** out);
}

extern "C" int tds_thomas(const double* lower, const double* diag, const double* upper,
                          int periodic, const double* rhs, double* out, int n, long long groups,
                          int sz, double pivot_floor, void* stream) {
    // A P=1 staged plan over a (groups, n, sz) field with the identity
    // stencil (its zero weights never see the halo), cached per operator and
    // device (plan.cpp thomas_plan): no allocation or copy per call. RhsBatch
    // (m, n) is the case groups=m, sz=1.
    if (groups < 0 || sz < 1) return set_err(TDS_ERR_INVALID, "bad field shape");
    const tds_plan* p = nullptr;
    int rc = tds::thomas_plan(lower, diag, upper, periodic, n, pivot_floor, &p);
    if (rc) return rc;
    tds::StagedArgs a = staged_args(p, groups * sz, sz);
    a.u = rhs;
    a.out = out;
    a.edge_mode = tds::EDGE_ZERO;
    return tds::launch_thomas(a, S(stream));
}

static int pack_common(const double* src, double* dst, int nx, int ny, int nz, int sz,
                       int direction, long long groups, bool to_field, void* stream) {
    if (direction < 0 || direction > 2 || sz < 1 || nx < 1 || ny < 1 || nz < 1)
        return set_err(TDS_ERR_INVALID, "bad layout");
    long long n = direction == 0 ? nx : (direction == 1 ? ny : nz);
    long long lines = (long long)nx * ny * nz / n;
    if (groups * sz < lines) return set_err(TDS_ERR_INVALID, "field has too few lines");
    return tds::launch_pack(src, dst, nx, ny, nz, sz, direction, groups, to_field, S(stream));
}

extern "C" int tds_pack(const double* cart, double* field, int nx, int ny, int nz, int sz,
                        int direction, long long groups, void* stream) {
    return pack_common(cart, field, nx, ny, nz, sz, direction, groups, true, stream);
}

extern "C" int tds_unpack(const double* field, double* cart, int nx, int ny, int nz, int sz,
                          int direction, long long groups, void* stream) {
    return pack_common(field, cart, nx, ny, nz, sz, direction, groups, false, stream);
}

// ------------------------------------------------ fused multi-GPU (k_dd)

namespace tds {
long long dd_mail_words(long long lines);
bool dd_eligible(int M, const FastArgs& a);
int launch_dd(int M, bool uniform, const FastArgs& a, double* mail, double* mail_prev,
              double* mail_next, unsigned long long epoch, int max_ctas, cudaStream_t s,
              bool query = false);
}  // namespace tds

extern "C" long long tds_mailbox_words(long long groups, int sz) {
    return tds::dd_mail_words(groups * sz);
}

extern "C" int tds_plan_restrict_fused(tds_plan* p, int mask) {
    if (!p) return -1;
    p->dd_defer[0] &= (mask & 1) ? 1 : 0;
    p->dd_defer[1] &= (mask & 2) ? 1 : 0;
    return (p->dd_defer[0] ? 1 : 0) | (p->dd_defer[1] ? 2 : 0);
}

extern "C" int tds_fused_eligible(const tds_plan* p, long long groups, int sz) {
    if (!p || p->rank < 0 || p->P < 2 || p->path != TDS_PATH_FAST) return 0;
    tds::FastArgs a = fast_args(p, groups * sz, sz);
    a.u = reinterpret_cast<const double*>(uintptr_t(256));   // alignment probe only
    return tds::dd_eligible(p->M, a) ? 1 : 0;
}

extern "C" long long tds_fused_grid(const tds_plan* p, long long groups, int sz, int max_ctas) {
    if (!tds_fused_eligible(p, groups, sz)) return -1;
    tds::FastArgs a = fast_args(p, groups * sz, sz);
    a.u = reinterpret_cast<const double*>(uintptr_t(256));   // no launch: shape only
    a.edge_mode = tds::EDGE_HALO;
    const int g = tds::launch_dd(p->M, p->uniform, a, nullptr, nullptr, nullptr, 0, max_ctas,
                                 nullptr, true);
    return g;
}

extern "C" int tds_fused_solve(const tds_plan* p, const double* u, double* out, long long groups,
                               int sz, double* mail, double* mail_prev, double* mail_next,
                               unsigned long long epoch, int max_ctas, void* stream) {
    int rc = check_field(p, groups, sz);
    if (rc) return rc;
    if (p->rank < 0 || p->P < 2 || p->path != TDS_PATH_FAST)
        return set_err(TDS_ERR_UNSUPPORTED, "fused solve needs a per-rank fast-path plan");
    if ((p->has_prev && !mail_prev) || (p->has_next && !mail_next) || !mail)
        return set_err(TDS_ERR_INVALID, "missing mailbox");
    const long long lines = groups * sz;
    tds::FastArgs a = fast_args(p, lines, sz);
    a.u = u;
    a.out = out;
    a.edge_mode = tds::EDGE_HALO;
    if (!tds::dd_eligible(p->M, a))
        return set_err(TDS_ERR_UNSUPPORTED, "field not eligible for the fused kernel");
    // dynamic item schedule (k_dd / k_dd2; deadlock-free with one counter per
    // rank, see k_dd). Knob TDS_DYN=0: round-robin.
    if (p->d_ctr && !(getenv("TDS_DYN") && getenv("TDS_DYN")[0] == '0')) {
        const unsigned slot = __atomic_fetch_add(&p->ctr_next, 1u, __ATOMIC_RELAXED);
        a.ctr = p->d_ctr + 2 * (slot % tds::CTR_SLOTS);
    }
    return tds::launch_dd(p->M, p->uniform, a, mail, p->has_prev ? mail_prev : nullptr,
                          p->has_next ? mail_next : nullptr, epoch, max_ctas, S(stream));
}

static int read_status(const double* mail, long long words, int* err) {
    if (!mail || words < 3 || !err) return set_err(TDS_ERR_INVALID, "null argument");
    unsigned long long v = 0;
    int rc = tds::cuda_check(cudaMemcpy(&v, mail + (words - 3), 8, cudaMemcpyDeviceToHost),
                             "read mailbox error word");
    *err = (v == 1ULL) ? 1 : 0;   // ERR_TIMEOUT
    return rc;
}

extern "C" int tds_mailbox_error(const double* mail, long long groups, int sz, int* err) {
    return read_status(mail, tds::dd_mail_words(groups * sz), err);
}

extern "C" int tds_mailbox_init(double* mail, long long words, void* stream) {
    if (!mail || words < 3) return set_err(TDS_ERR_INVALID, "bad mailbox");
    cudaStream_t s = S(stream);
    int rc = tds::cuda_check(cudaMemsetAsync(mail, 0xFF, size_t(words) * 8, s),
                             "cudaMemsetAsync(mailbox)");   // sentinel fill
    if (!rc)
        rc = tds::cuda_check(cudaMemsetAsync(mail + (words - 3), 0, 3 * 8, s),
                             "cudaMemsetAsync(mailbox status)");
    return rc;
}

extern "C" int tds_mailbox_status(const double* mail, long long words,
                                  unsigned long long* host_status, void* stream) {
    if (!mail || words < 3 || !host_status) return set_err(TDS_ERR_INVALID, "null argument");
    return tds::cuda_check(cudaMemcpyAsync(host_status, mail + (words - 3), 3 * 8,
                                           cudaMemcpyDeviceToHost, S(stream)),
                           "copy mailbox status");
}

extern "C" int tds_peer_access(int peer_device) {
    int dev = 0;
    int rc = tds::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    if (rc || peer_device == dev) return rc;
    int can = 0;
    rc = tds::cuda_check(cudaDeviceCanAccessPeer(&can, dev, peer_device), "cudaDeviceCanAccessPeer");
    if (rc) return rc;
    if (!can) return set_err(TDS_ERR_UNSUPPORTED, "no peer access between the devices");
    cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return TDS_OK;
    }
    return tds::cuda_check(e, "cudaDeviceEnablePeerAccess");
}

namespace tds {
long long dd_transport_mail_words(long long lines);
int launch_dd_transport(const FastArgs& f1, const FastArgs& f2, const double* ui,
                        const double* uj, double* out, double nu, long long lines, int sz,
                        double* mail, double* mail_prev, double* mail_next,
                        unsigned long long epoch, int max_ctas, cudaStream_t s, int nx = 0,
                        int ny = 0);
int launch_dd_transport_dir(const FastArgs& f1, const FastArgs& f2, const double* const* u,
                            double* const* out, double nu, int nx, int ny, int m, int sz,
                            double* mail, double* mail_prev, double* mail_next,
                            unsigned long long epoch, int max_ctas, cudaStream_t s);
}  // namespace tds

extern "C" long long tds_transport_mailbox_words(long long groups, int sz) {
    return tds::dd_transport_mail_words(groups * sz);
}

extern "C" int tds_transport_mailbox_error(const double* mail, long long groups, int sz,
                                           int* err) {
    return read_status(mail, tds::dd_transport_mail_words(groups * sz), err);
}

extern "C" int tds_fused_transport(const tds_plan* d1, const tds_plan* d2, const double* u_i,
                                   const double* u_j, double* out, double nu, long long groups,
                                   int sz, double* mail, double* mail_prev, double* mail_next,
                                   unsigned long long epoch, int max_ctas, void* stream) {
    int rc = check_field(d1, groups, sz);
    if (rc) return rc;
    if (!u_i || !u_j || !out || !mail) return set_err(TDS_ERR_INVALID, "null argument");
    // C >= 2: the kernel's edge threads hold either the first or the last
    // chunk of a block, never both
    auto ok = [&](const tds_plan* p) {
        return p->rank >= 0 && p->P >= 2 && p->path == TDS_PATH_FAST && p->M == 16 &&
               p->C >= 2 && p->uniform && !p->special_first && !p->special_last;
    };
    if (!ok(d1) || (nu != 0.0 && (!d2 || !ok(d2) || d2->C != d1->C || d2->rank != d1->rank ||
                                  d2->block_rows != d1->block_rows)))
        return set_err(TDS_ERR_UNSUPPORTED,
                       "fused distributed transport needs uniform per-rank 16-row-chunk plans");
    if ((d1->has_prev && !mail_prev) || (d1->has_next && !mail_next))
        return set_err(TDS_ERR_INVALID, "missing mailbox");
    if (reinterpret_cast<uintptr_t>(u_i) % 16 || reinterpret_cast<uintptr_t>(u_j) % 16 ||
        tds::box_rows(d1->block_rows, 16) == 0 || !tds::encode_fn())
        return set_err(TDS_ERR_UNSUPPORTED, "fused distributed transport: not TMA-eligible");
    const long long lines = groups * sz;
    tds::FastArgs f1 = fast_args(d1, lines, sz);
    tds::FastArgs f2 = nu != 0.0 ? fast_args(d2, lines, sz) : f1;
    return tds::launch_dd_transport(f1, f2, u_i, u_j, out, nu, lines, sz, mail,
                                    d1->has_prev ? mail_prev : nullptr,
                                    d1->has_next ? mail_next : nullptr, epoch, max_ctas,
                                    S(stream));
}

extern "C" int tds_fused_transport_in_x(const tds_plan* d1, const tds_plan* d2,
                                        const double* u_i, const double* u_j, double* acc,
                                        double nu, int nx, int ny, int m, int sz, double* mail,
                                        double* mail_prev, double* mail_next,
                                        unsigned long long epoch, int max_ctas, void* stream) {
    if (!d1 || !u_i || !u_j || !acc || !mail) return set_err(TDS_ERR_INVALID, "null argument");
    if (nx < 1 || ny < 1 || sz < 1 || ny % sz || m != d1->block_rows)
        return set_err(TDS_ERR_INVALID, "bad slab extents (sz | ny, m = the plan's block rows)");
    auto ok = [&](const tds_plan* p) {
        return p->rank >= 0 && p->P >= 2 && p->path == TDS_PATH_FAST && p->M == 16 &&
               p->C >= 2 && p->uniform && !p->special_first && !p->special_last;
    };
    if (!ok(d1) || (nu != 0.0 && (!d2 || !ok(d2) || d2->C != d1->C || d2->rank != d1->rank ||
                                  d2->block_rows != d1->block_rows)))
        return set_err(TDS_ERR_UNSUPPORTED,
                       "fused distributed transport needs uniform per-rank 16-row-chunk plans");
    if ((d1->has_prev && !mail_prev) || (d1->has_next && !mail_next))
        return set_err(TDS_ERR_INVALID, "missing mailbox");
    if (reinterpret_cast<uintptr_t>(u_i) % 16 || reinterpret_cast<uintptr_t>(u_j) % 16 ||
        tds::box_rows(m, 16) == 0 || !tds::encode_fn())
        return set_err(TDS_ERR_UNSUPPORTED, "fused distributed transport: not TMA-eligible");
    const long long lines = (long long)nx * ny;
    tds::FastArgs f1 = fast_args(d1, lines, sz);
    tds::FastArgs f2 = nu != 0.0 ? fast_args(d2, lines, sz) : f1;
    return tds::launch_dd_transport(f1, f2, u_i, u_j, acc, nu, lines, sz, mail,
                                    d1->has_prev ? mail_prev : nullptr,
                                    d1->has_next ? mail_next : nullptr, epoch, max_ctas,
                                    S(stream), nx, ny);
}

extern "C" int tds_fused_transport_direction(const tds_plan* d1, const tds_plan* d2,
                                             const double* u0, const double* u1,
                                             const double* u2, double* acc0, double* acc1,
                                             double* acc2, double nu, int nx, int ny, int m,
                                             int sz, double* mail, double* mail_prev,
                                             double* mail_next, unsigned long long epoch,
                                             int max_ctas, void* stream) {
    if (!d1 || !u0 || !u1 || !u2 || !acc0 || !acc1 || !acc2 || !mail)
        return set_err(TDS_ERR_INVALID, "null argument");
    if (nx < 1 || ny < 1 || sz < 1 || ny % sz || m != d1->block_rows)
        return set_err(TDS_ERR_INVALID, "bad slab extents (sz | ny, m = the plan's block rows)");
    auto ok = [&](const tds_plan* p) {
        return p->rank >= 0 && p->P >= 2 && p->path == TDS_PATH_FAST && p->M == 16 &&
               p->C >= 2 && p->uniform && !p->special_first && !p->special_last;
    };
    if (!ok(d1) || (nu != 0.0 && (!d2 || !ok(d2) || d2->C != d1->C || d2->rank != d1->rank ||
                                  d2->block_rows != d1->block_rows)))
        return set_err(TDS_ERR_UNSUPPORTED,
                       "fused distributed transport needs uniform per-rank 16-row-chunk plans");
    if ((d1->has_prev && !mail_prev) || (d1->has_next && !mail_next))
        return set_err(TDS_ERR_INVALID, "missing mailbox");
    if (tds::box_rows(m, 16) == 0 || !tds::encode_fn())
        return set_err(TDS_ERR_UNSUPPORTED, "fused distributed transport: not TMA-eligible");
    const long long lines = (long long)nx * ny;
    tds::FastArgs f1 = fast_args(d1, lines, sz);
    tds::FastArgs f2 = nu != 0.0 ? fast_args(d2, lines, sz) : f1;
    const double* u[3] = {u0, u1, u2};
    double* acc[3] = {acc0, acc1, acc2};
    return tds::launch_dd_transport_dir(f1, f2, u, acc, nu, nx, ny, m, sz, mail,
                                        d1->has_prev ? mail_prev : nullptr,
                                        d1->has_next ? mail_next : nullptr, epoch, max_ctas,
                                        S(stream));
}

extern "C" int tds_ipc_alloc(long long bytes, void** ptr, unsigned char* handle) {
    int rc = tds::cuda_check(cudaMalloc(ptr, size_t(bytes)), "cudaMalloc(mailbox)");
    if (rc) return rc;
    // sentinel fill + zeroed status words, complete BEFORE the handle is
    // shared: a neighbour may post as soon as it can map the mailbox
    rc = tds_mailbox_init(static_cast<double*>(*ptr), bytes / 8, nullptr);
    if (!rc) rc = tds::cuda_check(cudaDeviceSynchronize(), "mailbox fill");
    if (rc) return rc;
    cudaIpcMemHandle_t h;
    rc = tds::cuda_check(cudaIpcGetMemHandle(&h, *ptr), "cudaIpcGetMemHandle");
    if (rc) return rc;
    std::memcpy(handle, &h, sizeof(h));
    return TDS_OK;
}

extern "C" int tds_ipc_open(const unsigned char* handle, void** ptr) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    return tds::cuda_check(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess),
                           "cudaIpcOpenMemHandle");
}

extern "C" int tds_ipc_close(void* ptr) {
    return tds::cuda_check(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
}

extern "C" int tds_ipc_free(void* ptr) { return tds::cuda_check(cudaFree(ptr), "cudaFree"); }

// ------------------------------------------------- transport RHS (k_transport)

namespace tds {
struct TransportArgs;
int launch_reorder(const double* src, double* dst, int nx, int ny, int nz, int sz, int src_dir,
                   int dst_dir, int accumulate, cudaStream_t s);
int launch_transport_combine(const double* uj, const double* du, const double* dp,
                             const double* d2u, double nu, double* out, long long count,
                             int accumulate, cudaStream_t s);
int launch_axpy_mul(const double* a, const double* b, double w, int mul, double* out,
                    long long count, cudaStream_t s);
int transport_launch_from_plans(const tds_plan* d1, const tds_plan* d2, const double* ui,
                                const double* uj, double* out, double nu, int accumulate,
                                long long lines, int sz, cudaStream_t s, int geom, int nx = 0,
                                int ny = 0, int nz = 0);
int transport_direction_from_plans(const tds_plan* d1, const tds_plan* d2, const double* const* u,
                                   double* const* out, double nu, int nx, int ny, int nz, int sz,
                                   int dir, cudaStream_t s);
}  // namespace tds

extern "C" int tds_transport_contribution(const tds_plan* d1, const tds_plan* d2,
                                          const double* u_i, const double* u_j, double* out,
                                          double nu, int accumulate, long long groups, int sz,
                                          void* stream) {
    if (!d1 || !u_i || !u_j || !out) return set_err(TDS_ERR_INVALID, "null argument");
    const bool ok1 = d1->path == TDS_PATH_FAST && d1->uniform && (d1->M == 32 || d1->M == 16) &&
                     d1->P == 1 && d1->rank < 0 && !d1->special_first && !d1->special_last;
    const bool ok2 = !d2 || (d2->path == TDS_PATH_FAST && d2->uniform && d2->M == d1->M &&
                             d2->P == 1 && d2->rank < 0 && d2->C == d1->C &&
                             !d2->special_first && !d2->special_last);
    if (!ok1 || !ok2 || (nu != 0.0 && !d2))
        return set_err(TDS_ERR_UNSUPPORTED,
                       "fused transport needs uniform P=1 plans with 16- or 32-row chunks");
    return tds::transport_launch_from_plans(d1, nu != 0.0 ? d2 : nullptr, u_i, u_j, out, nu,
                                            accumulate, groups * sz, sz, S(stream), 0);
}

extern "C" int tds_transport_contribution_in_x(const tds_plan* d1, const tds_plan* d2,
                                               const double* u_i, const double* u_j, double* acc,
                                               double nu, int nx, int ny, int nz, int sz, int dir,
                                               void* stream) {
    if (!d1 || !u_i || !u_j || !acc) return set_err(TDS_ERR_INVALID, "null argument");
    if (dir != 1 && dir != 2) return set_err(TDS_ERR_INVALID, "dir must be 1 (y) or 2 (z)");
    if (nx < 1 || ny < 1 || nz < 1 || sz < 1 || ny % sz)
        return set_err(TDS_ERR_INVALID, "bad block extents (sz must divide ny)");
    const int rows = dir == 1 ? ny : nz;
    const bool ok1 = d1->path == TDS_PATH_FAST && d1->uniform && d1->M == 16 && d1->P == 1 &&
                     d1->rank < 0 && !d1->special_first && !d1->special_last &&
                     d1->block_rows == rows;
    const bool ok2 = !d2 || (d2->path == TDS_PATH_FAST && d2->uniform && d2->M == 16 &&
                             d2->P == 1 && d2->rank < 0 && d2->C == d1->C &&
                             !d2->special_first && !d2->special_last);
    if (!ok1 || !ok2 || (nu != 0.0 && !d2))
        return set_err(TDS_ERR_UNSUPPORTED,
                       "in-place transport needs uniform P=1 plans with 16-row chunks");
    const long long lines = dir == 1 ? (long long)nx * nz : (long long)nx * ny;
    return tds::transport_launch_from_plans(d1, nu != 0.0 ? d2 : nullptr, u_i, u_j, acc, nu, 1,
                                            lines, sz, S(stream), dir == 2 ? 1 : 2, nx, ny, nz);
}

extern "C" int tds_transport_direction(const tds_plan* d1, const tds_plan* d2, const double* u0,
                                       const double* u1, const double* u2, double* out0,
                                       double* out1, double* out2, double nu, int nx, int ny,
                                       int nz, int sz, int dir, void* stream) {
    if (!d1 || !u0 || !u1 || !u2 || !out0 || !out1 || !out2)
        return set_err(TDS_ERR_INVALID, "null argument");
    if (dir < 0 || dir > 2) return set_err(TDS_ERR_INVALID, "dir must be 0, 1 or 2");
    if (nx < 1 || ny < 1 || nz < 1 || sz < 1 || ny % sz)
        return set_err(TDS_ERR_INVALID, "bad block extents (sz must divide ny)");
    const int rows = dir == 0 ? nx : (dir == 1 ? ny : nz);
    const bool ok1 = d1->path == TDS_PATH_FAST && d1->uniform && d1->M == 16 && d1->P == 1 &&
                     d1->rank < 0 && !d1->special_first && !d1->special_last &&
                     d1->block_rows == rows;
    const bool ok2 = !d2 || (d2->path == TDS_PATH_FAST && d2->uniform && d2->M == 16 &&
                             d2->P == 1 && d2->rank < 0 && d2->C == d1->C &&
                             !d2->special_first && !d2->special_last);
    if (!ok1 || !ok2 || (nu != 0.0 && !d2))
        return set_err(TDS_ERR_UNSUPPORTED,
                       "direction transport needs uniform P=1 plans with 16-row chunks");
    const double* u[3] = {u0, u1, u2};
    double* out[3] = {out0, out1, out2};
    return tds::transport_direction_from_plans(d1, nu != 0.0 ? d2 : nullptr, u, out, nu, nx, ny,
                                               nz, sz, dir, S(stream));
}

extern "C" int tds_euler_update(const double* u, const double* rhs, double dt, double* out,
                                long long count, void* stream) {
    if (!u || !rhs || !out || count < 0) return set_err(TDS_ERR_INVALID, "bad argument");
    return tds::launch_axpy_mul(u, rhs, dt, 0, out, count, S(stream));
}

extern "C" int tds_multiply(const double* a, const double* b, double* out, long long count,
                            void* stream) {
    if (!a || !b || !out || count < 0) return set_err(TDS_ERR_INVALID, "bad argument");
    return tds::launch_axpy_mul(a, b, 0.0, 1, out, count, S(stream));
}

extern "C" int tds_reorder3(const double* src, double* dst, int nx, int ny, int nz, int sz,
                            int src_dir, int dst_dir, int accumulate, void* stream) {
    if (!src || !dst || nx < 1 || ny < 1 || nz < 1 || nz > 65535 || sz < 1 || src_dir < 0 ||
        src_dir > 2 || dst_dir < 0 || dst_dir > 2)
        return set_err(TDS_ERR_INVALID, "bad reorder arguments");
    const long long pts = (long long)nx * ny * nz;
    const int ns[3] = {nx, ny, nz};
    if (pts / ns[src_dir] % sz || pts / ns[dst_dir] % sz)
        return set_err(TDS_ERR_INVALID, "lines not divisible by sz");
    if (pts / ns[src_dir] > 0xffffffffLL || pts / ns[dst_dir] > 0xffffffffLL)
        return set_err(TDS_ERR_INVALID, "too many lines for 32-bit line indices");
    return tds::launch_reorder(src, dst, nx, ny, nz, sz, src_dir, dst_dir, accumulate, S(stream));
}

extern "C" int tds_reorder(const double* src, double* dst, int n, int sz, int src_dir,
                           int dst_dir, int accumulate, void* stream) {
    return tds_reorder3(src, dst, n, n, n, sz, src_dir, dst_dir, accumulate, stream);
}

extern "C" int tds_transport_combine(const double* uj, const double* du, const double* dp,
                                     const double* d2u, double nu, double* out, long long count,
                                     int accumulate, void* stream) {
    return tds::launch_transport_combine(uj, du, dp, d2u, nu, out, count, accumulate, S(stream));
}
