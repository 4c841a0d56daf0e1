// Internal declarations shared by the host plan builder and the kernels.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/tds_b200.h"

namespace tds {

constexpr double PIVOT_FLOOR = 1e-300;     // reference serial.py:21
constexpr double PAIR_DET_FLOOR = 1e-12;   // reference serial.py:22
constexpr int TL = 16;                     // lines per tile: 16 x fp64 = 128 B rows
constexpr int NCOEF = 10;                  // per-row table: st0..st4, f, r, w, sa, sc
constexpr int MMAX_UNIFORM = 32;
constexpr int MAX_CHUNKS = 32;             // C*TL <= 512 threads per tile
constexpr int CTR_SLOTS = 64;              // schedule counters per plan (launches in flight)

enum FastMode { MODE_SOLVE = 0, MODE_PASS_A = 1, MODE_PASS_B = 2 };
enum EdgeMode { EDGE_ZERO = 0, EDGE_WRAP = 1, EDGE_HALO = 2 };

int set_err(int code, const std::string& msg, int rank = -1);

// Per-chunk coefficient table shared by every chunk (kernel-parameter bank).
struct UniformTable {
    double st[5];
    double f[MMAX_UNIFORM], r[MMAX_UNIFORM], w[MMAX_UNIFORM];
    double sa[MMAX_UNIFORM], sc[MMAX_UNIFORM];
};

// Per-row table of one special chunk (first / last chunk of an otherwise
// uniform plan: one-sided closures of open operators). Row i holds the
// stencil s0..s4, f, r, w, sa, sc -- the layout of the global `tab`.
struct EdgeTable {
    double c[MMAX_UNIFORM][NCOEF];
    // 7-tap stencils of chunk rows 0, 1 (window rows i .. i+6, offsets -2..4)
    // and M-2, M-1 (rows i-2 .. i+4, offsets -4..2): the width-5 row placed
    // at its window shift (plan.cpp check_shift), zeros elsewhere -- shifted
    // one-sided closures cost two FMAs instead of per-row selects
    double x7[4][7];
};

// Coefficient source of the fast kernels (template parameter TAB): the
// global per-row table, the uniform table, or the uniform table with an
// EdgeTable for a special first / last chunk.
enum { TAB_GLOBAL = 0, TAB_UNIFORM = 1, TAB_EDGES = 2 };

struct FastArgs {
    const double* u;
    double* out;
    const double* halo_lo;
    const double* halo_hi;
    const double* d_first_in;
    const double* d_last_in;
    const double* prev_last;
    const double* next_first;
    double* d_first_out;
    double* d_last_out;
    const double* tab;     // rows x NCOEF (GLOBAL table)
    const double2* Hp;     // C x K pairs: Hp[k*K+q] = (H[2k][q], H[2k+1][q])
    const double2* Hb;     // banded Hp: C x nb pairs, columns bq0[k] + j (mod K)
    const int* bq0;
    int nb;
    int g_n0, g_n1;        // g0 . Y over q < g_n0, g1 . Y over q >= K - g_n1
    const double* g;       // 2 x K pass-A functionals
    long long lines;
    long long items;       // work items of tiles_per_cta tiles (persistent kernels)
    int rows;              // rows per line in u/out
    int sz;
    int chunks;            // C
    int tiles_per_cta;
    int edge_mode;
    int has_prev, has_next;
    int dd_defer16, dd_defer8;   // deferred-edge fused kernel allowed (see plan.cpp)
    int special_first, special_last;   // uniform plan whose first / last chunk uses e_first / e_last
    int has_shift;         // some stencil row is shifted (one-sided closures)
    int sh[4];             // window shift of block rows 0, 1, rows-2, rows-1
    double sa_first, sc_last, prev_sc_last, next_sa_first, det_prev, det_next;
    UniformTable ut;
    EdgeTable e_first, e_last;
    // dynamic item schedule of the single-GPU persistent kernels (k_tma):
    // ctr[0] hands out items past the grid's first, ctr[1] counts CTAs out
    // (the last one resets both); nullptr = static round-robin
    unsigned long long* ctr;
};

// Staged (reference-arithmetic) kernels: one thread per (line, block).
struct StagedArgs {
    const double* u;
    double* out;
    const double* halo_lo;
    const double* halo_hi;
    double* d_first;        // [nb][lines]
    double* d_last;
    const double* prev_last;
    const double* next_first;
    const double* st;       // rows x 5
    const double* w;        // rows: rank-level (DistD2) or Thomas tables
    const double* f;
    const double* r;
    const double* sa;
    const double* sc;
    const int* boff;        // [nb]
    const int* bsize;       // [nb]
    const double* bconst;   // [nb][6]: sa_first, sc_last, det_prev, det_next, has_prev, has_next
    long long lines;
    int rows;
    int sz;
    int nb;
    int edge_mode;          // EDGE_ZERO / EDGE_WRAP (block-global rows) / EDGE_HALO
    // Thomas (P=1) extras
    const double* th_a;
    const double* th_w;
    const double* th_cp;
    const double* th_z;
    double th_b0, th_qlast, th_den;
    int periodic;
    int has_shift;
    int sh[4];              // window shift of block rows 0, 1, rows-2, rows-1
};

// launchers (tds_kernels.cu)
int launch_fast(int M, int mode, bool uniform, const FastArgs& a, long long tiles,
                cudaStream_t s);
bool tma_eligible(int M, const FastArgs& a);
int launch_tma(int M, int mode, bool uniform, const FastArgs& a, long long tiles,
               cudaStream_t s);
int launch_staged_decouple(const StagedArgs& a, cudaStream_t s);
int launch_staged_finish(const StagedArgs& a, cudaStream_t s);
int launch_thomas(const StagedArgs& a, cudaStream_t s);
int launch_halo_rows(const double* u, double* first2, double* last2, long long lines,
                     int rows, int sz, cudaStream_t s);
int launch_decouple_pm(const double* u_ext, const double* st, const int* sh4, const double* w,
                       const double* f, const double* r, double* d, int m,
                       long long lanes, cudaStream_t s);
int launch_substitute_pm(const double* d, const double* sa, const double* sc,
                         const double* us, const double* ue, double* out, int m,
                         long long lanes, cudaStream_t s);
int launch_pair(const double* dl, const double* df, double sc, double sa, double det,
                double* ul, double* uf, long long lanes, cudaStream_t s);
int launch_pack(const double* src, double* dst, int nx, int ny, int nz, int sz,
                int dir, long long groups, bool to_field, cudaStream_t s);
int cuda_check(cudaError_t e, const char* what);

}  // namespace tds

struct tds_plan;
namespace tds {
// tds_plan_create with an explicit pivot floor (plan.cpp)
int plan_create_impl(const double* lower, const double* diag, const double* upper, int periodic,
                     const double* stencil, const int* stencil_shift, int n, const int* sizes_in,
                     int P, int rank, int flags, double pivot_floor, tds_plan** out);
}  // namespace tds

// Rank-level DistD2 coefficients (distributed.py:43-68), dropped couplings kept.
struct tds_rank_coeffs {
    std::vector<double> sa, sc, w, f, r;   // sc[0], sa[m-1] zeroed as the reference
    double drop_first = 0.0, drop_last = 0.0;  // signed values before zeroing
};

struct tds_plan {
    int n = 0;
    int periodic = 0;
    int P = 1;
    int rank = -1;
    int flags = 0;
    double pivot_floor = tds::PIVOT_FLOOR;   // P=1 Thomas tables (serial.py:26-90)
    int path = TDS_PATH_STAGED;
    int block_off = 0, block_rows = 0;   // rows of the global line held here
    std::vector<int> sizes, offs;
    std::vector<tds_rank_coeffs> rc;     // per rank (P>1)
    double max_dropped = 0.0, margin = 0.0;

    // fast path
    int M = 0, C = 0, K = 0;
    bool uniform = false;
    int special_first = 0, special_last = 0;
    tds::UniformTable ut{};
    tds::EdgeTable e_first{}, e_last{};
    double* d_tab = nullptr;
    double2* d_Hp = nullptr;
    double2* d_Hb = nullptr;   // banded H: C x band_n, columns d_bq0[k] + j (mod K)
    int* d_bq0 = nullptr;
    int band_n = 0;
    // k_tma dynamic-schedule counters: CTR_SLOTS pairs, one per launch in
    // flight (round-robin; a slot is reset by its launch's last CTA)
    unsigned long long* d_ctr = nullptr;
    mutable unsigned ctr_next = 0;
    int g_n0 = 0, g_n1 = 0;   // significant leading / trailing terms of g0 / g1
    double* d_g = nullptr;
    double sa_first = 0, sc_last = 0, prev_sc_last = 0, next_sa_first = 0;
    double det_prev = 1, det_next = 1;
    int has_prev = 0, has_next = 0;
    int dd_defer[2] = {0, 0};             // k_dd2 allowed for 16 / 8 lines per tile

    // staged path (device tables indexed by block row)
    double* d_st = nullptr;
    double* d_w = nullptr;
    double* d_f = nullptr;
    double* d_r = nullptr;
    double* d_sa = nullptr;
    double* d_sc = nullptr;
    int* d_boff = nullptr;
    int* d_bsize = nullptr;
    double* d_bconst = nullptr;
    int nb = 1;
    int has_staged = 0;   // fast plan that also carries staged tables (long lines)
    // P=1 Thomas tables
    double* d_tha = nullptr;
    double* d_thw = nullptr;
    double* d_thcp = nullptr;
    double* d_thz = nullptr;
    double th_b0 = 1, th_qlast = 0, th_den = 1;
    // stencil window shifts of block rows 0, 1, rows-2, rows-1 (one-sided
    // closures that reach past the width-5 window: open d2/dx2)
    int sh[4] = {0, 0, 0, 0};

    // banded reduced map of a block-circulant H (uniform periodic P=1 plan:
    // every chunk's band row is the same nb values, chunk k's window starting
    // at (band_q0 + 2k) mod K): the row, for kernels that keep it in the
    // kernel-parameter bank (k_transport_dir). band_circ = 0 otherwise.
    int band_circ = 0, band_q0 = 0;
    std::vector<double2> band_row;

    std::vector<void*> allocs;
};
