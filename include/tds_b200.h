/*
 * tds_b200.h -- C ABI of the B200-native DistD2 batched tridiagonal solver.
 *
 * Drop-in boundary for the reference package `tds` (arXiv 2411.13532,
 * /root/reference/pkg/src/tds). The reference is pure Python/NumPy and has
 * no FFI of its own; the entry points below are what its operator layer
 * would bind (ctypes stub in INTEGRATION.md). Every function:
 *   - takes plain pointers and sizes (no torch types);
 *   - takes DEVICE pointers for field data, owned by the caller;
 *   - takes an explicit cudaStream_t (passed as void*) and never synchronises
 *     the host with the device, except the functions marked SYNCHRONOUS
 *     (plan creation / destruction, IPC setup, tds_mailbox_error);
 *   - returns 0 (TDS_OK) or a TDS_ERR_* code; tds_last_error() gives text.
 * All error conditions the reference raises (SingularPivot, SingularPair,
 * SingularCorrection, ValueError) are coefficient-only and are raised by
 * tds_plan_create on the host; kernels are error-free.
 *
 * Field layout ("SZ-blocked", reference layout.py:1-13): a field is
 * (groups, n, sz) fp64, linear index lane + sz*pos + sz*n*group. A "line"
 * is one (group, lane) pair; line l lives at (l/sz)*n*sz + l%sz with row
 * stride sz. Position-major (n, lanes) arrays are the case groups=1, sz=lanes.
 */
#ifndef TDS_B200_H
#define TDS_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define TDS_ABI_VERSION 2

#define TDS_OK 0
#define TDS_ERR_INVALID 1             /* ValueError (shape/partition/size)  */
#define TDS_ERR_SINGULAR_PIVOT 2      /* errors.SingularPivot               */
#define TDS_ERR_SINGULAR_PAIR 3       /* errors.SingularPair                */
#define TDS_ERR_SINGULAR_CORRECTION 4 /* errors.SingularCorrection          */
#define TDS_ERR_CUDA 5                /* CUDA runtime error                 */
#define TDS_ERR_UNSUPPORTED 6         /* e.g. NotImplementedError           */

/* plan flags */
#define TDS_FLAG_STRICT 1   /* reference arithmetic order, no FMA: bit-identical
                               to the reference (staged kernels)              */
#define TDS_FLAG_STAGED 2   /* force the staged (multi-pass) kernels           */
#define TDS_FLAG_CHUNK16 4  /* prefer 16-row chunks (register-light consumers:
                               the TMA-staged fused transport kernel)         */

/* execution paths reported by tds_plan_query */
#define TDS_PATH_FAST 0     /* single-pass chunked kernel (16 B/pt)           */
#define TDS_PATH_STAGED 1   /* staged kernels (reference structure)           */

typedef struct tds_plan tds_plan;

typedef struct {
    int n;              /* global rows per line                               */
    int rank_count;     /* P of the partition                                 */
    int rank;           /* -1: all P ranks emulated on this device            */
    int block_rows;     /* rows per line held by this device                  */
    int path;           /* TDS_PATH_*                                         */
    int strict;         /* 1 if TDS_FLAG_STRICT                               */
    int chunk_rows;     /* M (fast path)                                      */
    int chunks;         /* C = block_rows / M (fast path)                     */
    int uniform;        /* 1: every chunk shares one coefficient table;       *
                         * 2: all but a special first / last chunk do       *
                         *    (one-sided closures); 0: per-row table        */
    int periodic;
    double max_dropped; /* max |dropped coupling| over ranks (audit)          */
    double dominance_margin; /* system.py:163-167 of the global system        */
} tds_plan_info;

int tds_abi_version(void);
const char* tds_last_error(void);
/* rank whose per-rank stage failed (-1: not rank-specific); the Python
 * shim wraps such errors in RankPanic like transport.spawn_ranks does. */
int tds_last_error_rank(void);

/*
 * Build a plan for one operator: the global system (lower, diag, upper,
 * periodic; system.py:31-51), its width-5 RHS stencil (n x 5 row-major,
 * NULL = identity; distributed.py:71-116) and a partition of the n rows
 * into `rank_count` blocks `sizes` (system.py:115-155).
 * stencil_shift (NULL = none) is an EXTENSION for one-sided closures that
 * need more than the width-5 window (the open d2/dx2 operator; the
 * reference has none, compact.py:79-81): row j's weights apply to
 * u[j + o + stencil_shift[j]], o = -2..2. Non-zero shifts are allowed only
 * on rows 0, 1 (0..2) and n-2, n-1 (-2..0) of an open line (n >= 8).
 *   rank == -1 : this device runs the whole operator, all ranks emulated
 *                (replaces distributed.run_distd2, distributed.py:399-449);
 *   rank == k  : this device owns rank k's rows only (replaces the per-rank
 *                preprocess + distd2_solve, distributed.py:144-199,327-366).
 * Host-side, O(n + C^3): runs Alg. 5 (preprocess) per rank and per chunk and
 * uploads the coefficient tables with cudaMemcpy on the current device.
 * SYNCHRONOUS.
 */
int tds_plan_create(const double* lower, const double* diag, const double* upper,
                    int periodic, const double* stencil, const int* stencil_shift, int n,
                    const int* sizes, int rank_count, int rank, int flags,
                    tds_plan** out);
/* Per-rank plan from rank-local data only, the reference's per-rank view:
 * a, b, c, stencil are rank k's local_slice bands (m rows; a[0] couples to
 * the previous rank's last row, c[m-1] to the next rank's first row; open
 * edges 0) and stencil rows (+ optional shifts, as above, on the rows of an
 * edge without a neighbour); prev_sc_last / next_sa_first are the cached
 * neighbour couplings of share_pair_coeffs (distributed.py:308-324, D16). */
int tds_plan_create_local(const double* a, const double* b, const double* c,
                          const double* stencil, const int* stencil_shift, int m,
                          int has_prev, int has_next, double prev_sc_last,
                          double next_sa_first, int flags, tds_plan** out);
int tds_plan_destroy(tds_plan* plan);
int tds_plan_query(const tds_plan* plan, tds_plan_info* info);

/* Rank-level DistCoeffs of rank k (distributed.py:43-68), host arrays of
 * length sizes[k]: s_a, s_c, w, f, r; dropped[2] = signed dropped couplings. */
int tds_plan_rank_coeffs(const tds_plan* plan, int k, double* s_a, double* s_c,
                         double* w, double* f, double* r, double* dropped);

/* Alg. 5 alone on one block of m rows (preprocess, distributed.py:144-199):
 * a[0] couples to the row before the block, c[m-1] to the row after it.
 * Outputs host arrays of length m, bit-identical to the reference; s_c[0]
 * and s_a[m-1] are zeroed and their signed values returned in dropped[2]. */
/* pivot_floor: |pivot| <= pivot_floor raises SingularPivot (reference
 * default 1e-300, distributed.py:144). */
int tds_preprocess(const double* a, const double* b, const double* c, int m,
                   double pivot_floor, double* s_a, double* s_c, double* w, double* f,
                   double* r, double* dropped);

/*
 * Whole-operator solve (rank == -1 plans): out = A^{-1} stencil(u) with the
 * reference's truncation at the partition's rank boundaries
 * (run_distd2, distributed.py:399-449). u, out: (groups, n, sz) device,
 * distinct (non-aliasing) buffers -- the reference returns fresh arrays.
 * The persistent kernels take their work items from schedule counters held
 * in the plan (reset by each launch's last CTA): up to 64 launches of one
 * plan may be in flight at once on different streams.
 */
int tds_solve(const tds_plan* plan, const double* u, double* out,
              long long groups, int sz, void* stream);

/* ---- per-rank distributed pipeline (rank == k plans) -------------------
 * ROUND 1 (halo, transport.py:142-171) and ROUND 2 (boundary rows,
 * transport.py:174-191) are done by the caller (NCCL send/recv) between
 * these calls. All arrays are device memory:
 *   u, out              (groups, m, sz)    this rank's block
 *   first2, last2       (groups, 2, sz)    rows {0,1} and {m-2,m-1} of u
 *   halo_lo, halo_hi    (groups, 2, sz)    prev's last 2 / next's first 2
 *                                          rows, NULL on an open edge
 *   d_first, d_last     (groups, sz)       decoupled rows d[0], d[m-1]
 *   prev_last, next_first (groups, sz)     neighbours' d[m-1] / d[0], NULL
 *                                          on an open edge                 */
int tds_halo_rows(const tds_plan* plan, const double* u, double* first2,
                  double* last2, long long groups, int sz, void* stream);
/* Alg. 6 boundary values d[0], d[m-1] of every line (decouple_fused,
 * distributed.py:257-276). `scratch` is (groups, m, sz); the fast path does
 * not touch it, the staged path keeps d there for tds_finish. */
int tds_boundary_rows(const tds_plan* plan, const double* u, const double* halo_lo,
                      const double* halo_hi, double* d_first, double* d_last,
                      double* scratch, long long groups, int sz, void* stream);
/* 2x2 boundary pairs + Alg. 7 substitution (distributed.py:279-305,345-366).
 * For the staged path `out` must be the `scratch` given to tds_boundary_rows. */
int tds_finish(const tds_plan* plan, const double* u, const double* halo_lo,
               const double* halo_hi, const double* d_first, const double* d_last,
               const double* prev_last, const double* next_first, double* out,
               long long groups, int sz, void* stream);

/* ---- fused per-rank solve over NVLink peer memory (k_dd) ----------------
 * One kernel per rank does the whole distd2_solve (distributed.py:327-366):
 * both neighbour rounds are peer stores into the neighbours' MAILBOXES,
 * fence-free (sentinel-armed slots). A mailbox is tds_mailbox_words(groups,
 * sz) 8-byte words prepared by tds_mailbox_init (tds_ipc_alloc does this);
 * neighbours map it with CUDA IPC (one process per GPU) or use the pointer
 * directly (several ranks in one process: same device, or peer access
 * enabled with tds_peer_access).
 * `epoch` must increase by one per solve (same value on every rank). All
 * ranks must have the same block size and the same `max_ctas`: the kernel is
 * persistent and every rank must run the same schedule. max_ctas == 0 uses
 * the device's resident capacity, max_ctas > 0 caps it, max_ctas = -k uses
 * capacity / k: ranks SHARING a device (k of them at most on any device)
 * must split it so that all of them are co-resident. A wait that exceeds 10 s (TDS_FUSED_TIMEOUT_MS) sets the
 * mailbox error word and yields NaN instead of hanging.
 * The last three words of every mailbox are STATUS words: [0] error
 * (1 = timeout), [1] / [2] cumulative halo / boundary-row words this rank
 * posted to its neighbours (measured message accounting). */
long long tds_mailbox_words(long long groups, int sz);
int tds_mailbox_init(double* mail, long long words, void* stream);
/* async copy of the three status words into host memory (pinned for true
 * asynchrony); `words` is the mailbox length */
int tds_mailbox_status(const double* mail, long long words, unsigned long long* host_status,
                       void* stream);
int tds_fused_eligible(const tds_plan* plan, long long groups, int sz);
/* The fused kernel variant (deferred edges or not, for 16 / 8-line tiles) is
 * a per-plan property, but all ranks MUST launch the same variant: AND the
 * plan's variant mask (bit 0: deferral allowed with 16-line tiles, bit 1:
 * with 8-line tiles) with `mask` and return the result. Ranks agree by
 * calling it with 3, reducing the results with AND over the group and
 * calling it again with the agreed mask (rank.DistD2Rank does this). */
int tds_plan_restrict_fused(tds_plan* plan, int mask);
/* The persistent grid tds_fused_solve would use for this plan and shape
 * (max_ctas as there; -1: not eligible). Ranks whose table variants differ
 * (edge ranks of open operators) can have different occupancies: they take
 * the MINIMUM over the group and pass it as max_ctas (rank.DistD2Rank). With
 * max_ctas <= 0 the launch itself uses the minimum over all variants. */
long long tds_fused_grid(const tds_plan* plan, long long groups, int sz, int max_ctas);
int tds_fused_solve(const tds_plan* plan, const double* u, double* out,
                    long long groups, int sz, double* mail, double* mail_prev,
                    double* mail_next, unsigned long long epoch, int max_ctas, void* stream);
/* SYNCHRONOUS convenience: *err = 1 if the mailbox recorded a timeout */
int tds_mailbox_error(const double* mail, long long groups, int sz, int* err);
/* CUDA IPC plumbing for mailboxes: handle is 64 bytes (cudaIpcMemHandle_t).
 * tds_ipc_alloc prepares the mailbox (tds_mailbox_init) and synchronises
 * before returning the handle. */
int tds_ipc_alloc(long long bytes, void** ptr, unsigned char* handle);
int tds_ipc_open(const unsigned char* handle, void** ptr);
int tds_ipc_close(void* ptr);
int tds_ipc_free(void* ptr);
/* enable access from the current device to peer_device (no-op if equal or
 * already enabled); TDS_ERR_UNSUPPORTED if the pair has no P2P path */
int tds_peer_access(int peer_device);

/* ---- phase-level kernels, reference arithmetic (bit-identical) ----------
 * Position-major (rows, lanes) device arrays, as the reference phase
 * functions take them. Coefficient arrays (stencil m x 5, w, f, r, s_a, s_c
 * of length m) are DEVICE arrays too: no allocation, copy or host
 * synchronisation per call. */
/* decouple_fused: u_ext (m+4, lanes) -> d (m, lanes); distributed.py:257-276.
 * shift4: NULL, or the HOST array of the window shifts of rows 0, 1, m-2,
 * m-1 (tds_plan_create's stencil_shift extension). */
int tds_decouple_fused(const double* u_ext, const double* stencil, const int* shift4,
                       const double* w, const double* f, const double* r, double* d, int m,
                       long long lanes, void* stream);
/* substitute: d (m, lanes) -> out (m, lanes); distributed.py:296-305 */
int tds_substitute(const double* d, const double* s_a, const double* s_c,
                   const double* u_start, const double* u_end, double* out, int m,
                   long long lanes, void* stream);
/* solve_boundary_pair over lanes; distributed.py:279-293 */
int tds_boundary_pair(const double* d_last, const double* d_first, double s_c_last,
                      double s_a_first, double* u_last, double* u_first,
                      long long lanes, void* stream);
/* thomas_solve / periodic_thomas_solve (serial.py:26-90) on a (groups, n, sz)
 * field; an RhsBatch (m, n) is groups = m, sz = 1. Bands are host arrays;
 * the multipliers are built once per (operator, pivot_floor, device) and
 * cached, so repeated calls allocate and copy nothing. */
int tds_thomas(const double* lower, const double* diag, const double* upper,
               int periodic, const double* rhs, double* out, int n,
               long long groups, int sz, double pivot_floor, void* stream);

/* ---- momentum-transport RHS (momentum.py:102-169) ------------------------
 * One (component i, direction j) contribution of the skew-symmetric
 * transport RHS, -1/2 (u_j du_i/dx_j + d(u_j u_i)/dx_j) + nu d2u_i/dx_j2, in
 * ONE fused pass over u_i and u_j (both in the j layout): d1 / d2 are P=1
 * plans of the periodic d/dx and d2/dx2 operators (d2 may be NULL when
 * nu == 0). accumulate = 1 adds into out. */
int tds_transport_contribution(const tds_plan* d1, const tds_plan* d2,
                               const double* u_i, const double* u_j, double* out,
                               double nu, int accumulate, long long groups, int sz,
                               void* stream);
/* elementwise combine of precomputed derivatives (rank-emulated path) */
int tds_transport_combine(const double* u_j, const double* du, const double* dp,
                          const double* d2u, double nu, double* out, long long count,
                          int accumulate, void* stream);
/* One (i, j) transport term along a direction split over the ranks
 * (one rank per GPU; SlabTransport's z terms): out = -1/2 (u_j d(u_i) +
 * d(u_j u_i)) + nu d2(u_i) on this rank's (groups, m, sz) block, the three
 * DistD2 solves fused in one kernel with their neighbour rounds done over
 * IPC-mapped mailboxes (tds_transport_mailbox_words words each, prepared by
 * tds_mailbox_init; same status words and max_ctas rule as tds_fused_solve). d1 / d2: this rank's d/dx and d2/dx2 plans with
 * 16-row chunks (TDS_FLAG_CHUNK16). Replaces directional_contribution
 * (momentum.py:102-126) with run_distd2 over the rank chain.
 * TDS_ERR_UNSUPPORTED when the plans / field do not allow it. */
long long tds_transport_mailbox_words(long long groups, int sz);
int tds_transport_mailbox_error(const double* mail, long long groups, int sz, int* err);
int tds_fused_transport(const tds_plan* d1, const tds_plan* d2, const double* u_i,
                        const double* u_j, double* out, double nu, long long groups, int sz,
                        double* mail, double* mail_prev, double* mail_next,
                        unsigned long long epoch, int max_ctas, void* stream);

/* The same distributed term read IN PLACE from a rank's x-layout z-slab
 * (nx, ny, m) -- the z lines of SlabTransport without re-layout passes --
 * and ADDED into the x-layout accumulator acc by TMA reduce-add. Same plans,
 * mailboxes (tds_transport_mailbox_words(nx ny / sz, sz) words) and epoch /
 * max_ctas rules as tds_fused_transport; sz | ny. Replaces reorder(x->z) +
 * directional_contribution + reorder/accumulate(z->x) of one term
 * (momentum.py:129-169) on the rank chain. */
int tds_fused_transport_in_x(const tds_plan* d1, const tds_plan* d2, const double* u_i,
                             const double* u_j, double* acc, double nu, int nx, int ny, int m,
                             int sz, double* mail, double* mail_prev, double* mail_next,
                             unsigned long long epoch, int max_ctas, void* stream);

/* All three z contributions of a rank's x-layout z-slab (nx, ny, m) in ONE
 * kernel per rank (k_dd_transport_dir): u0..u2 read once in place, the nine
 * DistD2 solves with their neighbour rounds over the mailboxes, each
 * component's term added into acc_i by TMA reduce-add. The distributed
 * counterpart of tds_transport_direction (dir = 2); plans, mailboxes
 * (tds_transport_mailbox_words(nx ny / sz, sz) words, shared with the
 * per-term kernels) and epoch / max_ctas rules as tds_fused_transport. */
int tds_fused_transport_direction(const tds_plan* d1, const tds_plan* d2, const double* u0,
                                  const double* u1, const double* u2, double* acc0, double* acc1,
                                  double* acc2, double nu, int nx, int ny, int m, int sz,
                                  double* mail, double* mail_prev, double* mail_next,
                                  unsigned long long epoch, int max_ctas, void* stream);

/* acc += the (i, dir) contribution, dir = 1 (y) or 2 (z), for an
 * (nx, ny, nz) block with everything in the x layout (groups = ny nz/sz, nx,
 * sz): the y / z lines are read in place through 4-D tensor maps and the
 * result is added into acc. Replaces the reference's reorder(x->dir) +
 * contribution + reorder/accumulate(dir->x) of one term (momentum.py:
 * 129-169); a rank's z-slab uses it for y. Plans: 16-row-chunk P=1 d/dx (d1)
 * and d2/dx2 (d2) operators of the line length (TDS_FLAG_CHUNK16); sz | ny;
 * y additionally needs sz = 32, 16 | nx. TDS_ERR_UNSUPPORTED otherwise. */
int tds_transport_contribution_in_x(const tds_plan* d1, const tds_plan* d2, const double* u_i,
                                    const double* u_j, double* acc, double nu, int nx, int ny,
                                    int nz, int sz, int dir, void* stream);
/* All three components' contributions along ONE direction `dir` (0 x, 1 y,
 * 2 z) for an (nx, ny, nz) block with every array in the x layout (groups =
 * ny nz/sz, rows, sz): out_i = (dir 0) or += (dir 1, 2) -1/2 (u_dir du_i +
 * d(u_dir u_i)) + nu d2u_i along dir, for i = 0, 1, 2, in one pass that reads
 * u0, u1, u2 once (k_transport_dir). Replaces the three
 * directional_contribution calls of one direction plus their reorders
 * (momentum.py:102-169): three launches evaluate the whole RHS. Plans as for
 * tds_transport_contribution_in_x (16-row-chunk P=1 d/dx and d2/dx2 of the
 * line length); y needs sz = 32 and 8 | nx. TDS_ERR_UNSUPPORTED otherwise. */
int tds_transport_direction(const tds_plan* d1, const tds_plan* d2, const double* u0,
                            const double* u1, const double* u2, double* out0, double* out1,
                            double* out2, double nu, int nx, int ny, int nz, int sz, int dir,
                            void* stream);
/* elementwise helpers of the transport demo: out = u + dt * rhs (the Euler
 * step, momentum.py:216-222) and out = a * b (the u_j u_i product of the
 * 3-solve fallback contribution, momentum.py:118) */
int tds_euler_update(const double* u, const double* rhs, double dt, double* out,
                     long long count, void* stream);
int tds_multiply(const double* a, const double* b, double* out, long long count, void* stream);

/* cubic n^3 field: SZ-blocked layout of src_dir -> dst_dir in one pass
 * (reorder, layout.py:144-152); accumulate = 1 adds into dst */
int tds_reorder(const double* src, double* dst, int n, int sz, int src_dir,
                int dst_dir, int accumulate, void* stream);
/* the same for an (nx, ny, nz) block (a rank's slab of the transport step);
 * both layouts must be unpadded (lines divisible by sz) */
int tds_reorder3(const double* src, double* dst, int nx, int ny, int nz, int sz,
                 int src_dir, int dst_dir, int accumulate, void* stream);

/* ---- layout (layout.py:82-152) -------------------------------------------
 * Cartesian (nx, ny, nz) C-order <-> SZ-blocked (groups, n, sz) field for
 * `direction` ('x'=0,'y'=1,'z'=2). groups*sz may exceed the line count:
 * the ghost lines are zero-filled by tds_pack (LayoutDescriptor pad=True). */
int tds_pack(const double* cart, double* field, int nx, int ny, int nz, int sz,
             int direction, long long groups, void* stream);
int tds_unpack(const double* field, double* cart, int nx, int ny, int nz, int sz,
               int direction, long long groups, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TDS_B200_H */
