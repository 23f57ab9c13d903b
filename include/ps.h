/* ps.h — C ABI of libps: the B200-native solve phase (and its O(N) setup) of the
 * two-term power-series method of Negi, Balakrishnan & Rao, "Fast Power Series
 * Solution of Large 3-D Electrodynamic Integral Equation for PEC Scatterers",
 * arXiv 2109.04129 (PAPER.md in the reference tree; line numbers "P:n").
 *
 * Problem statement (Eq. 9): [Z] x = b, Z dense N x N, here given as
 * the H-matrix Z = Z_N + Z_F (Eq. 13): dense symmetric near-field leaf
 * blocks Z_ij (Eq. 14; symmetric storage P:105) and ACA far
 * blocks Z_sub ~ U V^T (Eq. 11). Extended to a block of nrhs columns.
 *
 * Conventions (all entry points):
 *   - complex = interleaved complex128 (re, im) = C99 `double _Complex`;
 *   - matrices column-major with an explicit leading dimension; 0-based;
 *   - sizes are int64_t; B and X use the ORIGINAL RWG basis order of the
 *     generator (edges sorted by node pair); every internal permutation
 *     (octree/Morton order, nested-dissection elimination order) is private;
 *   - no exception crosses the ABI; every call returns a ps_status and, on
 *     failure, ps_last_error() holds a one-line message;
 *   - calls on one handle must not run concurrently (a handle owns streams,
 *     workspaces and cached solve plans).
 *
 * ---------------------------------------------------------------------------
 * H-matrix file (".hm", written by hmgen/build.py:write_hm), little-endian:
 *   header (128 B): "HMPS", u32 version=1, i64 N, i64 n_leaves, i64 n_near,
 *     i64 n_far, i64 flags (bit0 = symmetric), f64 lambda, f64 k, f64 leaf_edge,
 *     i64 L, f64 origin[3], f64 root_edge, i64 near_arena_len, i64 far_arena_len
 *   then u64 checksum(header) and, for each section, its bytes padded to 8 B
 *   followed by u64 checksum(section bytes):
 *     perm[N] i64        Morton position -> RWG index
 *     leaf_off[n_leaves+1] i64   leaf (Morton id) -> first Morton position
 *     leaf_ijk[n_leaves][3] i32  octree box index of the leaf
 *     elim_order[n_leaves] i32   elimination order (nested dissection)
 *     near_list[n_near][3] i64   (i, j, offset), i <= j; Z_ij column-major
 *                                n_i x n_j at near_arena[offset]; Z_ji = Z_ij^T
 *     near_arena[near_arena_len] complex128
 *     far_list[n_far][7] i64     (row0, m, col0, n, level, r, offset): block
 *                                rows [row0,row0+m) x cols [col0,col0+n) in
 *                                Morton positions ~ U V^T, U (m x r) at offset,
 *                                V (n x r) at offset + m r; the mirrored block
 *                                (cols x rows) = V U^T is implied, not stored
 *     far_arena[far_arena_len] complex128
 *   checksum64(bytes) = (sum_i w_i (2i+1) mod 2^64) XOR nbytes over the
 *   little-endian u64 words w_i of the zero-padded bytes.
 */
#ifndef PS_H_
#define PS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ps_handle ps_handle;

typedef enum {
  PS_OK = 0,
  PS_EINVAL = 1,     /* bad argument: NULL pointer, ldb < N, nrhs < 1, X aliases B, ... */
  PS_EIO = 2,        /* file cannot be opened / read */
  PS_EFORMAT = 3,    /* bad magic, version, size or checksum */
  PS_ENOMEM = 4,     /* host or device allocation failed */
  PS_ECUDA = 5,      /* CUDA runtime error (message carries cudaGetErrorString) */
  PS_ENCCL = 6,      /* reserved: collective failure (multi-GPU row partition) */
  PS_ESINGULAR = 7,  /* a scaled diagonal block Z~_kk had a pivot |u_ii| <= 1e-14 ||Z~_kk||_F;
                        the message names the leaf (Morton id) and its elimination position */
  PS_EDIVERGED = 8,  /* >= 1 RHS column had ||it_1|| / ||it_0|| >= ratio_threshold
                        (Eq. 45); X IS STILL FULLY WRITTEN */
  PS_ESTATE = 9      /* call order violated (ps_solve before ps_setup, ...) */
} ps_status;

/* Process placement.
 *   partition = 0 : replicated operator. Every rank loads the whole operator
 *                   and solves the RHS columns it is given (the caller splits
 *                   the columns); no collective. nccl_unique_id must be NULL.
 *   partition = 1 : row partition over nranks. Whole subtrees of the
 *                   elimination tree (leaf-cluster block rows: their alpha
 *                   panels, D^-1 and the far-field rows they own) are assigned
 *                   to ranks, the separator nodes above them are replicated.
 *                   One solve = 4 phases separated by collectives (sum
 *                   all-reduce of the separator rows after each interior forward
 *                   sweep, all-gather of w = R b_o before the far field — the
 *                   exchange between the two series terms — and of x at the end).
 *                   nccl_unique_id != NULL: 128-byte ncclUniqueId from
 *                   ps_nccl_unique_id() on rank 0, shared by the caller; hm_load
 *                   then joins the NCCL communicator (collective: all ranks must
 *                   call it) and ps_solve runs this rank's share (every rank
 *                   passes the full B and receives the full X).
 *                   nccl_unique_id == NULL: in-process group; the handles of all
 *                   ranks live in one process and are solved with ps_solve_group.
 *   device         : CUDA device of this rank. */
typedef struct {
  int rank, nranks, device;
  const void* nccl_unique_id;
  int partition;
} ps_dist;

typedef struct {
  int deterministic;        /* 1 (default): fixed summation order, bitwise repeatable (always true in v1) */
  int ordering;             /* 0 (default): elimination order from the file (nested dissection);
                               2: reverse Cuthill-McKee on the leaf near-field graph (recomputed in
                               ps_setup; not with a row partition). x is order-invariant, the
                               scaling (hence it_0 / it_1) is not. Others: PS_EINVAL. */
  int amalgamate_separators;/* reserved, must be 0 */
  double ratio_threshold;   /* divergence threshold of Eq. 45 / P:245; default 0.1; ratio >= thr => diverged */
} ps_setup_opts;

typedef struct {
  int64_t nrhs;             /* in: capacity of it0_norm / it1_norm (ignored if both NULL) */
  double* it0_norm;         /* out [nrhs] or NULL: ||it_0|| = ||b_o||_2 per column (Eq. 44) */
  double* it1_norm;         /* out [nrhs] or NULL: ||it_1|| = ||U b_o||_2 per column */
  int n_diverged;           /* out: columns with it1/it0 >= threshold */
  double t_solve_ms;        /* out: device time of the solve (CUDA events on the solve stream) */
  double bytes_moved;       /* out: algorithmic operator + vector bytes of this solve */
  double flops;             /* out: algorithmic flops of this solve */
  int64_t kernel_launches;  /* out: libps kernels launched by this call */
  double* ratio;            /* out [nrhs] or NULL: ||it_1|| / ||it_0|| per column (Eq. 45 LHS; 0 when
                               ||it_0|| = 0); the quantity compared with ratio_threshold */
} ps_report;

/* hm_load — read and verify an ".hm" file (layout above), copy the near and far
 * arenas to the device of `dist->device` (or the current device when dist is
 * NULL) and run the symbolic analysis (struct(k) with fill, elimination tree,
 * schedules; Eqs. 14-23 structure).
 *   path : NUL-terminated file name.            dist: NULL = single GPU.
 *   out  : receives the new handle (caller frees with ps_free); *out = NULL on error.
 * Errors: PS_EINVAL (NULL args), PS_EIO, PS_EFORMAT, PS_ENOMEM, PS_ECUDA. */
ps_status hm_load(const char* path, const ps_dist* dist, ps_handle** out);

/* ps_setup — the O(N) setup of P:105-171 (Eqs. 14-23) on the GPU: for every
 * leaf k in elimination order (level-parallel over the elimination tree):
 *   Z~_kk, Z~_kj after all Schur updates Z~_ij += alpha_ki^T Z~_kj (Eq. 21, fill
 *   included), D_k^{-1} = Z~_kk^{-1} (LU-type elimination with partial pivoting,
 *   explicit inverse), alpha_kj = -D_k^{-1} Z~_kj (Eq. 16).
 * opts: NULL = defaults. Frees the near-field input arena when done.
 * Row partition with NCCL (ps_dist.partition = 1, nccl_unique_id set): collective —
 * every rank calls it; each factors only its own interior subtrees and the separators,
 * with one NCCL sum all-reduce of the separator rows' partial W between the phases.
 * An in-process partition handle must use ps_setup_group (PS_ESTATE otherwise).
 * Errors: PS_EINVAL, PS_ESTATE (already set up), PS_ESINGULAR (message names
 * the leaf), PS_ENOMEM, PS_ECUDA. */
ps_status ps_setup(ps_handle* h, const ps_setup_opts* opts);

/* ps_setup_group — ps_setup of an in-process row partition (handles of ranks
 * 0..nranks-1 from hm_load with partition = 1 and nccl_unique_id = NULL, all on one
 * device): every rank runs its sharded setup (its own interior subtrees, then its
 * interior's Schur updates of the separator rows), the separator rows' partial W are
 * summed over the ranks in rank order (the in-process stand-in of the NCCL all-reduce
 * that ps_setup performs on an NCCL rank), then every rank eliminates the separators.
 * opts as ps_setup (ordering must be 0). Errors as ps_setup, plus PS_EINVAL when the
 * handles are not one consistent group. */
ps_status ps_setup_group(ps_handle* const* hs, int nranks, const ps_setup_opts* opts);

/* ps_solve — the two-term power-series solve (Eqs. 24, 26, 30-36):
 *   b~ = R^T b (Eq. 24), b_o = D^{-1} b~ (Eq. 32), u = U b_o = D^{-1} R^T Z_F R b_o
 *   (Eq. 31), x~ = b_o - u (Eq. 36, two terms), x = R x~ (Eq. 26),
 * with R = alpha_1 alpha_2 ... alpha_{n-1} applied as a block back-substitution
 * and R^T as a forward substitution over the stored alpha panels.
 *   nrhs      : number of columns, >= 1.
 *   B, ldb    : N x nrhs input, column-major, ldb >= N; read only.
 *   X, ldx    : N x nrhs output, column-major, ldx >= N; must not overlap B.
 *   on_device : 0 = B and X are host pointers (any host memory; pinned is
 *               faster); 1 = device pointers on this handle's GPU. Host blocks of
 *               >= 256 columns are solved as two column halves whose host<->device
 *               copies run on the handle's copy streams under the other half's
 *               kernels (columns are independent problems; same result as two
 *               ps_solve calls on the halves).
 *   cuda_stream : cudaStream_t to order the work on, or NULL for the handle's
 *               own stream. With on_device=1 the call returns once the work is
 *               queued AND complete (it synchronises the stream).
 *   rep       : optional report (see ps_report).
 * Errors: PS_EINVAL, PS_ESTATE (no ps_setup yet), PS_ENOMEM, PS_ECUDA,
 * PS_EDIVERGED (X fully written; see rep->n_diverged). */
ps_status ps_solve(ps_handle* h, int64_t nrhs, const void* B, int64_t ldb, void* X, int64_t ldx,
                   int on_device, void* cuda_stream, ps_report* rep);

/* ps_solve_async — ps_solve for DEVICE buffers without its host synchronisation: the same
 * kernels (Eqs. 24, 26, 30-36, and the per-column norms of Eqs. 44-45) are queued on
 * cuda_stream (NULL = the handle's own stream) and the call returns; X, the norms and the
 * ratios are complete when the stream reaches that point. Successive calls on ONE stream
 * pipeline (the host queues solve i + 1 while solve i runs); a handle must not be used
 * from two streams at once (its workspace is shared). The report of the LAST queued solve
 * is fetched with ps_solve_report. Single-GPU handles only (PS_ESTATE on a row-partition rank).
 * Arguments as ps_solve with on_device = 1. Errors: PS_EINVAL, PS_ESTATE, PS_ENOMEM, PS_ECUDA
 * (launch errors only; PS_EDIVERGED is reported by ps_solve_report). */
ps_status ps_solve_async(ps_handle* h, int64_t nrhs, const void* B, int64_t ldb, void* X, int64_t ldx,
                         void* cuda_stream);

/* ps_solve_report — synchronise the stream of the last ps_solve_async and fill its report
 * (rep may be NULL: status only): ||it_0||, ||it_1||, the Eq. 45 ratio per column,
 * n_diverged; t_solve_ms = device time of that last solve. Returns PS_EDIVERGED like ps_solve.
 * Errors: PS_EINVAL, PS_ESTATE (nothing pending), PS_ECUDA. */
ps_status ps_solve_report(ps_handle* h, ps_report* rep);

/* ps_solve_series — the n-term power series: Eqs. (35)-(36),
 * P:195-197, x~ = it_0 - it_1 + it_2 - ... (Eq. 44), it_0 = b_o = Z~_N^{-1} R^T b
 * (Eqs. 24, 32), it_n = U it_{n-1} (Eq. 31), x = R x~ (Eq. 26), with the per-term norm
 * ratio of Eq. 45 monitored on the device. Terms are added until
 *   - n == max_terms, or
 *   - tol > 0 and, after term n >= 1, every column has ||it_n|| <= tol ||x~_{n+1}||
 *     (x~_{n+1} = the partial sum through it_n; R25).
 * max_terms = 2, tol = 0 is the two-term solve of ps_solve (same result up to rounding
 * order: this path runs one launch set per operator, ps_solve one dataflow program).
 * A column DIVERGES when its last ratio ||it_n|| / ||it_{n-1}|| >= 1 (the terms do not
 * shrink, so the partial sums cannot converge: ||U|| <= 1 of P:203 fails).
 *   opts      : max_terms in [1, 4096]; tol >= 0 (NULL: max_terms = 2, tol = 0).
 *   B, X, ldb, ldx, on_device, cuda_stream : as ps_solve (single-GPU handles only).
 *   rep       : optional; rep->it_norm (capacity rep->nrhs columns x rep->max_terms
 *               terms, term-major it_norm[n * rep->nrhs + c]) receives ||it_n||_2 for
 *               every term computed; n_terms the terms summed; n_diverged as above.
 * Errors: PS_EINVAL (bad opts / arguments), PS_ESTATE (no ps_setup, or a row-partition
 * handle), PS_ENOMEM, PS_ECUDA, PS_EDIVERGED (X fully written). */
typedef struct {
  int max_terms;
  double tol;
} ps_series_opts;

typedef struct {
  int64_t nrhs;             /* in: column capacity of it_norm */
  int64_t max_terms;        /* in: term capacity of it_norm */
  double* it_norm;          /* out [max_terms x nrhs], term-major, or NULL */
  int n_terms;              /* out: terms summed (it_0 .. it_{n_terms-1}) */
  int n_diverged;           /* out: columns whose last ratio ||it_n|| / ||it_{n-1}|| >= 1 */
  double t_solve_ms;        /* out: device time (CUDA events on the solve stream) */
  double bytes_moved;       /* out: algorithmic bytes: 16 (2 n_R + n_D) + per extra term
                               16 (2 n_R + n_D + n_F), + vector passes */
  double flops;             /* out: algorithmic flops: 8 nrhs (2 n_R + n_D) + per extra term
                               8 nrhs (2 n_R + n_D + 2 n_F) */
  int64_t kernel_launches;  /* out: libps kernels launched by this call */
} ps_series_report;

ps_status ps_solve_series(ps_handle* h, const ps_series_opts* opts, int64_t nrhs, const void* B, int64_t ldb,
                          void* X, int64_t ldx, int on_device, void* cuda_stream, ps_series_report* rep);

/* ps_farfield — far field and radar cross section of RWG surface currents (SURVEY §8(f)
 * NEXT-4: the RCS curves of PAPER.md:333-341 computed from the solve's X on the GPU).
 *   F(r^, c) = sum_n I[n, c] int f_n(r') e^{+j k r^.r'} dS'  (7-point degree-5 rule per
 *   triangle), f_n the RWG function of P:71: +l_n/(2A+) (r' - v+) on T+, -l_n/(2A-) (r' - v-)
 *   on T-, l_n = the length of the edge T+ and T- share;
 *   sigma_theta / sigma_phi = (k eta)^2 / (4 pi) |F . theta^|^2, |F . phi^|^2 in m^2 for a
 *   unit-amplitude incident plane wave (theta^, phi^ of r^; phi = 0 on the z axis).
 * ALL arrays are DEVICE pointers on the current device (no handle is needed):
 *   nodes [nnodes x 3] f64 (m), tris [ntris x 3] i64 node ids;
 *   tp, tm, vp, vm [N] i64: triangles T+ / T- of basis n and their free vertices
 *                (node ids; the generator's RWG order = the order of I's rows);
 *   k (rad/m) >= 0, eta (ohm); I [N x nrhs] complex128 column-major, ldi >= N;
 *   rhat [ndir x 3] f64 unit observation directions;
 *   mono = 0: bistatic, F [ndir x nrhs x 3] complex128 (F[(d nrhs + c) 3 + xyz]) and
 *             sigma [ndir x nrhs x 2] f64 (theta, phi), every direction for every column;
 *   mono = 1: monostatic, ndir == nrhs, direction d paired with column d only:
 *             F [ndir x 3], sigma [ndir x 2];
 *   sigma may be NULL (F only). cuda_stream: cudaStream_t or NULL (legacy default stream);
 *   returns after the work completed. Index arrays are trusted (not range-checked).
 * Errors: PS_EINVAL (sizes, NULL pointers, mono with ndir != nrhs), PS_ENOMEM, PS_ECUDA;
 * message in ps_last_error(NULL). Deterministic (fixed split order). */
ps_status ps_farfield(int64_t nnodes, const double* nodes, int64_t ntris, const int64_t* tris, int64_t N,
                      const int64_t* tp, const int64_t* tm, const int64_t* vp, const int64_t* vm, double k,
                      double eta, const void* I, int64_t ldi, int64_t nrhs, int64_t ndir, const double* rhat,
                      int mono, void* F, double* sigma, void* cuda_stream);

/* ps_solve_group — one two-term solve of a row-partitioned problem whose ranks
 * are handles of THIS process (hm_load with partition = 1, nccl_unique_id =
 * NULL, ranks 0..nranks-1 in hs[0..nranks-1], all on one device). The phases
 * of every rank run in rank order on one stream and the collectives are
 * device copies / fixed-order sums between the ranks' workspaces — the same
 * per-rank work and exchange layout as the NCCL path, without concurrency.
 *   B, X : device pointers (N x nrhs, column-major, RWG order); X written from
 *          rank 0's gathered result. Other arguments as ps_solve.
 * Errors: PS_EINVAL (handles not one consistent group), PS_ESTATE, PS_ECUDA,
 * PS_EDIVERGED (X fully written). */
ps_status ps_solve_group(ps_handle* const* hs, int nranks, int64_t nrhs, const void* B, int64_t ldb,
                         void* X, int64_t ldx, void* cuda_stream, ps_report* rep);

/* ps_nccl_unique_id — ncclGetUniqueId into out[0..128) (call on rank 0, share
 * the bytes, pass them as ps_dist.nccl_unique_id on every rank). NCCL is
 * loaded at run time (libnccl.so.2). Errors: PS_EINVAL (cap < 128), PS_ENCCL. */
ps_status ps_nccl_unique_id(void* out, int64_t cap);

/* ps_partition — host-only: the row partition hm_load would use for nranks
 * ranks (no GPU needed). For every elimination position p (0..n_leaves-1):
 * owner[p] = rank owning the interior node p, or -1 for a replicated separator
 * node; far_owner[p] = rank computing the far-field rows of leaf p.
 * cap = capacity of both arrays. Returns n_leaves, or -ps_status on error. */
int64_t ps_partition(const char* path, int nranks, int32_t* owner, int32_t* far_owner, int64_t cap);

/* ps_n — number of unknowns N of the loaded H-matrix; -1 if h is NULL. */
int64_t ps_n(const ps_handle* h);

/* ps_last_error — message of the last failed call on h (or of the last failed
 * hm_load on this thread when h is NULL). Never NULL; owned by the library. */
const char* ps_last_error(const ps_handle* h);

/* ps_free — release all host and device memory of h. NULL-safe; legal after
 * hm_load without ps_setup. */
void ps_free(ps_handle* h);

/* ------------------------------------------------------------------------
 * Diagnostic entry points (parity tests of individual hot-path steps).
 * All vectors: N x nrhs column-major, ORIGINAL RWG order, DEVICE pointers on
 * the handle's GPU; ld = N. The call synchronises before returning.
 *   op = PS_OP_RT    : Y = R^T X            (forward sweep, Eq. 24)
 *        PS_OP_DINV  : Y = D^{-1} X         (Eq. 32)
 *        PS_OP_R     : Y = R X              (backward sweep, Eq. 26)
 *        PS_OP_ZF    : Y = Z_F X            (far field, Eq. 13; both halves of each pair)
 *        PS_OP_U     : Y = D^{-1} R^T Z_F R X (Eq. 31)
 * Errors: PS_EINVAL (bad op / nrhs), PS_ESTATE (PS_OP_ZF is legal before setup,
 * the others are not), PS_ECUDA. */
enum { PS_OP_RT = 1, PS_OP_DINV = 2, PS_OP_R = 3, PS_OP_ZF = 4, PS_OP_U = 5 };
ps_status ps_apply(ps_handle* h, int op, int64_t nrhs, const void* X, void* Y);

/* ps_info — structural statistics into out[0..n): see PS_INFO_* indices.
 * Returns the number of values written (<= n). */
enum {
  PS_INFO_N = 0, PS_INFO_NLEAVES, PS_INFO_NNEAR, PS_INFO_NFAR, PS_INFO_ALPHA_BLOCKS,
  PS_INFO_NR, PS_INFO_ND, PS_INFO_NF, PS_INFO_HEIGHT, PS_INFO_DEPTH, PS_INFO_SETUP_MADDS,
  PS_INFO_SETUP_DONE,
  PS_INFO_NRANKS,            /* ranks of the row partition (1 otherwise) */
  PS_INFO_OWN_ROWS,          /* unknowns in this rank's interior subtrees */
  PS_INFO_SEP_ROWS,          /* unknowns in the replicated separator nodes */
  PS_INFO_CHAINS,            /* elimination-tree chain pieces with >= 2 leaves (applied through T_c) */
  PS_INFO_CHAIN_HEIGHT,      /* levels of the chain graph (dependent stages of a sweep / 2) */
  PS_INFO_T_ENTRIES,         /* complex entries of all T_c (U_c x U_c each) */
  PS_INFO_OP_BYTES,          /* device bytes of the operator this handle holds (alpha panels, D^-1, T, far
                                stacks); a row-partition rank holds only its share */
  PS_INFO_SETUP_BYTES,       /* device bytes of the setup arenas of this handle (near blocks held, W, alpha
                                panels, D^-1): a row-partition rank holds its interior plus the separators */
  PS_INFO_COUNT
};
int ps_info(const ps_handle* h, double* out, int n);

/* ps_analyze — host-only: read + verify the file and run the symbolic analysis
 * (no GPU needed); writes the ps_info statistics of the would-be handle.
 * Returns the number of values written, or -ps_status on error (message in
 * ps_last_error(NULL)). */
int ps_analyze(const char* path, double* out, int n);

/* ps_validate — host-only check of the single-launch solve program for nrhs columns
 * (the task / segment / work-item tables ps_solve would launch): every
 * operand access inside its arena, no workspace element written by two tasks, every
 * read of a written range waiting on exactly that range's writer, and every item's
 * producers at smaller tickets (deadlock freedom of the persistent kernel). For nrhs
 * <= 8 the program is two launches around the one-pass far apply (far1p): tasks of
 * different launches are ordered by launch order, and the far1p tables are checked too
 * (factor ranges inside the FB arena, rows inside the vectors, every waiting item after
 * its producers). stats (optional, up to 7): tasks, segments, work items, write ranges,
 * read ranges, the largest ticket distance to a producer, far1p items (-1 / untouched:
 * none). Returns the number of work items, or
 * -ps_status (PS_ESTATE: a property is violated; the message names it). */
int64_t ps_validate(const char* path, int64_t nrhs, int64_t* stats, int nstats);

/* ps_analyze_rank — host-only, as ps_analyze for rank `rank` of a row partition over
 * nranks ranks (nranks = 1: the whole problem): the rank's own rows, separator rows,
 * and the device bytes its handle would hold (PS_INFO_OP_BYTES after setup,
 * PS_INFO_SETUP_BYTES during it). The near arena is skipped, not verified.
 * Returns the number of values written, or -ps_status. */
int ps_analyze_rank(const char* path, int rank, int nranks, double* out, int n);

/* ps_profile — enable (1) / disable (0) per-launch CUDA-event timing inside
 * ps_solve / ps_apply (events on the launching stream around every kernel;
 * adds a few microseconds per launch, so timed benchmarks run with it off).
 * Resets the accumulators. */
ps_status ps_profile(ps_handle* h, int enable);

/* ps_profile_read — accumulated since ps_profile(h,1): for each kernel class
 * c in {0 forward sweep, 1 backward sweep, 2 D^{-1}, 3 far stage 1,
 * 4 far stage 2, 5 permutations/combine/norms, 6 the whole-solve dataflow
 * program (default ps_solve path; two launches for nrhs <= 8), 7 the one-pass far
 * apply of nrhs <= 8 (Morton copy of w, far1p kernel, per-leaf sums)} four values
 * out[4c..4c+3] = (device ms, launches, algorithmic flops, algorithmic operator bytes).
 * Classes 0-4 and 6 are all the gather-GEMM kernel. Returns values written. */
int ps_profile_read(const ps_handle* h, double* out, int n);

/* ps_trace / ps_trace_read — debug instrumentation of the persistent dataflow
 * kernel: ps_trace(h, c) records, for the next launches of kernel class c
 * (as in ps_profile_read; -1 disables), per work item: item, SM id, and the
 * globaltimer (ns) at fetch, dependencies satisfied, compute done, published, and
 * (narrow warp-specialised kernel; else 0) when the scheduler warp took the item's
 * ticket and when it handed the prepared item over. ps_trace_read copies the last
 * traced launch, 14 int64 per item (those 8 plus task, row tile, column tile, chunk,
 * n_chunks, k-length); returns the item count. out: capacity 14 * cap_items. */
ps_status ps_trace(ps_handle* h, int cls);
int64_t ps_trace_read(ps_handle* h, int64_t* out, int64_t cap_items);

/* ps_get_dinv — copy D_k^{-1} of the leaf at elimination position `pos`
 * (n_k x n_k column-major, in the leaf's Morton-local unknown order) to host
 * memory `out` of capacity `cap` complex entries. Returns n_k on success;
 * -(n_k^2) without copying when cap < n_k^2 (call again with that capacity);
 * 0 on error (bad handle / position, no setup, or not this rank's block). */
int64_t ps_get_dinv(ps_handle* h, int64_t pos, void* out, int64_t cap);

/* ps_elim_leaf — Morton leaf id at elimination position pos; -1 if invalid. */
int64_t ps_elim_leaf(const ps_handle* h, int64_t pos);

#ifdef __cplusplus
}
#endif
#endif /* PS_H_ */
