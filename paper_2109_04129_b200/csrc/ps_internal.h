// ps_internal.h — structures shared by the host side (ps_host.cpp) and the
// sm_100a kernels (ps_kernels.cu) of libps. Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ps {

// One output block of the gathered batched complex GEMM ("gather-GEMM"):
//   O(i,c) = [I(i,c)] + sign * sum_{t in [t0,t1)} sum_k A_t(i,k) B_t(k,c),
// i < m, c < n. Every operand is addressed by (base pointer passed at launch)
// + element offset + two element strides, so the same table serves several
// buffers (e.g. both forward sweeps) and transposed views cost nothing.
struct GTask {
  int64_t oO, oI;          // element offsets into the O / I bases (oI < 0: no init)
  int64_t sOi, sOc, sIi, sIc;
  int32_t m, n;
  int32_t t0, t1;          // segment range
  int32_t K;               // total (virtual) K = sum of segment lengths
  int32_t sign;
  int32_t unit0;           // first completion counter of this task (one per column tile)
  int32_t n_mt;            // row tiles: column tile nt is complete when done[unit0+nt] == n_mt
  int32_t a_kmajor;        // 1: A's unit stride is along k (transposed views), 0: along i
  int32_t b_kmajor;        // 1: B's unit stride is along k, 0: along c
  int32_t idep;            // task (same launch) producing the init rows I; -1: none
                           // (device copy: that task's first completion unit, see Table::upload)
  int32_t osel;            // bit 0: O offsets address the scratch base S instead of O;
                           // bit 1: I offsets address S instead of I;
                           // bit 2: wide tile on the FP64 tensor-core consumer (per task)
  int32_t idep_nmt;        // device copy: the init producer's row tiles (its unit is complete at this count)
  int32_t idep_ntp;        // device copy: the init producer's column tiles (no wait for nt >= this)
};

// A segment of a task's K dimension: K_s consecutive k's starting at virtual
// position kstart; A(i, k) = A[oA + (k - kstart) sAk + i sAi],
// B(k, c) = B[oB + (k - kstart) sBk + c sBc].
struct GTerm {
  int64_t oA, oB;
  int64_t sAi, sAk, sBk, sBc;
  int32_t kstart, K;
  int32_t dep;             // task (same launch) producing this segment's B rows; -1: none
                           // (device copy: that task's first completion unit)
  int32_t bsel;            // bit 0: oB addresses the scratch base S instead of B; device copy adds
                           // the producer's row tiles (bits 1-15) and column tiles (bits 16-31)
};

// One CTA-sized piece of work: output tile (mt, nt) of `task`, virtual k in
// [ka, kb) touching segments [ta, tb). A tile whose K is split into
// nchunks > 1 pieces (split-K) writes partial sums to slots
// [slot, slot + nchunks); the last piece to arrive (counter arrive[tile]) adds
// them up in chunk order — deterministic.
struct GWork {
  int32_t task, mt, nt, ta, tb, ka, kb, chunk, nchunks, tile;
  int32_t crit;            // split-K combine: -1 = the tree root finalises; else the chunk that
                           // carries the latest dependency (queued last): it adds the published
                           // sum of all other chunks
  int32_t sub;             // combine subgroup of this chunk: members are the non-critical chunks
  int32_t sub_r0, sub_r1;  // of rank [sub_r0, sub_r1) (rank = chunk index skipping crit)
  int32_t nsub;            // number of subgroups of the tile
  int32_t sw_unit;         // slot reuse: the tile's partial-sum slots were last used by the
  int32_t sw_need;         // unit sw_unit (>= 0); wait until done[sw_unit] >= sw_need (all its
  int32_t pad;             // items precede this one in ticket order) before writing them
  int64_t slot;
};

// A batch = a contiguous range of work items launched as one kernel.
struct Batch {
  int64_t w0, nw;
};

// Arguments of one persistent dataflow launch over work[0..nwork): items are
// in topological order and fetched through a global ticket; an item waits
// (acquire) until the tasks producing its B operands have completed its column tile.
struct FlowArgs {
  const GWork* work;
  int64_t nwork;
  const GTask* tasks;
  const GTerm* terms;
  double2* O;
  const double2* I;
  const double2* A;
  const double2* B;
  double2* S;              // scratch vector base (chain stages of the sweeps)
  int32_t* counters;       // [0] ticket, [1 .. 1+n_units) done, then arrive[n_tiles]
  int32_t n_units;
  int32_t defer_fin;       // narrow WS items: split-K combine by the finisher warp (PS_DEFER_FIN)
  double2* partial;        // split-K partial tiles, GM_MT * GM_NT each
  int64_t* trace;          // optional: 8 x int64 per item (item, smid, t_fetch, t_ready, t_computed, t_done,
                           // narrow WS kernel: scheduler ticket taken, slot handed over), ns
  int32_t narrow;          // 1: narrow 64 x 8 tiles (small nrhs), 0: 32 x 64 tiles
  int32_t mma;             // wide tiles: 0 = DFMA consumer, 1 = FP64 tensor-core (DMMA) consumer
  int32_t ksplit;          // wide DFMA tiles: 1 = k-split two-column layout (item_body_ks), 0 = one column per lane
  int32_t gauss;           // wide DMMA tiles: 1 = three-multiplication complex product (item_body_dmma3)
};

// Tile geometry of the gather-GEMM kernel (ps_kernels.cu).
constexpr int GM_RMAX = 8;                  // rows per warp (register accumulators per thread)
constexpr int GM_WM = 4, GM_WN = 2;         // warp grid: 4 row groups x 2 column groups
constexpr int GM_MT = GM_WM * GM_RMAX;      // 32 rows per tile (max)
constexpr int GM_NT = GM_WN * 32;           // 64 columns per tile (one per lane)
constexpr int GM_KC = 16;
// narrow tile (small nrhs: GEMV-like, operator-streaming): 64 rows x 8 columns
constexpr int GN_MT = 64;
constexpr int GN_NT = 8;
constexpr int GM_CHUNK_K = 512;   // max virtual k per work item (shared-memory k tables)
constexpr int GN_CHUNK_K = 512;   // same for narrow tiles (warp-specialised kernel, two tables)
constexpr int GM_MAXSEG = 96;     // max segments per work item

// ---- one-pass far-field apply of narrow solves (nrhs <= 8; DESIGN.md §6 "far1p") ----
// Z_F w over every far block from ONE read of its factors (Eqs. 11, 13: the
// symmetric pair Z_ij = U V^T, Z_ji = V U^T). Per low-rank block, with F1 / F2 the factors
// (U / V or V / U, F1 the shorter one) copied rows-major (row a = r contiguous complex) into
// the FB arena and x = w in Morton order:
//   p1 = F1^T x1,  p2 = F2^T x2,  y2 = F2 p1,  y1 = F1 p2
// (y1 / y2 = that block's contribution to the rows of F1 / F2). A dense (rank-capped, R18)
// block D (m x n) is read as G = D or D^T, rows-major with the shorter row r = min(m, n):
//   y1 = G x2 (rows of G; x2 = the vector of G's columns),  y2 = G^T x1 (r rows).
// Contributions go to per-block pieces of P, summed per leaf in a fixed order (far_reduce):
// no float atomics. Work units: a pack of small blocks (each applied whole by one warp), or
// one big block, cut into row chunks applied in order by ONE CTA (F1 chunks -> p1; F2 chunks
// -> y2 rows and p2; F1 chunks again -> y1 rows), so no unit waits on another.
#ifndef PS_F1P_CH                 // -DPS_F1P_CH / -DPS_F1P_NS: tiling A/B builds (scripts/f1p_variants.sh)
#define PS_F1P_CH 2048
#endif
#ifndef PS_F1P_NS
#define PS_F1P_NS 2
#endif
constexpr int F1P_CH = PS_F1P_CH; // factor elements staged per item (32 KB; 2 stages + scratch: 2 CTAs / SM at 1 column, fits 227 KB at 8)
constexpr int F1P_RMAX = 64;      // max rank (dense: shorter side) of a block on this path
constexpr int F1P_XCH = 512;      // x rows x nrhs staged per item (complex elements)
constexpr int F1P_PACK = 32;      // max blocks per pack item
constexpr int F1P_NS = PS_F1P_NS;       // shared-memory ring stages of the far1p kernel
constexpr int F1P_CWARPS = 8;     // consumer warps of the far1p kernel
struct FBlk {
  int64_t o1, o2;          // element offsets (operator base) of F1 (n1 x r) / F2 (n2 x r); dense: G, -1
  int64_t x1, x2;          // first row of x1 / x2 in the Morton vector (rows, not elements)
  int64_t xa;              // first row of x1 in the gathered x arena XA (x2 follows: XA = [x1 | x2] per block)
  int64_t pad0;
  int64_t y1, y2;          // first row of the pieces y1 (n1 rows) / y2 (n2 rows; dense: r rows)
  int32_t n1, n2, r;
  int32_t dense;
  int32_t nc1, nc2;        // big blocks: row chunks of F1 / F2
  int32_t xo1, xo2;        // packed blocks: first row of x1 / x2 in the item's staged x rows
};
struct FItem {
  int64_t off;             // first element of the item's contiguous factor range (operator base)
  int64_t xa, xa2;         // staged x rows: XA rows [xa, xa + xn), then (dense big) [xa2, xa2 + xn2)
  int32_t xn, xn2;
  int32_t len;             // elements (<= F1P_CH)
  int32_t kind;            // 0 pack of whole blocks [b, b + nb); big block b, chunk nb, rows [a0, a1):
                           // 1 F1 rows (p1), 2 F2 rows (y2, p2), 3 F1 rows (y1), 4 dense G rows (y1, y2);
                           // -1 (kernel-internal) end of the CTA's work
  int32_t b, nb;           // pack: first block, count; big: block, chunk index
  int32_t a0, a1;          // big: row range of the chunk; pack: a0 = its staged x rows
};
struct FUnit {             // one ticket of work: items [i0, i0 + n) (a pack, or every chunk of a big block)
  int64_t i0;
  int32_t n, pad;
};
struct Far1pArgs {
  const FUnit* units;
  int64_t nunits;
  const FItem* items;
  const FBlk* blks;
  const double2* A;        // operator base (d_op)
  const double2* x;        // XA: the x rows of every block gathered from w ([x1 | x2] per block, row-major R)
  double2* y;              // pieces, rows x R row-major
  int32_t* cnt;            // [0]: unit ticket (zeroed per launch)
  int32_t R;
  int32_t minrows;         // big chunks: at least this many rows per consumer warp (PS_F1P_MINROWS)
};
void launch_far1p(const Far1pArgs& a, cudaStream_t st);
int far1p_resident_ctas(int R);
// Z[lrow[l] R + e] = sum_{q in [lptr[l], lptr[l+1])} y[poff[q] R + e], e < lsz[l] R (rows; list order)
void launch_far_reduce(int64_t nl, const int64_t* lptr, const int64_t* poff, const int64_t* lrow,
                       const int32_t* lsz, const double2* y, double2* Z, int R, cudaStream_t st);
// FB arena from the far stacks: run d copies rows x r elements, element (a, k) from
// src[so + a ss + k sk] to dst[do + a r + k] (operator base)
struct FCopy { int64_t dst, src, ss, sk; int32_t rows, r; };
void launch_fb_gather(int64_t n, const FCopy* runs, double2* base, cudaStream_t st);

// ---- kernel launchers (ps_kernels.cu) ----
// grid <= 0: one persistent CTA per resident slot (148 SMs x occupancy).
void launch_flow(const FlowArgs& a, int grid, cudaStream_t st);
int flow_resident_ctas();

// Batched in-place Gauss-Jordan inversion with partial pivoting:
// for each leaf l in [0,nl): src = Wbase + src_off[l] (n x n, ld = src_ld[l]),
// dst = Dbase + dst_off[l] (n x n, ld n). status[l] = 1 if singular.
void launch_inverse(int64_t nl, const int32_t* leaf_ids, const int32_t* sizes,
                    const int64_t* src_off, const int64_t* src_ld, const int64_t* dst_off,
                    const double2* Wbase, double2* Dbase, int32_t* status, int max_n,
                    cudaStream_t st);

// y[e*nrhs + c] = B[map[e] + c*ldb]   (gather rows of a column-major block; map[e] < 0: 0)
void launch_permute_in(int64_t N, int64_t nrhs, const int64_t* map, const double2* B, int64_t ldb,
                       double2* y, cudaStream_t st);
// X[map[e] + c*ldx] = y[e*nrhs + c]   (rows with map[e] < 0 are skipped)
void launch_permute_out(int64_t N, int64_t nrhs, const int64_t* map, const double2* y, double2* X,
                        int64_t ldx, cudaStream_t st);
// dst[e*nrhs + c] = src[map[e]*nrhs + c]  (row permutation, row-major blocks)
void launch_permute_rows(int64_t N, int64_t nrhs, const int64_t* map, const double2* src,
                         double2* dst, cudaStream_t st);
// xt = bo - u; part[chunk*nrhs + c] = (sum |bo|^2, sum |u|^2) over the chunk's rows
void launch_combine_norms(int64_t N, int64_t nrhs, const double2* bo, const double2* u, double2* xt,
                          double2* part, int64_t rows_per_chunk, cudaStream_t st);
// part[chunk*nrhs + c] = (sum |bo|^2, sum |bo - xt|^2) over the chunk's rows
void launch_norms2(int64_t N, int64_t nrhs, const double2* bo, const double2* xt, double2* part,
                   int64_t rows_per_chunk, cudaStream_t st);
// acc = (first ? 0 : acc) + sign it; part[chunk*nrhs + c] = (sum |it|^2, sum |acc|^2) (n-term series)
void launch_series_accum(int64_t N, int64_t nrhs, const double2* it, double2* acc, double sign, int first,
                         double2* part, int64_t rows_per_chunk, cudaStream_t st);
// norms[c] = (sqrt sum_chunks part.x, sqrt sum part.y); do_sqrt = 0: the sums themselves
void launch_finalize_norms(int64_t nchunks, int64_t nrhs, const double2* part, double2* norms,
                           cudaStream_t st, int do_sqrt = 1);
// dst[i] += src[i] (i < n), the in-process stand-in of a sum all-reduce (rank order fixed)
void launch_add(double* dst, const double* src, int64_t n, cudaStream_t st);
void launch_zero(double2* p, int64_t n, cudaStream_t st);
// far field / RCS of RWG currents (ps_rcs.cu, include/ps.h ps_farfield); returns the kernels
// launched, or -(partial entries needed) when part is NULL or smaller than that
int64_t launch_farfield(const double* nodes, const int64_t* tris, int64_t N, const int64_t* tp, const int64_t* tm,
                        const int64_t* vp, const int64_t* vm, double k, double eta, const double2* I, int64_t ldi,
                        int64_t nrhs, int64_t ndir, const double* rhat, int mono, double2* F, double* sigma,
                        double2* part, int64_t part_cap, cudaStream_t st);

// base[offs[e]] = 1 (e < n): identity diagonals of the chain matrices T_c
void launch_set_ones(double2* base, const int64_t* offs, int64_t n, cudaStream_t st);

}  // namespace ps
