// ps_kernels.cu — sm_100a kernels of libps (complex128 throughout).
//
// Every hot-path step of PAPER.md §III reduces to small dense complex block
// products over leaf-cluster lists:
//   * forward sweep  b~_j = b_j + sum_k alpha_kj^T b~_k      (Eq. 24, gather form)
//   * D^{-1} apply   b_o = Z~_N^{-1} b~                     (Eq. 32)
//   * backward sweep w_k = v_k + sum_j alpha_kj w_j          (Eq. 26)
//   * far field      t = U (V^T w), two stages               (Eqs. 11, 13, 31)
//   * setup          Z~_pj = Z_pj + sum_d alpha_dp^T Z~_dj   (Eq. 21, left-looking)
//                    alpha_pj = -D_p^{-1} Z~_pj              (Eq. 16)
// They all run through ONE gather-GEMM kernel driven by task/term tables built
// on the host (ps_host.cpp); D_p^{-1} comes from a batched Gauss-Jordan kernel.
// There are no float atomics: every output tile is owned by one CTA and its
// terms are summed in a fixed order, so results are bitwise repeatable.
//
// FP64 note: tcgen05 has no f64 kind; complex128 products run on the DFMA pipe
// (4 DFMA per complex multiply-add). DESIGN.md §Roofline derives the peak.
#include "ps_internal.h"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace ps {

__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

// ---------------------------------------------------------------------------
// Gather-GEMM, persistent dataflow form.
//
// CTA = 256 threads; output tile MT x NT = 32 x 32 complex; each thread owns a
// 2 x 2 register tile (rows ty, ty+16; cols tx, tx+16). Operand tiles (32 x KC
// of A, KC x 32 of B) go through two shared-memory buffers: the global loads of
// k-step s+1 are issued into registers before the FMAs of step s, so load
// latency overlaps compute. Loads follow the operand's unit-stride dimension
// (coalesced). A operands (operator panels) use the read-only path; B operands
// and inits are produced inside the same launch by other CTAs, so they are read
// with ld.global.cg (L2, never a stale L1 line).
//
// Scheduling: a CTA takes the next item from a global ticket (items are in
// topological order), waits with ld.acquire until every task producing its B
// rows has completed this column tile, computes, and publishes its tile with a
// release (threadfence + atomic). Deadlock-free: an item only waits on items
// with smaller tickets, which resident CTAs already hold.
constexpr int KC = GM_KC;

__device__ __forceinline__ int64_t gtimer() {
  int64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int smid() {
  int s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Per-item k tables: for the item's virtual k range [ka, kb) the A column
// base, A row stride, B row base and B column stride of every k (built from the
// segment list at item start), so k-steps run densely across segments.
template <int NK>
struct KTabT {
  int64_t kA[NK];
  const double2* kB[NK];             // absolute row pointer of B (base B or scratch S)
  int32_t kSi[NK];
  int32_t kSc[NK];
};
using KTab = KTabT<GM_CHUNK_K>;
using KTabN = KTabT<GN_CHUNK_K>;     // narrow (warp-specialised) items: <= GN_CHUNK_K k

constexpr int AS_LD = GM_MT;                // As[k][i]
constexpr int BS_LD = GM_NT;                // Bs[k][c]
constexpr int NSTAGE = 4;                   // cp.async pipeline depth (wide tiles)
constexpr int STAGE_A = KC * GM_MT;
constexpr int STAGE_B = KC * GM_NT;
static_assert(NSTAGE * STAGE_A >= GM_MT * GM_NT, "the k-half reductions reuse the A stages");

__device__ __forceinline__ void a_map(bool a_km, int e, int& i, int& k) {
  if (a_km) { k = e & (KC - 1); i = e / KC; } else { i = e % GM_MT; k = e / GM_MT; }
}
__device__ __forceinline__ void b_map(bool b_km, int e, int& c, int& k) {
  if (b_km) { k = e & (KC - 1); c = e / KC; } else { c = e & (GM_NT - 1); k = e / GM_NT; }
}

// 16-byte global -> shared async copy (L2 only, .cg); zero-fills when !valid.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}
// 16-byte global -> shared async copy, always valid (no zero-fill operand)
__device__ __forceinline__ void cp_async16_all(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// swz: the tensor-core consumer's stages are XOR-swizzled — element (k, i) of a stage at
// k LD + (i ^ 2 (k mod 4)) — so its fragment loads (lane (g, q) reads row g of k-row q) hit
// 8 distinct 16-byte bank groups per quarter warp instead of 2 (a 4-way conflict on every
// LDS.128 of an A or B fragment with the plain k-major layout).
template <int MT, int NT, class KT>
__device__ __forceinline__ void issue_a(const KT& kt, int k0, int klen, int i0, int mm, bool a_km,
                                        const double2* __restrict__ Ab, int tid, double2* As, bool swz = false) {
#pragma unroll
  for (int q = 0; q < MT * KC / 256; ++q) {
    const int e = tid + q * 256;
    int i, k;
    if (a_km) { k = e & (KC - 1); i = e / KC; } else { i = e % MT; k = e / MT; }
    const int kk = k0 + k;
    const bool v = (i < mm && kk < klen);
    const double2* src = v ? Ab + kt.kA[kk] + (int64_t)(i0 + i) * kt.kSi[kk] : Ab;
    cp_async16(As + k * MT + (swz ? (i ^ (2 * (k & 3))) : i), src, v);
  }
}
template <int MT, int NT, class KT>
__device__ __forceinline__ void issue_b(const KT& kt, int k0, int klen, int c0, int nn, bool b_km,
                                        const double2* __restrict__ Bb, int tid, double2* Bs, bool swz = false) {
  constexpr int NB = NT * KC;
#pragma unroll
  for (int q = 0; q < (NB + 255) / 256; ++q) {
    const int e = tid + q * 256;
    if (NB % 256 != 0 && e >= NB) break;
    int c, k;
    if (b_km) { k = e & (KC - 1); c = e / KC; } else { c = e % NT; k = e / NT; }
    const int kk = k0 + k;
    const bool v = (c < nn && kk < klen);
    const double2* src = v ? kt.kB[kk] + (int64_t)(c0 + c) * kt.kSc[kk] : Bb;
    cp_async16(Bs + k * NT + (swz ? (c ^ (2 * (k & 3))) : c), src, v);
  }
}

// release / acquire flag operations (one thread, after / before a CTA barrier)
__device__ __forceinline__ void red_release(int32_t* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_acq_rel(int32_t* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

constexpr size_t FLOW_SMEM = (size_t)NSTAGE * (STAGE_A + STAGE_B) * sizeof(double2) + sizeof(KTab);

// ---------------------------------------------------------------------------
// Split-K combine of one output tile, fixed summation order (deterministic).
// Each thread owns E tile elements at tile offsets off[e] with partial sums
// acc[e]. Non-critical chunks (all chunks except `crit`) are summed by a fixed
// two-level tree: subgroups of consecutive chunks (by rank; host-chosen), the last
// arriver of a subgroup sums its members in rank order, the last subgroup sums
// the subgroup sums in order. Counters of the tile: arrive[tile] (top) and
// arrive[tile + 1 + sg]. Slots: [slot, slot + nchunks) chunk partials,
// [slot + nchunks, ...) subgroup sums; the group sum goes to slot `crit`.
// crit >= 0: the critical chunk (queued last) waits for top == nsub + 1 and
// adds the group sum (p_0 + G, or G + p_last); crit < 0: the tree root finalises.
// Returns true when the caller must finalise with acc.


// CTA barrier of the compute threads: the whole CTA, or (warp-specialised
// kernel) the 8 compute warps only — the scheduler warp never joins it.
template <bool WS>
__device__ __forceinline__ void bsync() {
  if constexpr (WS) asm volatile("bar.sync 5, 256;" ::: "memory");
  else __syncthreads();
}

__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive_n(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// elements of one partial-sum slot: one output tile (narrow tiles are 4x smaller)
__device__ __forceinline__ int64_t slot_elems(const FlowArgs& a) {
  return a.narrow ? (int64_t)(GN_MT * GN_NT) : (int64_t)(GM_MT * GM_NT);
}

template <int E, bool WS = false>
__device__ __forceinline__ bool splitk_combine(const FlowArgs& a, const GWork& w, double2 (&acc)[E],
                                               const int (&off)[E], const bool (&own)[E], int tid,
                                               int* s_flag) {
  if (w.nchunks <= 1) return true;
  const int64_t TS = slot_elems(a);
  int32_t* ctr = a.counters + 1 + a.n_units + w.tile;
  const bool crit_mode = w.crit >= 0;
  const int nsub = w.nsub;
  if (crit_mode && w.chunk == w.crit) {
    if (tid == 0)
      while (ld_acquire(ctr) < nsub + 1) __nanosleep(32);
    bsync<WS>();
    const double2* Gs = a.partial + (w.slot + w.crit) * TS;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (own[e]) {
        const double2 v = __ldcg(Gs + off[e]);
        if (w.crit == 0) { acc[e].x = acc[e].x + v.x; acc[e].y = acc[e].y + v.y; }  // p_0 + G
        else { acc[e].x = v.x + acc[e].x; acc[e].y = v.y + acc[e].y; }              // G + p_last
      }
    return true;
  }
  auto chunk_of_rank = [&](int r) { return (crit_mode && r >= w.crit) ? r + 1 : r; };
  const int sg = w.sub;
  const int r0 = w.sub_r0, r1 = w.sub_r1;
  double2* P = a.partial + (w.slot + w.chunk) * TS;
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (own[e]) __stcg(P + off[e], acc[e]);
  bsync<WS>();
  if (tid == 0) *s_flag = (atom_acq_rel(ctr + 1 + sg, 1) == (r1 - r0) - 1);
  bsync<WS>();
  if (!*s_flag) return false;
  // last of its subgroup: sum the members in rank order (loads batched)
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = make_double2(0.0, 0.0);
  for (int r = r0; r < r1; ++r) {
    const double2* Q = a.partial + (w.slot + chunk_of_rank(r)) * TS;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (own[e]) {
        const double2 v = __ldcg(Q + off[e]);
        acc[e].x += v.x;
        acc[e].y += v.y;
      }
  }
  if (nsub > 1) {
    double2* S = a.partial + (w.slot + w.nchunks + sg) * TS;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (own[e]) __stcg(S + off[e], acc[e]);
    bsync<WS>();
    if (tid == 0) *s_flag = (atom_acq_rel(ctr, 1) == nsub - 1);
    bsync<WS>();
    if (!*s_flag) return false;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = make_double2(0.0, 0.0);
    for (int q = 0; q < nsub; ++q) {
      const double2* Q = a.partial + (w.slot + w.nchunks + q) * TS;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (own[e]) {
          const double2 v = __ldcg(Q + off[e]);
          acc[e].x += v.x;
          acc[e].y += v.y;
        }
    }
  } else if (crit_mode) {
    if (tid == 0) red_release(ctr, 1);       // top counts the (single) subgroup
  }
  if (!crit_mode) return true;                // the tree root finalises
  double2* Gs = a.partial + (w.slot + w.crit) * TS;
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (own[e]) __stcg(Gs + off[e], acc[e]);
  bsync<WS>();
  if (tid == 0) red_release(ctr, 1);          // top reaches nsub + 1: group sum published
  return false;
}

// A split tile's partial-sum slots are recycled (Table::assign_slots): the
// previous user's unit must be complete before this item writes them.
__device__ __forceinline__ void wait_slot_reuse(const FlowArgs& a, const GWork& w) {
  if (w.sw_unit < 0) return;
  const int32_t* flag = a.counters + 1 + w.sw_unit;
  while (ld_acquire(flag) < w.sw_need) __nanosleep(32);
}
// Wait (warp 0) until every producer task of this item's B rows (and of its init
// rows) has completed column tile nt, from the producer's completion unit, row tiles
// and column tiles precomputed at upload (Table::upload: no load of the producer's
// descriptor on the item's critical path). A producer with fewer columns than the
// consumer (chain setup: T row blocks widen up the chain) has no tile nt: the
// consumer's extra columns read zeros nobody writes, so there is no wait.
__device__ __forceinline__ void wait_unit(const FlowArgs& a, int unit, int nmt, int ntp, int nt) {
  if (nt >= ntp) return;
  const int32_t* flag = a.counters + 1 + unit + nt;
  while (ld_acquire(flag) < nmt) __nanosleep(32);
}
__device__ __forceinline__ void wait_term(const FlowArgs& a, const GTerm& g, int nt) {
  if (g.dep >= 0) wait_unit(a, g.dep, (g.bsel >> 1) & 0x7fff, (int)((unsigned)g.bsel >> 16), nt);
}
__device__ __forceinline__ void wait_deps(const FlowArgs& a, const GWork& w, const GTask& T, int tid) {
  if (tid == 0 && T.idep >= 0) wait_unit(a, T.idep, T.idep_nmt, T.idep_ntp, w.nt);
  if (tid == 1) wait_slot_reuse(a, w);
  for (int t = w.ta + tid; t < w.tb; t += 32) {
    wait_term(a, a.terms[t], w.nt);
  }
}

// Critical chunk: wait until the tile's non-critical group sum is published
// (top counter == nsub + 1). Never waits on a later ticket.
__device__ __forceinline__ void wait_group_sum(const FlowArgs& a, const GWork& w, int tid) {
  const int nsub = w.nsub;
  const int32_t* ctr = a.counters + 1 + a.n_units + w.tile;
  if (tid == 0)
    while (ld_acquire(ctr) < nsub + 1) __nanosleep(32);
  __syncthreads();
}


// Everything of one work item, for a compile-time rows-per-warp RM (so the
// FMA stream is branch-free). A operands (operator panels: immutable in the
// launch) of the first stages are requested before waiting for the producers
// of the B operands.
template <int RM>
__device__ __forceinline__ void item_body(const FlowArgs& a, const GWork& w, const GTask& T,
                                          const KTab& kt, double2* As0, double2* Bs0, int tid,
                                          int lane, int wm, int wn, int* s_last, int64_t* tr) {
  const int i0 = w.mt * GM_MT, c0 = w.nt * GM_NT;
  const int mm = min(GM_MT, T.m - i0), nn = min(GM_NT, T.n - c0);
  const int klen = w.kb - w.ka;
  const int rbase = wm * RM;
  const int col = wn * 32 + lane;
  int32_t* done = a.counters + 1;
  const bool a_km = T.a_kmajor != 0, b_km = T.b_kmajor != 0;
  const int nsteps = (klen + KC - 1) / KC;
  // ---- prologue part 1: A of stages 0..NSTAGE-2 (one group) ----
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s)
    if (s < nsteps) issue_a<GM_MT, GM_NT>(kt, s * KC, klen, i0, mm, a_km, a.A, tid, As0 + s * STAGE_A);
  cp_commit();
  // ---- accumulator start values that do not depend on the producers of B,
  // fetched before the wait: the chunk owning the init rows starts from
  // sign * I (rows no other task of the launch writes), and the critical chunk
  // adds the published group sum G of the other chunks (never a later ticket)
  const double sgn = (double)T.sign;
  const bool crit_fin = (w.nchunks > 1 && w.crit >= 0 && w.chunk == w.crit);
  const bool owns_init = (w.nchunks == 1) || (w.crit >= 0 ? w.chunk == w.crit : w.chunk == 0);
  double2 acc[RM];
#pragma unroll
  for (int r = 0; r < RM; ++r) acc[r] = make_double2(0.0, 0.0);
  if (crit_fin) {
    wait_group_sum(a, w, tid);
    const double2* Gs = a.partial + (w.slot + w.crit) * slot_elems(a);
#pragma unroll
    for (int r = 0; r < RM; ++r) acc[r] = __ldcg(Gs + (rbase + r) * GM_NT + col);
  }
  // init rows produced by an earlier task of this launch (idep >= 0) are read
  // only after that producer has published them (below, after the wait)
  auto load_init = [&]() {
    if (owns_init && T.oI >= 0 && col < nn) {
#pragma unroll
      for (int r = 0; r < RM; ++r)
        if (rbase + r < mm) {
          const double2 z = __ldcg(((T.osel & 2) ? (const double2*)a.S : a.I) + T.oI + (int64_t)(i0 + rbase + r) * T.sIi + (int64_t)(c0 + col) * T.sIc);
          acc[r].x += sgn * z.x;
          acc[r].y += sgn * z.y;
        }
    }
  };
  if (T.idep < 0) load_init();
  // ---- wait for the producers of B (warp 0, one segment per lane) ----
  if (tid < 32) wait_deps(a, w, T, tid);
  __syncthreads();
  if (T.idep >= 0) load_init();
  if (tr) tr[3] = gtimer();
  // ---- prologue part 2: B of stages 0..NSTAGE-2 (one group each) ----
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nsteps) issue_b<GM_MT, GM_NT>(kt, s * KC, klen, c0, nn, b_km, a.B, tid, Bs0 + s * STAGE_B);
    cp_commit();
  }

  for (int s = 0; s < nsteps; ++s) {
    cp_wait<NSTAGE - 2>();
    __syncthreads();
    const int st = s % NSTAGE;
    const double2* As = As0 + st * STAGE_A + rbase;
    const double2* Bs = Bs0 + st * STAGE_B + col;
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      const double2 b = Bs[k * BS_LD];
#pragma unroll
      for (int r = 0; r < RM; ++r) cfma(acc[r], As[k * AS_LD + r], b);
    }
    // refill the stage consumed one iteration ago (all threads are past the barrier above)
    const int sn = s + NSTAGE - 1;
    if (sn < nsteps) {
      const int stn = sn % NSTAGE;
      issue_a<GM_MT, GM_NT>(kt, sn * KC, klen, i0, mm, a_km, a.A, tid, As0 + stn * STAGE_A);
      issue_b<GM_MT, GM_NT>(kt, sn * KC, klen, c0, nn, b_km, a.B, tid, Bs0 + stn * STAGE_B);
    }
    cp_commit();
  }
  cp_wait<0>();
  __syncthreads();          // all warps done with the stage buffers before the next item
  if (tr) tr[4] = gtimer();
  // ---- split-K combine (fixed summation order => deterministic) ----
  int off[RM];
  bool own[RM];
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    off[r] = (rbase + r) * GM_NT + col;
    own[r] = true;
  }
  const bool finalize = crit_fin ? true : splitk_combine<RM>(a, w, acc, off, own, tid, s_last);
  if (finalize) {
    if (col < nn) {
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const int i = rbase + r;
        if (i < mm) {
          const double2 v = make_double2(sgn * acc[r].x, sgn * acc[r].y);   // O = I + sign * sum
          __stcg(((T.osel & 1) ? a.S : a.O) + T.oO + (int64_t)(i0 + i) * T.sOi + (int64_t)(c0 + col) * T.sOc, v);
        }
      }
    }
    __syncthreads();
    if (tid == 0) red_release(done + T.unit0 + w.nt, 1);
  }
}


// DFMA wide tile, k-split layout: 8 warps = 4 row groups (wm) x 2 k-halves (wk); lane
// owns columns lane and lane + 32 of the 64-column tile and RM rows. Per k a warp loads
// two B values (8 shared wavefronts) and RM broadcast A values for 2 RM complex FMAs —
// against 4 + RM wavefronts for RM FMAs in the one-column layout — so the shared-memory
// pipe, the binding limit of the DFMA consumer, carries ~25 % less per
// FMA. The two k-halves are summed through shared memory (kh 0 + kh 1, fixed order).
template <int RM>
__device__ __forceinline__ void item_body_ks(const FlowArgs& a, const GWork& w, const GTask& T,
                                             const KTab& kt, double2* As0, double2* Bs0, int tid,
                                             int lane, int warp, int* s_last, int64_t* tr) {
  const int wm = warp & 3, wk = warp >> 2;
  const int i0 = w.mt * GM_MT, c0 = w.nt * GM_NT;
  const int mm = min(GM_MT, T.m - i0), nn = min(GM_NT, T.n - c0);
  const int klen = w.kb - w.ka;
  const int rbase = wm * RM;
  int32_t* done = a.counters + 1;
  const bool a_km = T.a_kmajor != 0, b_km = T.b_kmajor != 0;
  const int nsteps = (klen + KC - 1) / KC;
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s)
    if (s < nsteps) issue_a<GM_MT, GM_NT>(kt, s * KC, klen, i0, mm, a_km, a.A, tid, As0 + s * STAGE_A);
  cp_commit();
  const double sgn = (double)T.sign;
  const bool crit_fin = (w.nchunks > 1 && w.crit >= 0 && w.chunk == w.crit);
  const bool owns_init = (w.nchunks == 1) || (w.crit >= 0 ? w.chunk == w.crit : w.chunk == 0);
  double2 acc[RM][2];
#pragma unroll
  for (int r = 0; r < RM; ++r) acc[r][0] = acc[r][1] = make_double2(0.0, 0.0);
  if (crit_fin) {
    wait_group_sum(a, w, tid);
    if (wk == 0) {
      const double2* Gs = a.partial + (w.slot + w.crit) * slot_elems(a);
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        acc[r][0] = __ldcg(Gs + (rbase + r) * GM_NT + lane);
        acc[r][1] = __ldcg(Gs + (rbase + r) * GM_NT + lane + 32);
      }
    }
  }
  auto load_init = [&]() {
    if (!(owns_init && T.oI >= 0 && wk == 0)) return;
    const double2* Ib = ((T.osel & 2) ? (const double2*)a.S : a.I) + T.oI;
#pragma unroll
    for (int r = 0; r < RM; ++r)
      if (rbase + r < mm)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = lane + 32 * e;
          if (col < nn) {
            const double2 z = __ldcg(Ib + (int64_t)(i0 + rbase + r) * T.sIi + (int64_t)(c0 + col) * T.sIc);
            acc[r][e].x += sgn * z.x;
            acc[r][e].y += sgn * z.y;
          }
        }
  };
  if (T.idep < 0) load_init();
  if (tid < 32) wait_deps(a, w, T, tid);
  __syncthreads();
  if (T.idep >= 0) load_init();
  if (tr) tr[3] = gtimer();
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nsteps) issue_b<GM_MT, GM_NT>(kt, s * KC, klen, c0, nn, b_km, a.B, tid, Bs0 + s * STAGE_B);
    cp_commit();
  }
  for (int s = 0; s < nsteps; ++s) {
    cp_wait<NSTAGE - 2>();
    __syncthreads();
    const int st = s % NSTAGE;
    const double2* As = As0 + st * STAGE_A + (KC / 2) * wk * AS_LD + rbase;
    const double2* Bs = Bs0 + st * STAGE_B + (KC / 2) * wk * BS_LD + lane;
#pragma unroll
    for (int k = 0; k < KC / 2; ++k) {
      const double2 b0 = Bs[k * BS_LD], b1 = Bs[k * BS_LD + 32];
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const double2 av = As[k * AS_LD + r];
        cfma(acc[r][0], av, b0);
        cfma(acc[r][1], av, b1);
      }
    }
    const int sn = s + NSTAGE - 1;
    if (sn < nsteps) {
      const int stn = sn % NSTAGE;
      issue_a<GM_MT, GM_NT>(kt, sn * KC, klen, i0, mm, a_km, a.A, tid, As0 + stn * STAGE_A);
      issue_b<GM_MT, GM_NT>(kt, sn * KC, klen, c0, nn, b_km, a.B, tid, Bs0 + stn * STAGE_B);
    }
    cp_commit();
  }
  cp_wait<0>();
  __syncthreads();
  if (tr) tr[4] = gtimer();
  // k-half reduction through shared memory (the stage buffers are free now)
  double2* red = As0;
  if (wk == 1) {
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      red[(rbase + r) * GM_NT + lane] = acc[r][0];
      red[(rbase + r) * GM_NT + lane + 32] = acc[r][1];
    }
  }
  __syncthreads();
  constexpr int E = 2 * RM;
  double2 accf[E];
  int off[E];
  bool own[E];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int x = 2 * r + e;
      off[x] = (rbase + r) * GM_NT + lane + 32 * e;
      own[x] = (wk == 0);
      if (wk == 0) {
        const double2 v = red[off[x]];
        accf[x] = make_double2(acc[r][e].x + v.x, acc[r][e].y + v.y);
      } else {
        accf[x] = make_double2(0.0, 0.0);
      }
    }
  __syncthreads();          // red (= stage buffers) free again before the next item
  const bool finalize = crit_fin ? true : splitk_combine<E>(a, w, accf, off, own, tid, s_last);
  if (finalize) {
    if (wk == 0) {
      double2* Ob = ((T.osel & 1) ? a.S : a.O) + T.oO;
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const int i = rbase + r;
        if (i < mm)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = lane + 32 * e;
            if (col < nn) {
              const double2 v = accf[2 * r + e];
              __stcg(Ob + (int64_t)(i0 + i) * T.sOi + (int64_t)(c0 + col) * T.sOc, make_double2(sgn * v.x, sgn * v.y));
            }
          }
      }
    }
    __syncthreads();
    if (tid == 0) red_release(done + T.unit0 + w.nt, 1);
  }
}

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col); per lane
// A[g][q], B[q][g], C[g][2q], C[g][2q+1] with g = lane / 4, q = lane % 4.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Wide tile on the FP64 tensor cores (mma.sync m8n8k4 f64; tcgen05 has no f64
// kind). 8 warps = 2 k-halves x 4 column groups: warp (kh, wc) computes rows
// [0, 8 MT) x columns [16 wc, 16 wc + 16) over k rows [8 kh, 8 kh + 8) of every
// KC = 16 stage; the two k-halves are summed through shared memory at the end
// (fixed order: kh 0 + kh 1). A complex k4-step is 4 real DMMAs per 8x8 block
// (re += Ar Br, im += Ar Bi, then re += (-Ai) Bi, im += Ai Br: dependent
// MMAs are MT*NT*2 instructions apart). One 16-byte shared load per lane per
// fragment (A[g][q], B[q][g] as (re, im)); per k4 a warp loads MT + 2
// fragments for 8 MT DMMAs, so the L1/shared pipe is no longer the bound it is
// for the DFMA tile.
__device__ __forceinline__ double dneg(double x) { return __longlong_as_double(__double_as_longlong(x) ^ (1ll << 63)); }

template <int MT>
__device__ __forceinline__ void item_body_dmma(const FlowArgs& a, const GWork& w, const GTask& T,
                                               const KTab& kt, double2* As0, double2* Bs0, int tid,
                                               int lane, int warp, int* s_last, int64_t* tr) {
  constexpr int NT = 2;
  const int i0 = w.mt * GM_MT, c0 = w.nt * GM_NT;
  const int mm = min(GM_MT, T.m - i0), nn = min(GM_NT, T.n - c0);
  const int klen = w.kb - w.ka;
  const int g = lane >> 2, q = lane & 3;
  const int kh = warp >> 2, wc = warp & 3;
  int32_t* done = a.counters + 1;
  const bool a_km = T.a_kmajor != 0, b_km = T.b_kmajor != 0;
  const int nsteps = (klen + KC - 1) / KC;
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s)
    if (s < nsteps) issue_a<GM_MT, GM_NT>(kt, s * KC, klen, i0, mm, a_km, a.A, tid, As0 + s * STAGE_A, true);
  cp_commit();
  const double sgn = (double)T.sign;
  const bool crit_fin = (w.nchunks > 1 && w.crit >= 0 && w.chunk == w.crit);
  const bool owns_init = (w.nchunks == 1) || (w.crit >= 0 ? w.chunk == w.crit : w.chunk == 0);
  // accumulators: block (m, n) rows m*8+g, columns 16 wc + 8 n + 2 q + {0, 1}
  double cre[MT][NT][2], cim[MT][NT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n) cre[m][n][0] = cre[m][n][1] = cim[m][n][0] = cim[m][n][1] = 0.0;
  auto tile_off = [&](int m, int n, int e) { return (m * 8 + g) * GM_NT + 16 * wc + 8 * n + 2 * q + e; };
  if (crit_fin) {
    wait_group_sum(a, w, tid);
    if (kh == 0) {
      const double2* Gs = a.partial + (w.slot + w.crit) * slot_elems(a);
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double2 v = __ldcg(Gs + tile_off(m, n, e));
            cre[m][n][e] = v.x;
            cim[m][n][e] = v.y;
          }
    }
  }
  auto load_init = [&]() {
    if (!(owns_init && T.oI >= 0 && kh == 0)) return;
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = m * 8 + g, c = 16 * wc + 8 * n + 2 * q + e;
          if (i < mm && c < nn) {
            const double2 z = __ldcg(((T.osel & 2) ? (const double2*)a.S : a.I) + T.oI + (int64_t)(i0 + i) * T.sIi + (int64_t)(c0 + c) * T.sIc);
            cre[m][n][e] += sgn * z.x;
            cim[m][n][e] += sgn * z.y;
          }
        }
  };
  if (T.idep < 0) load_init();
  if (tid < 32) wait_deps(a, w, T, tid);
  __syncthreads();
  if (T.idep >= 0) load_init();
  if (tr) tr[3] = gtimer();
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nsteps) issue_b<GM_MT, GM_NT>(kt, s * KC, klen, c0, nn, b_km, a.B, tid, Bs0 + s * STAGE_B, true);
    cp_commit();
  }
  for (int s = 0; s < nsteps; ++s) {
    cp_wait<NSTAGE - 2>();
    __syncthreads();
    const int st = s % NSTAGE;
    const int gs = g ^ (2 * q);                       // swizzled row / column of this lane's fragments
    const double2* As = As0 + st * STAGE_A + (8 * kh + q) * GM_MT + gs;
    const double2* Bs = Bs0 + st * STAGE_B + (8 * kh + q) * GM_NT + 16 * wc + gs;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      double2 av[MT], bv[NT];
#pragma unroll
      for (int m = 0; m < MT; ++m) av[m] = As[kk * 4 * GM_MT + m * 8];
#pragma unroll
      for (int n = 0; n < NT; ++n) bv[n] = Bs[kk * 4 * GM_NT + n * 8];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          dmma(cre[m][n][0], cre[m][n][1], av[m].x, bv[n].x);
          dmma(cim[m][n][0], cim[m][n][1], av[m].x, bv[n].y);
        }
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          dmma(cre[m][n][0], cre[m][n][1], dneg(av[m].y), bv[n].y);
          dmma(cim[m][n][0], cim[m][n][1], av[m].y, bv[n].x);
        }
    }
    const int sn = s + NSTAGE - 1;
    if (sn < nsteps) {
      const int stn = sn % NSTAGE;
      issue_a<GM_MT, GM_NT>(kt, sn * KC, klen, i0, mm, a_km, a.A, tid, As0 + stn * STAGE_A, true);
      issue_b<GM_MT, GM_NT>(kt, sn * KC, klen, c0, nn, b_km, a.B, tid, Bs0 + stn * STAGE_B, true);
    }
    cp_commit();
  }
  cp_wait<0>();
  __syncthreads();
  if (tr) tr[4] = gtimer();
  // k-half reduction through shared memory (stage buffers are free now)
  double2* red = As0;      // 32 x 64 complex = 32 KB <= NSTAGE * (STAGE_A + STAGE_B)
  if (kh == 1) {
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) red[tile_off(m, n, e)] = make_double2(cre[m][n][e], cim[m][n][e]);
  }
  __syncthreads();
  constexpr int E = MT * NT * 2;
  double2 acc[E];
  int off[E];
  bool own[E];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int x = (m * NT + n) * 2 + e;
        off[x] = tile_off(m, n, e);
        own[x] = (kh == 0);
        if (kh == 0) {
          const double2 v = red[off[x]];
          acc[x] = make_double2(cre[m][n][e] + v.x, cim[m][n][e] + v.y);
        } else {
          acc[x] = make_double2(0.0, 0.0);
        }
      }
  __syncthreads();          // red (= stage buffers) free again before the next item / partial reads
  const bool finalize = crit_fin ? true : splitk_combine<E>(a, w, acc, off, own, tid, s_last);
  if (finalize) {
    if (kh == 0) {
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = m * 8 + g, c = 16 * wc + 8 * n + 2 * q + e;
            if (i < mm && c < nn) {
              const double2 v = acc[(m * NT + n) * 2 + e];
              __stcg(((T.osel & 1) ? a.S : a.O) + T.oO + (int64_t)(i0 + i) * T.sOi + (int64_t)(c0 + c) * T.sOc,
                     make_double2(sgn * v.x, sgn * v.y));      // O = I + sign * sum
            }
          }
    }
    __syncthreads();
    if (tid == 0) red_release(done + T.unit0 + w.nt, 1);
  }
}

// Wide tile on the FP64 tensor cores with Gauss's three-multiplication complex product:
// (Ar + i Ai)(Br + i Bi) = (P1 - P2) + i (P3 - P1 - P2), P1 = Ar Br, P2 = Ai Bi,
// P3 = (Ar + Ai)(Br + Bi): 3 DMMAs per 8 x 8 complex block and k4 step instead of 4 (the
// consumer is tensor-pipe bound once its fragment loads are conflict-free). 8 warps = 8
// column groups of 8 columns, each warp all MT row blocks over the full KC of a stage
// (no k-half split, so no end-of-item reduction): three accumulator pairs per block
// (6 MT doubles per lane). The stages use the same swizzled layout as item_body_dmma.
template <int MT>
__device__ __forceinline__ void item_body_dmma3(const FlowArgs& a, const GWork& w, const GTask& T,
                                                const KTab& kt, double2* As0, double2* Bs0, int tid,
                                                int lane, int warp, int* s_last, int64_t* tr) {
  const int i0 = w.mt * GM_MT, c0 = w.nt * GM_NT;
  const int mm = min(GM_MT, T.m - i0), nn = min(GM_NT, T.n - c0);
  const int klen = w.kb - w.ka;
  const int g = lane >> 2, q = lane & 3;
  const int wc = warp;
  int32_t* done = a.counters + 1;
  const bool a_km = T.a_kmajor != 0, b_km = T.b_kmajor != 0;
  const int nsteps = (klen + KC - 1) / KC;
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s)
    if (s < nsteps) issue_a<GM_MT, GM_NT>(kt, s * KC, klen, i0, mm, a_km, a.A, tid, As0 + s * STAGE_A, true);
  cp_commit();
  const double sgn = (double)T.sign;
  const bool crit_fin = (w.nchunks > 1 && w.crit >= 0 && w.chunk == w.crit);
  const bool owns_init = (w.nchunks == 1) || (w.crit >= 0 ? w.chunk == w.crit : w.chunk == 0);
  double p1[MT][2], p2[MT][2], p3[MT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m) p1[m][0] = p1[m][1] = p2[m][0] = p2[m][1] = p3[m][0] = p3[m][1] = 0.0;
  auto tile_off = [&](int m, int e) { return (m * 8 + g) * GM_NT + 8 * wc + 2 * q + e; };
  // start values (init rows, critical chunk's group sum) enter as P1 += re, P3 += re + im, so
  // that re = P1 - P2 and im = P3 - P1 - P2 carry them exactly once
  auto add_start = [&](int m, int e, double re, double im) {
    p1[m][e] += re;
    p3[m][e] += re + im;
  };
  if (crit_fin) {
    wait_group_sum(a, w, tid);
    const double2* Gs = a.partial + (w.slot + w.crit) * slot_elems(a);
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double2 v = __ldcg(Gs + tile_off(m, e));
        add_start(m, e, v.x, v.y);
      }
  }
  auto load_init = [&]() {
    if (!(owns_init && T.oI >= 0)) return;
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = m * 8 + g, c = 8 * wc + 2 * q + e;
        if (i < mm && c < nn) {
          const double2 z = __ldcg(((T.osel & 2) ? (const double2*)a.S : a.I) + T.oI + (int64_t)(i0 + i) * T.sIi + (int64_t)(c0 + c) * T.sIc);
          add_start(m, e, sgn * z.x, sgn * z.y);
        }
      }
  };
  if (T.idep < 0) load_init();
  if (tid < 32) wait_deps(a, w, T, tid);
  __syncthreads();
  if (T.idep >= 0) load_init();
  if (tr) tr[3] = gtimer();
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nsteps) issue_b<GM_MT, GM_NT>(kt, s * KC, klen, c0, nn, b_km, a.B, tid, Bs0 + s * STAGE_B, true);
    cp_commit();
  }
  const int gs = g ^ (2 * q);                         // swizzled row / column of this lane's fragments
  for (int s = 0; s < nsteps; ++s) {
    cp_wait<NSTAGE - 2>();
    __syncthreads();
    const int st = s % NSTAGE;
    const double2* As = As0 + st * STAGE_A + q * GM_MT + gs;
    const double2* Bs = Bs0 + st * STAGE_B + q * GM_NT + 8 * wc + gs;
#pragma unroll
    for (int kk = 0; kk < KC / 4; ++kk) {
      double2 av[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) av[m] = As[kk * 4 * GM_MT + m * 8];
      const double2 bv = Bs[kk * 4 * GM_NT];
      const double bs = bv.x + bv.y;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        dmma(p1[m][0], p1[m][1], av[m].x, bv.x);
        dmma(p2[m][0], p2[m][1], av[m].y, bv.y);
        dmma(p3[m][0], p3[m][1], av[m].x + av[m].y, bs);
      }
    }
    const int sn = s + NSTAGE - 1;
    if (sn < nsteps) {
      const int stn = sn % NSTAGE;
      issue_a<GM_MT, GM_NT>(kt, sn * KC, klen, i0, mm, a_km, a.A, tid, As0 + stn * STAGE_A, true);
      issue_b<GM_MT, GM_NT>(kt, sn * KC, klen, c0, nn, b_km, a.B, tid, Bs0 + stn * STAGE_B, true);
    }
    cp_commit();
  }
  cp_wait<0>();
  __syncthreads();
  if (tr) tr[4] = gtimer();
  constexpr int E = MT * 2;
  double2 acc[E];
  int off[E];
  bool own[E];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      acc[m * 2 + e] = make_double2(p1[m][e] - p2[m][e], p3[m][e] - p1[m][e] - p2[m][e]);
      off[m * 2 + e] = tile_off(m, e);
      own[m * 2 + e] = true;
    }
  const bool finalize = crit_fin ? true : splitk_combine<E>(a, w, acc, off, own, tid, s_last);
  if (finalize) {
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = m * 8 + g, c = 8 * wc + 2 * q + e;
        if (i < mm && c < nn) {
          const double2 v = acc[m * 2 + e];
          __stcg(((T.osel & 1) ? a.S : a.O) + T.oO + (int64_t)(i0 + i) * T.sOi + (int64_t)(c0 + c) * T.sOc,
                 make_double2(sgn * v.x, sgn * v.y));      // O = I + sign * sum
        }
      }
    __syncthreads();
    if (tid == 0) red_release(done + T.unit0 + w.nt, 1);
  }
}

// Output tile: warp w = (wm, wn) = (w % 4, w / 4) owns rows
// [wm*RM, min(mm, (wm+1)*RM)) with RM = ceil(mm / 4) <= 8 (so the tile is
// only as tall as the task) and column wn*32 + lane. A values are broadcast
// shared loads, one B load feeds RM complex FMAs.
template <int MINB>
__global__ void __launch_bounds__(256, MINB)
flow_kernel(const FlowArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* As0 = reinterpret_cast<double2*>(smem_raw);
  double2* Bs0 = As0 + NSTAGE * STAGE_A;
  KTab& kt = *reinterpret_cast<KTab*>(Bs0 + NSTAGE * STAGE_B);
  __shared__ int s_item, s_last;
  __shared__ GWork s_w;
  __shared__ GTask s_T;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp % GM_WM, wn = warp / GM_WM;
  int32_t* ticket = a.counters;
  for (;;) {
    if (tid == 0) {
      const int it = atomicAdd(ticket, 1);
      s_item = it;
      if (it < a.nwork) s_w = a.work[it];
    }
    __syncthreads();
    const int64_t item = s_item;
    if (item >= a.nwork) return;
    int64_t* tr = (a.trace != nullptr && tid == 0) ? a.trace + 8 * item : nullptr;
    if (tr) { tr[0] = item; tr[1] = smid(); tr[2] = gtimer(); }
    const GWork& w = s_w;       // shared: one copy per CTA, not per-thread registers
    const GTask& T = s_T;
    // the task descriptor is loaded by the last warp while the others load the segments
    if (tid >= 256 - 32 && tid - (256 - 32) < (int)(sizeof(GTask) / 4))
      reinterpret_cast<int32_t*>(&s_T)[tid - (256 - 32)] =
          __ldg(reinterpret_cast<const int32_t*>(a.tasks + w.task) + (tid - (256 - 32)));
    // ---- k tables of this item (segments [ta, tb) clipped to [ka, kb)) ----
    for (int t = w.ta + tid; t < w.tb; t += 256) {
      const GTerm g = a.terms[t];
      const int lo = max(g.kstart, w.ka), hi = min(g.kstart + g.K, w.kb);
      for (int k = lo; k < hi; ++k) {
        const int64_t d = k - g.kstart;
        kt.kA[k - w.ka] = g.oA + d * g.sAk;
        kt.kB[k - w.ka] = ((g.bsel & 1) ? a.S : a.B) + g.oB + d * g.sBk;
        kt.kSi[k - w.ka] = (int32_t)g.sAi;
        kt.kSc[k - w.ka] = (int32_t)g.sBc;
      }
    }
    __syncthreads();
    const int mm = min(GM_MT, T.m - w.mt * GM_MT);
    const int RM = (mm + GM_WM - 1) / GM_WM;
    if (a.mma || (T.osel & 4)) {
      if (a.gauss) {
        switch ((mm + 7) / 8) {
          case 1: item_body_dmma3<1>(a, w, T, kt, As0, Bs0, tid, lane, warp, &s_last, tr); break;
          case 2: item_body_dmma3<2>(a, w, T, kt, As0, Bs0, tid, lane, warp, &s_last, tr); break;
          case 3: item_body_dmma3<3>(a, w, T, kt, As0, Bs0, tid, lane, warp, &s_last, tr); break;
          default: item_body_dmma3<4>(a, w, T, kt, As0, Bs0, tid, lane, warp, &s_last, tr); break;
        }
      } else {
        switch ((mm + 7) / 8) {
          case 1: item_body_dmma<1>(a, w, T, kt, As0, Bs0, tid, lane, warp, &s_last, tr); break;
          case 2: item_body_dmma<2>(a, w, T, kt, As0, Bs0, tid, lane, warp, &s_last, tr); break;
          case 3: item_body_dmma<3>(a, w, T, kt, As0, Bs0, tid, lane, warp, &s_last, tr); break;
          default: item_body_dmma<4>(a, w, T, kt, As0, Bs0, tid, lane, warp, &s_last, tr); break;
        }
      }
    } else
    switch (RM) {
#define PS_RM_CASE(R) \
      case R: if (a.ksplit) item_body_ks<R>(a, w, T, kt, As0, Bs0, tid, lane, warp, &s_last, tr); \
              else item_body<R>(a, w, T, kt, As0, Bs0, tid, lane, wm, wn, &s_last, tr); break;
      PS_RM_CASE(1) PS_RM_CASE(2) PS_RM_CASE(3) PS_RM_CASE(4) PS_RM_CASE(5)
#undef PS_RM_CASE
      // 6-8 rows per warp: 2 RM accumulator pairs would exceed the 128-register budget
      case 6: item_body<6>(a, w, T, kt, As0, Bs0, tid, lane, wm, wn, &s_last, tr); break;
      case 7: item_body<7>(a, w, T, kt, As0, Bs0, tid, lane, wm, wn, &s_last, tr); break;
      case 8: item_body<8>(a, w, T, kt, As0, Bs0, tid, lane, wm, wn, &s_last, tr); break;
      default: break;
    }
    if (tr) tr[5] = gtimer();
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Narrow tiles (nrhs <= 8, operator streaming): warp-specialised variant of the
// dataflow kernel. Warps 0-7 compute; warp 8 schedules: it takes the next
// ticket, copies the item's descriptors and segment list into a slot, builds
// the k table there (lanes over the k's of each segment) and waits (acquire)
// for the producers of the item's B / init rows and, for a critical chunk, for
// the group sum — while the compute warps stream the previous item. Two slots
// alternate; hand-over through named barriers FULL[s] = 1 + s / EMPTY[s] =
// 3 + s (288 threads); compute warps synchronise on barrier 5 (256).
// Deadlock-free: a handed-over item runs to completion without waiting, and the
// scheduler only waits on smaller tickets (the smallest unfinished ticket is
// always a running item or is handed over as soon as its CTA's item ends).
// (For the wide tiles this costs the compute warps registers — 2 CTAs x 288
// threads cap them at 112 — and measured slower.)
struct SlotWS {
  GWork w;
  GTask T;
  int64_t item;
  GTerm seg[GM_MAXSEG];
};
// Split-K hand-over from the compute warps to the finisher warp (deferred combine):
// the item's descriptor and output addressing, double-buffered (named barriers
// MAIL_FULL 6 + f / MAIL_EMPTY 8 + f, 288 threads).
struct MailWS {
  GWork w;
  int64_t oO, sOi, sOc;
  int32_t osel, sign, unit0, m, n, live;   // live 0: terminate
};

// Narrow item body of the warp-specialised kernel with a row-adaptive tile:
// MTW = 16 / 32 / 64 rows x KCW = 1024 / MTW k per stage. Thread t: row t % MTW,
// column pair 2 ((t / MTW) % 4), k slice (t / MTW) / 4 of NKS = 64 / MTW slices of
// 16 k; the slices are summed through shared memory at the end (fixed order).
// Variable-depth ring: a stage holds only the item's real rows (mm x KCW operator
// entries, B rows padded to the even column count), so a short task (a 4-8 or 17-24
// row leaf) keeps as many stages in flight as fit the 3 x 1024-entry A ring / the
// 1536-entry B ring (3..8) — the operator bytes in flight per CTA no longer shrink
// with the leaf size. Operand issue is lean: one k-table lookup per thread and stage
// for k-major A, elements outside the tile simply not copied (the ring is zeroed at
// kernel start and only ever holds finite values; B rows k >= klen are zero-filled,
// so stale A there contributes 0), B columns >= nn skipped.
constexpr int WS_ARING = 3 * KC * GN_MT;              // A ring: 3072 complex
constexpr int WS_BRING = 3 * 64 * GN_NT;              // B ring: 1536 complex
constexpr int WS_RING = WS_ARING + WS_BRING;
constexpr int WS_MAXNS = 8;

template <int N>
__device__ __forceinline__ void cp_wait_rt(int n) {   // cp.async.wait_group with a run-time count <= N
  if constexpr (N > 0) {
    if (n >= N) { cp_wait<N>(); return; }
    cp_wait_rt<N - 1>(n);
  } else {
    cp_wait<0>();
  }
}

template <int MTW>
__device__ __forceinline__ void item_body_nk(const FlowArgs& a, const GWork& w, const GTask& T,
                                             const KTabN& kt, double2* stages, int tid, int* s_last,
                                             int64_t* tr, MailWS* mail, int& jm) {
  constexpr int KCW = 1024 / MTW, NKS = 64 / MTW;
  const int i0 = w.mt * GN_MT, c0 = w.nt * GN_NT;
  const int mm = min(GN_MT, T.m - i0), nn = min(GN_NT, T.n - c0);
  const int klen = w.kb - w.ka;
  const int row = tid % MTW, rest = tid / MTW, cb = 2 * (rest & 3), ks = rest >> 2;
  int32_t* done = a.counters + 1;
  const bool a_km = T.a_kmajor != 0, b_km = T.b_kmajor != 0;
  const int nsteps = (klen + KCW - 1) / KCW;
  const int nnp = (nn + 1) & ~1;                       // B row stride in the ring (even column count)
  const int SA = mm * KCW, SB = nnp * KCW;             // stage sizes (complex)
  const int NS = min(WS_MAXNS, min(WS_ARING / SA, WS_BRING / SB));
  double2* Aring = stages;
  double2* Bring = stages + WS_ARING;
  auto issue_a = [&](int k0, double2* As) {
    if (a_km) {
      constexpr int QS = 256 / KCW;
      const int k = tid % KCW, i = tid / KCW, kk = k0 + k;
      if (kk < klen) {
        const int64_t si = kt.kSi[kk];
        const double2* base = a.A + kt.kA[kk] + (int64_t)(i0 + i) * si;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (i + q * QS < mm) cp_async16_all(As + k * mm + i + q * QS, base + q * QS * si);
      }
    } else {
      const int i = tid % MTW;
      if (i < mm) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int kk = k0 + tid / MTW + q * (256 / MTW);
          if (kk < klen) cp_async16_all(As + (kk - k0) * mm + i, a.A + kt.kA[kk] + (int64_t)(i0 + i) * kt.kSi[kk]);
        }
      }
    }
  };
  auto issue_b = [&](int k0, double2* Bs) {
    const int ne = KCW * nnp;
    for (int e = tid; e < ne; e += 256) {
      int c, k;
      if (b_km) { k = e % KCW; c = e / KCW; } else { c = e % nnp; k = e / nnp; }
      if (c < nn) {
        const int kk = k0 + k;
        const bool v = kk < klen;
        cp_async16(Bs + k * nnp + c, v ? kt.kB[kk] + (int64_t)(c0 + c) * kt.kSc[kk] : a.B, v);
      }
    }
  };
  for (int s = 0; s < NS - 1; ++s)
    if (s < nsteps) issue_a(s * KCW, Aring + s * SA);
  cp_commit();
  const double sgn = (double)T.sign;
  const bool crit_fin = (w.nchunks > 1 && w.crit >= 0 && w.chunk == w.crit);
  const bool owns_init = (w.nchunks == 1) || (w.crit >= 0 ? w.chunk == w.crit : w.chunk == 0);
  double2 acc[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  if (crit_fin && ks == 0) {
    const double2* Gs = a.partial + (w.slot + w.crit) * slot_elems(a);
    acc[0] = __ldcg(Gs + row * GN_NT + cb);
    acc[1] = __ldcg(Gs + row * GN_NT + cb + 1);
  }
  if (owns_init && T.oI >= 0 && row < mm && ks == 0) {
#pragma unroll
    for (int e = 0; e < 2; ++e)
      if (cb + e < nn) {
        const double2 z = __ldcg(((T.osel & 2) ? (const double2*)a.S : a.I) + T.oI + (int64_t)(i0 + row) * T.sIi +
                                 (int64_t)(c0 + cb + e) * T.sIc);
        acc[e].x += sgn * z.x;
        acc[e].y += sgn * z.y;
      }
  }
  if (tr) tr[3] = gtimer();
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nsteps) issue_b(s * KCW, Bring + s * SB);
    cp_commit();
  }
  const bool live = (row < mm) && (cb < nn);
  const bool two = cb + 1 < nn;                      // second column of the pair is a real column
  int st = 0, stn = NS - 1;                          // stage computed / stage refilled
  for (int s = 0; s < nsteps; ++s) {
    cp_wait_rt<WS_MAXNS - 2>(NS - 2);
    bsync<true>();
    if (live) {
      const double2* As = Aring + st * SA + (16 * ks) * mm + row;
      const double2* Bs = Bring + st * SB + (16 * ks) * nnp + cb;
      if (two) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const double2 av = As[k * mm];
          cfma(acc[0], av, Bs[k * nnp]);
          cfma(acc[1], av, Bs[k * nnp + 1]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) cfma(acc[0], As[k * mm], Bs[k * nnp]);
      }
    }
    const int sn = s + NS - 1;
    if (sn < nsteps) {
      issue_a(sn * KCW, Aring + stn * SA);
      issue_b(sn * KCW, Bring + stn * SB);
    }
    cp_commit();
    st = (st + 1 == NS) ? 0 : st + 1;
    stn = (stn + 1 == NS) ? 0 : stn + 1;
  }
  cp_wait<0>();
  bsync<true>();
  if (tr) tr[4] = gtimer();
  if constexpr (NKS > 1) {                           // sum the k slices: ks 0 + 1 + ... (fixed order)
    double2* red = stages;                           // NKS x MTW x 8 <= 512 complex
    if (ks > 0) {
      red[(ks * MTW + row) * GN_NT + cb] = acc[0];
      red[(ks * MTW + row) * GN_NT + cb + 1] = acc[1];
    }
    bsync<true>();
    if (ks == 0) {
#pragma unroll
      for (int q = 1; q < NKS; ++q) {
        const double2 v0 = red[(q * MTW + row) * GN_NT + cb], v1 = red[(q * MTW + row) * GN_NT + cb + 1];
        acc[0].x += v0.x; acc[0].y += v0.y;
        acc[1].x += v1.x; acc[1].y += v1.y;
      }
    }
    bsync<true>();
  }
  int off[2] = {row * GN_NT + cb, row * GN_NT + cb + 1};
  bool own[2] = {ks == 0, ks == 0 && two};           // no partial traffic for a padding column
  // publish the partial; the finisher warp combines (one warp: only for 1-2 column tiles,
  // at 8 columns it becomes the bottleneck, measured)
  if (a.defer_fin && w.nchunks > 1 && w.crit < 0 && nn <= 2) {
    double2* P = a.partial + (w.slot + w.chunk) * slot_elems(a);
    if (own[0]) __stcg(P + off[0], acc[0]);
    if (own[1]) __stcg(P + off[1], acc[1]);
    const int f = jm & 1;
    if (jm >= 2) bar_sync_n(8 + f, 288);             // mail f consumed by the finisher
    if (tid == 0) {
      MailWS& M = mail[f];
      M.w = w;
      M.oO = T.oO; M.sOi = T.sOi; M.sOc = T.sOc;
      M.osel = T.osel; M.sign = T.sign; M.unit0 = T.unit0; M.m = T.m; M.n = T.n; M.live = 1;
    }
    bar_arrive_n(6 + f, 288);                         // mail f full (partials stored before)
    ++jm;
    return;
  }
  const bool finalize = crit_fin ? true : splitk_combine<2, true>(a, w, acc, off, own, tid, s_last);
  if (finalize) {
    if (row < mm && ks == 0) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = cb + e;
        if (col < nn) {
          const double2 v = make_double2(sgn * acc[e].x, sgn * acc[e].y);   // O = I + sign * sum
          __stcg(((T.osel & 1) ? a.S : a.O) + T.oO + (int64_t)(i0 + row) * T.sOi + (int64_t)(c0 + col) * T.sOc, v);
        }
      }
    }
    bsync<true>();
    if (tid == 0) red_release(done + T.unit0 + w.nt, 1);
  }
}
constexpr size_t FLOW_WS_SMEM = (size_t)WS_RING * sizeof(double2) + 2 * sizeof(KTabN) + 2 * sizeof(SlotWS);
// two CTAs per SM (__launch_bounds__(320, 2)): dynamic + static shared memory (s_mail,
// s_last) + the 1 KB per-CTA reservation must fit twice in the SM's 228 KB
static_assert(2 * (FLOW_WS_SMEM + 2 * sizeof(MailWS) + 64 + 1024) <= 228 * 1024,
              "flow_kernel_ws no longer fits 2 CTAs per SM");
static_assert(2 * (FLOW_SMEM + sizeof(GWork) + sizeof(GTask) + 64 + 1024) <= 228 * 1024,
              "flow_kernel no longer fits 2 CTAs per SM");

__device__ void ws_scheduler(const FlowArgs& a, SlotWS* slots, KTabN* kts, int lane) {
  int32_t* ticket = a.counters;
  for (int64_t j = 0;; ++j) {
    const int s = (int)(j & 1);
    if (j >= 2) bar_sync_n(3 + s, 288);               // compute warps released slot s
    int it = 0;
    const int64_t t_s0 = a.trace ? gtimer() : 0;
    if (lane == 0) it = atomicAdd(ticket, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    SlotWS& sl = slots[s];
    if (it >= a.nwork) {
      if (lane == 0) sl.item = -1;
      __syncwarp();
      bar_arrive_n(1 + s, 288);
      return;
    }
    {
      const int32_t* src = reinterpret_cast<const int32_t*>(a.work + it);
      int32_t* dst = reinterpret_cast<int32_t*>(&sl.w);
      if (lane < (int)(sizeof(GWork) / 4)) dst[lane] = src[lane];
    }
    __syncwarp();
    const int ta = sl.w.ta, tb = sl.w.tb, ka = sl.w.ka, kb = sl.w.kb;
    {
      // task descriptor and segment list (<= GM_MAXSEG): all lanes' loads of the task and
      // of the first 4 x 32 segment words are issued before any store (one round trip)
      static_assert(sizeof(GTask) / 4 <= 32, "one task word per lane");
      const int32_t* src = reinterpret_cast<const int32_t*>(a.tasks + sl.w.task);
      const int32_t* ts = reinterpret_cast<const int32_t*>(a.terms + ta);
      const int n4 = (tb - ta) * (int)(sizeof(GTerm) / 4);
      int32_t tw = 0, r[4];
      if (lane < (int)(sizeof(GTask) / 4)) tw = __ldg(src + lane);
#pragma unroll
      for (int i = 0; i < 4; ++i) r[i] = (lane + 32 * i < n4) ? __ldg(ts + lane + 32 * i) : 0;
      int32_t* dst = reinterpret_cast<int32_t*>(&sl.T);
      int32_t* td = reinterpret_cast<int32_t*>(sl.seg);
      if (lane < (int)(sizeof(GTask) / 4)) dst[lane] = tw;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (lane + 32 * i < n4) td[lane + 32 * i] = r[i];
      for (int q = lane + 128; q < n4; q += 32) td[q] = ts[q];
    }
    if (lane == 0) sl.item = it;
    __syncwarp();
    KTabN& kt = kts[s];
    for (int t = 0; t < tb - ta; ++t) {
      const GTerm& g = sl.seg[t];
      const int lo = max(g.kstart, ka), hi = min(g.kstart + g.K, kb);
      const double2* bb = ((g.bsel & 1) ? a.S : a.B) + g.oB;
      for (int k = lo + lane; k < hi; k += 32) {
        const int64_t d = k - g.kstart;
        kt.kA[k - ka] = g.oA + d * g.sAk;
        kt.kB[k - ka] = bb + d * g.sBk;
        kt.kSi[k - ka] = (int32_t)g.sAi;
        kt.kSc[k - ka] = (int32_t)g.sBc;
      }
    }
    // producers (lanes over segments), init producer, split-K group sum
    const int nt = sl.w.nt;
    if (lane == 0 && sl.T.idep >= 0) wait_unit(a, sl.T.idep, sl.T.idep_nmt, sl.T.idep_ntp, nt);
    if (lane == 1) wait_slot_reuse(a, sl.w);
    for (int t = lane; t < tb - ta; t += 32)
      wait_term(a, sl.seg[t], nt);
    if (lane == 0 && sl.w.nchunks > 1 && sl.w.crit >= 0 && sl.w.chunk == sl.w.crit) {
      const int32_t* ctr = a.counters + 1 + a.n_units + sl.w.tile;
      while (ld_acquire(ctr) < sl.w.nsub + 1) __nanosleep(32);
    }
    __syncwarp();
    if (a.trace && lane == 0) {                       // scheduler: ticket taken, slot ready
      a.trace[8 * (int64_t)it + 6] = t_s0;
      a.trace[8 * (int64_t)it + 7] = gtimer();
    }
    bar_arrive_n(1 + s, 288);                         // slot s full
  }
}

// Finisher warp (deferred split-K combine): for each handed-over chunk, count it in
// its subgroup; the last arriver sums the subgroup's chunk slots in rank order
// (then, with several subgroups, the last subgroup sums the subgroup sums) and
// stores O = sign * sum — the same arithmetic and order as splitk_combine — and
// publishes the tile. Never waits on other items, so it cannot deadlock; the
// compute warps stream the next item meanwhile.
__device__ void ws_finisher(const FlowArgs& a, MailWS* mail, int lane) {
  int32_t* done = a.counters + 1;
  const int64_t TS = slot_elems(a);
  for (int64_t j = 0;; ++j) {
    const int f = (int)(j & 1);
    bar_sync_n(6 + f, 288);                           // mail f full
    const MailWS M = mail[f];
    bar_arrive_n(8 + f, 288);                         // mail f consumed
    if (!M.live) return;
    const GWork& w = M.w;
    int32_t* ctr = a.counters + 1 + a.n_units + w.tile;
    const int sg = w.sub, r0 = w.sub_r0, r1 = w.sub_r1, nsub = w.nsub;
    int last = 0;
    if (lane == 0) last = (atom_acq_rel(ctr + 1 + sg, 1) == (r1 - r0) - 1);
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) continue;
    const int i0 = w.mt * GN_MT, c0 = w.nt * GN_NT;
    const int mm = min(GN_MT, M.m - i0), nn = min(GN_NT, M.n - c0), ne = mm * nn;
    double2* Ob = ((M.osel & 1) ? a.S : a.O) + M.oO;
    const double sgn = (double)M.sign;
    auto store = [&](int row, int col, double2 v) {
      __stcg(Ob + (int64_t)(i0 + row) * M.sOi + (int64_t)(c0 + col) * M.sOc, make_double2(sgn * v.x, sgn * v.y));
    };
    for (int el = lane; el < ne; el += 32) {
      const int row = el / nn, col = el - row * nn, off = row * GN_NT + col;
      double2 acc = make_double2(0.0, 0.0);
      for (int r = r0; r < r1; ++r) {
        const double2 v = __ldcg(a.partial + (w.slot + r) * TS + off);
        acc.x += v.x;
        acc.y += v.y;
      }
      if (nsub > 1) __stcg(a.partial + (w.slot + w.nchunks + sg) * TS + off, acc);
      else store(row, col, acc);
    }
    if (nsub > 1) {
      __syncwarp();
      int last2 = 0;
      if (lane == 0) last2 = (atom_acq_rel(ctr, 1) == nsub - 1);
      last2 = __shfl_sync(0xffffffffu, last2, 0);
      if (!last2) continue;
      for (int el = lane; el < ne; el += 32) {
        const int row = el / nn, col = el - row * nn, off = row * GN_NT + col;
        double2 acc = make_double2(0.0, 0.0);
        for (int q = 0; q < nsub; ++q) {
          const double2 v = __ldcg(a.partial + (w.slot + w.nchunks + q) * TS + off);
          acc.x += v.x;
          acc.y += v.y;
        }
        store(row, col, acc);
      }
    }
    __syncwarp();
    if (lane == 0) red_release(done + M.unit0 + w.nt, 1);
  }
}

__global__ void __launch_bounds__(320, 2)
flow_kernel_ws(const FlowArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* stages = reinterpret_cast<double2*>(smem_raw);
  KTabN* kts = reinterpret_cast<KTabN*>(stages + WS_RING);
  SlotWS* slots = reinterpret_cast<SlotWS*>(kts + 2);
  __shared__ int s_last;
  __shared__ MailWS s_mail[2];
  const int tid = threadIdx.x;
  if (tid >= 288) {
    ws_finisher(a, s_mail, tid & 31);
    return;
  }
  if (tid >= 256) {
    ws_scheduler(a, slots, kts, tid & 31);
    return;
  }
  for (int e = tid; e < WS_RING; e += 256) stages[e] = make_double2(0.0, 0.0);
  bsync<true>();
  int jm = 0;                                         // mails handed to the finisher
  for (int64_t j = 0;; ++j) {
    const int s = (int)(j & 1);
    bar_sync_n(1 + s, 288);                           // slot s full
    const SlotWS& sl = slots[s];
    const int64_t item = sl.item;
    if (item < 0) {                                   // terminate the finisher
      const int f = jm & 1;
      if (jm >= 2) bar_sync_n(8 + f, 288);
      if (tid == 0) s_mail[f].live = 0;
      bar_arrive_n(6 + f, 288);
      return;
    }
    int64_t* tr = (a.trace != nullptr && tid == 0) ? a.trace + 8 * item : nullptr;
    if (tr) { tr[0] = item; tr[1] = smid(); tr[2] = gtimer(); }
    const int mrows = min(GN_MT, sl.T.m - sl.w.mt * GN_MT);
    if (mrows <= 16) item_body_nk<16>(a, sl.w, sl.T, kts[s], stages, tid, &s_last, tr, s_mail, jm);
    else if (mrows <= 32) item_body_nk<32>(a, sl.w, sl.T, kts[s], stages, tid, &s_last, tr, s_mail, jm);
    else item_body_nk<64>(a, sl.w, sl.T, kts[s], stages, tid, &s_last, tr, s_mail, jm);
    if (tr) tr[5] = gtimer();
    bsync<true>();                                    // every compute warp is done with slot s
    bar_arrive_n(3 + s, 288);                         // slot s empty
  }
}

int flow_ws_resident_ctas() {
  static int n = 0;
  if (n == 0) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(flow_kernel_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FLOW_WS_SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, flow_kernel_ws, 320, FLOW_WS_SMEM);
    n = sms * (per_sm > 0 ? per_sm : 1);
  }
  return n;
}

template <int MINB>
static int resident_of() {
  int per_sm = 0, dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(flow_kernel<MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FLOW_SMEM);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, flow_kernel<MINB>, 256, FLOW_SMEM);
  return sms * (per_sm > 0 ? per_sm : 1);
}
int flow_resident_ctas() {
  static int n = 0;
  if (n == 0) n = resident_of<2>();
  return n;
}
void launch_flow(const FlowArgs& a, int grid, cudaStream_t st) {
  if (a.nwork <= 0) return;
  if (a.narrow) {                                     // nrhs <= 8: warp-specialised narrow kernel
    int g = grid > 0 ? grid : flow_ws_resident_ctas();
    if (g > a.nwork) g = (int)a.nwork;
    flow_kernel_ws<<<g, 320, FLOW_WS_SMEM, st>>>(a);
    return;
  }
  const int resident = flow_resident_ctas();        // also sets the dynamic shared-memory attribute
  int g = grid > 0 ? grid : resident;
  if (g > a.nwork) g = (int)a.nwork;
  flow_kernel<2><<<g, 256, FLOW_SMEM, st>>>(a);
}

// ---------------------------------------------------------------------------
// One-pass far-field apply of narrow solves (far1p; ps_internal.h).
// Persistent, warp-specialised: a producer warp takes work units from a global ticket (a
// pack of small blocks, or ONE whole big block: its F1 chunks, F2 chunks, F1 chunks again) and
// stages every item of the unit into a ring of F1P_NS shared-memory stages with bulk async
// copies (cp.async.bulk -> UBLKCP; completion counted on the stage's mbarrier): the item's
// contiguous factor range, its block descriptors and the x rows it reads. Eight consumer
// warps compute out of shared memory, each walking the ring on its own (one arrival on the
// stage's empty barrier per warp): per block warp-level colsum (lane = (row group, column k),
// row groups added in a fixed order) and rowsum (lane per row). A big block never leaves its
// CTA: its column sums accumulate in per-warp shared-memory partials, summed in warp order at
// the two phase changes (consumer named barrier), so there are no inter-CTA waits; the second
// read of F1 follows its first by the block's own factor bytes (L2-resident for all but the
// largest blocks).
constexpr int F1P_THREADS = 32 * (F1P_CWARPS + 1);       // + the producer warp
constexpr int F1P_GK = 33 * 32;                          // colsum lane-map table entries (r = 0..32)
constexpr int F1P_STAGE_BYTES = 16 * (F1P_CH + F1P_XCH) + (int)sizeof(FBlk) * F1P_PACK + 64;
static_assert(sizeof(FBlk) % 16 == 0, "FBlk is bulk-copied");
static_assert(F1P_STAGE_BYTES % 16 == 0, "stages are bulk-copy destinations");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void f1p_cbar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * F1P_CWARPS) : "memory"); }

// dst[k ds + c] (+)= sum_{a in [a_lo, a_hi)} F[a r + k] x[a R + c], k < r, c < R (one warp; F and
// x in shared memory; accum: add to dst). r <= 32: lane = (g, k) with G = 32 / r row groups
// (rows a = a_lo + g mod G), two accumulators per lane (alternate rows), the G group sums added
// in g order through shuffles; r > 32: lane per k in two passes. Fixed order for a given r.
// Columns c in [R, NR) are computed on whatever follows in shared memory and never stored.
template <int NR>
__device__ __forceinline__ void f1p_colsum_w(const double2* F, int a_lo, int a_hi, int r, const double2* x, int R,
                                             double2* dst, int ds, bool accum, int lane, const uint16_t* gk) {
  // gk[r * 32 + lane] = (g << 8) | k for 1 <= r <= 32, gk[F1P_GK + r] = G = 32 / r (built once per CTA)
  const int G = r <= 32 ? gk[F1P_GK + r] : 1;
  for (int kk = 0; kk < r; kk += 32) {
    int g = 0, k = kk + lane;
    if (r <= 32) { const int e = gk[r * 32 + lane]; g = e >> 8; k = e & 255; }
    double2 s[NR], t[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) s[c] = t[c] = make_double2(0.0, 0.0);
    if (g < G && k < r) {
      const int fs = G * r, xs = G * R;
      const double2* fp = F + (a_lo + g) * r + k;
      const double2* xp = x + (a_lo + g) * R;
      int a = a_lo + g;
      for (; a + G < a_hi; a += 2 * G) {
        const double2 f0 = fp[0], f1 = fp[fs];
#pragma unroll
        for (int c = 0; c < NR; ++c) {
          cfma(s[c], f0, xp[c]);
          cfma(t[c], f1, xp[xs + c]);
        }
        fp += 2 * fs;
        xp += 2 * xs;
      }
      if (a < a_hi) {
        const double2 f0 = fp[0];
#pragma unroll
        for (int c = 0; c < NR; ++c) cfma(s[c], f0, xp[c]);
      }
#pragma unroll
      for (int c = 0; c < NR; ++c) { s[c].x += t[c].x; s[c].y += t[c].y; }
    }
    if (G > 1) {
#pragma unroll
      for (int c = 0; c < NR; ++c) t[c] = s[c];
      for (int g2 = 1; g2 < G; ++g2) {
        const int src = min(31, k + g2 * r);
#pragma unroll
        for (int c = 0; c < NR; ++c) {
          t[c].x += __shfl_sync(0xffffffffu, s[c].x, src);
          t[c].y += __shfl_sync(0xffffffffu, s[c].y, src);
        }
      }
#pragma unroll
      for (int c = 0; c < NR; ++c) s[c] = t[c];
    }
    if (g == 0 && k < r) {
      double2* d = dst + k * ds;
#pragma unroll
      for (int c = 0; c < NR; ++c)
        if (c < R) {
          double2 v = s[c];
          if (accum) { const double2 o = d[c]; v.x = o.x + v.x; v.y = o.y + v.y; }
          d[c] = v;
        }
    }
    if (r <= 32) break;
  }
}

// y[a R + c] = sum_k F[a r + k] q[k NR + c] for rows a in [a_lo, a_hi), c < R (one warp). L lanes
// per row (L = the power of two <= 8 that keeps the warp busy on few rows; k = sub, sub + L, ...,
// the L partial sums added by a fixed xor butterfly); with L = 1 (>= 32 rows) k is rotated per
// row for even r so a quarter warp's 16-byte loads hit distinct bank groups. Two accumulators.
template <int NR, bool MULTI>
__device__ __forceinline__ void f1p_rowsum(const double2* F, int a_lo, int a_hi, int r, const double2* qa, int R,
                                           double2* __restrict__ y, int lane, int nsplit = 1 << 30,
                                           const double2* qb = nullptr) {
  const int nrows = a_hi - a_lo;
  int L = 1;
  if (MULTI)
    while (L < 8 && 2 * L <= r && nrows * 2 * L <= 32) L *= 2;
  const int sub = lane & (L - 1), rpp = 32 / L;          // rows per pass
  for (int a = a_lo + lane / L; a - (lane / L) < a_hi; a += rpp) {
    double2 acc[NR], ac2[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) acc[c] = ac2[c] = make_double2(0.0, 0.0);
    if (a < a_hi) {
      const double2* Fa = F + a * r;
      const double2* q = a < nsplit ? qa : qb;           // stacked [F1; F2]: rows >= nsplit use qb
      if (L == 1) {
        int k = (r & 1) ? 0 : (a & 7);                   // any start < r; a & 7 spreads 8 rows over banks
        while (k >= r) k -= r;
        int j = 0;
        for (; j + 2 <= r; j += 2) {
          const int k1 = (k + 1 == r) ? 0 : k + 1;
          const double2 f0 = Fa[k], f1 = Fa[k1];
          const double2* q0 = q + k * NR;
          const double2* q1 = q + k1 * NR;
#pragma unroll
          for (int c = 0; c < NR; ++c) {
            cfma(acc[c], f0, q0[c]);
            cfma(ac2[c], f1, q1[c]);
          }
          k = (k1 + 1 == r) ? 0 : k1 + 1;
        }
        if (j < r) {
          const double2 f0 = Fa[k];
          const double2* q0 = q + k * NR;
#pragma unroll
          for (int c = 0; c < NR; ++c) cfma(acc[c], f0, q0[c]);
        }
      } else {
        int k = sub;
        for (; k + L < r; k += 2 * L) {
          const double2 f0 = Fa[k], f1 = Fa[k + L];
          const double2* q0 = q + k * NR;
          const double2* q1 = q + (k + L) * NR;
#pragma unroll
          for (int c = 0; c < NR; ++c) {
            cfma(acc[c], f0, q0[c]);
            cfma(ac2[c], f1, q1[c]);
          }
        }
        if (k < r) {
          const double2 f0 = Fa[k];
          const double2* q0 = q + k * NR;
#pragma unroll
          for (int c = 0; c < NR; ++c) cfma(acc[c], f0, q0[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < NR; ++c) { acc[c].x += ac2[c].x; acc[c].y += ac2[c].y; }
    }
    for (int o = L / 2; o > 0; o >>= 1)
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        acc[c].x += __shfl_xor_sync(0xffffffffu, acc[c].x, o);
        acc[c].y += __shfl_xor_sync(0xffffffffu, acc[c].y, o);
      }
    if (a < a_hi && sub == 0) {
      double2* ya = y + (int64_t)a * R;
#pragma unroll
      for (int c = 0; c < NR; ++c)
        if (c < R) ya[c] = acc[c];
    }
  }
}

// Stacked colsum of a small block's [F1; F2] (rows [0, n1) and [n1, n1 + n2), x stacked the same
// way): dst1[k NR + c] = sum over F1 rows, dst2 over F2 rows, in one pass of the warp's lanes
// (lane = (g, k) as f1p_colsum_w; two accumulators per side; the G group sums added in g order).
template <int NR>
__device__ __forceinline__ void f1p_colsum2_w(const double2* F, int n1, int n2, int r, const double2* x, int R,
                                              double2* dst1, double2* dst2, int lane, const uint16_t* gk) {
  const int G = r <= 32 ? gk[F1P_GK + r] : 1;
  for (int kk = 0; kk < r; kk += 32) {
    int g = 0, k = kk + lane;
    if (r <= 32) { const int e = gk[r * 32 + lane]; g = e >> 8; k = e & 255; }
    double2 s1[NR], s2[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) s1[c] = s2[c] = make_double2(0.0, 0.0);
    if (g < G && k < r) {
      const int fs = G * r, xs = G * R;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const int lo = side ? n1 : 0, hi = side ? n1 + n2 : n1;
        double2 u[NR], v[NR];
#pragma unroll
        for (int c = 0; c < NR; ++c) u[c] = v[c] = make_double2(0.0, 0.0);
        int a = lo + g;
        const double2* fp = F + a * r + k;
        const double2* xp = x + a * R;
        for (; a + G < hi; a += 2 * G) {
          const double2 f0 = fp[0], f1 = fp[fs];
#pragma unroll
          for (int c = 0; c < NR; ++c) {
            cfma(u[c], f0, xp[c]);
            cfma(v[c], f1, xp[xs + c]);
          }
          fp += 2 * fs;
          xp += 2 * xs;
        }
        if (a < hi) {
          const double2 f0 = fp[0];
#pragma unroll
          for (int c = 0; c < NR; ++c) cfma(u[c], f0, xp[c]);
        }
#pragma unroll
        for (int c = 0; c < NR; ++c) {
          const double2 w = make_double2(u[c].x + v[c].x, u[c].y + v[c].y);
          if (side) s2[c] = w; else s1[c] = w;
        }
      }
    }
    if (G > 1) {
      double2 t1[NR], t2[NR];
#pragma unroll
      for (int c = 0; c < NR; ++c) { t1[c] = s1[c]; t2[c] = s2[c]; }
      for (int g2 = 1; g2 < G; ++g2) {
        const int src = min(31, k + g2 * r);
#pragma unroll
        for (int c = 0; c < NR; ++c) {
          t1[c].x += __shfl_sync(0xffffffffu, s1[c].x, src);
          t1[c].y += __shfl_sync(0xffffffffu, s1[c].y, src);
          t2[c].x += __shfl_sync(0xffffffffu, s2[c].x, src);
          t2[c].y += __shfl_sync(0xffffffffu, s2[c].y, src);
        }
      }
#pragma unroll
      for (int c = 0; c < NR; ++c) { s1[c] = t1[c]; s2[c] = t2[c]; }
    }
    if (g == 0 && k < r)
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        dst1[k * NR + c] = s1[c];
        dst2[k * NR + c] = s2[c];
      }
    if (r <= 32) break;
  }
}

// rows [0, n) of x (stride R) -> q (stride NR), one warp
template <int NR>
__device__ __forceinline__ void f1p_to_q(const double2* x, int n, int R, double2* q, int lane) {
  for (int e = lane; e < n * NR; e += 32) {
    const int k = e / NR, c = e - k * NR;
    q[e] = c < R ? x[k * R + c] : make_double2(0.0, 0.0);
  }
  __syncwarp();
}

// A whole small block out of the staged pack, one warp (q1 / q2: this warp's scratch).
template <int NR>
__device__ void f1p_small(const Far1pArgs& a, const FBlk& b, const double2* F, int64_t off0, const double2* X,
                          double2* q1, double2* q2, int lane, const uint16_t* gk) {
  const int R = a.R;
  const double2* F1 = F + (b.o1 - off0);
  const double2* x1 = X + b.xo1 * R;
  const double2* x2 = X + b.xo2 * R;
  if (b.dense) {
    // G (n1 x r): y1 = G x2 (rows of G), y2 = G^T x1 (one per column of G)
    f1p_to_q<NR>(x2, b.r, R, q2, lane);
    f1p_rowsum<NR, false>(F1, 0, b.n1, b.r, q2, R, a.y + b.y1 * R, lane);
    f1p_colsum_w<NR>(F1, 0, b.n1, b.r, x1, R, a.y + b.y2 * R, R, false, lane, gk);
    __syncwarp();
    return;
  }
  // F2 follows F1 in the stage, x2 follows x1, and the piece y2 follows y1: one stacked pass each
  // (p1 = F1^T x1 -> q1, p2 = F2^T x2 -> q2; then rows of F1 take q2, rows of F2 take q1)
  f1p_colsum2_w<NR>(F1, b.n1, b.n2, b.r, x1, R, q1, q2, lane, gk);
  __syncwarp();
  f1p_rowsum<NR, false>(F1, 0, b.n1 + b.n2, b.r, q2, R, a.y + b.y1 * R, lane, b.n1, q1);
  __syncwarp();
}

// q[e] = sum over the consumer warps w (in order) of part_w[e], e < n (all consumer threads)
__device__ __forceinline__ void f1p_warp_sum(const double2* part, int wstride, int n, double2* q) {
  for (int e = threadIdx.x; e < n; e += 32 * F1P_CWARPS) {
    double2 s = part[e];
    for (int v = 1; v < F1P_CWARPS; ++v) {
      const double2 t = part[v * wstride + e];
      s.x += t.x; s.y += t.y;
    }
    q[e] = s;
  }
}

template <int NR>
__global__ void __launch_bounds__(F1P_THREADS, NR <= 2 ? 2 : 1) far1p_kernel(Far1pArgs a) {
  // ring stages: F1P_NS, two at 8 columns (the scratch grows with the columns)
  constexpr int NS = NR >= 8 ? 2 : F1P_NS;
  extern __shared__ __align__(128) unsigned char f1p_sm[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  // per consumer warp 2 x F1P_RMAX x NR (a pack's q1 / q2; a big block's column-sum partial is
  // the first half), then the big block's final column sums (F1P_RMAX x NR)
  double2* scr = (double2*)(f1p_sm + NS * F1P_STAGE_BYTES);
  double2* qf = scr + F1P_CWARPS * 2 * F1P_RMAX * NR;
  auto stF = [&](int s) { return (double2*)(f1p_sm + s * F1P_STAGE_BYTES); };
  auto stX = [&](int s) { return stF(s) + F1P_CH; };
  auto stB = [&](int s) { return (FBlk*)(stX(s) + F1P_XCH); };
  auto stI = [&](int s) { return (FItem*)(stB(s) + F1P_PACK); };
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int R = a.R;
  // colsum lane map for r <= 32: gk[r * 32 + lane] = (g << 8) | k, g = lane / r, k = lane % r;
  // gk[F1P_GK + r] = 32 / r (division-free lookups in the per-block loops)
  __shared__ uint16_t gk[F1P_GK + 33];
  for (int e = tid; e < F1P_GK + 33; e += blockDim.x) {
    if (e < F1P_GK) {
      const int rr = e >> 5, l = e & 31;
      gk[e] = rr ? (uint16_t)(((l / rr) << 8) | (l % rr)) : 0;
    } else {
      const int rr = e - F1P_GK;
      gk[e] = rr ? (uint16_t)(32 / rr) : 1;
    }
  }
  if (tid == 0)
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], F1P_CWARPS); }
  __syncthreads();
  if (w == F1P_CWARPS) {
    // ---- producer warp: descriptors come in batches (the unit's FItems, lane j holding item
    // j of a 32-item window, handed out by shuffles; the next unit's ticket is taken when a unit
    // starts); every item is 3-4 bulk copies (factor range, block descriptors, its x rows, which
    // are contiguous in the gathered arena XA), so no descriptor load sits between two fills ----
    int t = 0;
    int64_t u = 0, unext = 0;
    if (lane == 0) u = atomicAdd(a.cnt, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    auto shfl_item = [&](const FItem& L, int j) {
      FItem r;
      r.off = __shfl_sync(0xffffffffu, L.off, j);
      r.xa = __shfl_sync(0xffffffffu, L.xa, j);
      r.xa2 = __shfl_sync(0xffffffffu, L.xa2, j);
      r.xn = __shfl_sync(0xffffffffu, L.xn, j);
      r.xn2 = __shfl_sync(0xffffffffu, L.xn2, j);
      r.len = __shfl_sync(0xffffffffu, L.len, j);
      r.kind = __shfl_sync(0xffffffffu, L.kind, j);
      r.b = __shfl_sync(0xffffffffu, L.b, j);
      r.nb = __shfl_sync(0xffffffffu, L.nb, j);
      r.a0 = __shfl_sync(0xffffffffu, L.a0, j);
      r.a1 = __shfl_sync(0xffffffffu, L.a1, j);
      return r;
    };
    while (u < a.nunits) {
      if (lane == 0) unext = atomicAdd(a.cnt, 1);       // consumed when this unit ends
      const FUnit U = a.units[u];
      for (int base = 0; base < U.n; base += 32) {
        const int nw = min(32, U.n - base);
        FItem L{};
        if (lane < nw) L = a.items[U.i0 + base + lane];
        for (int j = 0; j < nw; ++j, ++t) {
          const FItem it = shfl_item(L, j);
          const int s = t % NS;
          const int nbl = it.kind == 0 ? it.nb : 1;
          const uint32_t bytes = 16u * it.len + (uint32_t)sizeof(FBlk) * nbl + 16u * R * (uint32_t)(it.xn + it.xn2);
          if (t >= NS) mbar_wait(&empty[s], ((t / NS) - 1) & 1);
          if (lane == 0) {
            *stI(s) = it;
            mbar_arrive_tx(&full[s], bytes);
            bulk_g2s(stF(s), a.A + it.off, 16u * it.len, &full[s]);
            bulk_g2s(stB(s), a.blks + it.b, (uint32_t)sizeof(FBlk) * nbl, &full[s]);
            if (it.xn > 0) bulk_g2s(stX(s), a.x + it.xa * R, 16u * R * it.xn, &full[s]);
            if (it.xn2 > 0) bulk_g2s(stX(s) + it.xn * R, a.x + it.xa2 * R, 16u * R * it.xn2, &full[s]);
          }
          __syncwarp();
        }
      }
      u = __shfl_sync(0xffffffffu, unext, 0);
    }
    // end marker for the consumers
    const int s = t % NS;
    if (t >= NS) mbar_wait(&empty[s], ((t / NS) - 1) & 1);
    if (lane == 0) {
      FItem end{};
      end.kind = -1;
      *stI(s) = end;
      mbar_arrive(&full[s]);
    }
    return;
  }
  // ---- consumer warps ----
  double2* q1 = scr + (w * 2) * F1P_RMAX * NR;           // pack q1 / big-block partial of this warp
  double2* q2 = q1 + F1P_RMAX * NR;
  for (int t = 0;; ++t) {
    const int s = t % NS;
    mbar_wait(&full[s], (t / NS) & 1);
    const FItem it = *stI(s);
    if (it.kind < 0) break;
    const double2* F = stF(s);
    const double2* X = stX(s);
    const FBlk* B = stB(s);
    if (it.kind == 0) {
      for (int j = w; j < it.nb; j += F1P_CWARPS) f1p_small<NR>(a, B[j], F, it.off, X, q1, q2, lane, gk);
    } else {
      const FBlk b = B[0];
      const int h = it.a1 - it.a0, ch = it.nb;
      // rows per warp: an even split, but at least minrows (fewer warps on a short chunk)
      const int per = max((h + F1P_CWARPS - 1) / F1P_CWARPS, a.minrows);
      const int lo = min(h, w * per), hi = min(h, lo + per);
      const int rR = b.r * NR;                           // partials / final sums: r x NR
      if (it.kind == 4) {                                // dense big: G rows [a0, a1)
        f1p_to_q<NR>(X + h * R, b.r, R, q2, lane);
        f1p_rowsum<NR, true>(F, lo, hi, b.r, q2, R, a.y + (b.y1 + it.a0) * R, lane);
        f1p_colsum_w<NR>(F, lo, hi, b.r, X, R, q1, NR, ch > 0, lane, gk);
        if (ch == b.nc1 - 1) {                           // y2 = G^T x1: the warps' partials in order
          __syncwarp();
          f1p_cbar();
          f1p_warp_sum(scr, 2 * F1P_RMAX * NR, rR, qf);
          f1p_cbar();
          for (int e = tid; e < b.r * R; e += 32 * F1P_CWARPS) {
            const int k = e / R, c = e - k * R;
            a.y[b.y2 * R + e] = qf[k * NR + c];
          }
          f1p_cbar();
        }
      } else if (it.kind == 1) {                         // F1 rows: p1 partial
        f1p_colsum_w<NR>(F, lo, hi, b.r, X, R, q1, NR, ch > 0, lane, gk);
      } else if (it.kind == 2) {                         // F2 rows: y2 = F2 p1, p2 partial
        if (ch == 0) {
          __syncwarp();
          f1p_cbar();
          f1p_warp_sum(scr, 2 * F1P_RMAX * NR, rR, qf);
          f1p_cbar();
        }
        f1p_rowsum<NR, true>(F, lo, hi, b.r, qf, R, a.y + (b.y2 + it.a0) * R, lane);
        f1p_colsum_w<NR>(F, lo, hi, b.r, X, R, q1, NR, ch > 0, lane, gk);
      } else {                                           // F1 rows again: y1 = F1 p2
        if (ch == 0) {
          __syncwarp();
          f1p_cbar();
          f1p_warp_sum(scr, 2 * F1P_RMAX * NR, rR, qf);
          f1p_cbar();
        }
        f1p_rowsum<NR, true>(F, lo, hi, b.r, qf, R, a.y + (b.y1 + it.a0) * R, lane);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// one column: 2 CTAs per SM (the shared-memory ring of each plus its static tables and barriers)
static_assert(2 * ((size_t)F1P_NS * F1P_STAGE_BYTES + sizeof(double2) * (F1P_CWARPS * 2 + 1) * F1P_RMAX +
                   2 * (F1P_GK + 33) + 64 + 1024) <= 228 * 1024, "far1p: two CTAs per SM at one column");
// eight columns: one CTA per SM, two stages plus the 8-column scratch inside the 227 KB opt-in limit
static_assert(2 * (size_t)F1P_STAGE_BYTES + sizeof(double2) * (F1P_CWARPS * 2 + 1) * F1P_RMAX * 8 +
                  2 * (F1P_GK + 33) + 64 + 1024 <= 227 * 1024, "far1p: one CTA per SM at eight columns");
template <int NR>
static size_t far1p_smem() {
  return (size_t)(NR >= 8 ? 2 : F1P_NS) * F1P_STAGE_BYTES + sizeof(double2) * ((size_t)F1P_CWARPS * 2 + 1) * F1P_RMAX * NR;
}
template <int NR>
static int far1p_resident_of() {
  static int n = 0;
  if (n == 0) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(far1p_kernel<NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)far1p_smem<NR>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, far1p_kernel<NR>, F1P_THREADS, far1p_smem<NR>());
    n = sms * (per_sm > 0 ? per_sm : 1);
  }
  return n;
}
int far1p_resident_ctas(int R) {
  return R <= 1 ? far1p_resident_of<1>() : R <= 2 ? far1p_resident_of<2>() : R <= 4 ? far1p_resident_of<4>()
                                                                                    : far1p_resident_of<8>();
}
template <int NR>
static void far1p_go(const Far1pArgs& a, cudaStream_t st) {
  int g = far1p_resident_of<NR>();
  if (g > a.nunits) g = (int)a.nunits;
  far1p_kernel<NR><<<g, F1P_THREADS, far1p_smem<NR>(), st>>>(a);
}
void launch_far1p(const Far1pArgs& a, cudaStream_t st) {
  if (a.nunits <= 0) return;
  if (a.R <= 1) far1p_go<1>(a, st);
  else if (a.R <= 2) far1p_go<2>(a, st);
  else if (a.R <= 4) far1p_go<4>(a, st);
  else far1p_go<8>(a, st);
}

// Per leaf: Z rows = sum of its pieces in list order (one warp per leaf, lanes over the
// leaf's rows x R elements).
__global__ void far_reduce_kernel(int64_t nl, const int64_t* __restrict__ lptr, const int64_t* __restrict__ poff,
                                  const int64_t* __restrict__ lrow, const int32_t* __restrict__ lsz,
                                  const double2* __restrict__ y, double2* __restrict__ Z, int R) {
  const int lane = threadIdx.x & 31;
  const int64_t l = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (l >= nl) return;
  const int64_t q0 = lptr[l], q1 = lptr[l + 1];
  const int n = lsz[l] * R;
  for (int e = lane; e < n; e += 32) {
    double2 s = make_double2(0.0, 0.0);
    int64_t q = q0;
    for (; q + 4 <= q1; q += 4) {
      const double2 t0 = y[poff[q] * R + e], t1 = y[poff[q + 1] * R + e];
      const double2 t2 = y[poff[q + 2] * R + e], t3 = y[poff[q + 3] * R + e];
      s.x += t0.x; s.y += t0.y; s.x += t1.x; s.y += t1.y;
      s.x += t2.x; s.y += t2.y; s.x += t3.x; s.y += t3.y;
    }
    for (; q < q1; ++q) {
      const double2 t = y[poff[q] * R + e];
      s.x += t.x; s.y += t.y;
    }
    Z[lrow[l] * R + e] = s;
  }
}
void launch_far_reduce(int64_t nl, const int64_t* lptr, const int64_t* poff, const int64_t* lrow,
                       const int32_t* lsz, const double2* y, double2* Z, int R, cudaStream_t st) {
  if (nl <= 0) return;
  const int64_t thr = nl * 32;
  far_reduce_kernel<<<(unsigned)((thr + 255) / 256), 256, 0, st>>>(nl, lptr, poff, lrow, lsz, y, Z, R);
}

__global__ void fb_gather_kernel(int64_t n, const FCopy* __restrict__ runs, double2* __restrict__ base) {
  for (int64_t d = blockIdx.x; d < n; d += gridDim.x) {
    const FCopy c = runs[d];
    const int64_t tot = (int64_t)c.rows * c.r;
    for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
      const int64_t row = e / c.r, k = e - row * c.r;
      base[c.dst + e] = base[c.src + row * c.ss + k * c.sk];
    }
  }
}
void launch_fb_gather(int64_t n, const FCopy* runs, double2* base, cudaStream_t st) {
  if (n <= 0) return;
  fb_gather_kernel<<<(unsigned)(n < 148 * 64 ? n : 148 * 64), 128, 0, st>>>(n, runs, base);
}

// ---------------------------------------------------------------------------
// Batched explicit inverse of the scaled diagonal blocks (Eqs. 23, 30):
// in-place Gauss-Jordan with partial pivoting (max |z|^2, lowest row on ties),
// one CTA per leaf. Blocks up to SMEM_N fit shared memory; larger ones are
// eliminated in place in the destination buffer (L2-resident).
constexpr int SMEM_N = 117;     // n^2 + n complex + n int + the static reductions <= 227 KB

__global__ void __launch_bounds__(512)
inverse_kernel(const int32_t* __restrict__ leaf_ids, const int32_t* __restrict__ sizes,
               const int64_t* __restrict__ src_off, const int64_t* __restrict__ src_ld,
               const int64_t* __restrict__ dst_off, const double2* __restrict__ Wb,
               double2* __restrict__ Db, int32_t* __restrict__ status, int use_smem, int n_lo, int n_hi) {
  extern __shared__ double2 sm[];
  __shared__ double red_v[512];
  __shared__ int red_i[512];
  __shared__ double s_fro;
  __shared__ int s_piv;
  __shared__ int s_sing;
  const int l = blockIdx.x;
  const int n = sizes[l];
  if (n < n_lo || n > n_hi) return;                   // another launch of this level takes it
  const int64_t ld_src = src_ld[l];
  const double2* src = Wb + src_off[l];
  double2* dst = Db + dst_off[l];
  const bool in_smem = use_smem != 0;
  double2* a = in_smem ? sm : dst;       // working matrix, column-major, ld n
  double2* colk = in_smem ? sm + n * n : sm;  // column k factors (n)
  int* piv = (int*)(colk + n);
  const int tid = threadIdx.x, nt = blockDim.x;
  double fro = 0.0;
  for (int e = tid; e < n * n; e += nt) {
    const int i = e % n, j = e / n;
    const double2 v = src[i + (int64_t)j * ld_src];
    a[e] = v;
    fro += v.x * v.x + v.y * v.y;
  }
  red_v[tid] = fro;
  __syncthreads();
  for (int s = nt / 2; s > 0; s >>= 1) {
    if (tid < s) red_v[tid] += red_v[tid + s];
    __syncthreads();
  }
  if (tid == 0) { s_fro = sqrt(red_v[0]); s_sing = 0; }
  __syncthreads();
  const double tol2 = (1e-14 * s_fro) * (1e-14 * s_fro);
  const int lane = tid & 31, w = tid >> 5, nw = nt >> 5;
  // per pivot: 3 CTA barriers (pivot reduction, swap + column k copy, elimination); the pivot
  // search is a warp-shuffle argmax (max |z|^2, lowest row on ties), every column j is owned by
  // one warp (rows over lanes: coalesced, no index division), which scales row k itself
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int bi = n;
    for (int i = k + tid; i < n; i += nt) {
      const double2 v = a[i + k * n];
      const double m2 = v.x * v.x + v.y * v.y;
      if (m2 > best) { best = m2; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double vo = __shfl_xor_sync(0xffffffffu, best, o);
      const int io = __shfl_xor_sync(0xffffffffu, bi, o);
      if (vo > best || (vo == best && io < bi)) { best = vo; bi = io; }
    }
    if (lane == 0) { red_v[w] = best; red_i[w] = bi; }
    __syncthreads();
    if (w == 0) {
      best = lane < nw ? red_v[lane] : -1.0;
      bi = lane < nw ? red_i[lane] : n;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double vo = __shfl_xor_sync(0xffffffffu, best, o);
        const int io = __shfl_xor_sync(0xffffffffu, bi, o);
        if (vo > best || (vo == best && io < bi)) { best = vo; bi = io; }
      }
      if (lane == 0) {
        s_piv = bi;
        piv[k] = bi;
        if (!(best > tol2)) s_sing = 1;
      }
    }
    __syncthreads();
    if (s_sing) break;
    const int r = s_piv;
    // rows k <-> r (column k is rewritten whole by the elimination: not swapped), and column
    // k as it reads after the swap saved as the elimination factors
    for (int j = tid; j < n; j += nt) {
      if (r != k && j != k) {
        const double2 t = a[k + j * n];
        a[k + j * n] = a[r + j * n];
        a[r + j * n] = t;
      }
    }
    for (int i = tid; i < n; i += nt) colk[i] = a[(i == k ? r : i == r ? k : i) + k * n];
    __syncthreads();
    const double2 p = colk[k];
    const double pm = p.x * p.x + p.y * p.y;
    const double2 inv = make_double2(p.x / pm, -p.y / pm);
    for (int j = w; j < n; j += nw) {
      const double2 v = (j == k) ? make_double2(1.0, 0.0) : a[k + j * n];
      const double2 rk = make_double2(v.x * inv.x - v.y * inv.y, v.x * inv.y + v.y * inv.x);
      __syncwarp();                                     // every lane has read row k of column j
      for (int i = lane; i < n; i += 32) {
        if (i == k) { a[k + j * n] = rk; continue; }
        const double2 f = colk[i];
        double2 base = (j == k) ? make_double2(0.0, 0.0) : a[i + j * n];
        base.x -= f.x * rk.x - f.y * rk.y;
        base.y -= f.x * rk.y + f.y * rk.x;
        a[i + j * n] = base;
      }
    }
    __syncthreads();
  }
  if (s_sing) {
    if (tid == 0) status[l] = 1;
    return;
  }
  // undo the row interchanges as column interchanges, in reverse order
  for (int k = n - 1; k >= 0; --k) {
    const int r = piv[k];
    if (r != k)
      for (int i = tid; i < n; i += nt) {
        const double2 t = a[i + k * n];
        a[i + k * n] = a[i + r * n];
        a[i + r * n] = t;
      }
    __syncthreads();
  }
  if (in_smem)
    for (int e = tid; e < n * n; e += nt) dst[e] = a[e];
  if (tid == 0) status[l] = 0;
}

// Blocks too large for one CTA's shared memory (C3's and C5's separator leaves, up to 375
// unknowns): one thread-block CLUSTER of CL CTAs per block, CTA r holding columns
// [r w, min(n, (r + 1) w)) of the working matrix in its own shared memory (w = ceil(n / CL)).
// Per pivot k the CTA owning column k picks the pivot (the same rule: max |z|^2, lowest row on
// ties) and writes column k as it reads after the row swap, and the pivot row, into every CTA's
// shared memory (distributed shared memory, double-buffered by the parity of k); one cluster
// barrier; every CTA then swaps, scales and eliminates its own columns (a warp per column).
// The final column interchanges become one permuted store per column.
constexpr int INVC_T = 256;

__global__ void __launch_bounds__(INVC_T)
inverse_cluster_kernel(const int32_t* __restrict__ sizes, const int64_t* __restrict__ src_off,
                       const int64_t* __restrict__ src_ld, const int64_t* __restrict__ dst_off,
                       const double2* __restrict__ Wb, double2* __restrict__ Db, int32_t* __restrict__ status,
                       int n_lo, int n_hi) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double2 smc[];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ double s_part[16];                        // Frobenius partials of the CTAs (rank 0's copy used)
  __shared__ double s_tol2;
  __shared__ int s_r, s_sing;
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks(), rk = (int)cl.block_rank();
  const int l = blockIdx.x / CL;
  const int n = sizes[l];
  if (n < n_lo || n > n_hi) return;                    // the whole cluster returns
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  const int w = (n + CL - 1) / CL;
  const int j0 = min(n, rk * w), j1 = min(n, j0 + w), nj = j1 - j0;
  double2* a = smc;                                    // n x w, column-major, ld n
  double2* cbuf = smc + (size_t)n * w;                 // 2 x n: column k after the swap, by parity of k
  int* meta = (int*)(cbuf + 2 * n);                    // [par]: pivot row, [2 + par]: singular
  int* piv = meta + 4;                                 // n pivot rows
  int* loc = piv + n;                                  // n: final column c <- working column loc[c]
  const int64_t ld_src = src_ld[l];
  const double2* src = Wb + src_off[l];
  double2* dst = Db + dst_off[l];
  double fro = 0.0;
  for (int jj = wid; jj < nj; jj += nw)
    for (int i = lane; i < n; i += 32) {
      const double2 v = src[i + (int64_t)(j0 + jj) * ld_src];
      a[i + jj * n] = v;
      fro += v.x * v.x + v.y * v.y;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  if (lane == 0) red_v[wid] = fro;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int v = 0; v < nw; ++v) t += red_v[v];
    *cl.map_shared_rank(&s_part[rk], 0) = t;
  }
  cl.sync();
  if (tid == 0) {
    const double* p0 = cl.map_shared_rank(s_part, 0);
    double t = 0.0;
    for (int v = 0; v < CL; ++v) t += p0[v];          // fixed rank order: the same tolerance everywhere
    const double f = sqrt(t);
    s_tol2 = (1e-14 * f) * (1e-14 * f);
  }
  __syncthreads();
  const double tol2 = s_tol2;
  bool sing = false;
  for (int k = 0; k < n; ++k) {
    const int par = k & 1;
    if (k / w == rk) {                                 // this CTA owns column k
      __syncthreads();                                 // its columns are up to date
      const double2* ck = a + (k - j0) * n;
      double best = -1.0;
      int bi = n;
      for (int i = k + tid; i < n; i += nt) {
        const double m2 = ck[i].x * ck[i].x + ck[i].y * ck[i].y;
        if (m2 > best) { best = m2; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double vo = __shfl_xor_sync(0xffffffffu, best, o);
        const int io = __shfl_xor_sync(0xffffffffu, bi, o);
        if (vo > best || (vo == best && io < bi)) { best = vo; bi = io; }
      }
      if (lane == 0) { red_v[wid] = best; red_i[wid] = bi; }
      __syncthreads();
      if (wid == 0) {
        best = lane < nw ? red_v[lane] : -1.0;
        bi = lane < nw ? red_i[lane] : n;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double vo = __shfl_xor_sync(0xffffffffu, best, o);
          const int io = __shfl_xor_sync(0xffffffffu, bi, o);
          if (vo > best || (vo == best && io < bi)) { best = vo; bi = io; }
        }
        if (lane == 0) { s_r = bi; s_sing = !(best > tol2); }
      }
      __syncthreads();
      const int r = s_r;
      for (int e = tid; e < n * CL; e += nt) {
        const int q = e / n, i = e - q * n;
        *cl.map_shared_rank(cbuf + par * n + i, q) = ck[i == k ? r : i == r ? k : i];
      }
      if (tid < CL) {
        *cl.map_shared_rank(meta + par, tid) = r;
        *cl.map_shared_rank(meta + 2 + par, tid) = s_sing;
        *cl.map_shared_rank(piv + k, tid) = r;
      }
    }
    cl.sync();
    if (meta[2 + par]) { sing = true; break; }
    const int r = meta[par];
    const double2* colk = cbuf + par * n;
    const double2 p = colk[k];
    const double pm = p.x * p.x + p.y * p.y;
    const double2 inv = make_double2(p.x / pm, -p.y / pm);
    for (int jj = wid; jj < nj; jj += nw) {
      const int j = j0 + jj;
      double2* c = a + jj * n;
      const double2 old_k = c[k];                      // row k before the swap (becomes row r)
      const double2 v = (j == k) ? make_double2(1.0, 0.0) : c[r];
      const double2 rkv = make_double2(v.x * inv.x - v.y * inv.y, v.x * inv.y + v.y * inv.x);
      __syncwarp();
      for (int i = lane; i < n; i += 32) {
        if (i == k) { c[k] = rkv; continue; }
        const double2 f = colk[i];
        double2 base = (j == k) ? make_double2(0.0, 0.0) : (i == r ? old_k : c[i]);
        base.x -= f.x * rkv.x - f.y * rkv.y;
        base.y -= f.x * rkv.y + f.y * rkv.x;
        c[i] = base;
      }
    }
  }
  if (!sing) {
    if (tid == 0) {                                    // the column interchanges, composed
      for (int c = 0; c < n; ++c) loc[c] = c;
      for (int k = n - 1; k >= 0; --k) {
        const int t = loc[k];
        loc[k] = loc[piv[k]];
        loc[piv[k]] = t;
      }
    }
    __syncthreads();
    for (int c = wid; c < n; c += nw) {
      const int jw = loc[c];
      if (jw < j0 || jw >= j1) continue;
      const double2* col = a + (jw - j0) * n;
      for (int i = lane; i < n; i += 32) dst[i + (int64_t)c * n] = col[i];
    }
  }
  if (rk == 0 && tid == 0) status[l] = sing ? 1 : 0;
  cl.sync();                                           // no CTA leaves while its shared memory may be written
}

static size_t inv_cluster_smem(int n, int CL) {
  const int w = (n + CL - 1) / CL;
  return (size_t)n * w * sizeof(double2) + 2 * (size_t)n * sizeof(double2) + (4 + 2 * (size_t)n) * sizeof(int) + 16;
}

void launch_inverse(int64_t nl, const int32_t* leaf_ids, const int32_t* sizes, const int64_t* src_off,
                    const int64_t* src_ld, const int64_t* dst_off, const double2* Wbase,
                    double2* Dbase, int32_t* status, int max_n, cudaStream_t st) {
  if (nl <= 0) return;
  static int max_dyn = -1, max_dyn_c = -1;
  if (max_dyn < 0) {                                   // opt-in limit minus the kernels' static shared memory
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, inverse_kernel);
    max_dyn = optin - (int)fa.sharedSizeBytes;
    cudaFuncSetAttribute(inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
    cudaFuncAttributes fc{};
    cudaFuncGetAttributes(&fc, inverse_cluster_kernel);
    max_dyn_c = optin - (int)fc.sharedSizeBytes;
    cudaFuncSetAttribute(inverse_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_c);
    cudaFuncSetAttribute(inverse_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  auto smem_of = [](int nn, int mn) {
    return (size_t)nn * nn * sizeof(double2) + (size_t)mn * sizeof(double2) + (size_t)mn * sizeof(int) + 16;
  };
  // sizes >= cmin go to the cluster kernel (default: the ones shared memory of one CTA cannot hold)
  static const int cmin = [] {
    const char* e = std::getenv("PS_INV_CLUSTER_MIN");
    return e ? std::max(1, std::atoi(e)) : SMEM_N + 1;
  }();
  const int ns = std::min(max_n, std::min(SMEM_N, cmin - 1));
  if (ns >= 1)
    inverse_kernel<<<(unsigned)nl, 512, smem_of(ns, ns), st>>>(leaf_ids, sizes, src_off, src_ld, dst_off, Wbase,
                                                               Dbase, status, 1, 0, ns);
  if (max_n <= ns) return;
  int CL = 0;
  for (int c : {8, 16})
    if ((int64_t)inv_cluster_smem(max_n, c) <= max_dyn_c) { CL = c; break; }
  if (CL) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nl * CL));
    cfg.blockDim = dim3(INVC_T);
    cfg.dynamicSmemBytes = inv_cluster_smem(max_n, CL);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, inverse_cluster_kernel, sizes, src_off, src_ld, dst_off, Wbase, Dbase, status,
                       ns + 1, max_n);
  } else {                                             // larger still: in place in the destination (L2)
    inverse_kernel<<<(unsigned)nl, 512, smem_of(0, max_n), st>>>(leaf_ids, sizes, src_off, src_ld, dst_off,
                                                                 Wbase, Dbase, status, 0, ns + 1, max_n);
  }
}

// ---------------------------------------------------------------------------
// Permutations between the caller's RWG order (column-major N x nrhs) and the
// internal leaf-row-major layout (row = unknown, nrhs contiguous complex).
// The column-major side is touched 16 bytes at a time at scattered rows, so the elements are
// walked in panels of PERM_PW columns (panel, row, column in panel): the rows x PERM_PW slab
// of B / X a panel touches stays in L2 while every row is visited, and each of its 32-byte
// sectors moves to or from HBM once (column-fastest order over all nrhs columns left half-used
// sectors: 1.1 TB/s at 360 columns).
constexpr int64_t PERM_PW = 16;
__device__ __forceinline__ void perm_index(int64_t e, int64_t N, int64_t nrhs, int64_t& r, int64_t& c) {
  const int64_t np = (nrhs + PERM_PW - 1) / PERM_PW;
  int64_t p = e / (N * PERM_PW);                       // only the last panel is narrower
  if (p > np - 1) p = np - 1;
  const int64_t rem = e - p * N * PERM_PW;
  const int64_t w = p == np - 1 ? nrhs - p * PERM_PW : PERM_PW;
  r = rem / w;
  c = p * PERM_PW + (rem - r * w);
}
__global__ void permute_in_kernel(int64_t N, int64_t nrhs, const int64_t* __restrict__ map,
                                  const double2* __restrict__ B, int64_t ldb, double2* __restrict__ y) {
  const int64_t tot = N * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r, c;
    perm_index(e, N, nrhs, r, c);
    const int64_t m = map[r];
    y[r * nrhs + c] = m >= 0 ? B[m + c * ldb] : make_double2(0.0, 0.0);
  }
}
__global__ void permute_out_kernel(int64_t N, int64_t nrhs, const int64_t* __restrict__ map,
                                   const double2* __restrict__ y, double2* __restrict__ X, int64_t ldx) {
  const int64_t tot = N * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r, c;
    perm_index(e, N, nrhs, r, c);
    const int64_t m = map[r];
    if (m >= 0) X[m + c * ldx] = y[r * nrhs + c];
  }
}
__global__ void permute_rows_kernel(int64_t N, int64_t nrhs, const int64_t* __restrict__ map,
                                    const double2* __restrict__ src, double2* __restrict__ dst) {
  const int64_t tot = N * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / nrhs, c = e - r * nrhs;
    dst[e] = src[map[r] * nrhs + c];
  }
}

static unsigned grid_for(int64_t tot) {
  int64_t g = (tot + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

void launch_permute_in(int64_t N, int64_t nrhs, const int64_t* map, const double2* B, int64_t ldb,
                       double2* y, cudaStream_t st) {
  permute_in_kernel<<<grid_for(N * nrhs), 256, 0, st>>>(N, nrhs, map, B, ldb, y);
}
void launch_permute_out(int64_t N, int64_t nrhs, const int64_t* map, const double2* y, double2* X,
                        int64_t ldx, cudaStream_t st) {
  permute_out_kernel<<<grid_for(N * nrhs), 256, 0, st>>>(N, nrhs, map, y, X, ldx);
}
void launch_permute_rows(int64_t N, int64_t nrhs, const int64_t* map, const double2* src,
                         double2* dst, cudaStream_t st) {
  permute_rows_kernel<<<grid_for(N * nrhs), 256, 0, st>>>(N, nrhs, map, src, dst);
}

// ---------------------------------------------------------------------------
// x~ = b_o - u (Eq. 36) fused with the per-column squared norms of it_0 = b_o
// and it_1 = u (Eq. 44). Deterministic two-stage reduction (fixed chunking).
__global__ void combine_norms_kernel(int64_t N, int64_t nrhs, const double2* __restrict__ bo,
                                     const double2* __restrict__ u, double2* __restrict__ xt,
                                     double2* __restrict__ part, int64_t rpc) {
  const int64_t c = blockIdx.y * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nrhs) return;
  const int64_t r0 = blockIdx.x * rpc, r1 = min(N, r0 + rpc);
  double s0 = 0.0, s1 = 0.0;
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t e = r * nrhs + c;
    const double2 a = bo[e], b = u[e];
    s0 += a.x * a.x + a.y * a.y;
    s1 += b.x * b.x + b.y * b.y;
    xt[e] = make_double2(a.x - b.x, a.y - b.y);
  }
  part[blockIdx.x * nrhs + c] = make_double2(s0, s1);
}
// ||b_o||^2 and ||u||^2 = ||b_o - x~||^2 per column (Eq. 44), fixed chunking
__global__ void norms2_kernel(int64_t N, int64_t nrhs, const double2* __restrict__ bo,
                              const double2* __restrict__ xt, double2* __restrict__ part, int64_t rpc) {
  const int64_t c = blockIdx.y * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nrhs) return;
  const int64_t r0 = blockIdx.x * rpc, r1 = min(N, r0 + rpc);
  double s0 = 0.0, s1 = 0.0;
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t e = r * nrhs + c;
    const double2 a = bo[e], x = xt[e];
    const double ux = a.x - x.x, uy = a.y - x.y;
    s0 += a.x * a.x + a.y * a.y;
    s1 += ux * ux + uy * uy;
  }
  part[blockIdx.x * nrhs + c] = make_double2(s0, s1);
}
void launch_norms2(int64_t N, int64_t nrhs, const double2* bo, const double2* xt, double2* part,
                   int64_t rpc, cudaStream_t st) {
  dim3 g((unsigned)((N + rpc - 1) / rpc), (unsigned)((nrhs + 127) / 128));
  norms2_kernel<<<g, 128, 0, st>>>(N, nrhs, bo, xt, part, rpc);
}

// Per-column sums of the chunk partials (fixed order: thread (cx, ky) adds chunks ky, ky + KY, ...
// in turn, then the KY sums are added pairwise by a fixed halving tree). CW columns per CTA:
// 32 for wide blocks (coalesced over the columns), 1 for narrow ones (all threads over chunks).
template <int CW>
__global__ void __launch_bounds__(256) finalize_norms_kernel(int64_t nch, int64_t nrhs, const double2* __restrict__ part,
                                                             double2* __restrict__ norms, int do_sqrt) {
  constexpr int KY = 256 / CW;
  __shared__ double2 sm[256];
  const int cx = threadIdx.x % CW, ky = threadIdx.x / CW;
  const int64_t c = blockIdx.x * (int64_t)CW + cx;
  double s0 = 0.0, s1 = 0.0;
  if (c < nrhs)
    for (int64_t k = ky; k < nch; k += KY) {
      const double2 p = part[k * nrhs + c];
      s0 += p.x;
      s1 += p.y;
    }
  sm[threadIdx.x] = make_double2(s0, s1);
  __syncthreads();
  for (int h = KY / 2; h > 0; h >>= 1) {
    if (ky < h) {
      const double2 o = sm[(ky + h) * CW + cx];
      double2 v = sm[ky * CW + cx];
      v.x += o.x;
      v.y += o.y;
      sm[ky * CW + cx] = v;
    }
    __syncthreads();
  }
  if (ky == 0 && c < nrhs) {
    const double2 v = sm[cx];
    norms[c] = do_sqrt ? make_double2(sqrt(v.x), sqrt(v.y)) : v;
  }
}
void launch_combine_norms(int64_t N, int64_t nrhs, const double2* bo, const double2* u, double2* xt,
                          double2* part, int64_t rpc, cudaStream_t st) {
  dim3 g((unsigned)((N + rpc - 1) / rpc), (unsigned)((nrhs + 127) / 128));
  combine_norms_kernel<<<g, 128, 0, st>>>(N, nrhs, bo, u, xt, part, rpc);
}
void launch_finalize_norms(int64_t nch, int64_t nrhs, const double2* part, double2* norms,
                           cudaStream_t st, int do_sqrt) {
  if (nrhs >= 32) finalize_norms_kernel<32><<<(unsigned)((nrhs + 31) / 32), 256, 0, st>>>(nch, nrhs, part, norms, do_sqrt);
  else finalize_norms_kernel<1><<<(unsigned)nrhs, 256, 0, st>>>(nch, nrhs, part, norms, do_sqrt);
}

// One term of the n-term series (Eq. 44): acc += sign it_n, fused with the per-column squared
// norms of it_n and of the new partial sum (Eqs. 44-45); fixed chunking as combine_norms.
__global__ void series_accum_kernel(int64_t N, int64_t nrhs, const double2* __restrict__ it,
                                    double2* __restrict__ acc, double sign, int first,
                                    double2* __restrict__ part, int64_t rpc) {
  const int64_t c = blockIdx.y * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nrhs) return;
  const int64_t r0 = blockIdx.x * rpc, r1 = min(N, r0 + rpc);
  double s0 = 0.0, s1 = 0.0;
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t e = r * nrhs + c;
    const double2 t = it[e];
    double2 a = first ? make_double2(0.0, 0.0) : acc[e];
    a.x += sign * t.x;
    a.y += sign * t.y;
    s0 += t.x * t.x + t.y * t.y;
    s1 += a.x * a.x + a.y * a.y;
    acc[e] = a;
  }
  part[blockIdx.x * nrhs + c] = make_double2(s0, s1);
}
void launch_series_accum(int64_t N, int64_t nrhs, const double2* it, double2* acc, double sign, int first,
                         double2* part, int64_t rpc, cudaStream_t st) {
  dim3 g((unsigned)((N + rpc - 1) / rpc), (unsigned)((nrhs + 127) / 128));
  series_accum_kernel<<<g, 128, 0, st>>>(N, nrhs, it, acc, sign, first, part, rpc);
}

__global__ void set_ones_kernel(double2* __restrict__ base, const int64_t* __restrict__ offs, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    base[offs[e]] = make_double2(1.0, 0.0);
}
void launch_set_ones(double2* base, const int64_t* offs, int64_t n, cudaStream_t st) {
  if (n > 0) set_ones_kernel<<<grid_for(n), 256, 0, st>>>(base, offs, n);
}

__global__ void add_kernel(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] += src[e];
}
void launch_add(double* dst, const double* src, int64_t n, cudaStream_t st) {
  if (n > 0) add_kernel<<<grid_for(n), 256, 0, st>>>(dst, src, n);
}

__global__ void zero_kernel(double2* p, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    p[e] = make_double2(0.0, 0.0);
}
void launch_zero(double2* p, int64_t n, cudaStream_t st) {
  if (n > 0) zero_kernel<<<grid_for(n), 256, 0, st>>>(p, n);
}

}  // namespace ps
