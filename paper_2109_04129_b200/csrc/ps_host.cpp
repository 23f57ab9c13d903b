// ps_host.cpp — host side of libps: the C ABI of include/ps.h.
//
//   hm_load  : read + verify the .hm file, upload the near/far arenas, symbolic
//              analysis of the scaling (Eqs. 14-23): struct(k) with
//              fill-in, elimination tree, level schedules, arena layout.
//   ps_setup : GPU, level by level over the elimination tree (left-looking):
//              Z~_p* = Z_p* + sum_d alpha_dp^T Z~_d*     (Eq. 21)
//              D_p^{-1} = (Z~_pp)^{-1}                  (Eqs. 23, 30)
//              alpha_p* = -D_p^{-1} Z~_p*               (Eq. 16)
//   ps_solve : GPU, two-term series (Eqs. 24, 26, 31, 32, 36, 44-45).
//
// Everything that runs per leaf/block is expressed as rows of the gather-GEMM
// task tables consumed by ps_kernels.cu; this file only builds tables (once per
// handle / per nrhs) and enqueues launches. No numerical work happens here.
#include "../../include/ps.h"
#include "ps_internal.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>
#include <queue>
#include <condition_variable>
#include <exception>
#include <mutex>
#include <thread>
#include <tuple>

using namespace ps;

namespace {

thread_local std::string g_err;

struct PsError {
  ps_status st;
  std::string msg;
};

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      throw PsError{e_ == cudaErrorMemoryAllocation ? PS_ENOMEM : PS_ECUDA,                     \
                    std::string(#x) + ": " + cudaGetErrorString(e_)};                           \
  } while (0)

// Pinned host staging of a handle's table uploads: a cudaMemcpyAsync from pageable
// memory synchronises the stream and stages / pins the pages on every call (measured
// 16-500 ms of a C2 setup); copying through one pinned ring keeps the uploads cheap and
// asynchronous. All copies of a ring go to one stream (the handle's), so the event of
// the latest copy covers every earlier one when the ring wraps.
struct PinnedRing {
  char* p = nullptr;
  size_t cap = 0, off = 0;
  cudaEvent_t ev = nullptr;
  bool pending = false;
  PinnedRing() = default;
  PinnedRing(const PinnedRing&) = delete;
  PinnedRing& operator=(const PinnedRing&) = delete;
  ~PinnedRing() {
    if (pending) cudaEventSynchronize(ev);
    if (p) cudaFreeHost(p);
    if (ev) cudaEventDestroy(ev);
  }
  void copy(void* dst, const void* src, size_t bytes, cudaStream_t st);
};

// Device buffer; alloc() keeps the allocation when it is large enough (tables rebuilt
// level by level in ps_setup reuse their buffers instead of a cudaMalloc / cudaFree pair each).
template <class T>
struct DevBuf {
  T* p = nullptr;
  int64_t n = 0, cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), cap(o.cap) { o.p = nullptr; o.n = o.cap = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; cap = o.cap; o.p = nullptr; o.n = o.cap = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = cap = 0;
  }
  void alloc(int64_t count) {
    if (p && count > 0 && count <= cap) { n = count; return; }
    release();
    if (count <= 0) return;
    const cudaError_t e = cudaMalloc(&p, sizeof(T) * (size_t)count);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      throw PsError{e == cudaErrorMemoryAllocation ? PS_ENOMEM : PS_ECUDA,
                    std::string("device allocation of ") + std::to_string((sizeof(T) * (size_t)count) >> 20) +
                        " MiB failed (" + cudaGetErrorString(e) + "; " + std::to_string(fr >> 20) + " of " +
                        std::to_string(tot >> 20) + " MiB free)"};
    }
    n = cap = count;
  }
  void upload(const std::vector<T>& v, cudaStream_t st, PinnedRing* ring = nullptr) {
    alloc((int64_t)v.size());
    if (v.empty()) return;
    if (ring) ring->copy(p, v.data(), sizeof(T) * v.size(), st);
    else CK(cudaMemcpyAsync(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st));
  }
};

void PinnedRing::copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  const size_t need = (bytes + 255) & ~(size_t)255;
  if (need > cap || off + need > cap) {                 // wrap or grow: the ring's copies must be done
    if (pending) CK(cudaEventSynchronize(ev));
    pending = false;
    off = 0;
    if (need > cap) {
      if (p) CK(cudaFreeHost(p));
      p = nullptr;
      cap = std::max<size_t>(need, std::max<size_t>(2 * cap, (size_t)64 << 20));
      CK(cudaMallocHost(&p, cap));
    }
  }
  if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  std::memcpy(p + off, src, bytes);
  CK(cudaMemcpyAsync(dst, p + off, bytes, cudaMemcpyHostToDevice, st));
  CK(cudaEventRecord(ev, st));
  pending = true;
  off += need;
}

uint64_t checksum64(const uint8_t* b, size_t nbytes) {
  uint64_t h = 0;
  size_t nw = nbytes / 8;
  for (size_t i = 0; i < nw; ++i) {
    uint64_t w;
    std::memcpy(&w, b + 8 * i, 8);
    h += w * (2 * (uint64_t)i + 1);
  }
  if (nbytes % 8) {
    uint64_t w = 0;
    std::memcpy(&w, b + 8 * nw, nbytes % 8);
    h += w * (2 * (uint64_t)nw + 1);
  }
  return h ^ (uint64_t)nbytes;
}

// Optional per-launch CUDA-event profiling (ps_profile): events are recorded on
// the launching stream around every kernel; elapsed times are accumulated per
// kernel class after the solve's final synchronisation.
enum { PC_FWD = 0, PC_BWD, PC_DINV, PC_FAR1, PC_FAR2, PC_AUX, PC_PROG, PC_F1P, PC_COUNT };
struct Prof {
  bool on = false;
  // debug trace of the LAST profiled flow launch of class trace_cls
  bool trace_on = false;
  int trace_cls = 0;
  DevBuf<int64_t> trace_buf;
  const std::vector<GWork>* trace_work = nullptr;
  const std::vector<GTask>* trace_tasks = nullptr;
  int64_t trace_w0 = 0, trace_nw = 0;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, size_t>> marks;
  size_t used = 0;
  double ms[PC_COUNT] = {0}, flops[PC_COUNT] = {0}, bytes[PC_COUNT] = {0};
  int64_t n[PC_COUNT] = {0};
  void begin(int cls, cudaStream_t s) {
    if (!on) return;
    if (used + 2 > pool.size()) {
      size_t old = pool.size();
      pool.resize(std::max<size_t>(64, 2 * pool.size()));
      for (size_t i = old; i < pool.size(); ++i) CK(cudaEventCreate(&pool[i]));
    }
    marks.push_back({cls, used});
    CK(cudaEventRecord(pool[used], s));
    used += 2;
  }
  void end(cudaStream_t s) {
    if (!on) return;
    CK(cudaEventRecord(pool[marks.back().second + 1], s));
  }
  void collect() {  // after a stream sync
    for (auto& m : marks) {
      float t = 0;
      CK(cudaEventElapsedTime(&t, pool[m.second], pool[m.second + 1]));
      ms[m.first] += t;
      n[m.first] += 1;
    }
    marks.clear();
    used = 0;
  }
  void reset() {
    for (int c = 0; c < PC_COUNT; ++c) ms[c] = flops[c] = bytes[c] = 0, n[c] = 0;
  }
  ~Prof() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// Tuning knobs (environment, read once; defaults are the measured choices).
int env_int(const char* name, int def) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : def;
}

// split-K chunk (k-steps) of the narrow (small nrhs, operator-streaming) tiles
int NARROW_STEPS() {
  static const int v = env_int("PS_NARROW_STEPS", 16);
  return v;
}

// Tile mode of a plan with nrhs columns: 1 = narrow 64 x 8 tiles (nrhs <= 8, operator
// streaming), 0 = wide 32 x 64 tiles.
int narrow_mode(int64_t R) { return R <= 8 ? 1 : 0; }
// concurrent work units of a launch (the split-K chunk heuristics aim at about one item
// per unit per stage) and rows of a tile
bool g_host_only = false;        // ps_validate: plans built on the host only (no device)
int resident_units(int) { return g_host_only ? 296 : flow_resident_ctas(); }
int mode_rows(int mode) { return mode ? GN_MT : GM_MT; }

// A gather-GEMM table: tasks, segments, work items and batches (one launch each).
constexpr int CHUNK_STEPS = 16;    // target k-steps (of GM_KC) per split-K work item

struct Table {
  std::vector<GTask> tasks;
  std::vector<GTerm> terms;
  std::vector<GWork> work;
  std::vector<Batch> batches;
  DevBuf<GTask> d_tasks;
  DevBuf<GTerm> d_terms;
  DevBuf<GWork> d_work;
  DevBuf<int32_t> d_counters;
  DevBuf<double2> d_partial;
  int64_t cur_batch_start = 0;
  // completion units, split-K tiles and partial slots are numbered per batch (one
  // launch each; counters are cleared per launch), the buffers sized for the largest
  int32_t n_units = 0, n_tiles = 0;
  int64_t n_slots = 0;
  int32_t max_units = 0, max_tiles = 0;
  int64_t max_slots = 0;
  int chunk_steps = CHUNK_STEPS;
  int narrow = 0;          // 1: 64 x 8 tiles (small nrhs), 0: 32 x 64 tiles
  double2* S = nullptr;    // scratch vector base of osel / bsel offsets (chain stages)
  int mma = 0;             // wide-tile consumer: 0 DFMA, 1 FP64 mma.sync (DMMA)
  // optional global ordering of work items (ticket order): key = key_base + nt * key_stagger,
  // stable-sorted by sort_by_key() (valid when every dependency has a smaller key)
  double key_base = 0, key_stagger = 0;
  std::vector<double> keys, keys_late;
  std::vector<double> task_key;      // key_base of every task at creation
  // early_keys: a chunk is keyed just after the latest of its producers' tasks
  // (not at its own task's key), so a gather's bulk chunks enter the ticket
  // order as soon as their inputs can exist; the critical chunk (which adds the
  // group sum) keeps the task's key. Every item still follows its producers.
  bool early_keys = false;
  // sorts the items of the open batch (keys hold one entry per item since cur_batch_start)
  void sort_by_key() {
    const int64_t w0 = cur_batch_start, nw = (int64_t)work.size() - w0;
    if ((int64_t)keys.size() != nw) throw PsError{PS_ECUDA, "internal: ticket keys out of step with the batch"};
    std::vector<int64_t> idx(nw);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t x, int64_t y) { return keys[x] < keys[y]; });
    std::vector<GWork> w2(nw);
    for (int64_t i = 0; i < nw; ++i) w2[i] = work[w0 + idx[i]];
    std::copy(w2.begin(), w2.end(), work.begin() + w0);
    keys.clear();
    keys_late.clear();
  }
  // sort_by_key + close_batch for a one-batch table, bounded partial-slot memory: with
  // early keys a split tile's chunks spread over the ticket order and its slots stay
  // live meanwhile; if the recycled pool still exceeds the budget (C5), the batch is
  // re-ordered by its tasks' own keys (chunks of a tile adjacent) and re-assigned.
  void sort_close_bounded() {
    static const int64_t budget_mb = env_int("PS_SLOT_BUDGET_MB", 4096);   // < 0: always task-keyed
    const int64_t budget = budget_mb < 0 ? 0 : budget_mb << 20;
    const bool can_redo = early_keys && budget_mb != 0;
    std::vector<GWork> w0;
    std::vector<double> kl;
    if (can_redo) { w0 = work; kl = keys_late; }
    const int32_t nu = n_units, ntl = n_tiles, mu = max_units, mtl = max_tiles;
    const int64_t ns = n_slots, ms = max_slots, cb0 = cur_batch_start;
    sort_by_key();
    close_batch();
    if (can_redo && max_slots * slot_elems() * 16 >= budget) {
      work.swap(w0);
      keys = kl;
      batches.pop_back();
      task_end.pop_back();
      n_units = nu; n_tiles = ntl; max_units = mu; max_tiles = mtl;
      n_slots = ns; max_slots = ms; cur_batch_start = cb0;
      sort_by_key();
      close_batch();
      late_keys_used = true;
    }
  }
  bool late_keys_used = false;
  // empty the table for a new level, keeping its device buffers (ps_setup)
  void reset_keep_device() {
    Table f;
    f.d_tasks = std::move(d_tasks); f.d_terms = std::move(d_terms); f.d_work = std::move(d_work);
    f.d_counters = std::move(d_counters); f.d_partial = std::move(d_partial);
    f.S = S; f.narrow = narrow; f.chunk_steps = chunk_steps; f.mma = mma;
    *this = std::move(f);
  }
  int MT() const { return narrow ? GN_MT : GM_MT; }
  int64_t slot_elems() const { return narrow ? (int64_t)GN_MT * GN_NT : (int64_t)GM_MT * GM_NT; }
  int NT() const { return narrow ? GN_NT : GM_NT; }

  int32_t add_task(int64_t oO, int64_t sOi, int64_t sOc, int64_t oI, int64_t sIi, int64_t sIc, int m,
                   int n, int sign) {
    GTask t;
    t.oO = oO; t.sOi = sOi; t.sOc = sOc;
    t.oI = oI; t.sIi = sIi; t.sIc = sIc;
    t.m = m; t.n = n; t.sign = sign;
    t.t0 = t.t1 = (int32_t)terms.size();
    t.K = 0;
    t.unit0 = 0; t.n_mt = (m + GM_MT - 1) / GM_MT;
    t.a_kmajor = 0; t.b_kmajor = 0; t.idep = -1; t.osel = 0; t.idep_nmt = 0; t.idep_ntp = 0;
    tasks.push_back(t);
    task_key.push_back(key_base);
    return (int32_t)tasks.size() - 1;
  }
  // append a K-segment: A(i,k) = A[oA + k sAk + i sAi], B(k,c) = B[oB + k sBk + c sBc]
  void add_term(int32_t task, int64_t oA, int64_t sAi, int64_t sAk, int64_t oB, int64_t sBk,
                int64_t sBc, int K, int32_t dep = -1, int32_t bsel = 0) {
    if (task != (int32_t)tasks.size() - 1)
      throw PsError{PS_ECUDA, "internal: terms must be added to the newest task"};
    if (K <= 0) return;
    GTask& t = tasks[task];
    if (t.t1 == t.t0) {
      t.a_kmajor = (sAi != 1) ? 1 : 0;
      t.b_kmajor = (sBc != 1) ? 1 : 0;
    }
    GTerm g;
    g.oA = oA; g.sAi = sAi; g.sAk = sAk;
    g.oB = oB; g.sBk = sBk; g.sBc = sBc;
    g.kstart = t.K; g.K = K; g.dep = dep; g.bsel = bsel;
    terms.push_back(g);
    t.K += K;
    t.t1 = (int32_t)terms.size();
  }
  // work items of a task: every (mt, nt) tile, its virtual K split into chunks
  // of ~chunk_steps k-steps (split-K); also assigns the task's completion units.
  // chunks (ka, kb, ta, tb) covering virtual k in [k_lo, k_hi) = segments [s0, s1)
  void chunk_range(int32_t s0, int32_t s1, std::vector<std::array<int32_t, 4>>& ch, int steps) const {
    if (s0 >= s1) return;
    const int32_t k_lo = terms[s0].kstart, k_hi = terms[s1 - 1].kstart + terms[s1 - 1].K;
    const int target = std::min(steps * GM_KC, narrow ? GN_CHUNK_K : GM_CHUNK_K);
    int32_t ka = k_lo, ta = s0;
    while (ka < k_hi) {
      int32_t kb = std::min(k_hi, ka + target);
      int32_t tb = ta;
      while (tb < s1 && terms[tb].kstart < kb) ++tb;
      if (tb - ta > GM_MAXSEG) {          // too many tiny segments: stop earlier
        tb = ta + GM_MAXSEG;
        kb = terms[tb - 1].kstart + terms[tb - 1].K;
        kb = ka + std::max<int32_t>(GM_KC, ((kb - ka) / GM_KC) * GM_KC);
        kb = std::min(kb, k_hi);
        tb = ta;
        while (tb < s1 && terms[tb].kstart < kb) ++tb;
      }
      ch.push_back({ka, kb, ta, tb});
      ka = kb;
      while (ta < s1 && terms[ta].kstart + terms[ta].K <= ka) ++ta;
    }
  }
  // Work items of a task: every (mt, nt) tile, its virtual K split into chunks
  // of ~chunk_steps k-steps (split-K); also assigns the task's completion units.
  // isolate = +1 / -1 puts the first / last segment (the dependency expected to
  // complete last: the parent in the backward sweep, the last child in the
  // forward sweep) in a chunk of its own, so a chain hop waits on a short chunk.
  // Work items of a task: every (mt, nt) tile, its virtual K split into chunks
  // of ~steps k-steps (split-K); also assigns the task's completion units.
  // isolate = +1 / -1: the first / last segment (the dependency expected to
  // complete last: the parent in the backward sweep, the last child in the
  // forward sweep) becomes the critical chunk (queued last, adds the sum of
  // the others); the NEAR - 1 segments next to it (the next-latest
  // dependencies) become single-segment chunks in subgroups of their own, the
  // bulk is chunked normally and combined in subgroups of SUBG.
  static inline const int NEAR = env_int("PS_NEAR", 1), SUBG = env_int("PS_SUBG", 16);
  // segments in the critical chunk: the chain predecessor AND the one before it,
  // so the group sum the critical chunk adds never waits on a just-finished
  // producer (its latest input is >= 2 hops old)
  static inline const int CRITSEG = env_int("PS_CRITSEG", 2);
  void tile(int32_t task, int isolate = 0, int steps = 0) {
    if (steps <= 0) steps = chunk_steps;
    GTask& t = tasks[task];
    // narrow items of short tasks (<= 32 rows: 16/32-row tiles stream 64/32 k per stage) take
    // twice the k per chunk in stages big enough to hit the chunk cap, so an item streams as
    // many operator bytes as a 64-row one (C4-1 -5 %; in small stages it would cost parallelism)
    static const int short_x2 = env_int("PS_NARROW_SHORT_X2", 1);
    if (narrow && short_x2 && t.m <= 32 && steps >= NARROW_STEPS()) steps *= 2;   // only where the stage is capped
    // consumer per task: every wide task on the FP64 tensor cores (with the swizzled,
    // conflict-free fragment loads the DMMA consumer beats DFMA even on 4-20-row leaves
    // padded to 8-row blocks: C4-360 100.6 -> 91.7 ms); PS_MMA_MINROWS=n keeps tasks
    // shorter than n rows on the DFMA consumer (PS_MMA=dfma: all of them)
    static const int auto_mma = env_int("PS_AUTO_MMA", 1), mma_rows = env_int("PS_MMA_MINROWS", 1);
    if (auto_mma && !narrow && t.m >= mma_rows) t.osel |= 4;
    static const int iso_env = env_int("PS_ISOLATE", 0);
    if (!iso_env) isolate = 0;
    t.n_mt = (t.m + MT() - 1) / MT();
    const int nmt = t.n_mt, nnt = (t.n + NT() - 1) / NT();
    t.unit0 = n_units;
    n_units += nnt;
    std::vector<std::array<int32_t, 4>> ch;   // (ka, kb, ta, tb)
    std::vector<char> single;                 // chunk forms its own subgroup
    auto add = [&](int32_t s0, int32_t s1, bool one) {
      const size_t before = ch.size();
      chunk_range(s0, s1, ch, steps);
      single.resize(ch.size(), one ? 1 : 0);
      (void)before;
    };
    const int nseg = t.t1 - t.t0;
    int32_t crit = -1;
    if (isolate != 0 && nseg >= 2) {
      const int cs = std::max(1, std::min(CRITSEG, nseg - 1));       // segments in the critical chunk
      const int nnear = std::max(0, std::min(NEAR - 1, nseg - cs));
      auto add_one = [&](int32_t s0, int32_t s1) {                    // one chunk, however long
        chunk_range(s0, s1, ch, 1 << 20);
        single.resize(ch.size(), 1);
      };
      if (isolate > 0) {
        add_one(t.t0, t.t0 + cs);                                    // critical
        for (int q = 0; q < nnear; ++q) add(t.t0 + cs + q, t.t0 + cs + q + 1, true);
        add(t.t0 + cs + nnear, t.t1, false);
        crit = 0;
      } else {
        add(t.t0, t.t1 - cs - nnear, false);
        for (int q = nnear - 1; q >= 0; --q) add(t.t1 - cs - 1 - q, t.t1 - cs - q, true);
        add_one(t.t1 - cs, t.t1);                                    // critical
        crit = (int32_t)ch.size() - 1;
      }
    } else {
      add(t.t0, t.t1, false);
    }
    if (ch.empty()) {
      ch.push_back({0, 0, t.t0, t.t0});
      single.push_back(0);
    }
    const int nch = (int)ch.size();
    if (nch < 2) crit = -1;
    // subgroups over the non-critical chunks in rank order
    std::vector<int32_t> rank_chunk;
    for (int c = 0; c < nch; ++c)
      if (c != crit) rank_chunk.push_back(c);
    const int G = (int)rank_chunk.size();
    std::vector<int32_t> sub_of(nch, -1), sub_r0, sub_r1;
    for (int r = 0; r < G;) {
      int r1 = r + 1;
      if (!single[rank_chunk[r]])
        while (r1 < G && r1 - r < SUBG && !single[rank_chunk[r1]]) ++r1;
      for (int q = r; q < r1; ++q) sub_of[rank_chunk[q]] = (int32_t)sub_r0.size();
      sub_r0.push_back(r);
      sub_r1.push_back(r1);
      r = r1;
    }
    const int nsub = (int)sub_r0.size();
    for (int a = 0; a < nmt; ++a)
      for (int b = 0; b < nnt; ++b) {
        // split-K tiles: counters [top, subgroups...], slots [chunks..., subgroup sums...]
        const int32_t tile_id = n_tiles;
        if (nch > 1) n_tiles += 1 + nsub;
        const int64_t slot = nch > 1 ? n_slots : 0;
        if (nch > 1) n_slots += nch + nsub;
        auto push = [&](int c) {
          const int sg = sub_of[c];
          work.push_back({task, a, b, ch[c][2], ch[c][3], ch[c][0], ch[c][1], c, nch, tile_id, crit,
                          sg, sg >= 0 ? sub_r0[sg] : 0, sg >= 0 ? sub_r1[sg] : 0, nsub, -1, 0, 0, slot});
          double k = key_base;
          if (early_keys && c != crit) {
            double kp = -1.0;
            for (int32_t q = ch[c][2]; q < ch[c][3]; ++q)
              if (terms[q].dep >= 0) kp = std::max(kp, task_key[terms[q].dep]);
            if (t.idep >= 0) kp = std::max(kp, task_key[t.idep]);
            static const double early_off = 0.01 * env_int("PS_EARLY_OFF", 50);   // key levels after the producer
            k = std::min(key_base, kp + early_off);
          }
          keys.push_back(k + b * key_stagger);
          keys_late.push_back(key_base + b * key_stagger);
        };
        for (int c = 0; c < nch; ++c)
          if (c != crit) push(c);
        if (crit >= 0) push(crit);
      }
  }
  // Partial-sum slots of the batch's split tiles, recycled in ticket order: a
  // tile takes a block (power-of-two size class >= nchunks + nsub) whose previous
  // tile's unit has ALL its items at least SLOT_SLACK tickets before this tile's
  // first item; the tile's items wait for that unit (ticket-ordered, so
  // deadlock-free) before writing. Bounds the partial buffer by the tiles in
  // flight instead of every split tile of the launch (C5: >100 GB otherwise).
  static inline const int SLOT_REUSE = env_int("PS_SLOT_REUSE", 1);
  static inline const int SLOT_SLACK = env_int("PS_SLOT_SLACK", 2048);
  void assign_slots(int64_t w0, int64_t w1) {
    if (!SLOT_REUSE || w1 <= w0) return;
    std::vector<int64_t> ulast(n_units, -1);
    for (int64_t i = w0; i < w1; ++i) ulast[tasks[work[i].task].unit0 + work[i].nt] = i;
    struct Blk { int64_t base; int32_t unit, need; };
    std::vector<std::vector<Blk>> free_(32);
    using Pend = std::tuple<int64_t, int, Blk>;             // (release ticket, class, block)
    auto cmp = [](const Pend& x, const Pend& y) { return std::get<0>(x) > std::get<0>(y); };
    std::priority_queue<Pend, std::vector<Pend>, decltype(cmp)> pend(cmp);
    std::unordered_map<int32_t, Blk> of_tile;                 // tile -> (slot base, wait unit, need)
    int64_t pool = 0;
    for (int64_t i = w0; i < w1; ++i) {
      GWork& w = work[i];
      if (w.nchunks <= 1) continue;
      auto it = of_tile.find(w.tile);
      if (it == of_tile.end()) {
        while (!pend.empty() && std::get<0>(pend.top()) + SLOT_SLACK < i) {
          free_[std::get<1>(pend.top())].push_back(std::get<2>(pend.top()));
          pend.pop();
        }
        const int64_t len = (int64_t)w.nchunks + w.nsub;
        int c = 0;
        while ((int64_t(1) << c) < len) ++c;
        Blk b;
        if (!free_[c].empty()) {
          b = free_[c].back();
          free_[c].pop_back();
        } else {
          b = {pool, -1, 0};
          pool += int64_t(1) << c;
        }
        it = of_tile.emplace(w.tile, b).first;
        const GTask& T = tasks[w.task];
        const int32_t u = T.unit0 + w.nt;
        pend.push({ulast[u], c, Blk{b.base, u, T.n_mt}});
      }
      w.slot = it->second.base;
      w.sw_unit = it->second.unit;
      w.sw_need = it->second.need;
    }
    n_slots = pool;
  }
  std::vector<int32_t> task_end;      // tasks.size() at each close_batch (task -> batch)
  int batch_of_task(int32_t t) const {
    return (int)(std::upper_bound(task_end.begin(), task_end.end(), t) - task_end.begin());
  }
  void close_batch() {
    task_end.push_back((int32_t)tasks.size());
    keys.clear();
    keys_late.clear();
    int64_t n = (int64_t)work.size() - cur_batch_start;
    batches.push_back({cur_batch_start, n});
    assign_slots(cur_batch_start, (int64_t)work.size());
    cur_batch_start = (int64_t)work.size();
    max_units = std::max(max_units, n_units);
    max_tiles = std::max(max_tiles, n_tiles);
    max_slots = std::max(max_slots, n_slots);
    static const int per_batch = env_int("PS_BATCH_SLOTS", 1);
    if (per_batch) {
      n_units = n_tiles = 0;
      n_slots = 0;
    }
  }
  double alg_flops = 0, alg_bytes = 0;   // useful flops / operator (A) bytes of one full pass
  void upload(cudaStream_t st, PinnedRing* ring = nullptr) {
    alg_flops = alg_bytes = 0;
    for (const GTask& t : tasks)
      for (int32_t k = t.t0; k < t.t1; ++k) {
        alg_flops += 8.0 * t.m * (double)t.n * terms[k].K;
        alg_bytes += 16.0 * t.m * (double)terms[k].K;
      }
    // device copies: dependencies as the producer's completion unit, row tiles and
    // column tiles (the kernels wait without loading the producer's descriptor)
    std::vector<GTask> dtasks = tasks;
    std::vector<GTerm> dterms = terms;
    auto ntp_of = [&](const GTask& P) { return (P.n + NT() - 1) / NT(); };
    for (GTask& t : dtasks) {
      t.idep_nmt = t.idep_ntp = 0;
      if (t.idep >= 0) {
        const GTask& P = tasks[t.idep];
        t.idep_nmt = P.n_mt;
        t.idep_ntp = ntp_of(P);
        t.idep = P.unit0;
      }
    }
    for (GTerm& g : dterms)
      if (g.dep >= 0) {
        const GTask& P = tasks[g.dep];
        if (P.n_mt >= (1 << 15) || ntp_of(P) >= (1 << 16))
          throw PsError{PS_ECUDA, "internal: dependency descriptor out of range"};
        g.bsel = (g.bsel & 1) | (P.n_mt << 1) | (int32_t)((uint32_t)ntp_of(P) << 16);
        g.dep = P.unit0;
      }
    d_tasks.upload(dtasks, st, ring);
    d_terms.upload(dterms, st, ring);
    d_work.upload(work, st, ring);
    d_counters.alloc(1 + (int64_t)max_units + max_tiles);
    d_partial.alloc(std::max<int64_t>(max_slots, 1) * slot_elems());
    static const int verbose = env_int("PS_VERBOSE", 0);
    if (verbose)
      std::fprintf(stderr, "[ps] table: %zu tasks, %zu terms, %zu items, %zu batches, %lld partial slots (%lld MiB)%s\n",
                   tasks.size(), terms.size(), work.size(), batches.size(), (long long)max_slots,
                   (long long)((max_slots * slot_elems() * 16) >> 20), late_keys_used ? ", task-keyed" : "");
  }
  int64_t launch(int b, double2* O, const double2* I, const double2* A, const double2* B,
                 cudaStream_t st, Prof* pf = nullptr, int cls = 0) const {
    const Batch& bt = batches[b];
    if (bt.nw <= 0) return 0;
    if (pf) pf->begin(cls, st);
    CK(cudaMemsetAsync(d_counters.p, 0, sizeof(int32_t) * d_counters.n, st));
    FlowArgs fa;
    fa.work = d_work.p + bt.w0;
    fa.nwork = bt.nw;
    fa.tasks = d_tasks.p;
    fa.terms = d_terms.p;
    fa.O = O; fa.I = I; fa.A = A; fa.B = B; fa.S = S;
    fa.counters = d_counters.p;
    fa.n_units = max_units;
    static const int defer_fin = env_int("PS_DEFER_FIN", 1);
    fa.defer_fin = defer_fin;
    fa.partial = d_partial.p;
    fa.trace = nullptr;
    fa.narrow = narrow;
    // consumer: PS_MMA=dmma / dfma forces one for every table, else the table's own
    // choice (far-field tables: FP64 tensor cores; sweeps / D^-1 / setup: DFMA)
    static const int mma_env = [] {
      const char* e = std::getenv("PS_MMA");
      if (e && std::string(e) == "dmma") return 1;
      if (e && std::string(e) == "dfma") return 0;
      return -1;
    }();
    fa.mma = mma_env >= 0 ? mma_env : mma;
    static const int ksplit = env_int("PS_KSPLIT", 1);
    fa.ksplit = ksplit;
    static const int gauss = env_int("PS_GAUSS", 1);
    fa.gauss = gauss;
    if (pf && pf->trace_on && cls == pf->trace_cls) {
      pf->trace_buf.alloc(8 * bt.nw);
      CK(cudaMemsetAsync(pf->trace_buf.p, 0, 8 * sizeof(int64_t) * bt.nw, st));
      fa.trace = pf->trace_buf.p;
      pf->trace_work = &work;
      pf->trace_tasks = &tasks;
      pf->trace_w0 = bt.w0;
      pf->trace_nw = bt.nw;
    }
    launch_flow(fa, 0, st);
    if (pf) pf->end(st);
    return 1;
  }
  int64_t launch_all(double2* O, const double2* I, const double2* A, const double2* B,
                     cudaStream_t st, Prof* pf = nullptr, int cls = 0) const {
    int64_t n = 0;
    for (size_t b = 0; b < batches.size(); ++b) n += launch((int)b, O, I, A, B, st, pf, cls);
    if (pf && pf->on) {
      pf->flops[cls] += alg_flops;
      pf->bytes[cls] += alg_bytes;
    }
    return n;
  }
};

// Per-nrhs solve plan: tables + workspaces.
struct SolvePlan {
  int64_t nrhs = 0;
  int64_t ws_len = 0;                      // program workspace (complex entries)
  Table fwd, bwd, dinv, far1, far2;        // per-operator tables (ps_apply, PS_SOLVE=stages)
  Table prog;                              // the whole two-term solve as one dataflow program
  DevBuf<double2> ws;                      // program workspace: Y BO W Z XT X TMP SC (offsets below)
  int64_t oY = 0, oBO = 0, oW = 0, oZ = 0, oXT = 0, oX = 0, oTMP = 0, oSC = 0;
  DevBuf<double2> y, bo, w, u, xt, wm, tm, part, norms, stage, sc;
  int64_t nchunks = 0, rpc = 64;
  int64_t launches_per_solve = 0;
  bool stages_built = false;
  // far1p (narrow solves): the program is two batches (S1-S3 | S6-S8) around the one-pass
  // far apply (Morton copy of w, far1p items -> pieces, per-leaf sums -> Z)
  bool f1p = false;
  std::vector<FBlk> f1p_blk;               // the handle's blocks with this nrhs' packing / chunking
  std::vector<FItem> f1p_item;
  std::vector<FUnit> f1p_unit;
  DevBuf<FBlk> d_f1p_blk;
  DevBuf<FItem> d_f1p_item;
  DevBuf<FUnit> d_f1p_unit;
  DevBuf<int32_t> d_f1p_cnt;
  DevBuf<double2> f1p_y, f1p_xa;
};

// Per-nrhs plan of the row-partitioned solve: this rank's tables
// over one workspace arena ws = [Y | BO | W | Z | XT | X | TMP] in the
// partitioned row layout (doff), every table addressing it through offsets.
struct DistPlan {
  int64_t nrhs = 0;
  Table fwdIA, fwdSA, dinvA, bwdA, far1, far2, fwdIC, fwdSC, dinvC, bwdC;
  DevBuf<double2> ws, part, sums, scratch;
  int64_t oY = 0, oBO = 0, oW = 0, oZ = 0, oXT = 0, oX = 0, oTMP = 0, oSC = 0;
  int64_t rpc = 64, nchI = 0, nchS = 0;
};

}  // namespace

struct ps_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t ustream = nullptr;          // ps_setup: table uploads (overlapping the level kernels)
  std::string err;
  // ---- file ----
  int64_t N = 0, nl = 0, nnear = 0, nfar = 0;
  std::vector<int64_t> perm, leaf_off;
  std::vector<int32_t> leaf_ijk, elim;
  std::vector<int64_t> near_list;   // 3 per block
  std::vector<int64_t> far_list;    // 7 per block
  int64_t near_len = 0, far_len = 0;
  // ---- symbolic (positions p = elimination order) ----
  std::vector<int32_t> pos_of, leaf_at, nsz, parent, height, depth;
  std::vector<int64_t> eoff;                          // first unknown of p (E order)
  std::vector<std::vector<int32_t>> st;               // struct(p), sorted
  std::vector<std::vector<int64_t>> pcol;             // column offset of st[p][i] inside P_p
  std::vector<int64_t> S;                             // sum of sizes in struct(p)
  std::vector<std::vector<std::pair<int32_t, int32_t>>> gath;  // q -> (d, idx of q in st[d])
  std::vector<int64_t> Woff, Poff, Doff;
  int64_t Wlen = 0, Plen = 0, Dlen = 0;
  int max_height = 0, max_depth = 0;
  std::vector<int64_t> e2rwg, e2mort, m2e;
  // far field restacked per cluster (Morton range): S_c = [factor^T of every
  // block side whose rows are cluster c] (sum_r x len, column-major)
  std::vector<int64_t> cl_start, cl_len, cl_sr, cl_soff;
  std::vector<int64_t> fb_ct, fb_cs, fb_rbt, fb_rbs;   // per block: clusters, row offsets in stacks
  std::vector<int64_t> fb_dense;                       // per block: offset of dense D (m x n) or -1
  int64_t stack_len = 0;
  double setup_madds = 0;
  int64_t alpha_blocks = 0;
  // ---- elimination-tree chains: maximal paths p_1 -> ... -> p_L
  // (p_{i+1} = parent(p_i) with p_i its only child), cut into pieces of at most
  // PS_TMAX unknowns. A piece with L >= 2 has T_c = (I - A_c^T)^{-1}, A_c the
  // strictly upper block matrix of its internal alpha blocks (U_c x U_c,
  // column-major, in the T region of the operator arena), so each sweep over
  // the piece is one parallel block product instead of L dependent hops.
  std::vector<int32_t> chain_of;                 // per position
  std::vector<std::vector<int32_t>> chains;      // positions p_1..p_L, bottom to top
  std::vector<int64_t> ch_U, ch_Toff;            // unknowns; offset of T_c (-1: L = 1)
  std::vector<int64_t> cpos;                     // per position: first row inside its chain
  std::vector<int32_t> ch_height, ch_depth;
  int max_ch_height = 0, max_ch_depth = 0;
  int64_t Tlen = 0, Tbase = 0;
  bool use_chains = true;
  // near block lookup: (leaf a, leaf b) -> index into near_list
  std::unordered_map<uint64_t, int64_t> near_idx;
  // ---- device ----
  // operator arena: [ alpha panels P (Plen) | D^-1 (Dlen) | far stacks + dense far blocks ]
  DevBuf<double2> d_near, d_W, d_op;
  // far stacks and chain matrices live in their own allocations, made after the
  // setup-only arenas (W, near) are freed (peak device memory of ps_setup); tables
  // address them from the d_op base through the pointer differences Fbase / Tbase
  DevBuf<double2> d_farbuf, d_T;
  std::vector<double2> far_host;            // restacked far factors until uploaded
  struct RawBuf { double2* p = nullptr; } d_P, d_D, d_far;   // views into d_op
  int64_t Pbase = 0, Dbase = 0, Fbase = 0;
  DevBuf<int64_t> d_e2rwg, d_e2mort, d_m2e;
  bool setup_done = false;
  double ratio_threshold = 0.1;
  std::unique_ptr<SolvePlan> plan;
  DevBuf<double2> series_norms;            // ps_solve_series: per term (||it_n||, ||x~||) per column
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaStream_t cs_in = nullptr, cs_out = nullptr;   // ps_solve on host buffers, pipelined halves:
  cudaEvent_t hp_ev[6] = {};                        // copy streams, ordering events, staging
  DevBuf<double2> hp_in[2], hp_out[2], hp_norms;
  int64_t pend_nrhs = 0;               // ps_solve_async: columns of the solve whose report is pending
  cudaStream_t pend_stream = nullptr;  //                 and the stream it was queued on
  Prof prof;
  // ---- row partition (ps_dist.partition = 1) ----
  int rank = 0, nranks = 1, part_mode = 0;
  bool sharded = false;                    // operator held for this rank's share only (sharded setup)
  std::vector<char> need;                  // per position: this rank holds its rows (own interior or separator)
  std::vector<int64_t> near_dev;           // per near block: element offset in d_near, -1 if not held
  int64_t near_dev_len = 0;
  int64_t Wsep0 = 0, Wsep_len = 0;         // separator rows of the W arena (one contiguous range, summed
                                           // over the ranks between the two setup phases)
  int64_t near_file_off = -1;              // byte offset of the near arena in the .hm file (deferred read)
  uint64_t near_file_ck = 0;
  std::string path;
  PinnedRing ring;                         // pinned staging of the table uploads (h->stream)
  std::vector<int32_t> owner, far_owner;   // per position: interior rank (-1 separator); far-row rank
  std::vector<int64_t> doff;               // first row of position p in the partitioned layout:
                                           // [rank 0 interior | ... | rank P-1 interior | separators],
                                           // each interior block padded to maxI rows
  int64_t own_rows = 0, maxI = 0, Nsep = 0, Npad = 0;
  std::vector<int64_t> d2rwg;              // layout row -> RWG index (-1: padding)
  DevBuf<int64_t> d_d2rwg;
  void* nccl = nullptr;                    // ncclComm_t; nullptr: in-process group (ps_solve_group)
  std::unique_ptr<DistPlan> dplan;
  // ---- one-pass far apply of narrow solves (far1p, ps_internal.h) ----
  int f1p_state = 0;                       // 0 not built, 1 ready, -1 unavailable on this handle
  std::vector<FBlk> f1p_blk;                // blocks: [0, f1p_nsmall) small (pack candidates), then big
  int64_t f1p_nsmall = 0, f1p_ch = F1P_CH;
  std::vector<int64_t> f1p_lptr, f1p_poff, f1p_lrow;   // per Morton leaf: its pieces (rows), first E row
  std::vector<int64_t> f1p_xmap;                        // XA row -> elimination row of w
  std::vector<int32_t> f1p_lsz;
  int64_t f1p_prows = 0, f1p_len = 0, FBbase = 0;
  double f1p_alg_bytes = 0, f1p_alg_flops1 = 0;        // factor bytes read once; flops per column
  DevBuf<double2> d_fb;                    // FB arena: factors rows-major, small blocks first
  DevBuf<int64_t> d_f1p_lptr, d_f1p_poff, d_f1p_lrow, d_f1p_xmap;
  DevBuf<int32_t> d_f1p_lsz;
};

namespace {

ps_status fail(ps_handle* h, ps_status s, const std::string& msg) {
  if (h) h->err = msg;
  g_err = msg;
  return s;
}

// ------------------------------------------------------------------ file
void read_file(ps_handle* h, const char* path, std::vector<double2>& near_arena,
               std::vector<double2>& far_arena, bool defer_near = false) {
  FILE* f = std::fopen(path, "rb");
  if (!f) throw PsError{PS_EIO, std::string("cannot open ") + path};
  std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
  auto rd = [&](void* dst, size_t n) {
    if (n && std::fread(dst, 1, n, f) != n) throw PsError{PS_EFORMAT, "truncated file"};
  };
  uint8_t hdr[128];
  rd(hdr, 128);
  if (std::memcmp(hdr, "HMPS", 4) != 0) throw PsError{PS_EFORMAT, "bad magic (not an .hm file)"};
  uint32_t ver;
  std::memcpy(&ver, hdr + 4, 4);
  if (ver != 1) throw PsError{PS_EFORMAT, "unsupported .hm version " + std::to_string(ver)};
  int64_t v5[5];
  std::memcpy(v5, hdr + 8, 40);
  h->N = v5[0]; h->nl = v5[1]; h->nnear = v5[2]; h->nfar = v5[3];
  if (!(v5[4] & 1)) throw PsError{PS_EFORMAT, "only symmetric H-matrices are supported"};
  std::memcpy(&h->near_len, hdr + 112, 8);
  std::memcpy(&h->far_len, hdr + 120, 8);
  if (h->N <= 0 || h->nl <= 0 || h->nl > h->N || h->nnear < h->nl || h->nfar < 0 ||
      h->near_len < 0 || h->far_len < 0)
    throw PsError{PS_EFORMAT, "inconsistent header sizes"};
  uint64_t ck;
  rd(&ck, 8);
  if (ck != checksum64(hdr, 128)) throw PsError{PS_EFORMAT, "header checksum mismatch"};
  auto section = [&](void* dst, size_t nbytes, const char* name) {
    rd(dst, nbytes);
    size_t pad = (8 - nbytes % 8) % 8;
    uint8_t z[8];
    rd(z, pad);
    uint64_t c;
    rd(&c, 8);
    if (c != checksum64((const uint8_t*)dst, nbytes))
      throw PsError{PS_EFORMAT, std::string("checksum mismatch in section ") + name};
  };
  h->perm.resize(h->N);
  section(h->perm.data(), 8 * h->N, "perm");
  h->leaf_off.resize(h->nl + 1);
  section(h->leaf_off.data(), 8 * (h->nl + 1), "leaf_off");
  h->leaf_ijk.resize(3 * h->nl);
  section(h->leaf_ijk.data(), 12 * h->nl, "leaf_ijk");
  h->elim.resize(h->nl);
  section(h->elim.data(), 4 * h->nl, "elim_order");
  h->near_list.resize(3 * h->nnear);
  section(h->near_list.data(), 24 * h->nnear, "near_list");
  if (defer_near) {            // read later, only this rank's blocks (load_near)
    h->near_file_off = (int64_t)std::ftell(f);
    const int64_t nb = 16 * h->near_len, pad = (8 - nb % 8) % 8;
    if (std::fseek(f, nb + pad, SEEK_CUR) != 0) throw PsError{PS_EFORMAT, "truncated file"};
    rd(&h->near_file_ck, 8);
  } else {
    near_arena.resize(h->near_len);
    section(near_arena.data(), 16 * h->near_len, "near_arena");
  }
  h->far_list.resize(7 * h->nfar);
  section(h->far_list.data(), 56 * h->nfar, "far_list");
  far_arena.resize(h->far_len);
  section(far_arena.data(), 16 * h->far_len, "far_arena");
  // validation of indices
  if (h->leaf_off[0] != 0 || h->leaf_off[h->nl] != h->N) throw PsError{PS_EFORMAT, "bad leaf_off"};
  for (int64_t l = 0; l < h->nl; ++l)
    if (h->leaf_off[l + 1] <= h->leaf_off[l]) throw PsError{PS_EFORMAT, "empty leaf"};
  std::vector<char> seen(h->N, 0);
  for (int64_t p : h->perm) {
    if (p < 0 || p >= h->N || seen[p]) throw PsError{PS_EFORMAT, "perm is not a permutation"};
    seen[p] = 1;
  }
  std::vector<char> seenl(h->nl, 0);
  for (int32_t l : h->elim) {
    if (l < 0 || l >= h->nl || seenl[l]) throw PsError{PS_EFORMAT, "elim_order is not a permutation"};
    seenl[l] = 1;
  }
  for (int64_t b = 0; b < h->nnear; ++b) {
    int64_t i = h->near_list[3 * b], j = h->near_list[3 * b + 1], o = h->near_list[3 * b + 2];
    if (i < 0 || j < i || j >= h->nl) throw PsError{PS_EFORMAT, "bad near pair"};
    int64_t ni = h->leaf_off[i + 1] - h->leaf_off[i], nj = h->leaf_off[j + 1] - h->leaf_off[j];
    if (o < 0 || o + ni * nj > h->near_len) throw PsError{PS_EFORMAT, "near block out of arena"};
  }
  for (int64_t b = 0; b < h->nfar; ++b) {
    const int64_t* F = &h->far_list[7 * b];
    if (F[0] < 0 || F[1] <= 0 || F[0] + F[1] > h->N || F[2] < 0 || F[3] <= 0 || F[2] + F[3] > h->N ||
        F[5] < 0 || F[6] < 0 || F[6] + F[5] * (F[1] + F[3]) > h->far_len)
      throw PsError{PS_EFORMAT, "bad far block"};
  }
}

// Streamed read of the near arena (deferred by read_file): the whole section is read
// in chunks for its checksum, and only the blocks with keep[b] != 0 are copied into
// `out` (compact, in near-list order; h->near_dev[b] = element offset or -1). A rank
// of a row partition thus never holds the other ranks' near field in host memory.
void load_near(ps_handle* h, const std::vector<char>& keep, std::vector<double2>& out) {
  FILE* f = std::fopen(h->path.c_str(), "rb");
  if (!f) throw PsError{PS_EIO, "cannot reopen " + h->path};
  std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
  if (std::fseek(f, h->near_file_off, SEEK_SET) != 0) throw PsError{PS_EFORMAT, "truncated file"};
  const int64_t nb = h->nnear;
  std::vector<std::array<int64_t, 3>> blk;            // (arena offset, length, block)
  h->near_dev.assign(nb, -1);
  int64_t tot = 0;
  for (int64_t b = 0; b < nb; ++b) {
    if (!keep[b]) continue;
    const int64_t i = h->near_list[3 * b], j = h->near_list[3 * b + 1];
    const int64_t len = (h->leaf_off[i + 1] - h->leaf_off[i]) * (h->leaf_off[j + 1] - h->leaf_off[j]);
    blk.push_back({h->near_list[3 * b + 2], len, b});
    h->near_dev[b] = tot;
    tot += len;
  }
  out.assign(std::max<int64_t>(tot, 1), double2{0.0, 0.0});
  h->near_dev_len = tot;
  std::sort(blk.begin(), blk.end());
  const int64_t CH = 1 << 22;                          // elements per chunk (64 MB)
  std::vector<double2> buf(std::min<int64_t>(CH, std::max<int64_t>(h->near_len, 1)));
  uint64_t ck = 0;
  size_t bi = 0;
  for (int64_t c0 = 0; c0 < h->near_len; c0 += CH) {
    const int64_t n = std::min(CH, h->near_len - c0);
    if (std::fread(buf.data(), 16, (size_t)n, f) != (size_t)n) throw PsError{PS_EFORMAT, "truncated file"};
    const uint8_t* b8 = reinterpret_cast<const uint8_t*>(buf.data());
    const uint64_t w0 = (uint64_t)c0 * 2;              // 8-byte words before this chunk
    for (int64_t q = 0; q < 2 * n; ++q) {
      uint64_t w;
      std::memcpy(&w, b8 + 8 * q, 8);
      ck += w * (2 * (w0 + (uint64_t)q) + 1);
    }
    while (bi < blk.size() && blk[bi][0] + blk[bi][1] <= c0) ++bi;
    for (size_t k = bi; k < blk.size() && blk[k][0] < c0 + n; ++k) {
      const int64_t lo = std::max(blk[k][0], c0), hi = std::min(blk[k][0] + blk[k][1], c0 + n);
      std::copy(buf.data() + (lo - c0), buf.data() + (hi - c0), out.data() + h->near_dev[blk[k][2]] + (lo - blk[k][0]));
    }
  }
  ck ^= (uint64_t)(16 * h->near_len);
  if (ck != h->near_file_ck) throw PsError{PS_EFORMAT, "checksum mismatch in section near_arena"};
}

// Chains of the elimination tree (see ps_handle), bottom-up by position. With a row
// partition (owner != NULL) a chain never crosses an owner change (rank interior /
// separator), so every T_c belongs entirely to one owner class.
void build_chains(ps_handle* h, const std::vector<int32_t>* owner) {
  const int64_t nl = h->nl;
  {
    const int64_t tmax = env_int("PS_TMAX", 4096);
    h->use_chains = env_int("PS_CHAINS", 1) != 0;
    std::vector<int32_t> nch(nl, 0);
    for (int64_t p = 0; p < nl; ++p)
      if (h->parent[p] >= 0) ++nch[h->parent[p]];
    h->chain_of.assign(nl, -1);
    h->cpos.assign(nl, 0);
    h->chains.clear();
    h->ch_U.clear();
    for (int64_t p = 0; p < nl; ++p) {
      if (h->chain_of[p] >= 0) continue;
      std::vector<int32_t> c{(int32_t)p};
      int64_t U = h->nsz[p];
      int32_t q = (int32_t)p;
      while (h->parent[q] >= 0 && nch[h->parent[q]] == 1 && h->chain_of[h->parent[q]] < 0 &&
             U + h->nsz[h->parent[q]] <= tmax && (!owner || (*owner)[h->parent[q]] == (*owner)[q])) {
        q = h->parent[q];
        h->cpos[q] = U;
        U += h->nsz[q];
        c.push_back(q);
      }
      static const int cmin = env_int("PS_CHAIN_MIN", 2);
      if ((int)c.size() < cmin) {                   // too short to pay for a T_c: single nodes
        for (int32_t x : c) {
          h->chain_of[x] = (int32_t)h->chains.size();
          h->cpos[x] = 0;
          h->chains.push_back({x});
          h->ch_U.push_back(h->nsz[x]);
        }
        continue;
      }
      const int32_t id = (int32_t)h->chains.size();
      for (int32_t x : c) h->chain_of[x] = id;
      h->chains.push_back(std::move(c));
      h->ch_U.push_back(U);
    }
    const int64_t nc = (int64_t)h->chains.size();
    h->ch_Toff.assign(nc, -1);
    h->Tlen = 0;
    for (int64_t c = 0; c < nc; ++c)
      if (h->chains[c].size() >= 2) {
        h->ch_Toff[c] = h->Tlen;
        h->Tlen += h->ch_U[c] * h->ch_U[c];
      }
    // chain-graph levels: the parent of a piece's top is the first node of another piece
    std::vector<int32_t> order(nc);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return h->chains[x].back() < h->chains[y].back(); });
    h->ch_height.assign(nc, 0);
    h->ch_depth.assign(nc, 0);
    for (int32_t c : order) {
      const int32_t up = h->parent[h->chains[c].back()];
      if (up >= 0) h->ch_height[h->chain_of[up]] = std::max(h->ch_height[h->chain_of[up]], h->ch_height[c] + 1);
    }
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
      const int32_t up = h->parent[h->chains[*it].back()];
      if (up >= 0) h->ch_depth[*it] = h->ch_depth[h->chain_of[up]] + 1;
    }
    h->max_ch_height = h->max_ch_depth = 0;
    for (int64_t c = 0; c < nc; ++c) {
      h->max_ch_height = std::max(h->max_ch_height, h->ch_height[c]);
      h->max_ch_depth = std::max(h->max_ch_depth, h->ch_depth[c]);
    }
    if (!h->use_chains) {                          // every node its own piece (no T_c)
      h->Tlen = 0;
      std::vector<std::vector<int32_t>> single;
      for (int64_t p = 0; p < nl; ++p) single.push_back({(int32_t)p});
      h->chains.swap(single);
      h->ch_U.assign(nl, 0);
      h->ch_Toff.assign(nl, -1);
      h->ch_height.assign(nl, 0);
      h->ch_depth.assign(nl, 0);
      for (int64_t p = 0; p < nl; ++p) {
        h->chain_of[p] = (int32_t)p;
        h->cpos[p] = 0;
        h->ch_U[p] = h->nsz[p];
        h->ch_height[p] = h->height[p];
        h->ch_depth[p] = h->depth[p];
      }
      h->max_ch_height = h->max_height;
      h->max_ch_depth = h->max_depth;
    }
  }
}

// ------------------------------------------------------------------ symbolic
void build_chains(ps_handle* h, const std::vector<int32_t>* owner);
void symbolic(ps_handle* h) {
  const int64_t nl = h->nl;
  h->pos_of.assign(nl, 0);
  h->leaf_at.assign(nl, 0);
  for (int64_t p = 0; p < nl; ++p) {
    h->leaf_at[p] = h->elim[p];
    h->pos_of[h->elim[p]] = (int32_t)p;
  }
  h->nsz.resize(nl);
  h->eoff.assign(nl + 1, 0);
  for (int64_t p = 0; p < nl; ++p) {
    int32_t l = h->leaf_at[p];
    h->nsz[p] = (int32_t)(h->leaf_off[l + 1] - h->leaf_off[l]);
    h->eoff[p + 1] = h->eoff[p] + h->nsz[p];
  }
  // adjacency (upper, by position) from the near list
  std::vector<std::vector<int32_t>> up(nl);
  bool has_diag_missing = false;
  std::vector<char> diag(nl, 0);
  for (int64_t b = 0; b < h->nnear; ++b) {
    int64_t i = h->near_list[3 * b], j = h->near_list[3 * b + 1];
    h->near_idx[(uint64_t)i * (uint64_t)nl + (uint64_t)j] = b;
    int32_t p = h->pos_of[i], q = h->pos_of[j];
    if (p == q) { diag[p] = 1; continue; }
    if (p > q) std::swap(p, q);
    up[p].push_back(q);
  }
  for (int64_t p = 0; p < nl; ++p) has_diag_missing |= !diag[p];
  if (has_diag_missing) throw PsError{PS_EFORMAT, "near list lacks a diagonal block"};
  // struct(p) = up(p) U (U_children struct(c) \ {p}); parent = min struct(p)
  h->st.assign(nl, {});
  h->parent.assign(nl, -1);
  std::vector<std::vector<int32_t>> children(nl);
  for (int64_t p = 0; p < nl; ++p) {
    std::vector<int32_t> s = up[p];
    for (int32_t c : children[p])
      for (int32_t x : h->st[c])
        if (x != p) s.push_back(x);
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    h->st[p] = std::move(s);
    if (!h->st[p].empty()) {
      h->parent[p] = h->st[p][0];
      children[h->st[p][0]].push_back((int32_t)p);
    }
  }
  // levels: height (forward sweep / setup), depth (backward sweep)
  h->height.assign(nl, 0);
  for (int64_t p = 0; p < nl; ++p)
    if (h->parent[p] >= 0) h->height[h->parent[p]] = std::max(h->height[h->parent[p]], h->height[p] + 1);
  h->depth.assign(nl, 0);
  for (int64_t p = nl - 1; p >= 0; --p)
    if (h->parent[p] >= 0) h->depth[p] = h->depth[h->parent[p]] + 1;
  h->max_height = 0;
  h->max_depth = 0;
  for (int64_t p = 0; p < nl; ++p) {
    h->max_height = std::max(h->max_height, h->height[p]);
    h->max_depth = std::max(h->max_depth, h->depth[p]);
  }
  // panel column offsets, arena layout, gather lists, setup cost
  h->pcol.assign(nl, {});
  h->S.assign(nl, 0);
  h->gath.assign(nl, {});
  h->Woff.assign(nl, 0);
  h->Poff.assign(nl, 0);
  h->Doff.assign(nl, 0);
  int64_t W = 0, P = 0, D = 0;
  h->setup_madds = 0;
  h->alpha_blocks = 0;
  for (int64_t p = 0; p < nl; ++p) {
    int64_t c = 0;
    h->pcol[p].resize(h->st[p].size());
    for (size_t i = 0; i < h->st[p].size(); ++i) {
      h->pcol[p][i] = c;
      c += h->nsz[h->st[p][i]];
      h->gath[h->st[p][i]].push_back({(int32_t)p, (int32_t)i});
    }
    h->S[p] = c;
    h->alpha_blocks += (int64_t)h->st[p].size();
    const int64_t n = h->nsz[p];
    h->Woff[p] = W;
    W += n * (n + c);
    h->Poff[p] = P;
    P += n * c;
    h->Doff[p] = D;
    D += n * n;
    h->setup_madds += (double)n * n * n + (double)n * n * c + 0.5 * (double)n * c * (c + n);
  }
  h->Wlen = W;
  h->Plen = P;
  h->Dlen = D;
  build_chains(h, nullptr);
  // unknown maps
  h->e2mort.resize(h->N);
  h->e2rwg.resize(h->N);
  h->m2e.resize(h->N);
  for (int64_t p = 0; p < nl; ++p) {
    int32_t l = h->leaf_at[p];
    for (int64_t t = 0; t < h->nsz[p]; ++t) {
      int64_t e = h->eoff[p] + t, m = h->leaf_off[l] + t;
      h->e2mort[e] = m;
      h->e2rwg[e] = h->perm[m];
      h->m2e[m] = e;
    }
  }
}

// ------------------------------------------------------------------ row partition
// Row partition of the solve over P ranks (SURVEY §8(e) option 1).
// The elimination tree decouples disjoint subtrees: struct(p) only holds
// ancestors of p, so the forward sweep of a subtree needs nothing from outside
// it, and the backward sweep of a subtree needs only its ancestors. Whole
// subtrees are assigned to ranks ("interior"); the nodes above them
// ("separators") are replicated on every rank. Starting from the roots, the
// heaviest subtree is split (its root becomes a separator) and the resulting
// subtrees are bin-packed (largest first) onto the ranks; the split count that
// minimises max-rank-load + replicated-separator load is kept.
//   owner[p]     : rank owning interior position p, -1 for separators
//   far_owner[p] : rank computing the far-field rows t_p (owner for interior
//                  nodes; separators spread greedily by far-field work)
void partition(const ps_handle* h, int P, std::vector<int32_t>& owner, std::vector<int32_t>& far_owner) {
  const int64_t nl = h->nl;
  owner.assign(nl, 0);
  far_owner.assign(nl, 0);
  if (P <= 1) return;
  // per-position weights ~ operator entries touched per solve (4 sweeps, 2 D^-1; far 2 stages)
  std::vector<double> wn(nl), wf(nl, 0.0);
  for (int64_t p = 0; p < nl; ++p) wn[p] = 4.0 * h->nsz[p] * (double)h->S[p] + 2.0 * h->nsz[p] * (double)h->nsz[p];
  auto leaf_of_m = [&](int64_t m) {
    return (int64_t)(std::upper_bound(h->leaf_off.begin(), h->leaf_off.end(), m) - h->leaf_off.begin()) - 1;
  };
  for (int64_t b = 0; b < h->nfar; ++b) {
    const int64_t* F = &h->far_list[7 * b];
    const int64_t r0 = F[0], m = F[1], c0 = F[2], n = F[3], r = F[5];
    for (int side = 0; side < 2; ++side) {
      const int64_t a0 = side ? c0 : r0, len = side ? n : m, other = side ? m : n;
      for (int64_t l = leaf_of_m(a0); l < nl && h->leaf_off[l] < a0 + len; ++l) {
        const int64_t lo = std::max(a0, h->leaf_off[l]), hi = std::min(a0 + len, h->leaf_off[l + 1]);
        wf[h->pos_of[l]] += (double)(hi - lo) * (double)std::min<int64_t>(2 * r, other);
      }
    }
  }
  std::vector<std::vector<int32_t>> children(nl);
  std::vector<int32_t> roots;
  for (int64_t p = 0; p < nl; ++p) {
    if (h->parent[p] >= 0) children[h->parent[p]].push_back((int32_t)p);
    else roots.push_back((int32_t)p);
  }
  std::vector<double> W(nl);   // subtree weight (children have smaller positions)
  for (int64_t p = 0; p < nl; ++p) W[p] = wn[p] + wf[p];
  for (int64_t p = 0; p < nl; ++p)
    if (h->parent[p] >= 0) W[h->parent[p]] += W[p];
  std::vector<int32_t> subs = roots, sep;
  double sep_near = 0, sep_far = 0;
  double best = 1e300;
  std::vector<int32_t> best_subs, best_sep, best_bin;
  const size_t max_subs = (size_t)(32 * P);
  for (int it = 0; it < 64 * P + 64; ++it) {
    // LPT bin packing of the current subtrees
    std::vector<int32_t> ord = subs;
    std::sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) { return W[x] > W[y] || (W[x] == W[y] && x < y); });
    std::vector<double> load(P, 0.0);
    std::vector<int32_t> bin(nl, -1);
    for (int32_t s : ord) {
      int g = (int)(std::min_element(load.begin(), load.end()) - load.begin());
      load[g] += W[s];
      bin[s] = g;
    }
    const double cost = *std::max_element(load.begin(), load.end()) + sep_near + sep_far / P;
    if (cost < best) {
      best = cost;
      best_subs = subs;
      best_sep = sep;
      best_bin = bin;
    }
    if (subs.size() >= max_subs) break;
    // split the heaviest subtree that has children
    int32_t hv = -1;
    for (int32_t s : subs)
      if (!children[s].empty() && (hv < 0 || W[s] > W[hv])) hv = s;
    if (hv < 0) break;
    subs.erase(std::find(subs.begin(), subs.end(), hv));
    for (int32_t c : children[hv]) subs.push_back(c);
    sep.push_back(hv);
    sep_near += wn[hv];
    sep_far += wf[hv];
  }
  // interior owners: every node of an assigned subtree (children have smaller
  // positions, so a reverse sweep propagates the owner down from the subtree roots)
  owner.assign(nl, -2);
  for (int32_t s : best_sep) owner[s] = -1;
  for (int32_t s : best_subs) owner[s] = best_bin[s];
  for (int64_t p = nl - 1; p >= 0; --p)
    if (owner[p] == -2) owner[p] = owner[h->parent[p]];
  // far rows of the separators: greedy by far work onto the least-loaded rank
  std::vector<double> load(P, 0.0);
  for (int64_t p = 0; p < nl; ++p)
    if (owner[p] >= 0) load[owner[p]] += wn[p] + wf[p];
  std::vector<int32_t> sp_ord;
  for (int64_t p = 0; p < nl; ++p) {
    far_owner[p] = owner[p];
    if (owner[p] < 0) sp_ord.push_back((int32_t)p);
  }
  std::sort(sp_ord.begin(), sp_ord.end(), [&](int32_t x, int32_t y) { return wf[x] > wf[y] || (wf[x] == wf[y] && x < y); });
  for (int32_t p : sp_ord) {
    int g = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    far_owner[p] = g;
    load[g] += wf[p];
  }
}

// Restack the far factors per cluster (DESIGN.md §Far field): block b ~ U V^T
// with rows t = [r0, r0+m), cols s = [c0, c0+n) contributes U^T (r x m) to the
// stack of t and V^T (r x n) to the stack of s. Stage 1 is then one GEMM per
// cluster, S_c w_c, and stage 2 reads U/V rows from the same stacks.
static bool is_identity(const double2* M, int64_t n) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) {
      const double2 v = M[i + j * n];
      if (v.y != 0.0 || v.x != (i == j ? 1.0 : 0.0)) return false;
    }
  return true;
}

void far_layout(ps_handle* h, const std::vector<double2>& far_arena, std::vector<double2>& stacked) {
  std::map<std::pair<int64_t, int64_t>, int64_t> cid;
  auto get = [&](int64_t a, int64_t l) {
    auto it = cid.find({a, l});
    if (it != cid.end()) return it->second;
    int64_t id = (int64_t)h->cl_start.size();
    cid[{a, l}] = id;
    h->cl_start.push_back(a);
    h->cl_len.push_back(l);
    h->cl_sr.push_back(0);
    return id;
  };
  const int64_t nf = h->nfar;
  h->fb_ct.assign(nf, 0); h->fb_cs.assign(nf, 0); h->fb_rbt.assign(nf, 0); h->fb_rbs.assign(nf, 0);
  h->fb_dense.assign(nf, -1);
  // Row partition: a rank keeps only the blocks with a row range (either side) of a leaf
  // whose far-field rows it computes (far_owner); the others are never read there.
  std::vector<char> keep(nf, 1);
  if (h->part_mode) {
    auto leaf_of_m = [&](int64_t m) {
      return (int64_t)(std::upper_bound(h->leaf_off.begin(), h->leaf_off.end(), m) - h->leaf_off.begin()) - 1;
    };
    auto mine = [&](int64_t a0, int64_t len) {
      for (int64_t l = leaf_of_m(a0); l < h->nl && h->leaf_off[l] < a0 + len; ++l)
        if (h->far_owner[h->pos_of[l]] == h->rank) return true;
      return false;
    };
    for (int64_t b = 0; b < nf; ++b) {
      const int64_t* F = &h->far_list[7 * b];
      keep[b] = (mine(F[0], F[1]) || mine(F[2], F[3])) ? 1 : 0;
    }
  }
  // Blocks stored exactly as dense x I (ACA rank cap, R18) are applied as the
  // dense block D (m x n) itself: multiplying by an exact identity is exact, so
  // this only removes work. D lives after the stacks in the same arena.
  std::vector<int64_t> dense_src(nf, -1);   // 0: D = U, 1: D = V^T
  int64_t dense_len = 0;
  for (int64_t b = 0; b < nf; ++b) {
    const int64_t* F = &h->far_list[7 * b];
    const int64_t m = F[1], n = F[3], r = F[5], fo = F[6];
    if (!keep[b]) continue;
    if (r == n && is_identity(&far_arena[fo + m * r], n)) dense_src[b] = 0;
    else if (r == m && is_identity(&far_arena[fo], m)) dense_src[b] = 1;
    if (dense_src[b] >= 0) {
      h->fb_dense[b] = dense_len;
      dense_len += m * n;
    }
  }
  for (int64_t b = 0; b < nf; ++b) {
    const int64_t* F = &h->far_list[7 * b];
    const int64_t t = get(F[0], F[1]), c = get(F[2], F[3]), r = F[5];
    h->fb_ct[b] = t;
    h->fb_cs[b] = c;
    if (dense_src[b] >= 0 || !keep[b]) continue;
    h->fb_rbt[b] = h->cl_sr[t];
    h->cl_sr[t] += r;
    h->fb_rbs[b] = h->cl_sr[c];
    h->cl_sr[c] += r;
  }
  const int64_t nc = (int64_t)h->cl_start.size();
  h->cl_soff.assign(nc, 0);
  int64_t off = 0;
  for (int64_t c = 0; c < nc; ++c) {
    h->cl_soff[c] = off;
    off += h->cl_sr[c] * h->cl_len[c];
  }
  h->stack_len = off;
  for (int64_t b = 0; b < nf; ++b)
    if (h->fb_dense[b] >= 0) h->fb_dense[b] += off;
  stacked.assign(std::max<int64_t>(off + dense_len, 1), double2{0.0, 0.0});
  for (int64_t b = 0; b < nf; ++b) {
    const int64_t* F = &h->far_list[7 * b];
    const int64_t m = F[1], n = F[3], r = F[5], fo = F[6];
    if (!keep[b]) continue;
    if (dense_src[b] == 0) {          // D = U (m x n)
      std::copy(&far_arena[fo], &far_arena[fo] + m * n, &stacked[h->fb_dense[b]]);
      continue;
    }
    if (dense_src[b] == 1) {          // D = V^T: D(i, k) = V(k, i), V n x m
      for (int64_t k = 0; k < n; ++k)
        for (int64_t i = 0; i < m; ++i) stacked[h->fb_dense[b] + i + k * m] = far_arena[fo + m * r + k + i * n];
      continue;
    }
    const int64_t t = h->fb_ct[b], c = h->fb_cs[b];
    const int64_t srt = h->cl_sr[t], src = h->cl_sr[c];
    for (int64_t j = 0; j < r; ++j) {
      for (int64_t k = 0; k < m; ++k)   // U(k, j) -> S_t(rb_t + j, k)
        stacked[h->cl_soff[t] + (h->fb_rbt[b] + j) + k * srt] = far_arena[fo + k + j * m];
      for (int64_t k = 0; k < n; ++k)   // V(k, j) -> S_s(rb_s + j, k)
        stacked[h->cl_soff[c] + (h->fb_rbs[b] + j) + k * src] = far_arena[fo + m * r + k + j * n];
    }
  }
}

int64_t wcol(const ps_handle* h, int32_t p, int32_t j) {
  // column offset of block j inside W_p = [Z~_pp | Z~_p,struct(p)]
  if (j == p) return 0;
  const auto& s = h->st[p];
  auto it = std::lower_bound(s.begin(), s.end(), j);
  if (it == s.end() || *it != j) throw PsError{PS_ECUDA, "internal: struct lookup failed"};
  return h->nsz[p] + h->pcol[p][it - s.begin()];
}

// ------------------------------------------------------------------ setup
// Setup tables of ONE elimination level (built, launched and freed level by
// level, so the host/device work lists never hold more than one level: C5's
// whole-setup lists would be several GB).
struct SetupLevel {
  Table asmb, panel;
  DevBuf<int32_t> d_ids, d_sz;
  DevBuf<int64_t> d_src, d_ld, d_dst;
  std::vector<int32_t> ids, sz;                       // host side of the inverse launch
  std::vector<int64_t> src, ld, dst;
  int64_t nlev = 0;
  int maxn = 0;
  double t_upload = 0;
  void reset() {
    asmb.reset_keep_device();
    panel.reset_keep_device();
    asmb.S = panel.S = nullptr;
    nlev = 0;
    maxn = 0;
  }
  // take the host tables built (by a worker thread) into `o`, keeping this level's device buffers
  void adopt(SetupLevel& o) {
    auto keep = [](Table& dst, Table& src) {
      src.d_tasks = std::move(dst.d_tasks); src.d_terms = std::move(dst.d_terms); src.d_work = std::move(dst.d_work);
      src.d_counters = std::move(dst.d_counters); src.d_partial = std::move(dst.d_partial);
      dst = std::move(src);
    };
    keep(asmb, o.asmb);
    keep(panel, o.panel);
    ids.swap(o.ids); sz.swap(o.sz); src.swap(o.src); ld.swap(o.ld); dst.swap(o.dst);
    nlev = o.nlev;
    maxn = o.maxn;
  }
};

// mode 0: every descendant's update, near-block init (the whole tree on one rank, or a
//         rank's own interior); mode 1: separator rows, updates from this rank's own
//         interior only, near-block init where this rank holds the block (rank 0), no
//         panels (phase B of the sharded setup); mode 2: separator rows, updates from
//         separator descendants only, added in place to the rank-summed W (phase C).
void build_setup_level(ps_handle* h, const std::vector<int32_t>& leaves, SetupLevel& sp, int mode = 0) {
  const int64_t nl = h->nl;
  if (mode == 2) sp.asmb.S = h->d_W.p;
  {
    for (int32_t p : leaves) {
      const int64_t np_ = h->nsz[p];
      const int32_t lp = h->leaf_at[p];
      // targets j in {p} U struct(p): W_pj = Z_pj + sum_d alpha_dp^T W_dj
      std::vector<int32_t> targets;
      targets.push_back(p);
      for (int32_t j : h->st[p]) targets.push_back(j);
      // terms of each target, from descendants d with p in struct(d), in increasing d
      std::map<int32_t, std::vector<std::array<int64_t, 3>>> terms_of;  // j -> (oA, oB, nd)
      for (auto [d, idx] : h->gath[p]) {
        if (mode == 1 && h->owner[d] != h->rank) continue;
        if (mode == 2 && h->owner[d] >= 0) continue;
        const int64_t nd = h->nsz[d];
        const auto& sd = h->st[d];
        const int64_t oA = h->Poff[d] + h->pcol[d][idx] * nd;   // alpha_dp (nd x np), transposed view
        for (size_t jj = idx; jj < sd.size(); ++jj) {
          const int64_t oB = h->Woff[d] + (nd + h->pcol[d][jj]) * nd;  // W_dj (nd x nj)
          terms_of[sd[jj]].push_back({oA, oB, nd});
        }
      }
      for (int32_t j : targets) {
        const int64_t nj = h->nsz[j];
        const int32_t lj = h->leaf_at[j];
        // near block init (file stores i <= j by leaf id; Z_ji = Z_ij^T)
        int64_t oI = -1, sIi = 0, sIc = 0;
        uint64_t key_a = (uint64_t)std::min(lp, lj) * (uint64_t)nl + (uint64_t)std::max(lp, lj);
        auto it = h->near_idx.find(key_a);
        if (it != h->near_idx.end() && mode != 2) {
          const int64_t* nb = &h->near_list[3 * it->second];
          const int64_t n_first = h->leaf_off[nb[0] + 1] - h->leaf_off[nb[0]];
          oI = h->near_dev.empty() ? nb[2] : h->near_dev[it->second];   // -1: block not held here
          if (lp == nb[0]) { sIi = 1; sIc = n_first; }   // Z_{lp,lj} as stored
          else { sIi = n_first; sIc = 1; }               // transpose view
        }
        const int64_t oO = h->Woff[p] + wcol(h, p, j) * np_;
        if (mode == 2) { oI = oO; sIi = 1; sIc = np_; }  // in place: the rank-summed W_pj
        int32_t t = sp.asmb.add_task(oO, 1, np_, oI, sIi, sIc, (int)np_, (int)nj, +1);
        if (mode == 2) sp.asmb.tasks[t].osel |= 2;
        auto tj = terms_of.find(j);
        if (tj != terms_of.end())
          for (auto& c : tj->second) sp.asmb.add_term(t, c[0], c[2], 1, c[1], 1, c[2], (int)c[2]);
        sp.asmb.tile(t);
      }
    }
    sp.asmb.close_batch();
    // panel: P_p = -Dinv_p W_p[:, n_p:]
    for (int32_t p : leaves) {
      const int64_t np_ = h->nsz[p];
      if (h->S[p] == 0 || mode == 1) continue;
      int32_t t = sp.panel.add_task(h->Poff[p], 1, np_, -1, 0, 0, (int)np_, (int)h->S[p], -1);
      sp.panel.add_term(t, h->Doff[p], 1, np_, h->Woff[p] + np_ * np_, 1, np_, (int)np_);
      sp.panel.tile(t);
    }
    sp.panel.close_batch();
  }
  sp.ids = leaves;
  sp.sz.clear(); sp.src.clear(); sp.ld.clear(); sp.dst.clear();
  for (int32_t p : leaves) {
    sp.sz.push_back(h->nsz[p]);
    sp.src.push_back(h->Woff[p]);
    sp.ld.push_back(h->nsz[p]);
    sp.dst.push_back(h->Doff[p]);
    sp.maxn = std::max(sp.maxn, h->nsz[p]);
  }
  sp.nlev = (int64_t)leaves.size();
}

// Device side of a level: its tables and inverse lists, through the pinned ring on the upload
// stream u (the caller orders u after the kernels that last used these buffers)
void upload_setup_level(ps_handle* h, SetupLevel& sp, cudaStream_t u) {
  const auto tu0 = std::chrono::steady_clock::now();
  sp.asmb.upload(u, &h->ring);
  sp.panel.upload(u, &h->ring);
  sp.d_ids.upload(sp.ids, u, &h->ring);
  sp.d_sz.upload(sp.sz, u, &h->ring);
  sp.d_src.upload(sp.src, u, &h->ring);
  sp.d_ld.upload(sp.ld, u, &h->ring);
  sp.d_dst.upload(sp.dst, u, &h->ring);
  sp.t_upload = std::chrono::duration<double>(std::chrono::steady_clock::now() - tu0).count();
}

// Upload the restacked far factors (once) and point Fbase at them.
void ensure_far(ps_handle* h, cudaStream_t s) {
  if (!h->d_farbuf.p) {
    h->d_farbuf.alloc(std::max<int64_t>((int64_t)h->far_host.size(), 1));
    if (!h->far_host.empty())
      CK(cudaMemcpyAsync(h->d_farbuf.p, h->far_host.data(), sizeof(double2) * h->far_host.size(),
                         cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    std::vector<double2>().swap(h->far_host);
  }
  h->d_far.p = h->d_farbuf.p;
  h->Fbase = (int64_t)(h->d_farbuf.p - h->d_op.p);
}

// One-pass far apply of narrow solves (far1p; ps_internal.h): the block,
// item and piece tables (once per handle) and the FB arena (every far factor copied
// rows-major out of the stacks by one gather launch). Returns false (and the program keeps
// the two-stage far field) when a block's rank exceeds F1P_RMAX or on a row-partition rank.
bool build_far1p(ps_handle* h, cudaStream_t s) {
  if (h->f1p_state) return h->f1p_state > 0;
  h->f1p_state = -1;
  // PS_FAR1P: 1 always, 0 never, -1 (default) where it pays: splitting the program at the far
  // field costs the overlap of the far products with the sweeps' dependency bubbles and a
  // launch gap, so the one-pass apply is taken when the far factors are large (>= 1 GiB) and a
  // large share (>= 30 %) of the sweeps' operator (C4: 2.6 GB vs 4 x 1.1 GB: 3.75 vs 4.42 ms per
  // 1-RHS solve; C3's 0.4 GB / C2's 0.3 GB far fields measured equal or slower)
  const int mode = env_int("PS_FAR1P", -1);
  if (h->part_mode || mode == 0) return false;
  const int64_t nf = h->nfar, nl = h->nl;
  if (mode < 0) {
    double far_el = 0;
    for (int64_t b = 0; b < nf; ++b) {
      const int64_t* F = &h->far_list[7 * b];
      far_el += h->fb_dense[b] >= 0 ? (double)F[1] * F[3] : (double)(F[1] + F[3]) * F[5];
    }
    if (far_el < (double)(1 << 26) || far_el < 0.3 * 4.0 * (double)h->Plen) return false;
  }
  for (int64_t b = 0; b < nf; ++b) {
    const int64_t* F = &h->far_list[7 * b];
    const int64_t r = F[5];
    if (r == 0) continue;
    if (h->fb_dense[b] >= 0 ? std::min(F[1], F[3]) > F1P_RMAX : r > F1P_RMAX) return false;
  }
  auto leaf_of_pos = [&](int64_t m) {
    return (int64_t)(std::upper_bound(h->leaf_off.begin(), h->leaf_off.end(), m) - h->leaf_off.begin()) - 1;
  };
  // elements per item (staged); PS_F1P_CHUNK < F1P_CH (tests) cuts more blocks into chunks
  const int64_t CH = std::max<int64_t>(F1P_RMAX, std::min<int64_t>(F1P_CH, env_int("PS_F1P_CHUNK", F1P_CH)));
  // blocks: small ones first in block order (packed), then the big ones
  struct Src { int64_t src, ss, sk; };
  std::vector<FBlk> small, big;
  std::vector<std::array<Src, 2>> src_small, src_big;
  int64_t prow = 0;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> leaf_pieces(nl);   // (order key, piece row)
  auto add_piece = [&](int64_t x0, int64_t len, int64_t y0) {
    for (int64_t l = leaf_of_pos(x0); l < nl && h->leaf_off[l] < x0 + len; ++l)
      leaf_pieces[l].push_back({y0 + (h->leaf_off[l] - x0), 0});
  };
  double alg = 0, fl1 = 0;
  for (int64_t b = 0; b < nf; ++b) {
    const int64_t* F = &h->far_list[7 * b];
    const int64_t r0 = F[0], m = F[1], c0 = F[2], n = F[3], r = F[5];
    if (r == 0) continue;
    FBlk k{};
    std::array<Src, 2> sr{};
    if (h->fb_dense[b] >= 0) {
      const int64_t D = h->Fbase + h->fb_dense[b];      // m x n column-major
      k.dense = 1;
      k.o2 = -1;
      k.n2 = 0;
      if (m <= n) {   // G = D^T: rows = the column cluster (n), row length m
        k.n1 = (int32_t)n; k.r = (int32_t)m; k.x1 = c0; k.x2 = r0;
        sr[0] = {D, m, 1};
      } else {        // G = D: rows = the row cluster (m), row length n
        k.n1 = (int32_t)m; k.r = (int32_t)n; k.x1 = r0; k.x2 = c0;
        sr[0] = {D, 1, m};
      }
      k.y1 = prow; prow += k.n1;
      k.y2 = prow; prow += k.r;
      alg += 16.0 * m * n;
      fl1 += 16.0 * m * n;   // two complex products per entry, 8 flop each
    } else {
      const int64_t ct = h->fb_ct[b], cs = h->fb_cs[b];
      const Src U{h->Fbase + h->cl_soff[ct] + h->fb_rbt[b], h->cl_sr[ct], 1};
      const Src V{h->Fbase + h->cl_soff[cs] + h->fb_rbs[b], h->cl_sr[cs], 1};
      const bool u_first = m <= n;                       // F1 = the shorter factor (read twice if big)
      k.r = (int32_t)r;
      k.n1 = (int32_t)(u_first ? m : n); k.x1 = u_first ? r0 : c0;
      k.n2 = (int32_t)(u_first ? n : m); k.x2 = u_first ? c0 : r0;
      sr[0] = u_first ? U : V;
      sr[1] = u_first ? V : U;
      k.y1 = prow; prow += k.n1;
      k.y2 = prow; prow += k.n2;
      alg += 16.0 * (m + n) * r;
      fl1 += 16.0 * (m + n) * r;
    }
    const int64_t elems = (int64_t)(k.n1 + k.n2) * k.r;
    (elems <= CH ? small : big).push_back(k);
    (elems <= CH ? src_small : src_big).push_back(sr);
  }
  std::vector<FBlk> blk;
  std::vector<FCopy> runs;
  int64_t fb = 0;
  auto place = [&](FBlk& k, const std::array<Src, 2>& sr) {
    k.o1 = h->FBbase + fb;
    runs.push_back({k.o1, sr[0].src, sr[0].ss, sr[0].sk, k.n1, k.r});
    fb += (int64_t)k.n1 * k.r;
    if (!k.dense) {
      k.o2 = h->FBbase + fb;
      runs.push_back({k.o2, sr[1].src, sr[1].ss, sr[1].sk, k.n2, k.r});
      fb += (int64_t)k.n2 * k.r;
    }
  };
  // FB layout: the small blocks (candidates for packs) first, in block order, then the big ones
  for (size_t i = 0; i < small.size(); ++i) {
    FBlk k = small[i];
    place(k, src_small[i]);
    blk.push_back(k);
  }
  h->f1p_nsmall = (int64_t)small.size();
  for (size_t i = 0; i < big.size(); ++i) {
    FBlk k = big[i];
    place(k, src_big[i]);
    blk.push_back(k);
  }
  // gathered x arena XA: per block (FB order) its x1 rows then its x2 rows, as elimination rows
  h->f1p_xmap.clear();
  for (FBlk& k : blk) {
    k.xa = (int64_t)h->f1p_xmap.size();
    for (int32_t i = 0; i < k.n1; ++i) h->f1p_xmap.push_back(h->m2e[k.x1 + i]);
    const int32_t n2x = k.dense ? k.r : k.n2;
    for (int32_t i = 0; i < n2x; ++i) h->f1p_xmap.push_back(h->m2e[k.x2 + i]);
  }
  h->f1p_blk = std::move(blk);
  h->f1p_len = fb;
  h->f1p_prows = prow;
  h->f1p_alg_bytes = alg;
  h->f1p_alg_flops1 = fl1;
  h->f1p_ch = CH;
  // per Morton leaf: its pieces in block order (the fixed summation order)
  for (const FBlk& k : h->f1p_blk) {
    add_piece(k.x1, k.n1, k.y1);
    add_piece(k.x2, k.dense ? k.r : k.n2, k.y2);
  }
  h->f1p_lptr.assign(nl + 1, 0);
  h->f1p_poff.clear();
  h->f1p_lrow.assign(nl, 0);
  h->f1p_lsz.assign(nl, 0);
  for (int64_t l = 0; l < nl; ++l) {
    for (auto& pc : leaf_pieces[l]) h->f1p_poff.push_back(pc.first);
    h->f1p_lptr[l + 1] = (int64_t)h->f1p_poff.size();
    h->f1p_lrow[l] = h->eoff[h->pos_of[l]];
    h->f1p_lsz[l] = (int32_t)(h->leaf_off[l + 1] - h->leaf_off[l]);
  }
  if (!g_host_only) {
    h->d_fb.alloc(std::max<int64_t>(fb, 1));
    // the FB arena is addressed from the operator base like every other operator region
    const int64_t shift = (int64_t)(h->d_fb.p - h->d_op.p) - h->FBbase;
    for (FBlk& k : h->f1p_blk) { k.o1 += shift; if (k.o2 >= 0) k.o2 += shift; }
    for (FCopy& c : runs) c.dst += shift;
    h->FBbase += shift;
    DevBuf<FCopy> d_runs;
    d_runs.upload(runs, s);
    launch_fb_gather((int64_t)runs.size(), d_runs.p, h->d_op.p, s);
    CK(cudaGetLastError());
    h->d_f1p_xmap.upload(h->f1p_xmap, s);
    h->d_f1p_lptr.upload(h->f1p_lptr, s);
    h->d_f1p_poff.upload(h->f1p_poff, s);
    h->d_f1p_lrow.upload(h->f1p_lrow, s);
    h->d_f1p_lsz.upload(h->f1p_lsz, s);
    CK(cudaStreamSynchronize(s));
  }
  h->f1p_state = 1;
  return true;
}

// Per-plan far1p work for nrhs R (build_far1p made the blocks): packs of consecutive small
// blocks (<= CH factor elements, <= F1P_XCH / R staged x rows, <= F1P_PACK blocks) and one unit per
// other block, cut into row chunks (<= CH elements and <= F1P_XCH / R x rows each): F1 chunks,
// F2 chunks, F1 chunks again (dense: G chunks). Units are taken from a ticket, the big ones
// first (largest first: the tail of the launch is packs).
void build_far1p_items(const ps_handle* h, SolvePlan& sp, int64_t R) {
  const int64_t CH = h->f1p_ch, XR = F1P_XCH / R;
  std::vector<FBlk> blk = h->f1p_blk;
  std::vector<std::vector<FItem>> bigu;                   // per big unit: its items
  std::vector<int64_t> bigsz;
  std::vector<FItem> packs;
  auto xrows = [](const FBlk& k) { return (int64_t)k.n1 + (k.dense ? k.r : k.n2); };
  auto add_big = [&](int32_t id) {
    FBlk& k = blk[id];
    const int64_t cap = k.dense ? XR - k.r : XR;         // dense chunks also stage the r column rows
    const int32_t hr = (int32_t)std::max<int64_t>(1, std::min<int64_t>(CH / k.r, cap));
    k.nc1 = (k.n1 + hr - 1) / hr;
    k.nc2 = k.dense ? 0 : (k.n2 + hr - 1) / hr;
    k.xo1 = k.xo2 = 0;
    std::vector<FItem> its;
    // chunk c of a side: factor rows [a0, a1) and (except the F1-again pass) their x rows
    auto chunk = [&](int kind, int64_t o, int64_t xa, int32_t c, int32_t a0, int32_t a1) {
      FItem it{};
      it.off = o + (int64_t)a0 * k.r;
      it.len = (a1 - a0) * k.r;
      it.kind = kind; it.b = id; it.nb = c; it.a0 = a0; it.a1 = a1;
      if (kind != 3) { it.xa = xa + a0; it.xn = a1 - a0; }
      if (kind == 4) { it.xa2 = k.xa + k.n1; it.xn2 = k.r; }
      its.push_back(it);
    };
    for (int32_t c = 0; c < k.nc1; ++c)
      chunk(k.dense ? 4 : 1, k.o1, k.xa, c, c * hr, std::min(k.n1, (c + 1) * hr));
    for (int32_t c = 0; c < k.nc2; ++c) chunk(2, k.o2, k.xa + k.n1, c, c * hr, std::min(k.n2, (c + 1) * hr));
    if (!k.dense)
      for (int32_t c = 0; c < k.nc1; ++c) chunk(3, k.o1, k.xa, c, c * hr, std::min(k.n1, (c + 1) * hr));
    bigsz.push_back((int64_t)(k.n1 + k.n2) * k.r);
    bigu.push_back(std::move(its));
  };
  {
    int64_t p0 = -1, plen = 0, px = 0;
    int32_t pb = 0, pnb = 0;
    auto flush = [&] {
      if (pnb > 0) {
        FItem it{};
        it.off = p0; it.len = (int32_t)plen; it.kind = 0; it.b = pb; it.nb = pnb;
        it.a0 = (int32_t)px;                                // x rows (consecutive blocks: one XA range)
        it.xa = blk[pb].xa; it.xn = (int32_t)px;
        packs.push_back(it);
      }
      pnb = 0; plen = 0; px = 0;
    };
    for (int64_t i = 0; i < h->f1p_nsmall; ++i) {
      FBlk& k = blk[i];
      const int64_t e = (int64_t)(k.n1 + k.n2) * k.r, xr = xrows(k);
      if (xr > XR) {                                     // its x rows do not fit a stage: chunked
        flush();
        add_big((int32_t)i);
        continue;
      }
      if (plen + e > CH || px + xr > XR || pnb == F1P_PACK) flush();
      if (pnb == 0) { p0 = k.o1; pb = (int32_t)i; }
      k.xo1 = (int32_t)px;
      k.xo2 = (int32_t)(px + k.n1);
      px += xr;
      plen += e;
      ++pnb;
    }
    flush();
  }
  for (int64_t i = h->f1p_nsmall; i < (int64_t)blk.size(); ++i) add_big((int32_t)i);
  std::vector<int64_t> ord(bigu.size());
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return bigsz[x] > bigsz[y]; });
  sp.f1p_item.clear();
  sp.f1p_unit.clear();
  for (int64_t u : ord) {
    sp.f1p_unit.push_back(FUnit{(int64_t)sp.f1p_item.size(), (int32_t)bigu[u].size(), 0});
    sp.f1p_item.insert(sp.f1p_item.end(), bigu[u].begin(), bigu[u].end());
  }
  // packs: F1P_PACKS_PER_UNIT consecutive packs per ticket (the producer loads a unit's
  // descriptors in one batch; a ticket per pack would put a descriptor round trip on every fill)
  static const int ppu = std::max(1, env_int("PS_F1P_PACKS_PER_UNIT", 8));
  for (size_t i = 0; i < packs.size(); i += ppu) {
    const int n = (int)std::min<size_t>(ppu, packs.size() - i);
    sp.f1p_unit.push_back(FUnit{(int64_t)sp.f1p_item.size(), n, 0});
    sp.f1p_item.insert(sp.f1p_item.end(), packs.begin() + i, packs.begin() + i + n);
  }
  sp.f1p_blk = std::move(blk);
}

// T_c = (I - A_c^T)^{-1} of every chain piece with L >= 2 (see ps_handle): the
// forward sweep (Eq. 24) restricted to the piece, applied to the identity:
//   X_i = delta_i + sum_{k < i, p_i in struct(p_k)} alpha_{p_k p_i}^T X_k,
// row block i of T_c = X_i (columns beyond the diagonal block stay 0). One
// dataflow launch; pieces are independent, hops within a piece are ordered.
void chain_setup(ps_handle* h, cudaStream_t s) {
  if (h->Tlen == 0) return;
  // T lives in its own allocation: its rows are addressed through the table's
  // scratch base (offsets >= 0; a negative offset would read as "no init")
  double2* Tp = h->d_T.p;
  CK(cudaMemsetAsync(Tp, 0, sizeof(double2) * h->Tlen, s));
  std::vector<int64_t> ones;
  Table Tt;
  Tt.S = Tp;
  std::vector<int32_t> tk(h->nl, -1);
  const int64_t Pb = h->Pbase;
  for (size_t c = 0; c < h->chains.size(); ++c) {
    if (h->ch_Toff[c] < 0) continue;
    const int64_t U = h->ch_U[c], To = h->ch_Toff[c];
    for (int64_t i = 0; i < U; ++i) ones.push_back(To + i + i * U);
    for (int32_t p : h->chains[c]) {
      const int64_t np_ = h->nsz[p], cp = h->cpos[p];
      int32_t t = Tt.add_task(To + cp, 1, U, To + cp, 1, U, (int)np_, (int)(cp + np_), +1);
      Tt.tasks[t].osel = 1 | 2;                      // O and I in T (scratch base)
      for (auto [d, idx] : h->gath[p]) {
        if (h->chain_of[d] != (int32_t)c) continue;
        const int64_t nd = h->nsz[d];
        Tt.add_term(t, Pb + h->Poff[d] + h->pcol[d][idx] * nd, nd, 1, To + h->cpos[d], 1, U, (int)nd, tk[d], 1);
      }
      Tt.tile(t, -1, 8);
      tk[p] = t;
    }
  }
  Tt.close_batch();
  Tt.upload(s);
  DevBuf<int64_t> d_ones;
  d_ones.upload(ones, s);
  launch_set_ones(Tp, d_ones.p, (int64_t)ones.size(), s);
  Tt.launch_all(h->d_op.p, h->d_op.p, h->d_op.p, h->d_op.p, s);
  CK(cudaStreamSynchronize(s));
}

// Chain-aware sweeps. Pieces are processed in chain-graph order
// (forward: by chain height; backward: by chain depth). A single-node piece is
// an ordinary gather task. A piece with L >= 2 is two stages:
//   forward   E_i: e_{p_i} = y_{p_i} + sum_{d outside} alpha_{d p_i}^T y_d   (-> scratch)
//             Y_i: y_{p_i} = sum_{j <= i} T_c[i, j] e_{p_j}
//   backward  F_i: f_{p_i} = v_{p_i} + sum_{j outside} alpha_{p_i j} w_j      (-> scratch)
//             W_i: w_{p_i} = sum_{j >= i} T_c[j, i]^T f_{p_j}
// so a piece costs 2 dependent hops instead of L. Exact reformulation of
// Eqs. 24 / 26: T_c is the piece's product of the elementary factors (Eq. 15).
void build_chain_sweeps(ps_handle* h, SolvePlan& sp, int64_t R, int narrow, int resident) {
  const int64_t nl = h->nl, nc = (int64_t)h->chains.size();
  const int64_t Pb = h->Pbase, Tb = h->Tbase;
  sp.fwd.S = sp.bwd.S = sp.sc.p;
  sp.fwd.early_keys = sp.bwd.early_keys = env_int("PS_EARLY", 1) != 0;
  // split-K chunk size per stage: ~ipc items per resident CTA, clamped to
  // [2, maxs] k-steps (a stage lasts as long as its longest item)
  static const int maxs = env_int("PS_SWEEP_MAXSTEPS", 16), ipc = env_int("PS_SWEEP_IPC", 2);
  auto steps_of = [&](const std::vector<std::pair<int64_t, int64_t>>& mk) {   // (m, K) of a stage's tasks
    if (narrow) {   // operator streaming: enough items per stage to occupy every CTA
      static const int nadapt = env_int("PS_NARROW_ADAPT", 1);
      if (!nadapt) return NARROW_STEPS();
      double ks = 0;
      for (auto [m, K] : mk) ks += std::ceil((double)m / mode_rows(narrow)) * std::ceil((double)K / GM_KC);
      return std::max(2, std::min(NARROW_STEPS(), (int)std::ceil(ks / (double)resident)));
    }
    double ks = 0;
    for (auto [m, K] : mk) ks += std::ceil((double)m / GM_MT) * std::ceil((double)R / GM_NT) * std::ceil((double)K / GM_KC);
    return std::max(2, std::min(maxs, (int)std::ceil(ks / ((double)ipc * resident))));
  };
  // ticket order: (stage + column tile * stagger), so the column tiles enter the
  // stage sequence staggered and the window of fetched items holds ready work
  static const int stag_pct = env_int("PS_STAGGER", 0);
  const int ntw = narrow ? GN_NT : GM_NT;
  const int nnt = (int)((R + ntw - 1) / ntw);
  const double nst_f = 2.0 * (h->max_ch_height + 1), nst_b = 2.0 * (h->max_ch_depth + 1);
  sp.fwd.key_stagger = nnt > 1 ? 0.01 * stag_pct * nst_f / nnt : 0.0;
  sp.bwd.key_stagger = nnt > 1 ? 0.01 * stag_pct * nst_b / nnt : 0.0;
  double stage = 0;
  auto by_height = [&](const std::vector<std::pair<int32_t, int32_t>>& gl) {
    auto v = gl;
    std::stable_sort(v.begin(), v.end(), [&](const std::pair<int32_t, int32_t>& x, const std::pair<int32_t, int32_t>& y) {
      return h->height[x.first] < h->height[y.first];
    });
    return v;
  };
  std::vector<std::vector<int32_t>> lev_f(h->max_ch_height + 1), lev_b(h->max_ch_depth + 1);
  for (int64_t c = 0; c < nc; ++c) {
    lev_f[h->ch_height[c]].push_back((int32_t)c);
    lev_b[h->ch_depth[c]].push_back((int32_t)c);
  }
  // ---- forward sweep (in place on v; e in scratch) ----
  std::vector<int32_t> yt(nl, -1), et(nl, -1);
  for (const auto& cl : lev_f) {
    std::vector<std::pair<int64_t, int64_t>> mk;
    for (int32_t c : cl)
      for (int32_t p : h->chains[c]) {
        int64_t K = 0;
        for (auto [d, idx] : h->gath[p])
          if (h->chain_of[d] != c) K += h->nsz[d];
        mk.push_back({h->nsz[p], K});
      }
    const int stpE = steps_of(mk);
    sp.fwd.key_base = stage++;
    for (int32_t c : cl) {
      const bool single = h->chains[c].size() == 1;
      for (int32_t p : h->chains[c]) {
        std::vector<std::pair<int32_t, int32_t>> gl;
        for (auto [d, idx] : h->gath[p])
          if (h->chain_of[d] != c) gl.push_back({d, idx});
        if (single && gl.empty()) continue;          // y_p = b_p: nothing to do
        const int64_t np_ = h->nsz[p];
        int32_t t = sp.fwd.add_task(h->eoff[p] * R, R, 1, h->eoff[p] * R, R, 1, (int)np_, (int)R, +1);
        if (!single) sp.fwd.tasks[t].osel = 1;        // e_p -> scratch
        for (auto [d, idx] : by_height(gl)) {
          const int64_t nd = h->nsz[d];
          sp.fwd.add_term(t, Pb + h->Poff[d] + h->pcol[d][idx] * nd, nd, 1, h->eoff[d] * R, R, 1, (int)nd, yt[d]);
        }
        sp.fwd.tile(t, -1, stpE);
        (single ? yt : et)[p] = t;
      }
    }
    mk.clear();
    for (int32_t c : cl)
      if (h->chains[c].size() > 1)
        for (int32_t p : h->chains[c]) mk.push_back({h->nsz[p], h->cpos[p]});
    const int stpY = steps_of(mk);
    sp.fwd.key_base = stage++;
    for (int32_t c : cl) {
      if (h->chains[c].size() == 1) continue;
      const int64_t U = h->ch_U[c], To = Tb + h->ch_Toff[c];
      for (size_t i = 0; i < h->chains[c].size(); ++i) {
        const int32_t p = h->chains[c][i];
        const int64_t np_ = h->nsz[p];
        int32_t t = sp.fwd.add_task(h->eoff[p] * R, R, 1, h->eoff[p] * R, R, 1, (int)np_, (int)R, +1);
        sp.fwd.tasks[t].osel = 2;                     // init e_p (T_c[i, i] = I) from scratch
        sp.fwd.tasks[t].idep = et[p];
        for (size_t j = 0; j < i; ++j) {
          const int32_t q = h->chains[c][j];
          sp.fwd.add_term(t, To + h->cpos[p] + h->cpos[q] * U, 1, U, h->eoff[q] * R, R, 1, (int)h->nsz[q], et[q], 1);
        }
        sp.fwd.tile(t, 0, stpY);
        yt[p] = t;
      }
    }
  }
  sp.fwd.sort_close_bounded();
  stage = 0;
  // ---- backward sweep (O = out, I = in, B = out; f in scratch) ----
  std::vector<int32_t> wt(nl, -1), ft(nl, -1);
  for (const auto& cl : lev_b) {
    std::vector<std::pair<int64_t, int64_t>> mk;
    for (int32_t c : cl)
      for (int32_t p : h->chains[c]) {
        int64_t K = 0;
        for (int32_t j : h->st[p])
          if (h->chain_of[j] != c) K += h->nsz[j];
        mk.push_back({h->nsz[p], K});
      }
    const int stpF = steps_of(mk);
    sp.bwd.key_base = stage++;
    for (int32_t c : cl) {
      const bool single = h->chains[c].size() == 1;
      for (int32_t p : h->chains[c]) {
        const int64_t np_ = h->nsz[p];
        int32_t t = sp.bwd.add_task(h->eoff[p] * R, R, 1, h->eoff[p] * R, R, 1, (int)np_, (int)R, +1);
        if (!single) sp.bwd.tasks[t].osel = 1;        // f_p -> scratch
        for (size_t i = 0; i < h->st[p].size(); ++i) {
          const int32_t j = h->st[p][i];
          if (h->chain_of[j] == c) continue;
          sp.bwd.add_term(t, Pb + h->Poff[p] + h->pcol[p][i] * np_, 1, np_, h->eoff[j] * R, R, 1, (int)h->nsz[j], wt[j]);
        }
        sp.bwd.tile(t, +1, stpF);
        (single ? wt : ft)[p] = t;
      }
    }
    mk.clear();
    for (int32_t c : cl)
      if (h->chains[c].size() > 1)
        for (int32_t p : h->chains[c]) mk.push_back({h->nsz[p], h->ch_U[c] - h->cpos[p] - h->nsz[p]});
    const int stpW = steps_of(mk);
    sp.bwd.key_base = stage++;
    for (int32_t c : cl) {
      if (h->chains[c].size() == 1) continue;
      const int64_t U = h->ch_U[c], To = Tb + h->ch_Toff[c];
      const auto& ch = h->chains[c];
      for (size_t i = 0; i < ch.size(); ++i) {
        const int32_t p = ch[i];
        const int64_t np_ = h->nsz[p];
        int32_t t = sp.bwd.add_task(h->eoff[p] * R, R, 1, h->eoff[p] * R, R, 1, (int)np_, (int)R, +1);
        sp.bwd.tasks[t].osel = 2;                     // init f_p (T_c[i, i] = I) from scratch
        sp.bwd.tasks[t].idep = ft[p];
        for (size_t j = i + 1; j < ch.size(); ++j) {  // T_c[j, i]^T: A(r, k) = T_c[cpos_j + k + (cpos_i + r) U]
          const int32_t q = ch[j];
          sp.bwd.add_term(t, To + h->cpos[q] + h->cpos[p] * U, U, 1, h->eoff[q] * R, R, 1, (int)h->nsz[q], ft[q], 1);
        }
        sp.bwd.tile(t, 0, stpW);
        wt[p] = t;
      }
    }
  }
  sp.bwd.sort_close_bounded();
}

// Elimination order = reverse Cuthill-McKee on the leaf near-field graph (ps_setup
// ordering = 2; PAPER.md P:171 names a bandwidth-reducing (Sloan) order). x does
// not depend on the order; the scaling, hence it_0 / it_1, does.
// Re-runs the symbolic analysis and re-lays the operator arena (the far stacks move).
void reorder_rcm(ps_handle* h, cudaStream_t s) {
  const int64_t nl = h->nl;
  std::vector<std::vector<int32_t>> adj(nl);
  for (int64_t b = 0; b < h->nnear; ++b) {
    const int32_t i = (int32_t)h->near_list[3 * b], j = (int32_t)h->near_list[3 * b + 1];
    if (i == j) continue;
    adj[i].push_back(j);
    adj[j].push_back(i);
  }
  auto deg = [&](int32_t v) { return adj[v].size(); };
  for (auto& a : adj) std::sort(a.begin(), a.end(), [&](int32_t x, int32_t y) { return deg(x) < deg(y) || (deg(x) == deg(y) && x < y); });
  std::vector<char> seen(nl, 0);
  std::vector<int32_t> order;
  order.reserve(nl);
  while ((int64_t)order.size() < nl) {
    int32_t start = -1;
    for (int32_t v = 0; v < nl; ++v)
      if (!seen[v] && (start < 0 || deg(v) < deg(start))) start = v;
    size_t head = order.size();
    order.push_back(start);
    seen[start] = 1;
    while (head < order.size()) {
      const int32_t u = order[head++];
      for (int32_t v : adj[u])
        if (!seen[v]) { seen[v] = 1; order.push_back(v); }
    }
  }
  std::reverse(order.begin(), order.end());
  // rebuild everything that depends on the order (the far stacks do not)
  h->elim = order;
  symbolic(h);
  h->Pbase = 0;
  h->Dbase = h->Plen;
  h->d_op.alloc(h->Plen + h->Dlen);
  h->d_P.p = h->d_op.p + h->Pbase;
  h->d_D.p = h->d_op.p + h->Dbase;
  if (h->d_farbuf.p) ensure_far(h, s);
  h->d_e2rwg.upload(h->e2rwg, s);
  h->d_e2mort.upload(h->e2mort, s);
  h->d_m2e.upload(h->m2e, s);
  CK(cudaStreamSynchronize(s));
  h->plan.reset();
}

// ------------------------------------------------------------------ solve plan
void build_solve_plan(ps_handle* h, SolvePlan& sp, int64_t nrhs) {
  const int64_t nl = h->nl;
  const int64_t R = nrhs;
  sp.nrhs = nrhs;
  const int narrow = narrow_mode(R);
  sp.sc.alloc(h->N * R);                           // chain-stage scratch (e / f)
  for (Table* tb : {&sp.fwd, &sp.bwd, &sp.dinv, &sp.far1, &sp.far2}) {
    tb->narrow = narrow;
    if (narrow) tb->chunk_steps = NARROW_STEPS();
  }
  if (!narrow) {
    sp.far1.chunk_steps = sp.far2.chunk_steps = env_int("PS_FAR_STEPS", 32);
    sp.far1.mma = sp.far2.mma = env_int("PS_FAR_MMA", 1);
  }
  const int resident = resident_units(narrow);
  // forward sweep (gather form of Eq. 24) and backward sweep (Eq. 26), chain-collapsed
  build_chain_sweeps(h, sp, R, narrow, resident);     // PS_CHAINS=0: every node its own piece
  // D^{-1} (Eq. 32), one batch
  for (int64_t p = 0; p < nl; ++p) {
    const int64_t np_ = h->nsz[p];
    int32_t t = sp.dinv.add_task(h->eoff[p] * R, R, 1, -1, 0, 0, (int)np_, (int)R, +1);
    sp.dinv.add_term(t, h->Doff[p], 1, np_, h->eoff[p] * R, R, 1, (int)np_);
    sp.dinv.tile(t);
  }
  sp.dinv.close_batch();
  // far field, Morton order (DESIGN.md §Far field). Workspace `wm` holds the
  // Morton-ordered w (N x R) followed by the stage-1 products (one buffer, so
  // stage 2 reads both through one base).
  const int64_t NRw = h->N * R;
  // stage 1, one task per cluster c: tmp_c (sum_r x R) = S_c w[c]
  const int64_t ncl = (int64_t)h->cl_start.size();
  std::vector<int64_t> toff(ncl);
  int64_t T = 0;
  for (int64_t c = 0; c < ncl; ++c) {
    toff[c] = NRw + T;
    T += h->cl_sr[c] * R;
    if (h->cl_sr[c] == 0) continue;
    int32_t t1 = sp.far1.add_task(toff[c], R, 1, -1, 0, 0, (int)h->cl_sr[c], (int)R, +1);
    sp.far1.add_term(t1, h->cl_soff[c], 1, h->cl_sr[c], h->cl_start[c] * R, R, 1, (int)h->cl_len[c]);
    sp.far1.tile(t1);
  }
  sp.far1.close_batch();
  // stage 2 per Morton leaf l: t_l = sum_b U_b[rows of l] (V_b^T w_s) + sum_b V_b[rows of l] (U_b^T w_t)
  //                                 + dense blocks D w_s / D^T w_t
  std::vector<std::vector<std::array<int64_t, 6>>> contrib(nl);  // (oA, sAi, sAk, oB, K, -)
  auto leaf_of_pos = [&](int64_t m) {
    return (int64_t)(std::upper_bound(h->leaf_off.begin(), h->leaf_off.end(), m) - h->leaf_off.begin()) - 1;
  };
  for (int64_t b = 0; b < h->nfar; ++b) {
    const int64_t* F = &h->far_list[7 * b];
    const int64_t r0 = F[0], m = F[1], c0 = F[2], n = F[3], r = F[5];
    if (r == 0) continue;
    const int64_t ct = h->fb_ct[b], cs = h->fb_cs[b];
    if (h->fb_dense[b] >= 0) {
      const int64_t D = h->fb_dense[b];
      for (int64_t l = leaf_of_pos(r0); l < nl && h->leaf_off[l] < r0 + m; ++l)   // D w_s
        contrib[l].push_back({D + (h->leaf_off[l] - r0), 1, m, c0 * R, n, 0});
      for (int64_t l = leaf_of_pos(c0); l < nl && h->leaf_off[l] < c0 + n; ++l)   // D^T w_t
        contrib[l].push_back({D + (h->leaf_off[l] - c0) * m, m, 1, r0 * R, m, 0});
      continue;
    }
    for (int64_t l = leaf_of_pos(r0); l < nl && h->leaf_off[l] < r0 + m; ++l)
      contrib[l].push_back({h->cl_soff[ct] + h->fb_rbt[b] + (h->leaf_off[l] - r0) * h->cl_sr[ct],
                            h->cl_sr[ct], 1, toff[cs] + h->fb_rbs[b] * R, r, 0});
    for (int64_t l = leaf_of_pos(c0); l < nl && h->leaf_off[l] < c0 + n; ++l)
      contrib[l].push_back({h->cl_soff[cs] + h->fb_rbs[b] + (h->leaf_off[l] - c0) * h->cl_sr[cs],
                            h->cl_sr[cs], 1, toff[ct] + h->fb_rbt[b] * R, r, 0});
  }
  for (int64_t l = 0; l < nl; ++l) {
    const int64_t nlf = h->leaf_off[l + 1] - h->leaf_off[l];
    int32_t t = sp.far2.add_task(h->leaf_off[l] * R, R, 1, -1, 0, 0, (int)nlf, (int)R, +1);
    for (auto& c : contrib[l]) sp.far2.add_term(t, c[0], c[1], c[2], c[3], R, 1, (int)c[4]);
    sp.far2.tile(t);
  }
  sp.far2.close_batch();
  for (Table* tb : {&sp.fwd, &sp.bwd, &sp.dinv, &sp.far1, &sp.far2}) tb->upload(h->stream, &h->ring);
  const int64_t NR = h->N * R;
  sp.y.alloc(NR); sp.bo.alloc(NR); sp.w.alloc(NR); sp.u.alloc(NR); sp.xt.alloc(NR);
  sp.wm.alloc(NR + std::max<int64_t>(T, 1)); sp.tm.alloc(NR);
  CK(cudaStreamSynchronize(h->stream));
}

// buffers every solve path needs: host staging, norm partial sums
void build_common(ps_handle* h, SolvePlan& sp, int64_t nrhs) {
  sp.nrhs = nrhs;
  sp.stage.alloc(h->N * nrhs);
  sp.nchunks = (h->N + sp.rpc - 1) / sp.rpc;
  sp.part.alloc(sp.nchunks * nrhs);
  sp.norms.alloc(nrhs);
}


// ------------------------------------------------------------------ solve program
// The whole two-term solve (Eqs. 24, 32, 26, 31, 36, 26) as ONE task
// table for one persistent launch. Stages and their dependencies (per column
// tile nt; B = segment producers, I = init producer):
//   S1 fwd    y_q  = y_q + sum_d a_dq^T y_d              B: S1(d)
//   S2 dinv   bo_p = D_p^-1 y_p                          B: S1(p)
//   S3 bwd    w_p  = bo_p + sum_j a_pj w_j               I: S2(p)  B: S3(j)
//   S4 far1   tmp_c = S_c w[c]  (per cluster, rows gathered per leaf)   B: S3
//   S5 far2   z_l  = sum U tmp + V tmp + dense D w       B: S4 / S3
//   S6 fwd    z_q  = z_q + sum_d a_dq^T z_d              I: S5(q)  B: S6(d) or S5(d)
//   S7 dinv   xt_p = bo_p - D_p^-1 z_p                   I: S2(p)  B: S6(p) or S5(p)
//   S8 bwd    x_p  = xt_p + sum_j a_pj x_j               I: S7(p)  B: S8(j)
// Work items are ordered by (stage, level) + nt * stagger: every dependency has
// a smaller key (deadlock-free ticket order), and the column tiles enter the
// pipeline staggered, so one tile's thin elimination-chain phase overlaps
// another tile's bulk work. Vectors live in one workspace arena, operators in
// one operator arena, so a single set of base pointers serves every task.
void build_program(ps_handle* h, SolvePlan& sp, int64_t R) {
  const int64_t nl = h->nl;
  Table& P = sp.prog;
  P.narrow = narrow_mode(R);
  if (P.narrow) P.chunk_steps = NARROW_STEPS();
  const int64_t NR = h->N * R;
  sp.oY = 0; sp.oBO = NR; sp.oW = 2 * NR; sp.oZ = 3 * NR; sp.oXT = 4 * NR; sp.oX = 5 * NR; sp.oTMP = 6 * NR;
  const int64_t ncl = (int64_t)h->cl_start.size();
  std::vector<int64_t> toff(ncl);
  int64_t Ttot = 0;
  for (int64_t c = 0; c < ncl; ++c) { toff[c] = sp.oTMP + Ttot; Ttot += h->cl_sr[c] * R; }
  const int resident = resident_units(P.narrow);
  // narrow solves: the far field as the one-pass far1p apply between two program batches
  sp.f1p = P.narrow && build_far1p(h, h->stream);
  if (sp.f1p) build_far1p_items(h, sp, R);
  P.key_stagger = env_int("PS_PROG_STAGGER", 0);     // column tile b enters b * this many key levels later
  P.early_keys = true;
  // far field on the tensor-core consumer with long chunks, as in the stage tables
  const bool far_mma = !P.narrow && env_int("PS_FAR_MMA", 1) != 0;
  const int far_steps = P.narrow ? NARROW_STEPS() : env_int("PS_FAR_STEPS", 32);
  sp.oSC = sp.oTMP + Ttot;                             // chain scratch (e / f), N x R
  double lev = 0;
  const int64_t Fb = h->Fbase, Pb = h->Pbase, Db = h->Dbase;
  auto leaf_of_pos = [&](int64_t m) {
    return (int64_t)(std::upper_bound(h->leaf_off.begin(), h->leaf_off.end(), m) - h->leaf_off.begin()) - 1;
  };
  std::vector<int32_t> s1(nl, -1), s2(nl, -1), s3(nl, -1), s4(ncl, -1), s5(nl, -1), s6(nl, -1), s7(nl, -1),
      s8(nl, -1);
  // Chain-collapsed sweeps inside the program (as build_chain_sweeps, all vectors and
  // the chain scratch in the one workspace arena): per chain level an E / F stage
  // (gathers from outside the piece, to scratch) and a Y / W stage (T_c products).
  const int64_t Tb = h->Tbase, nc = (int64_t)h->chains.size();
  // each sweep of the program owns a scratch region: with all stages in one launch a
  // later sweep's gathers (F / E tasks) may run while an earlier sweep's T products
  // still read their e / f rows (write-after-read across sweeps)
  int64_t SC = sp.oSC;
  std::vector<std::vector<int32_t>> lev_f(h->max_ch_height + 1), lev_b(h->max_ch_depth + 1);
  for (int64_t c = 0; c < nc; ++c) {
    lev_f[h->ch_height[c]].push_back((int32_t)c);
    lev_b[h->ch_depth[c]].push_back((int32_t)c);
  }
  auto steps_of = [&](const std::vector<std::pair<int64_t, int64_t>>& mk) {
    double ks = 0;
    if (P.narrow) {
      for (auto [m, K] : mk) ks += std::ceil((double)m / mode_rows(P.narrow)) * std::ceil((double)K / GM_KC);
      return std::max(2, std::min(NARROW_STEPS(), (int)std::ceil(ks / (double)resident)));
    }
    static const int pmax = env_int("PS_SWEEP_MAXSTEPS", 32), pipc = env_int("PS_SWEEP_IPC", 1);
    for (auto [m, K] : mk) ks += std::ceil((double)m / GM_MT) * std::ceil((double)R / GM_NT) * std::ceil((double)K / GM_KC);
    return std::max(2, std::min(pmax, (int)std::ceil(ks / ((double)pipc * resident))));
  };
  auto by_height = [&](std::vector<std::pair<int32_t, int32_t>> v) {
    std::stable_sort(v.begin(), v.end(), [&](const std::pair<int32_t, int32_t>& x, const std::pair<int32_t, int32_t>& y) {
      return h->height[x.first] < h->height[y.first];
    });
    return v;
  };
  // forward sweep in place on `buf`; init_dep[p] produces the initial rows p (or none)
  static const int direct_ends = env_int("PS_DIRECT_ENDS", 1);   // chain end pieces skip the identity T copy
  auto fwd_stage = [&](int64_t buf, std::vector<int32_t>& out, const std::vector<int32_t>* init_dep) {
    auto prod = [&](int32_t d) { return out[d] >= 0 ? out[d] : (init_dep ? (*init_dep)[d] : -1); };
    std::vector<int32_t> et(nl, -1);
    std::vector<char> in_buf(nl, 0);
    for (const auto& cl : lev_f) {
      std::vector<std::pair<int64_t, int64_t>> mk;
      for (int32_t c : cl)
        for (int32_t p : h->chains[c]) {
          int64_t K = 0;
          for (auto [d, idx] : h->gath[p])
            if (h->chain_of[d] != c) K += h->nsz[d];
          mk.push_back({h->nsz[p], K});
        }
      const int stpE = steps_of(mk);
      P.key_base = lev++;
      for (int32_t c : cl) {
        const bool single = h->chains[c].size() == 1;
        for (int32_t p : h->chains[c]) {
          std::vector<std::pair<int32_t, int32_t>> gl;
          for (auto [d, idx] : h->gath[p])
            if (h->chain_of[d] != c) gl.push_back({d, idx});
          // the chain's first piece has no T product (T_c[0, 0] = I): its e is its y, written in place
          const bool direct = single || (direct_ends && p == h->chains[c][0]);
          if (direct) in_buf[p] = 1;
          if (direct && gl.empty()) continue;            // y_p = its input rows: nothing to do
          const int64_t np_ = h->nsz[p];
          const int64_t o = (direct ? buf : SC) + h->eoff[p] * R;
          int32_t t = P.add_task(o, R, 1, buf + h->eoff[p] * R, R, 1, (int)np_, (int)R, +1);
          if (init_dep) P.tasks[t].idep = (*init_dep)[p];
          for (auto [d, idx] : by_height(gl)) {
            const int64_t nd = h->nsz[d];
            P.add_term(t, Pb + h->Poff[d] + h->pcol[d][idx] * nd, nd, 1, buf + h->eoff[d] * R, R, 1, (int)nd, prod(d));
          }
          P.tile(t, -1, stpE);
          (direct ? out : et)[p] = t;
        }
      }
      mk.clear();
      for (int32_t c : cl)
        if (h->chains[c].size() > 1)
          for (int32_t p : h->chains[c]) mk.push_back({h->nsz[p], h->cpos[p]});
      const int stpY = steps_of(mk);
      P.key_base = lev++;
      for (int32_t c : cl) {
        if (h->chains[c].size() == 1) continue;
        const int64_t U = h->ch_U[c], To = Tb + h->ch_Toff[c];
        for (size_t i = 0; i < h->chains[c].size(); ++i) {
          const int32_t p = h->chains[c][i];
          if (in_buf[p]) continue;                       // first piece: y written by its E task (or input)
          const int64_t np_ = h->nsz[p];
          int32_t t = P.add_task(buf + h->eoff[p] * R, R, 1, SC + h->eoff[p] * R, R, 1, (int)np_, (int)R, +1);
          P.tasks[t].idep = et[p];
          for (size_t j = 0; j < i; ++j) {
            const int32_t q = h->chains[c][j];
            P.add_term(t, To + h->cpos[p] + h->cpos[q] * U, 1, U, (in_buf[q] ? buf : SC) + h->eoff[q] * R, R, 1,
                       (int)h->nsz[q], in_buf[q] ? prod(q) : et[q]);
          }
          P.tile(t, 0, stpY);
          out[p] = t;
        }
      }
    }
  };
  auto dinv_stage = [&](int64_t src, int64_t dst, int64_t init, int sign, std::vector<int32_t>& out,
                        const std::vector<int32_t>& src_dep, const std::vector<int32_t>* init_dep) {
    P.key_base = lev++;
    for (int64_t p = 0; p < nl; ++p) {
      const int64_t np_ = h->nsz[p];
      int32_t t = P.add_task(dst + h->eoff[p] * R, R, 1, init >= 0 ? init + h->eoff[p] * R : -1, R, 1,
                             (int)np_, (int)R, sign);
      if (init_dep) P.tasks[t].idep = (*init_dep)[p];
      P.add_term(t, Db + h->Doff[p], 1, np_, src + h->eoff[p] * R, R, 1, (int)np_, src_dep[p]);
      P.tile(t);
      out[p] = t;
    }
  };
  // backward sweep out_buf = R init; init_dep[p] produces the rows p of init
  auto bwd_stage = [&](int64_t init, int64_t out_buf, std::vector<int32_t>& out,
                       const std::vector<int32_t>& init_dep) {
    std::vector<int32_t> ft(nl, -1);
    std::vector<char> in_buf(nl, 0);
    for (const auto& cl : lev_b) {
      std::vector<std::pair<int64_t, int64_t>> mk;
      for (int32_t c : cl)
        for (int32_t p : h->chains[c]) {
          int64_t K = 0;
          for (int32_t j : h->st[p])
            if (h->chain_of[j] != c) K += h->nsz[j];
          mk.push_back({h->nsz[p], K});
        }
      const int stpF = steps_of(mk);
      P.key_base = lev++;
      for (int32_t c : cl) {
        const bool single = h->chains[c].size() == 1;
        for (int32_t p : h->chains[c]) {
          const int64_t np_ = h->nsz[p];
          // the chain's top piece has no T product: its f is its w, written directly
          const bool direct = single || (direct_ends && p == h->chains[c].back());
          if (direct) in_buf[p] = 1;
          const int64_t o = (direct ? out_buf : SC) + h->eoff[p] * R;
          int32_t t = P.add_task(o, R, 1, init + h->eoff[p] * R, R, 1, (int)np_, (int)R, +1);
          P.tasks[t].idep = init_dep[p];
          for (size_t i = 0; i < h->st[p].size(); ++i) {
            const int32_t j = h->st[p][i];
            if (h->chain_of[j] == c) continue;
            P.add_term(t, Pb + h->Poff[p] + h->pcol[p][i] * np_, 1, np_, out_buf + h->eoff[j] * R, R, 1,
                       (int)h->nsz[j], out[j]);
          }
          P.tile(t, +1, stpF);
          (direct ? out : ft)[p] = t;
        }
      }
      mk.clear();
      for (int32_t c : cl)
        if (h->chains[c].size() > 1)
          for (int32_t p : h->chains[c]) mk.push_back({h->nsz[p], h->ch_U[c] - h->cpos[p] - h->nsz[p]});
      const int stpW = steps_of(mk);
      P.key_base = lev++;
      for (int32_t c : cl) {
        if (h->chains[c].size() == 1) continue;
        const int64_t U = h->ch_U[c], To = Tb + h->ch_Toff[c];
        const auto& ch = h->chains[c];
        for (size_t i = 0; i < ch.size(); ++i) {
          const int32_t p = ch[i];
          if (in_buf[p]) continue;                       // top piece: w written by its F task
          const int64_t np_ = h->nsz[p];
          int32_t t = P.add_task(out_buf + h->eoff[p] * R, R, 1, SC + h->eoff[p] * R, R, 1, (int)np_, (int)R, +1);
          P.tasks[t].idep = ft[p];
          for (size_t j = i + 1; j < ch.size(); ++j) {
            const int32_t q = ch[j];
            P.add_term(t, To + h->cpos[q] + h->cpos[p] * U, U, 1, (in_buf[q] ? out_buf : SC) + h->eoff[q] * R, R, 1,
                       (int)h->nsz[q], in_buf[q] ? out[q] : ft[q]);
          }
          P.tile(t, 0, stpW);
          out[p] = t;
        }
      }
    }
  };
  SC = sp.oSC;
  fwd_stage(sp.oY, s1, nullptr);                                         // S1
  dinv_stage(sp.oY, sp.oBO, -1, +1, s2, s1, nullptr);                    // S2
  SC = sp.oSC + NR;
  bwd_stage(sp.oBO, sp.oW, s3, s2);                                      // S3
  if (sp.f1p) {
    // batch 0 ends here; S4 / S5 are the far1p launches (Z complete before batch 1, whose
    // tasks therefore carry no dependency on batch 0 or the far field)
    P.sort_close_bounded();
  } else {
  // S4 far stage 1: per cluster, rows gathered per leaf from W (elimination order)
  P.key_base = lev++;
  for (int64_t c = 0; c < ncl; ++c) {
    if (h->cl_sr[c] == 0) continue;
    const int64_t sr = h->cl_sr[c], a0 = h->cl_start[c], len = h->cl_len[c];
    int32_t t = P.add_task(toff[c], R, 1, -1, 0, 0, (int)sr, (int)R, +1);
    if (far_mma) P.tasks[t].osel |= 4;
    for (int64_t l = leaf_of_pos(a0); l < nl && h->leaf_off[l] < a0 + len; ++l) {
      const int32_t pos = h->pos_of[l];
      P.add_term(t, Fb + h->cl_soff[c] + (h->leaf_off[l] - a0) * sr, 1, sr, sp.oW + h->eoff[pos] * R, R, 1,
                 (int)(h->leaf_off[l + 1] - h->leaf_off[l]), s3[pos]);
    }
    P.tile(t, 0, far_steps);
    s4[c] = t;
  }
  // S5 far stage 2: per leaf, written in elimination order into Z
  P.key_base = lev++;
  {
    struct Seg { int64_t oA, sAi, sAk, oB; int K; int32_t dep; };
    std::vector<std::vector<Seg>> contrib(nl);
    for (int64_t b = 0; b < h->nfar; ++b) {
      const int64_t* F = &h->far_list[7 * b];
      const int64_t r0 = F[0], m = F[1], c0 = F[2], n = F[3], r = F[5];
      if (r == 0) continue;
      const int64_t ct = h->fb_ct[b], cs = h->fb_cs[b];
      if (h->fb_dense[b] >= 0) {
        const int64_t D = Fb + h->fb_dense[b];
        // t rows: D w_s, K over the source leaves;  s rows: D^T w_t, K over the target leaves
        for (int64_t l = leaf_of_pos(r0); l < nl && h->leaf_off[l] < r0 + m; ++l)
          for (int64_t g = leaf_of_pos(c0); g < nl && h->leaf_off[g] < c0 + n; ++g) {
            const int32_t pg = h->pos_of[g];
            contrib[l].push_back({D + (h->leaf_off[l] - r0) + (h->leaf_off[g] - c0) * m, 1, m,
                                  sp.oW + h->eoff[pg] * R, (int)(h->leaf_off[g + 1] - h->leaf_off[g]), s3[pg]});
          }
        for (int64_t l = leaf_of_pos(c0); l < nl && h->leaf_off[l] < c0 + n; ++l)
          for (int64_t g = leaf_of_pos(r0); g < nl && h->leaf_off[g] < r0 + m; ++g) {
            const int32_t pg = h->pos_of[g];
            contrib[l].push_back({D + (h->leaf_off[g] - r0) + (h->leaf_off[l] - c0) * m, m, 1,
                                  sp.oW + h->eoff[pg] * R, (int)(h->leaf_off[g + 1] - h->leaf_off[g]), s3[pg]});
          }
        continue;
      }
      for (int64_t l = leaf_of_pos(r0); l < nl && h->leaf_off[l] < r0 + m; ++l)
        contrib[l].push_back({Fb + h->cl_soff[ct] + h->fb_rbt[b] + (h->leaf_off[l] - r0) * h->cl_sr[ct],
                              h->cl_sr[ct], 1, toff[cs] + h->fb_rbs[b] * R, (int)r, s4[cs]});
      for (int64_t l = leaf_of_pos(c0); l < nl && h->leaf_off[l] < c0 + n; ++l)
        contrib[l].push_back({Fb + h->cl_soff[cs] + h->fb_rbs[b] + (h->leaf_off[l] - c0) * h->cl_sr[cs],
                              h->cl_sr[cs], 1, toff[ct] + h->fb_rbt[b] * R, (int)r, s4[ct]});
    }
    for (int64_t l = 0; l < nl; ++l) {
      const int32_t pos = h->pos_of[l];
      const int64_t nlf = h->leaf_off[l + 1] - h->leaf_off[l];
      int32_t t = P.add_task(sp.oZ + h->eoff[pos] * R, R, 1, -1, 0, 0, (int)nlf, (int)R, +1);
      if (far_mma) P.tasks[t].osel |= 4;
      for (auto& g : contrib[l]) P.add_term(t, g.oA, g.sAi, g.sAk, g.oB, R, 1, g.K, g.dep);
      P.tile(t, 0, far_steps);
      s5[pos] = t;
    }
  }
  }
  SC = sp.oSC + 2 * NR;
  fwd_stage(sp.oZ, s6, &s5);                                             // S6
  std::vector<int32_t> zfin(nl);
  for (int64_t p = 0; p < nl; ++p) zfin[p] = s6[p] >= 0 ? s6[p] : s5[p];
  const std::vector<int32_t> none(nl, -1);
  dinv_stage(sp.oZ, sp.oXT, sp.oBO, -1, s7, zfin, sp.f1p ? &none : &s2); // S7: xt = bo - D^-1 z
  SC = sp.oSC + 3 * NR;
  bwd_stage(sp.oXT, sp.oX, s8, s7);                                      // S8
  P.sort_close_bounded();
  sp.ws_len = 10 * NR + std::max<int64_t>(Ttot, 1);
  if (g_host_only) return;                           // ps_validate: tables only
  P.upload(h->stream, &h->ring);
  sp.ws.alloc(sp.ws_len);
  if (sp.f1p) {
    sp.d_f1p_blk.upload(sp.f1p_blk, h->stream);
    sp.d_f1p_item.upload(sp.f1p_item, h->stream);
    sp.d_f1p_unit.upload(sp.f1p_unit, h->stream);
    sp.d_f1p_cnt.alloc(1);
    sp.f1p_y.alloc(std::max<int64_t>(h->f1p_prows * R, 1));
    sp.f1p_xa.alloc(std::max<int64_t>((int64_t)h->f1p_xmap.size() * R, 1));
  }
  // the tables were copied from pageable host memory on h->stream (non-blocking):
  // complete them before ps_solve launches the program on the caller's stream
  CK(cudaStreamSynchronize(h->stream));
}

// Host-only check of a solve program (ps_validate): the properties the persistent
// dataflow kernel relies on, for every task, segment and work item of the table.
//   bounds      every operand access lies inside its arena: O / I / B in the
//               workspace, A inside one operator region (panels, D^-1, far, T);
//   races       happens-before = the transitive closure of the dependencies (init
//               producer, segment producers): any two tasks writing one element, and
//               any task reading a range (segments B, init rows I) and any task
//               writing into it, are ordered by it — no unordered write/write or
//               read/write pair, so the kernel has no data race on the workspace;
//   tickets     every item's producers (and the previous user of its partial slots)
//               have all their items at smaller tickets: with all CTAs resident the
//               smallest unfinished ticket can always run (deadlock freedom).
std::string validate_program(const ps_handle* h, const SolvePlan& sp, std::vector<int64_t>& stats) {
  const Table& P = sp.prog;
  const int64_t WS = sp.ws_len;
  struct Reg { int64_t lo, hi; };
  const std::vector<Reg> opr = {{h->Pbase, h->Pbase + h->Plen}, {h->Dbase, h->Dbase + h->Dlen},
                                {h->Fbase, h->Fbase + (int64_t)h->far_host.size()}, {h->Tbase, h->Tbase + h->Tlen}};
  auto op_ok = [&](int64_t lo, int64_t hi) {
    for (const Reg& r : opr)
      if (lo >= r.lo && hi <= r.hi) return true;
    return false;
  };
  auto msg = [](const char* what, int64_t a, int64_t b) {
    return std::string(what) + " (" + std::to_string(a) + ", " + std::to_string(b) + ")";
  };
  struct Iv { int64_t lo, hi; int32_t task; };
  std::vector<Iv> wr;
  const int64_t nt = (int64_t)P.tasks.size();
  // rows of a row-major block: [o + i s, o + i s + n) for i < m (contiguous when s == n)
  auto rows = [&](int64_t o, int64_t si, int64_t sc, int m, int n, int32_t task, std::vector<Iv>& out) -> bool {
    if (sc != 1) return false;
    if (si == n) { out.push_back({o, o + (int64_t)m * n, task}); return true; }
    for (int i = 0; i < m; ++i) out.push_back({o + i * si, o + i * si + n, task});
    return true;
  };
  for (int64_t t = 0; t < nt; ++t) {
    const GTask& T = P.tasks[t];
    if (T.osel & 3) return msg("task addresses the scratch base (not used by the program)", t, T.osel);
    if (!rows(T.oO, T.sOi, T.sOc, T.m, T.n, (int32_t)t, wr)) return msg("non-unit column stride of O", t, T.sOc);
  }
  for (const Iv& v : wr)
    if (v.lo < 0 || v.hi > WS) return msg("write outside the workspace", v.task, v.lo);
  std::sort(wr.begin(), wr.end(), [](const Iv& a, const Iv& b) { return a.lo < b.lo; });
  // happens-before: b (transitively) waits on a through init / segment dependencies
  std::vector<std::vector<int32_t>> deps(nt);
  for (int64_t t = 0; t < nt; ++t) {
    const GTask& T = P.tasks[t];
    if (T.idep >= 0) deps[t].push_back(T.idep);
    for (int32_t k = T.t0; k < T.t1; ++k)
      if (P.terms[k].dep >= 0) deps[t].push_back(P.terms[k].dep);
  }
  std::vector<int64_t> seen(nt, -1);
  int64_t gen = 0;
  std::vector<int32_t> stack;
  auto before = [&](int32_t a, int32_t b) -> bool {  // a happens before b
    if (a == b) return false;
    if (P.batch_of_task(a) != P.batch_of_task(b)) return P.batch_of_task(a) < P.batch_of_task(b);  // launch order
    ++gen;
    stack.assign(1, b);
    while (!stack.empty()) {
      const int32_t x = stack.back();
      stack.pop_back();
      for (int32_t d : deps[x]) {
        if (d == a) return true;
        if (d > a && seen[d] != gen) { seen[d] = gen; stack.push_back(d); }   // producers have smaller ids
      }
    }
    return false;
  };
  auto ordered = [&](int32_t a, int32_t b) { return a == b || before(a, b) || before(b, a); };
  {
    std::vector<Iv> open_;                               // sweep over sorted starts
    for (const Iv& v : wr) {
      open_.erase(std::remove_if(open_.begin(), open_.end(), [&](const Iv& o) { return o.hi <= v.lo; }), open_.end());
      for (const Iv& o : open_)
        if (!ordered(o.task, v.task)) return msg("two unordered tasks write one element", o.task, v.task);
      open_.push_back(v);
    }
  }
  // writers overlapping [lo, hi)
  auto writers = [&](int64_t lo, int64_t hi, std::vector<int32_t>& out) {
    out.clear();
    auto it = std::upper_bound(wr.begin(), wr.end(), lo, [](int64_t x, const Iv& v) { return x < v.lo; });
    if (it != wr.begin()) --it;
    for (; it != wr.end() && it->lo < hi; ++it)
      if (it->hi > lo) out.push_back(it->task);
  };
  std::vector<int32_t> ws;
  std::vector<Iv> rd;
  int64_t nread = 0;
  for (int64_t t = 0; t < nt; ++t) {
    const GTask& T = P.tasks[t];
    if (T.oI >= 0) {
      rd.clear();
      if (!rows(T.oI, T.sIi, T.sIc, T.m, T.n, (int32_t)t, rd)) return msg("non-unit column stride of I", t, T.sIc);
      for (const Iv& v : rd) {
        if (v.lo < 0 || v.hi > WS) return msg("init read outside the workspace", t, v.lo);
        writers(v.lo, v.hi, ws);
        for (int32_t w : ws)
          if (!ordered(w, (int32_t)t)) return msg("init rows written by a task unordered with the reader", t, w);
        ++nread;
      }
    }
    for (int32_t k = T.t0; k < T.t1; ++k) {
      const GTerm& g = P.terms[k];
      if (g.bsel & 1) return msg("segment addresses the scratch base", t, k);
      const int64_t alo = g.oA, ahi = g.oA + (int64_t)(g.K - 1) * g.sAk + (int64_t)(T.m - 1) * g.sAi + 1;
      if (g.sAk < 0 || g.sAi < 0 || !op_ok(alo, ahi)) return msg("operator read outside its region", t, k);
      rd.clear();
      if (!rows(g.oB, g.sBk, g.sBc, g.K, T.n, (int32_t)t, rd)) return msg("non-unit column stride of B", t, k);
      for (const Iv& v : rd) {
        if (v.lo < 0 || v.hi > WS) return msg("segment read outside the workspace", t, k);
        writers(v.lo, v.hi, ws);
        for (int32_t w : ws)
          if (!ordered(w, (int32_t)t)) return msg("segment rows written by a task unordered with the reader", t, w);
        ++nread;
      }
    }
  }
  // ticket order
  const int64_t nw = (int64_t)P.work.size();
  std::vector<int64_t> last(nt, -1);
  for (int64_t i = 0; i < nw; ++i) last[P.work[i].task] = std::max(last[P.work[i].task], i);
  // completion units are numbered per batch (launch)
  const int nbat = (int)P.task_end.size();
  std::vector<std::vector<int32_t>> unit_task(std::max(nbat, 1), std::vector<int32_t>(std::max<int32_t>(P.max_units, 1), -1));
  for (int64_t t = 0; t < nt; ++t)
    for (int32_t u = 0; u < (P.tasks[t].n + P.NT() - 1) / P.NT(); ++u)
      unit_task[P.batch_of_task((int32_t)t)][P.tasks[t].unit0 + u] = (int32_t)t;
  int64_t max_back = 0;
  for (int64_t i = 0; i < nw; ++i) {
    const GWork& w = P.work[i];
    const GTask& T = P.tasks[w.task];
    auto need_before = [&](int32_t task) -> bool {
      if (task < 0) return true;
      max_back = std::max(max_back, i - last[task]);
      return last[task] < i;
    };
    const int bt = P.batch_of_task(w.task);
    auto same_batch = [&](int32_t task) { return task < 0 || P.batch_of_task(task) == bt; };
    if (!same_batch(T.idep)) return msg("init producer in another launch", i, T.idep);
    if (!need_before(T.idep)) return msg("item precedes its init producer", i, T.idep);
    for (int32_t k = w.ta; k < w.tb; ++k) {
      if (!same_batch(P.terms[k].dep)) return msg("segment producer in another launch", i, P.terms[k].dep);
      if (!need_before(P.terms[k].dep)) return msg("item precedes a segment producer", i, P.terms[k].dep);
    }
    if (w.sw_unit >= 0 && !need_before(unit_task[bt][w.sw_unit])) return msg("item precedes its slots' previous user", i, w.sw_unit);
  }
  stats = {nt, (int64_t)P.terms.size(), nw, (int64_t)wr.size(), nread, max_back};
  return "";
}

// Host-only check of the far1p tables (ps_validate): every item's factor range inside the
// FB arena and every pack block inside its item's staged range; x / y rows inside the Morton
// vector / the pieces; partial slots inside their area; every gamma (beta) item of a big
// block after all its alpha (gamma) items in item order (the only waits: deadlock-free).
std::string validate_far1p(const ps_handle* h, const SolvePlan& sp, std::vector<int64_t>& stats) {
  const int64_t lo = h->FBbase, hi = h->FBbase + h->f1p_len, N = h->N, R = sp.nrhs;
  auto msg = [](const char* what, int64_t a) { return std::string("far1p: ") + what + " (" + std::to_string(a) + ")"; };
  const int64_t nb = (int64_t)sp.f1p_blk.size(), ni = (int64_t)sp.f1p_item.size();
  std::vector<int64_t> covered(nb, 0);
  std::vector<char> item_seen(ni, 0);
  for (int64_t u = 0; u < (int64_t)sp.f1p_unit.size(); ++u) {
    const FUnit& U = sp.f1p_unit[u];
    if (U.i0 < 0 || U.n < 1 || U.i0 + U.n > ni) return msg("unit items out of range", u);
    const FItem& f = sp.f1p_item[U.i0];
    if (f.kind == 0)
      for (int j = 0; j < U.n; ++j)
        if (sp.f1p_item[U.i0 + j].kind != 0) return msg("pack unit holding a chunk", u);
    if (f.kind != 0) {
      // one big block, its chunks in phase order: F1 (or dense G) chunks, F2 chunks, F1 chunks
      const FBlk& k = sp.f1p_blk[f.b];
      std::vector<std::pair<int, int>> want;
      for (int c = 0; c < k.nc1; ++c) want.push_back({k.dense ? 4 : 1, c});
      for (int c = 0; c < k.nc2; ++c) want.push_back({2, c});
      if (!k.dense)
        for (int c = 0; c < k.nc1; ++c) want.push_back({3, c});
      if ((int64_t)want.size() != U.n) return msg("big unit does not hold its block's chunks", u);
      for (int j = 0; j < U.n; ++j) {
        const FItem& it = sp.f1p_item[U.i0 + j];
        if (it.b != f.b || it.kind != want[j].first || it.nb != want[j].second) return msg("big unit chunks out of order", u);
      }
    }
    for (int j = 0; j < U.n; ++j) {
      if (item_seen[U.i0 + j]) return msg("item in two units", U.i0 + j);
      item_seen[U.i0 + j] = 1;
    }
  }
  for (int64_t i = 0; i < ni; ++i) {
    if (!item_seen[i]) return msg("item in no unit", i);
    const FItem& it = sp.f1p_item[i];
    if (it.len <= 0 || it.len > F1P_CH || it.off < lo || it.off + it.len > hi) return msg("item range outside the FB arena", i);
    if (it.kind == 0) {
      if (it.b < 0 || it.nb < 1 || it.nb > F1P_PACK || it.b + it.nb > nb) return msg("pack blocks out of range", i);
      int64_t xr = 0;
      for (int32_t j = it.b; j < it.b + it.nb; ++j) {
        const FBlk& k = sp.f1p_blk[j];
        const int64_t e1 = (int64_t)k.n1 * k.r, e2 = (int64_t)k.n2 * k.r;
        if (k.o1 < it.off || k.o1 + e1 > it.off + it.len) return msg("pack block outside its item", j);
        if (!k.dense && (k.o2 < it.off || k.o2 + e2 > it.off + it.len)) return msg("pack block outside its item", j);
        const int64_t x2n = k.dense ? k.r : k.n2;
        if (k.xo1 != xr || k.xo2 != xr + k.n1) return msg("pack x rows not consecutive", j);
        xr += k.n1 + x2n;
        covered[j] += e1 + e2;
      }
      if (xr * R > F1P_XCH || xr != it.a0 || xr != it.xn || it.xa != sp.f1p_blk[it.b].xa)
        return msg("pack x rows exceed the stage or miscounted", i);
      for (int32_t j = it.b; j < it.b + it.nb; ++j)
        if (sp.f1p_blk[j].xa != it.xa + sp.f1p_blk[j].xo1) return msg("pack x rows not one XA range", j);
      continue;
    }
    if (it.b < 0 || it.b >= nb) return msg("big item block out of range", i);
    const FBlk& k = sp.f1p_blk[it.b];
    const bool on2 = it.kind == 2;
    const int64_t o = on2 ? k.o2 : k.o1;
    const int32_t rows = on2 ? k.n2 : k.n1;
    if (it.a0 < 0 || it.a1 > rows || it.a0 >= it.a1 || it.off != o + (int64_t)it.a0 * k.r ||
        it.len != (it.a1 - it.a0) * k.r)
      return msg("big item rows inconsistent with its block", i);
    if (((int64_t)(it.a1 - it.a0) + (it.kind == 4 ? k.r : 0)) * R > F1P_XCH) return msg("chunk x rows exceed the stage", i);
    {
      const int64_t want = it.kind == 3 ? -1 : (it.kind == 2 ? k.xa + k.n1 : k.xa) + it.a0;
      const int32_t wn = it.kind == 3 ? 0 : it.a1 - it.a0;
      if ((wn > 0 && it.xa != want) || it.xn != wn || (it.kind == 4 ? (it.xa2 != k.xa + k.n1 || it.xn2 != k.r) : it.xn2 != 0))
        return msg("chunk x rows inconsistent with its block", i);
    }
    if (it.kind != 3) covered[it.b] += it.len;
  }
  for (int64_t j = 0; j < nb; ++j) {
    const FBlk& k = sp.f1p_blk[j];
    const int64_t e = (int64_t)(k.n1 + k.n2) * k.r;
    if (covered[j] != e) return msg("block factors not covered exactly once", j);
    if (k.r < 1 || k.r > F1P_RMAX) return msg("block rank outside (0, F1P_RMAX]", j);
    // the kernel applies a small low-rank block as the stacked [F1; F2]: F2, x2 and y2 follow F1, x1, y1
    if (!k.dense && (k.o2 != k.o1 + (int64_t)k.n1 * k.r || k.y2 != k.y1 + k.n1 || k.xa + k.n1 < 0))
      return msg("low-rank block sides not stacked", j);
    if (k.x1 < 0 || k.x1 + k.n1 > N || k.x2 < 0 || k.x2 + (k.dense ? k.r : k.n2) > N) return msg("x rows outside N", j);
    if (k.xa < 0 || k.xa + k.n1 + (k.dense ? k.r : k.n2) > (int64_t)h->f1p_xmap.size()) return msg("XA rows out of range", j);
    if (k.y1 < 0 || k.y1 + k.n1 > h->f1p_prows || k.y2 < 0 || k.y2 + (k.dense ? k.r : k.n2) > h->f1p_prows)
      return msg("piece rows out of range", j);
  }
  stats.push_back(ni);
  return "";
}

bool use_stages() {
  static const bool v = [] {
    const char* e = std::getenv("PS_SOLVE");
    return e && std::string(e) == "stages";
  }();
  return v;
}

// Per-nrhs plan, built on first use: the single-launch program for ps_solve and,
// only when needed (ps_apply, PS_SOLVE=stages), the per-operator stage tables.
SolvePlan& get_plan(ps_handle* h, int64_t nrhs, bool need_stages = false) {
  if (!h->plan || h->plan->nrhs != nrhs) {
    h->plan.reset();
    auto sp = std::make_unique<SolvePlan>();
    build_common(h, *sp, nrhs);
    if (!use_stages()) build_program(h, *sp, nrhs);
    h->plan = std::move(sp);
  }
  if ((need_stages || use_stages()) && !h->plan->stages_built) {
    build_solve_plan(h, *h->plan, nrhs);
    h->plan->stages_built = true;
  }
  return *h->plan;
}

// individual operators on internal (E-order, row-major) vectors --------------
int64_t op_Rt(ps_handle* h, SolvePlan& sp, double2* v, cudaStream_t s) {   // in place
  return sp.fwd.launch_all(v, v, h->d_P.p, v, s, &h->prof, PC_FWD);
}
int64_t op_R(ps_handle* h, SolvePlan& sp, const double2* in, double2* out, cudaStream_t s) {
  return sp.bwd.launch_all(out, in, h->d_P.p, out, s, &h->prof, PC_BWD);
}
int64_t op_Dinv(ps_handle* h, SolvePlan& sp, const double2* in, double2* out, cudaStream_t s) {
  return sp.dinv.launch_all(out, nullptr, h->d_D.p, in, s, &h->prof, PC_DINV);
}
template <class F>
int64_t aux(ps_handle* h, cudaStream_t s, F f) {
  h->prof.begin(PC_AUX, s);
  f();
  h->prof.end(s);
  return 1;
}
int64_t op_ZF(ps_handle* h, SolvePlan& sp, const double2* in, double2* out, cudaStream_t s) {
  const int64_t N = h->N, R = sp.nrhs;
  int64_t n = 0;
  n += aux(h, s, [&] { launch_permute_rows(N, R, h->d_m2e.p, in, sp.wm.p, s); });      // E -> Morton
  n += sp.far1.launch_all(sp.wm.p, nullptr, h->d_far.p, sp.wm.p, s, &h->prof, PC_FAR1);
  n += sp.far2.launch_all(sp.tm.p, nullptr, h->d_far.p, sp.wm.p, s, &h->prof, PC_FAR2);
  n += aux(h, s, [&] { launch_permute_rows(N, R, h->d_e2mort.p, sp.tm.p, out, s); });  // Morton -> E
  return n;
}

// far1p: Z (E order) = Z_F W over every far block, one read of the factors (build_far1p)
int64_t far1p_apply(ps_handle* h, SolvePlan& sp, const double2* W, double2* Z, cudaStream_t s) {
  const int64_t N = h->N, R = sp.nrhs;
  h->prof.begin(PC_F1P, s);
  CK(cudaMemsetAsync(sp.d_f1p_cnt.p, 0, sizeof(int32_t), s));
  launch_permute_rows((int64_t)h->f1p_xmap.size(), R, h->d_f1p_xmap.p, W, sp.f1p_xa.p, s);   // w -> XA
  Far1pArgs fa;
  fa.units = sp.d_f1p_unit.p;
  fa.nunits = (int64_t)sp.f1p_unit.size();
  fa.items = sp.d_f1p_item.p;
  fa.blks = sp.d_f1p_blk.p;
  fa.A = h->d_op.p;
  fa.x = sp.f1p_xa.p;
  fa.y = sp.f1p_y.p;
  fa.cnt = sp.d_f1p_cnt.p;
  fa.R = (int32_t)R;
  static const int minrows = env_int("PS_F1P_MINROWS", 0);
  fa.minrows = minrows;
  launch_far1p(fa, s);
  launch_far_reduce(h->nl, h->d_f1p_lptr.p, h->d_f1p_poff.p, h->d_f1p_lrow.p, h->d_f1p_lsz.p, sp.f1p_y.p, Z,
                    (int)R, s);
  h->prof.end(s);
  if (h->prof.on) {
    h->prof.flops[PC_F1P] += h->f1p_alg_flops1 * (double)R;
    h->prof.bytes[PC_F1P] += h->f1p_alg_bytes;
  }
  return 3;
}

double solve_bytes(const ps_handle* h, int64_t nrhs) {
  double nR = 0, nD = 0, nF = 0;
  for (int64_t p = 0; p < h->nl; ++p) {
    nR += (double)h->nsz[p] * h->S[p];
    nD += (double)h->nsz[p] * h->nsz[p];
  }
  for (int64_t b = 0; b < h->nfar; ++b) nF += (double)h->far_list[7 * b + 5] * (h->far_list[7 * b + 1] + h->far_list[7 * b + 3]);
  // operator: 4 alpha sweeps, 2 D^{-1}, far factors once;
  // vectors: each of ~12 N x nrhs passes (read or write)
  return 16.0 * (4 * nR + 2 * nD + nF) + 16.0 * 12.0 * (double)h->N * nrhs;
}
double solve_flops(const ps_handle* h, int64_t nrhs) {
  double nR = 0, nD = 0, nF = 0;
  for (int64_t p = 0; p < h->nl; ++p) {
    nR += (double)h->nsz[p] * h->S[p];
    nD += (double)h->nsz[p] * h->nsz[p];
  }
  for (int64_t b = 0; b < h->nfar; ++b) nF += (double)h->far_list[7 * b + 5] * (h->far_list[7 * b + 1] + h->far_list[7 * b + 3]);
  return 8.0 * nrhs * (4 * nR + 2 * nD + 2 * nF);
}

// ------------------------------------------------------------------ NCCL (run-time loaded)
// libps does not link NCCL: it is opened on first use (the copy torch already
// loaded when present, else the system one), so single-GPU users need none.
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  static std::string why;
  if (!tried) {
    tried = true;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      why = std::string("cannot load libnccl.so.2: ") + dlerror();
    } else {
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(lib, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(lib, "ncclCommInitRank");
      api.allReduce = (decltype(api.allReduce))dlsym(lib, "ncclAllReduce");
      api.allGather = (decltype(api.allGather))dlsym(lib, "ncclAllGather");
      api.commDestroy = (decltype(api.commDestroy))dlsym(lib, "ncclCommDestroy");
      api.errStr = (decltype(api.errStr))dlsym(lib, "ncclGetErrorString");
      if (!api.getUniqueId || !api.commInitRank || !api.allReduce || !api.allGather || !api.commDestroy)
        why = "libnccl.so.2 lacks a required symbol";
    }
  }
  if (!why.empty()) throw PsError{PS_ENCCL, why};
  return api;
}

#define NCK(x)                                                                                  \
  do {                                                                                          \
    ncclResult_t r_ = (x);                                                                      \
    if (r_ != ncclSuccess)                                                                      \
      throw PsError{PS_ENCCL, std::string(#x) + ": " +                                          \
                                  (nccl_api().errStr ? nccl_api().errStr(r_) : "nccl error")};  \
  } while (0)

// ------------------------------------------------------------------ row-partitioned solve
// Vector layout of the partitioned mode: rank g's interior positions (in
// elimination order) at rows [g maxI, g maxI + own_g), the separators (in
// elimination order) at rows [P maxI, P maxI + Nsep). The separator block and
// every rank block are contiguous, so the exchanges are plain all-reduce /
// all-gather calls on sub-ranges of one buffer.
void dist_layout(ps_handle* h) {
  const int P = h->nranks;
  partition(h, P, h->owner, h->far_owner);
  std::vector<int64_t> cnt(P, 0);
  h->Nsep = 0;
  for (int64_t p = 0; p < h->nl; ++p) {
    if (h->owner[p] >= 0) cnt[h->owner[p]] += h->nsz[p];
    else h->Nsep += h->nsz[p];
  }
  h->maxI = *std::max_element(cnt.begin(), cnt.end());
  h->own_rows = cnt[h->rank];
  h->Npad = P * h->maxI + h->Nsep;
  h->doff.assign(h->nl, 0);
  std::vector<int64_t> next(P);
  for (int g = 0; g < P; ++g) next[g] = g * h->maxI;
  int64_t sn = P * h->maxI;
  for (int64_t p = 0; p < h->nl; ++p) {
    if (h->owner[p] >= 0) { h->doff[p] = next[h->owner[p]]; next[h->owner[p]] += h->nsz[p]; }
    else { h->doff[p] = sn; sn += h->nsz[p]; }
  }
  h->d2rwg.assign(h->Npad, -1);
  for (int64_t p = 0; p < h->nl; ++p) {
    const int32_t l = h->leaf_at[p];
    for (int64_t t = 0; t < h->nsz[p]; ++t) h->d2rwg[h->doff[p] + t] = h->perm[h->leaf_off[l] + t];
  }
}

// Sharded layout of a row-partition rank: the rank holds the rows of
// its own interior positions and of the replicated separators only — W, alpha panels
// and D^-1 in compact arenas (W: interior first, then the separators as one contiguous
// range, summed over the ranks between the two setup phases), the near blocks whose
// row position it assembles (separator rows' near blocks on rank 0 only), and T_c of
// the chains it uses (chains are cut where the owner changes).
void shard_layout(ps_handle* h, std::vector<char>& keep_near) {
  const int64_t nl = h->nl;
  const int g = h->rank;
  h->need.assign(nl, 0);
  for (int64_t p = 0; p < nl; ++p) h->need[p] = (h->owner[p] == g || h->owner[p] < 0) ? 1 : 0;
  build_chains(h, &h->owner);
  int64_t W = 0, P = 0, D = 0;
  h->Woff.assign(nl, -1);
  h->Poff.assign(nl, -1);
  h->Doff.assign(nl, -1);
  for (int pass = 0; pass < 2; ++pass) {               // interior rows, then the separators
    if (pass == 1) h->Wsep0 = W;
    for (int64_t p = 0; p < nl; ++p) {
      if (!(pass == 0 ? h->owner[p] == g : h->owner[p] < 0)) continue;
      h->Woff[p] = W;
      W += (int64_t)h->nsz[p] * (h->nsz[p] + h->S[p]);
    }
  }
  h->Wsep_len = W - h->Wsep0;
  for (int64_t p = 0; p < nl; ++p) {
    if (!h->need[p]) continue;
    h->Poff[p] = P;
    P += (int64_t)h->nsz[p] * h->S[p];
    h->Doff[p] = D;
    D += (int64_t)h->nsz[p] * h->nsz[p];
  }
  h->Wlen = W; h->Plen = P; h->Dlen = D;
  h->Tlen = 0;
  for (size_t c = 0; c < h->chains.size(); ++c) {
    h->ch_Toff[c] = -1;
    if (h->chains[c].size() >= 2 && h->need[h->chains[c][0]]) {
      h->ch_Toff[c] = h->Tlen;
      h->Tlen += h->ch_U[c] * h->ch_U[c];
    }
  }
  keep_near.assign(h->nnear, 0);
  for (int64_t b = 0; b < h->nnear; ++b) {
    const int32_t pi = h->pos_of[h->near_list[3 * b]], pj = h->pos_of[h->near_list[3 * b + 1]];
    const int32_t r = std::min(pi, pj);
    keep_near[b] = (h->owner[r] == g || (h->owner[r] < 0 && g == 0)) ? 1 : 0;
  }
  h->sharded = true;
}

// This rank's tables. Phases and the exchange after each:
//   0  y = B; y[S] = 0 on ranks != 0; forward sweep of the interior subtrees
//      plus their contributions to the separator rows            -> all-reduce y[S]
//   1  separator forward sweep; b_o = D^-1 y; w = R b_o (separators, then
//      interior)                                                  -> all-gather w
//   2  z = Z_F w on this rank's far rows (z[S] = 0 elsewhere); interior forward
//      sweep of z + separator contributions                       -> all-reduce z[S]
//   3  separator forward sweep of z; xt = b_o - D^-1 z; norms of this rank's
//      rows; x = R xt                                             -> all-gather x, all-reduce norms
//   4  X = x in RWG order
void build_dist_plan(ps_handle* h, DistPlan& dp, int64_t R) {
  const int64_t nl = h->nl;
  const int g = h->rank;
  dp.nrhs = R;
  const int64_t NP = h->Npad * R;
  dp.oY = 0; dp.oBO = NP; dp.oW = 2 * NP; dp.oZ = 3 * NP; dp.oXT = 4 * NP; dp.oX = 5 * NP; dp.oTMP = 6 * NP;
  const int64_t ncl = (int64_t)h->cl_start.size();
  std::vector<int64_t> toff(ncl);
  int64_t Ttot = 0;
  for (int64_t c = 0; c < ncl; ++c) { toff[c] = dp.oTMP + Ttot; Ttot += h->cl_sr[c] * R; }
  dp.oSC = dp.oTMP + Ttot;                           // chain scratch (e / f) of the sweeps
  const int narrow = narrow_mode(R);
  for (Table* tb : {&dp.fwdIA, &dp.fwdSA, &dp.dinvA, &dp.bwdA, &dp.far1, &dp.far2, &dp.fwdIC, &dp.fwdSC,
                    &dp.dinvC, &dp.bwdC}) {
    tb->narrow = narrow;
    if (narrow) tb->chunk_steps = NARROW_STEPS();
  }
  auto mine = [&](int64_t p) { return h->owner[p] == g; };
  auto sep = [&](int64_t p) { return h->owner[p] < 0; };
  const int64_t Pb = h->Pbase, Db = h->Dbase, Fb = h->Fbase;
  static const int direct_ends = env_int("PS_DIRECT_ENDS", 1);   // as build_program
  // Chain-collapsed sweeps of the partitioned solve (as build_chain_sweeps): the
  // chain pieces are cut where the owner changes (interior of this rank / another
  // rank / separator); a cut piece uses the principal sub-block of its chain's T_c
  // (the inverse of a block-triangular matrix restricted to a contiguous range of
  // block rows is the inverse of that range's block). Every table gets producer keys.
  struct DPiece { int32_t c, i0, i1, own; };           // chain c nodes [i0, i1), owner value
  std::vector<DPiece> dpieces;
  std::vector<int32_t> dpiece_of(nl, -1);
  for (size_t c = 0; c < h->chains.size(); ++c) {
    const auto& ch = h->chains[c];
    size_t i = 0;
    while (i < ch.size()) {
      size_t j = i + 1;
      while (j < ch.size() && h->owner[ch[j]] == h->owner[ch[i]]) ++j;
      for (size_t q = i; q < j; ++q) dpiece_of[ch[q]] = (int32_t)dpieces.size();
      dpieces.push_back({(int32_t)c, (int32_t)i, (int32_t)j, h->owner[ch[i]]});
      i = j;
    }
  }
  const int64_t SCo = dp.oSC;
  const int wsteps = narrow ? NARROW_STEPS() : 16;
  auto piece_nodes = [&](const DPiece& P) {
    std::vector<int32_t> v;
    for (int32_t i = P.i0; i < P.i1; ++i) v.push_back(h->chains[P.c][i]);
    return v;
  };
  // forward sweep in place on `buf`; interior: this rank's pieces (gathers from its own
  // subtrees) and then the partial sums into separator rows; else the separator pieces
  // (gathers from separator descendants; interior partial sums are already in buf)
  auto fwd = [&](Table& T, int64_t buf, bool interior) {
    T.early_keys = true;
    double key = 0;
    std::vector<int32_t> ft(nl, -1), et(nl, -1);
    std::vector<char> in_buf(nl, 0);
    std::vector<int32_t> order;
    for (size_t k = 0; k < dpieces.size(); ++k)
      if (interior ? dpieces[k].own == g : dpieces[k].own < 0) order.push_back((int32_t)k);
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
      return h->height[h->chains[dpieces[x].c][dpieces[x].i0]] < h->height[h->chains[dpieces[y].c][dpieces[y].i0]];
    });
    for (int32_t k : order) {
      const DPiece& Pc = dpieces[k];
      const auto nodes = piece_nodes(Pc);
      const bool single = nodes.size() == 1;
      T.key_base = key++;
      for (int32_t p : nodes) {
        std::vector<std::pair<int32_t, int32_t>> gl;
        for (auto [d, idx] : h->gath[p])
          if (dpiece_of[d] != k && (interior ? mine(d) : sep(d))) gl.push_back({d, idx});
        const bool direct = single || (direct_ends && p == nodes[0]);   // no T product: write y directly
        if (direct) in_buf[p] = 1;
        if (direct && gl.empty()) continue;
        const int64_t np_ = h->nsz[p];
        int32_t t = T.add_task((direct ? buf : SCo) + h->doff[p] * R, R, 1, buf + h->doff[p] * R, R, 1, (int)np_,
                               (int)R, +1);
        for (auto [d, idx] : gl) {
          const int64_t nd = h->nsz[d];
          T.add_term(t, Pb + h->Poff[d] + h->pcol[d][idx] * nd, nd, 1, buf + h->doff[d] * R, R, 1, (int)nd, ft[d]);
        }
        T.tile(t, 0, wsteps);
        (direct ? ft : et)[p] = t;
      }
      if (single) continue;
      const int64_t U = h->ch_U[Pc.c], To = h->Tbase + h->ch_Toff[Pc.c];
      T.key_base = key++;
      for (size_t i = 0; i < nodes.size(); ++i) {
        const int32_t p = nodes[i];
        if (in_buf[p]) continue;
        const int64_t np_ = h->nsz[p];
        int32_t t = T.add_task(buf + h->doff[p] * R, R, 1, SCo + h->doff[p] * R, R, 1, (int)np_, (int)R, +1);
        T.tasks[t].idep = et[p];
        for (size_t j = 0; j < i; ++j) {
          const int32_t q = nodes[j];
          T.add_term(t, To + h->cpos[p] + h->cpos[q] * U, 1, U, (in_buf[q] ? buf : SCo) + h->doff[q] * R, R, 1,
                     (int)h->nsz[q], in_buf[q] ? ft[q] : et[q]);
        }
        T.tile(t, 0, wsteps);
        ft[p] = t;
      }
    }
    if (interior) {                                   // partial sums into the separator rows
      T.key_base = key++;
      for (int64_t q = 0; q < nl; ++q) {
        if (!sep(q)) continue;
        std::vector<std::pair<int32_t, int32_t>> gl;
        for (auto [d, idx] : h->gath[q])
          if (mine(d)) gl.push_back({d, idx});
        if (gl.empty()) continue;
        const int64_t nq = h->nsz[q];
        int32_t t = T.add_task(buf + h->doff[q] * R, R, 1, buf + h->doff[q] * R, R, 1, (int)nq, (int)R, +1);
        for (auto [d, idx] : gl) {
          const int64_t nd = h->nsz[d];
          T.add_term(t, Pb + h->Poff[d] + h->pcol[d][idx] * nd, nd, 1, buf + h->doff[d] * R, R, 1, (int)nd, ft[d]);
        }
        T.tile(t, 0, wsteps);
      }
    }
    T.sort_close_bounded();
  };
  // D^-1 on this rank's interior and the separators: dst = init + sign D^-1 src
  auto dinv = [&](Table& T, int64_t src, int64_t dst, int64_t init, int sign) {
    for (int64_t p = 0; p < nl; ++p) {
      if (!(mine(p) || sep(p))) continue;
      const int64_t np_ = h->nsz[p];
      int32_t t = T.add_task(dst + h->doff[p] * R, R, 1, init >= 0 ? init + h->doff[p] * R : -1, R, 1, (int)np_,
                             (int)R, sign);
      T.add_term(t, Db + h->Doff[p], 1, np_, src + h->doff[p] * R, R, 1, (int)np_);
      T.tile(t);
    }
    T.close_batch();
  };
  // backward sweep (Eq. 26): separator pieces, then this rank's pieces, top-down; the
  // struct of a node lies in its own subtree's ancestors: this rank or the separators
  auto bwd = [&](Table& T, int64_t in, int64_t out) {
    T.early_keys = true;
    double key = 0;
    std::vector<int32_t> wt(nl, -1), ft(nl, -1);
    std::vector<char> in_buf(nl, 0);
    std::vector<int32_t> order;
    for (size_t k = 0; k < dpieces.size(); ++k)
      if (dpieces[k].own == g || dpieces[k].own < 0) order.push_back((int32_t)k);
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
      return h->height[h->chains[dpieces[x].c][dpieces[x].i1 - 1]] > h->height[h->chains[dpieces[y].c][dpieces[y].i1 - 1]];
    });
    for (int32_t k : order) {
      const DPiece& Pc = dpieces[k];
      const auto nodes = piece_nodes(Pc);
      const bool single = nodes.size() == 1;
      T.key_base = key++;
      for (int32_t p : nodes) {
        const int64_t np_ = h->nsz[p];
        const bool direct = single || (direct_ends && p == nodes.back());   // no T product: write w directly
        if (direct) in_buf[p] = 1;
        int32_t t = T.add_task((direct ? out : SCo) + h->doff[p] * R, R, 1, in + h->doff[p] * R, R, 1, (int)np_,
                               (int)R, +1);
        for (size_t i = 0; i < h->st[p].size(); ++i) {
          const int32_t j = h->st[p][i];
          if (!(mine(j) || sep(j))) throw PsError{PS_ECUDA, "internal: struct leaves the rank's subtree"};
          if (dpiece_of[j] == k) continue;
          T.add_term(t, Pb + h->Poff[p] + h->pcol[p][i] * np_, 1, np_, out + h->doff[j] * R, R, 1,
                     (int)h->nsz[j], wt[j]);
        }
        T.tile(t, 0, wsteps);
        (direct ? wt : ft)[p] = t;
      }
      if (single) continue;
      const int64_t U = h->ch_U[Pc.c], To = h->Tbase + h->ch_Toff[Pc.c];
      T.key_base = key++;
      for (size_t i = 0; i < nodes.size(); ++i) {
        const int32_t p = nodes[i];
        if (in_buf[p]) continue;
        const int64_t np_ = h->nsz[p];
        int32_t t = T.add_task(out + h->doff[p] * R, R, 1, SCo + h->doff[p] * R, R, 1, (int)np_, (int)R, +1);
        T.tasks[t].idep = ft[p];
        for (size_t j = i + 1; j < nodes.size(); ++j) {
          const int32_t q = nodes[j];
          T.add_term(t, To + h->cpos[q] + h->cpos[p] * U, U, 1, (in_buf[q] ? out : SCo) + h->doff[q] * R, R, 1,
                     (int)h->nsz[q], in_buf[q] ? wt[q] : ft[q]);
        }
        T.tile(t, 0, wsteps);
        wt[p] = t;
      }
    }
    T.sort_close_bounded();
  };
  fwd(dp.fwdIA, dp.oY, true);
  fwd(dp.fwdSA, dp.oY, false);
  dinv(dp.dinvA, dp.oY, dp.oBO, -1, +1);
  bwd(dp.bwdA, dp.oBO, dp.oW);
  fwd(dp.fwdIC, dp.oZ, true);
  fwd(dp.fwdSC, dp.oZ, false);
  dinv(dp.dinvC, dp.oZ, dp.oXT, dp.oBO, -1);
  bwd(dp.bwdC, dp.oXT, dp.oX);
  // far field z = Z_F w for the leaves whose far rows this rank computes: stage 2
  // per leaf (as build_program's S5), stage 1 only for the stacked rows it reads
  auto leaf_of_pos = [&](int64_t m) {
    return (int64_t)(std::upper_bound(h->leaf_off.begin(), h->leaf_off.end(), m) - h->leaf_off.begin()) - 1;
  };
  struct Seg { int64_t oA, sAi, sAk, oB; int K; };
  std::vector<std::vector<Seg>> contrib(nl);
  std::vector<std::vector<std::pair<int64_t, int64_t>>> need(ncl);   // stage-1 rows [a, a + r) per cluster
  auto target = [&](int64_t l) { return h->far_owner[h->pos_of[l]] == g; };
  for (int64_t b = 0; b < h->nfar; ++b) {
    const int64_t* F = &h->far_list[7 * b];
    const int64_t r0 = F[0], m = F[1], c0 = F[2], n = F[3], r = F[5];
    if (r == 0) continue;
    const int64_t ct = h->fb_ct[b], cs = h->fb_cs[b];
    if (h->fb_dense[b] >= 0) {
      const int64_t D = Fb + h->fb_dense[b];
      for (int64_t l = leaf_of_pos(r0); l < nl && h->leaf_off[l] < r0 + m; ++l) {
        if (!target(l)) continue;
        for (int64_t q = leaf_of_pos(c0); q < nl && h->leaf_off[q] < c0 + n; ++q)
          contrib[l].push_back({D + (h->leaf_off[l] - r0) + (h->leaf_off[q] - c0) * m, 1, m,
                                dp.oW + h->doff[h->pos_of[q]] * R, (int)(h->leaf_off[q + 1] - h->leaf_off[q])});
      }
      for (int64_t l = leaf_of_pos(c0); l < nl && h->leaf_off[l] < c0 + n; ++l) {
        if (!target(l)) continue;
        for (int64_t q = leaf_of_pos(r0); q < nl && h->leaf_off[q] < r0 + m; ++q)
          contrib[l].push_back({D + (h->leaf_off[q] - r0) + (h->leaf_off[l] - c0) * m, m, 1,
                                dp.oW + h->doff[h->pos_of[q]] * R, (int)(h->leaf_off[q + 1] - h->leaf_off[q])});
      }
      continue;
    }
    bool used_s = false, used_t = false;
    for (int64_t l = leaf_of_pos(r0); l < nl && h->leaf_off[l] < r0 + m; ++l)
      if (target(l)) {
        contrib[l].push_back({Fb + h->cl_soff[ct] + h->fb_rbt[b] + (h->leaf_off[l] - r0) * h->cl_sr[ct],
                              h->cl_sr[ct], 1, toff[cs] + h->fb_rbs[b] * R, (int)r});
        used_s = true;
      }
    for (int64_t l = leaf_of_pos(c0); l < nl && h->leaf_off[l] < c0 + n; ++l)
      if (target(l)) {
        contrib[l].push_back({Fb + h->cl_soff[cs] + h->fb_rbs[b] + (h->leaf_off[l] - c0) * h->cl_sr[cs],
                              h->cl_sr[cs], 1, toff[ct] + h->fb_rbt[b] * R, (int)r});
        used_t = true;
      }
    if (used_s) need[cs].push_back({h->fb_rbs[b], r});    // V_b^T w_s
    if (used_t) need[ct].push_back({h->fb_rbt[b], r});    // U_b^T w_t
  }
  for (int64_t c = 0; c < ncl; ++c) {
    auto& v = need[c];
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    std::vector<std::pair<int64_t, int64_t>> merged;   // (a, end)
    for (auto [a, r] : v) {
      if (!merged.empty() && a <= merged.back().second) merged.back().second = std::max(merged.back().second, a + r);
      else merged.push_back({a, a + r});
    }
    const int64_t sr = h->cl_sr[c], a0 = h->cl_start[c], len = h->cl_len[c];
    for (auto [a, e] : merged) {
      int32_t t = dp.far1.add_task(toff[c] + a * R, R, 1, -1, 0, 0, (int)(e - a), (int)R, +1);
      for (int64_t l = leaf_of_pos(a0); l < nl && h->leaf_off[l] < a0 + len; ++l)
        dp.far1.add_term(t, Fb + h->cl_soff[c] + a + (h->leaf_off[l] - a0) * sr, 1, sr,
                         dp.oW + h->doff[h->pos_of[l]] * R, R, 1, (int)(h->leaf_off[l + 1] - h->leaf_off[l]));
      dp.far1.tile(t);
    }
  }
  dp.far1.close_batch();
  for (int64_t l = 0; l < nl; ++l) {
    if (!target(l)) continue;
    const int32_t pos = h->pos_of[l];
    int32_t t = dp.far2.add_task(dp.oZ + h->doff[pos] * R, R, 1, -1, 0, 0, (int)h->nsz[pos], (int)R, +1);
    for (auto& q : contrib[l]) dp.far2.add_term(t, q.oA, q.sAi, q.sAk, q.oB, R, 1, q.K);
    dp.far2.tile(t);
  }
  dp.far2.close_batch();
  for (Table* tb : {&dp.fwdIA, &dp.fwdSA, &dp.dinvA, &dp.bwdA, &dp.far1, &dp.far2, &dp.fwdIC, &dp.fwdSC,
                    &dp.dinvC, &dp.bwdC})
    tb->upload(h->stream, &h->ring);
  dp.ws.alloc(7 * NP + std::max<int64_t>(Ttot, 1));
  CK(cudaMemsetAsync(dp.ws.p, 0, sizeof(double2) * dp.ws.n, h->stream));   // padding rows stay 0
  dp.nchI = (h->own_rows + dp.rpc - 1) / dp.rpc;
  dp.nchS = h->rank == 0 ? (h->Nsep + dp.rpc - 1) / dp.rpc : 0;
  dp.part.alloc(std::max<int64_t>(dp.nchI + dp.nchS, 1) * R);
  dp.sums.alloc(R);
  dp.scratch.alloc(std::max<int64_t>(std::max(h->Nsep, h->maxI) * R, R));
  CK(cudaStreamSynchronize(h->stream));
}

DistPlan& get_dist_plan(ps_handle* h, int64_t nrhs) {
  if (!h->dplan || h->dplan->nrhs != nrhs) {
    h->dplan.reset();
    auto dp = std::make_unique<DistPlan>();
    build_dist_plan(h, *dp, nrhs);
    h->dplan = std::move(dp);
  }
  return *h->dplan;
}

// One phase of this rank's partitioned solve (see build_dist_plan).
int64_t dist_phase(ps_handle* h, DistPlan& dp, int k, const double2* Bd, int64_t ldb, double2* Xd, int64_t ldx,
                   cudaStream_t s) {
  const int64_t R = dp.nrhs;
  double2* ws = dp.ws.p;
  const double2* A = h->d_op.p;
  const int64_t sep0 = h->nranks * h->maxI;
  Prof* pf = &h->prof;
  int64_t n = 0;
  switch (k) {
    case 0:
      n += aux(h, s, [&] { launch_permute_in(h->Npad, R, h->d_d2rwg.p, Bd, ldb, ws + dp.oY, s); });
      if (h->rank != 0 && h->Nsep > 0)
        CK(cudaMemsetAsync(ws + dp.oY + sep0 * R, 0, sizeof(double2) * h->Nsep * R, s));
      n += dp.fwdIA.launch_all(ws, ws, A, ws, s, pf, PC_FWD);
      break;
    case 1:
      n += dp.fwdSA.launch_all(ws, ws, A, ws, s, pf, PC_FWD);
      n += dp.dinvA.launch_all(ws, ws, A, ws, s, pf, PC_DINV);
      n += dp.bwdA.launch_all(ws, ws, A, ws, s, pf, PC_BWD);
      break;
    case 2:
      if (h->Nsep > 0) CK(cudaMemsetAsync(ws + dp.oZ + sep0 * R, 0, sizeof(double2) * h->Nsep * R, s));
      n += dp.far1.launch_all(ws, ws, A, ws, s, pf, PC_FAR1);
      n += dp.far2.launch_all(ws, ws, A, ws, s, pf, PC_FAR2);
      n += dp.fwdIC.launch_all(ws, ws, A, ws, s, pf, PC_FWD);
      break;
    case 3:
      n += dp.fwdSC.launch_all(ws, ws, A, ws, s, pf, PC_FWD);
      n += dp.dinvC.launch_all(ws, ws, A, ws, s, pf, PC_DINV);
      n += aux(h, s, [&] {    // ||b_o||^2, ||u||^2 = ||b_o - xt||^2 over this rank's rows (Eq. 44)
        const int64_t r0 = h->rank * h->maxI;
        if (h->own_rows > 0)
          launch_norms2(h->own_rows, R, ws + dp.oBO + r0 * R, ws + dp.oXT + r0 * R, dp.part.p, dp.rpc, s);
        if (dp.nchS > 0)
          launch_norms2(h->Nsep, R, ws + dp.oBO + sep0 * R, ws + dp.oXT + sep0 * R, dp.part.p + dp.nchI * R,
                        dp.rpc, s);
        if (dp.nchI + dp.nchS > 0) launch_finalize_norms(dp.nchI + dp.nchS, R, dp.part.p, dp.sums.p, s, 0);
        else CK(cudaMemsetAsync(dp.sums.p, 0, sizeof(double2) * R, s));
      }) + 2;
      n += dp.bwdC.launch_all(ws, ws, A, ws, s, pf, PC_BWD);
      break;
    case 4:
      n += aux(h, s, [&] { launch_permute_out(h->Npad, R, h->d_d2rwg.p, ws + dp.oX, Xd, ldx, s); });
      break;
  }
  return n;
}

// The exchange after phase k, as (offset, count) sub-ranges of the workspace
// (complex elements): kind 0 = sum all-reduce, 1 = all-gather of equal blocks
// (rank g's block at off + g * count), 2 = sum all-reduce of the norm sums.
struct Xchg { int kind; int64_t off, count; };
std::vector<Xchg> dist_exchanges(const ps_handle* h, const DistPlan& dp, int k) {
  const int64_t R = dp.nrhs, sep0 = h->nranks * h->maxI;
  switch (k) {
    case 0: return {{0, dp.oY + sep0 * R, h->Nsep * R}};
    case 1: return {{1, dp.oW, h->maxI * R}};
    case 2: return {{0, dp.oZ + sep0 * R, h->Nsep * R}};
    case 3: return {{1, dp.oX, h->maxI * R}, {2, 0, R}};
  }
  return {};
}

void nccl_exchange(ps_handle* h, DistPlan& dp, int k, cudaStream_t s) {
  NcclApi& api = nccl_api();
  ncclComm_t comm = (ncclComm_t)h->nccl;
  for (const Xchg& x : dist_exchanges(h, dp, k)) {
    if (x.count <= 0) continue;
    if (x.kind == 1) {
      double2* base = dp.ws.p + x.off;
      NCK(api.allGather(base + h->rank * x.count, base, 2 * x.count, ncclDouble, comm, s));
    } else {
      double2* p = x.kind == 2 ? dp.sums.p : dp.ws.p + x.off;
      NCK(api.allReduce(p, p, 2 * x.count, ncclDouble, ncclSum, comm, s));
    }
  }
}

// The partitioned solve over `nh` handles: nh = 1 with an NCCL communicator
// (this rank's share, collectives through NCCL), or nh = nranks handles of an
// in-process group (phases in rank order, group_exchange between them).
void group_exchange(ps_handle* const* hs, int P, int k, cudaStream_t s);
void dist_solve(ps_handle* const* hs, int nh, int64_t nrhs, const void* B, int64_t ldb, void* X, int64_t ldx,
                int on_device, cudaStream_t s, std::vector<double2>& norms, int64_t& launches, float& ms) {
  ps_handle* h0 = hs[0];
  const int64_t N = h0->N, R = nrhs;
  for (int i = 0; i < nh; ++i) get_dist_plan(hs[i], nrhs);
  DistPlan& d0 = *h0->dplan;
  const double2* Bd = (const double2*)B;
  double2* Xd = (double2*)X;
  int64_t ldb_d = ldb, ldx_d = ldx;
  if (!on_device) {          // stage through d0.ws's TMP tail is not safe; use a dedicated buffer
    if (d0.scratch.n < 2 * N * R) d0.scratch.alloc(std::max<int64_t>(2 * N * R, d0.scratch.n));
    CK(cudaMemcpy2DAsync(d0.scratch.p, 16 * N, B, 16 * ldb, 16 * N, nrhs, cudaMemcpyHostToDevice, s));
    Bd = d0.scratch.p;
    Xd = d0.scratch.p + N * R;
    ldb_d = ldx_d = N;
  }
  CK(cudaEventRecord(h0->ev0, s));
  launches = 0;
  for (int k = 0; k < 5; ++k) {
    for (int i = 0; i < nh; ++i)
      if (k < 4 || i == 0) launches += dist_phase(hs[i], *hs[i]->dplan, k, Bd, ldb_d, Xd, ldx_d, s);
    if (k < 4) {
      if (nh == 1) nccl_exchange(h0, d0, k, s);
      else group_exchange(hs, nh, k, s);
    }
  }
  CK(cudaEventRecord(h0->ev1, s));
  CK(cudaGetLastError());
  if (!on_device)
    CK(cudaMemcpy2DAsync(X, 16 * ldx, Xd, 16 * N, 16 * N, nrhs, cudaMemcpyDeviceToHost, s));
  norms.assign(R, double2{0.0, 0.0});
  CK(cudaMemcpyAsync(norms.data(), d0.sums.p, 16 * R, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (auto& v : norms) v = double2{std::sqrt(v.x), std::sqrt(v.y)};
  CK(cudaEventElapsedTime(&ms, h0->ev0, h0->ev1));
  for (int i = 0; i < nh; ++i)
    if (hs[i]->prof.on) hs[i]->prof.collect();
}

// In-process group (ps_solve_group): the same exchanges between the ranks'
// workspaces on one device, summing in rank order.
void group_exchange(ps_handle* const* hs, int P, int k, cudaStream_t s) {
  const std::vector<Xchg> xs = dist_exchanges(hs[0], *hs[0]->dplan, k);
  for (const Xchg& x : xs) {
    if (x.count <= 0) continue;
    const size_t bytes = sizeof(double2) * x.count;
    auto at = [&](int g) { DistPlan& d = *hs[g]->dplan; return x.kind == 2 ? d.sums.p : d.ws.p + x.off; };
    if (x.kind == 1) {
      for (int src = 0; src < P; ++src)
        for (int dst = 0; dst < P; ++dst)
          if (dst != src)
            CK(cudaMemcpyAsync(at(dst) + src * x.count, at(src) + src * x.count, bytes, cudaMemcpyDeviceToDevice, s));
    } else {
      double2* acc = hs[0]->dplan->scratch.p;
      CK(cudaMemcpyAsync(acc, at(0), bytes, cudaMemcpyDeviceToDevice, s));
      for (int g = 1; g < P; ++g) launch_add((double*)acc, (const double*)at(g), 2 * x.count, s);
      for (int g = 0; g < P; ++g) CK(cudaMemcpyAsync(at(g), acc, bytes, cudaMemcpyDeviceToDevice, s));
    }
  }
}

}  // namespace

namespace {
ps_status finish_dist(ps_handle* const* hs, int nh, int64_t nrhs, const void* B, int64_t ldb, void* X,
                      int64_t ldx, int on_device, void* cuda_stream, ps_report* rep, const char* who) {
  ps_handle* h = hs[0];
  try {
    CK(cudaSetDevice(h->device));
    cudaStream_t s = cuda_stream ? (cudaStream_t)cuda_stream : h->stream;
    std::vector<double2> norms;
    int64_t launches = 0;
    float ms = 0;
    dist_solve(hs, nh, nrhs, B, ldb, X, ldx, on_device, s, norms, launches, ms);
    int ndiv = 0;
    for (int64_t c = 0; c < nrhs; ++c) {
      const double r = norms[c].x > 0 ? norms[c].y / norms[c].x : 0.0;
      if (!(r < h->ratio_threshold)) ++ndiv;
    }
    if (rep) {
      rep->t_solve_ms = ms;
      rep->n_diverged = ndiv;
      rep->bytes_moved = solve_bytes(h, nrhs);
      rep->flops = solve_flops(h, nrhs);
      rep->kernel_launches = launches;
      const int64_t cap = std::min<int64_t>(rep->nrhs, nrhs);
      for (int64_t c = 0; c < cap; ++c) {
        if (rep->it0_norm) rep->it0_norm[c] = norms[c].x;
        if (rep->it1_norm) rep->it1_norm[c] = norms[c].y;
        if (rep->ratio) rep->ratio[c] = norms[c].x > 0 ? norms[c].y / norms[c].x : 0.0;
      }
    }
    if (ndiv > 0)
      return fail(h, PS_EDIVERGED, std::string(who) + ": " + std::to_string(ndiv) + " of " + std::to_string(nrhs) +
                                       " columns have ||it_1||/||it_0|| >= " + std::to_string(h->ratio_threshold));
  } catch (const PsError& e) {
    return fail(h, e.st, std::string(who) + ": " + e.msg);
  } catch (const std::bad_alloc&) {
    return fail(h, PS_ENOMEM, std::string(who) + ": host allocation failed");
  }
  return PS_OK;
}

// ------------------------------------------------------------------ setup driver
// The positions, elimination level by elimination level (setup tables are built,
// launched and freed per level): mode as build_setup_level; modes 0 and 2 also invert
// the scaled diagonal blocks (Eqs. 23, 30) and form the alpha panels (Eq. 16).
// The elimination levels of ps_setup, bottom-up. Each level's host tables (assembly, panel,
// inverse lists) depend only on the structure, so worker threads build them ahead of the GPU
// (at most PS_SETUP_AHEAD levels ahead); the main thread uploads and launches level after level
// without waiting for the device (stream order protects the reused device buffers), and the
// singular-block flags of every level are checked once at the end.
void setup_levels(ps_handle* h, cudaStream_t s, const std::vector<int32_t>& pos, int mode) {
  if (pos.empty()) return;
  using clk = std::chrono::steady_clock;
  static const int verbose = env_int("PS_VERBOSE", 0);
  double t_wait_host = 0, t_up = 0;
  const auto t00 = clk::now();
  std::vector<std::vector<int32_t>> lv(h->max_height + 1);
  for (int32_t p : pos) lv[mode == 1 ? 0 : h->height[p]].push_back(p);   // phase B: one batch
  std::vector<const std::vector<int32_t>*> order;
  for (const auto& l : lv)
    if (!l.empty()) order.push_back(&l);
  const int L = (int)order.size();
  DevBuf<int32_t> d_status;
  d_status.alloc(std::max<int64_t>((int64_t)pos.size(), 1));
  CK(cudaMemsetAsync(d_status.p, 0, sizeof(int32_t) * d_status.n, s));
  static const int nthreads = std::max(1, std::min(env_int("PS_SETUP_THREADS", 8),
                                                   (int)std::thread::hardware_concurrency()));
  static const int ahead = std::max(1, env_int("PS_SETUP_AHEAD", 32));
  std::vector<std::unique_ptr<SetupLevel>> built(L);
  std::vector<char> ready(L, 0);
  std::mutex mu;
  std::condition_variable cv;
  int next = 0, consumed = 0;
  bool stop = false;
  std::exception_ptr err;
  auto worker = [&] {
    for (;;) {
      int i;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || (next < L && next < consumed + ahead); });
        if (stop || next >= L) return;
        i = next++;
      }
      auto lvl = std::make_unique<SetupLevel>();
      try {
        build_setup_level(h, *order[i], *lvl, mode);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err) err = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        built[i] = std::move(lvl);
        ready[i] = 1;
      }
      cv.notify_all();
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < std::min(nthreads, L); ++t) pool.emplace_back(worker);
  auto finish = [&] {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& th : pool) th.join();
    pool.clear();
  };
  // two device table sets used by alternate levels: level i's uploads (upload stream) wait for
  // the kernels of level i - 2 (the previous user of the set); its kernels wait for its uploads
  SetupLevel dev[2];
  if (!h->ustream) CK(cudaStreamCreateWithFlags(&h->ustream, cudaStreamNonBlocking));
  cudaEvent_t kdone[2], udone;
  for (auto& e : kdone) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&udone, cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t* k; cudaEvent_t u;
    ~EvGuard() { cudaEventDestroy(k[0]); cudaEventDestroy(k[1]); cudaEventDestroy(u); }
  } evg{kdone, udone};
  int64_t off = 0;
  try {
    for (int i = 0; i < L; ++i) {
      SetupLevel& sp = dev[i & 1];
      const auto t0 = clk::now();
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return ready[i] || err; });
        if (err) std::rethrow_exception(err);
        sp.adopt(*built[i]);
        built[i].reset();
        consumed = i + 1;
      }
      cv.notify_all();
      t_wait_host += std::chrono::duration<double>(clk::now() - t0).count();
      if (mode == 2) sp.asmb.S = h->d_W.p;
      if (i >= 2) CK(cudaStreamWaitEvent(h->ustream, kdone[i & 1], 0));
      upload_setup_level(h, sp, h->ustream);
      CK(cudaEventRecord(udone, h->ustream));
      CK(cudaStreamWaitEvent(s, udone, 0));
      t_up += sp.t_upload;
      // Eq. 21 (left-looking): assemble W_p = [Z~_pp | Z~_p,struct(p)]
      sp.asmb.launch_all(h->d_W.p, h->d_near.p, h->d_P.p, h->d_W.p, s);
      if (mode != 1) {
        // Eqs. 23/30: D_p^{-1}
        launch_inverse(sp.nlev, sp.d_ids.p, sp.d_sz.p, sp.d_src.p, sp.d_ld.p, sp.d_dst.p, h->d_W.p, h->d_D.p,
                       d_status.p + off, sp.maxn, s);
        // Eq. 16: alpha_p* = -D_p^{-1} Z~_p*
        sp.panel.launch_all(h->d_P.p, nullptr, h->d_D.p, h->d_W.p, s);
      }
      CK(cudaEventRecord(kdone[i & 1], s));
      off += sp.nlev;
    }
  } catch (...) {
    finish();
    throw;
  }
  finish();
  std::vector<int32_t> status(pos.size(), 0);
  CK(cudaMemcpyAsync(status.data(), d_status.p, sizeof(int32_t) * status.size(), cudaMemcpyDeviceToHost, s));
  const auto t1 = clk::now();
  CK(cudaStreamSynchronize(s));
  const double t_wait = std::chrono::duration<double>(clk::now() - t1).count();
  if (mode != 1) {
    int64_t o = 0;
    for (int i = 0; i < L; ++i)
      for (size_t j = 0; j < order[i]->size(); ++j, ++o)
        if (status[o]) {
          const int32_t p = (*order[i])[j];
          throw PsError{PS_ESINGULAR, "singular scaled diagonal block at elimination position " + std::to_string(p) +
                                          " (leaf " + std::to_string(h->leaf_at[p]) + ")"};
        }
  }
  if (verbose)
    std::fprintf(stderr, "[ps] setup mode %d: %zu positions, %d levels, %.1f ms (waiting on host tables %.1f ms, "
                 "uploads %.1f ms, final wait on the GPU %.1f ms, %d builder threads)\n", mode, pos.size(), L,
                 1e3 * std::chrono::duration<double>(clk::now() - t00).count(), 1e3 * t_wait_host, 1e3 * t_up,
                 1e3 * t_wait, nthreads);
}

// After the scaling: free the setup-only arenas, upload the far stacks, form T_c.
void setup_finish(ps_handle* h, cudaStream_t s) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  h->d_W.release();
  h->d_near.release();
  const auto t1 = clk::now();
  ensure_far(h, s);
  const auto t2 = clk::now();
  h->d_T.alloc(std::max<int64_t>(h->Tlen, 1));
  h->Tbase = (int64_t)(h->d_T.p - h->d_op.p);
  chain_setup(h, s);
  CK(cudaStreamSynchronize(s));
  static const int verbose = env_int("PS_VERBOSE", 0);
  if (verbose)
    std::fprintf(stderr, "[ps] setup finish: %.1f ms (free W / near %.1f, far upload %.1f, chain matrices %.1f)\n",
                 1e3 * std::chrono::duration<double>(clk::now() - t0).count(),
                 1e3 * std::chrono::duration<double>(t1 - t0).count(), 1e3 * std::chrono::duration<double>(t2 - t1).count(),
                 1e3 * std::chrono::duration<double>(clk::now() - t2).count());
  h->plan.reset();                                  // plans made before setup (ps_apply Z_F) are stale
  h->dplan.reset();
  h->setup_done = true;
}

// Sharded setup of a row-partition rank, phase 0: the rank's own
// interior subtrees completely (their updates never leave the subtree), then its
// interior's partial Schur updates of every separator row (phase B; rank 0 adds the
// separator rows' near blocks). Phase 1, after the W separator range has been summed
// over the ranks: the separators themselves, level by level, replicated.
void setup_sharded(ps_handle* h, cudaStream_t s, int phase) {
  std::vector<int32_t> own, sep;
  for (int64_t p = 0; p < h->nl; ++p) {
    if (h->owner[p] == h->rank) own.push_back((int32_t)p);
    else if (h->owner[p] < 0) sep.push_back((int32_t)p);
  }
  if (phase == 0) {
    h->d_W.alloc(std::max<int64_t>(h->Wlen, 1));
    if (h->Wsep_len > 0) CK(cudaMemsetAsync(h->d_W.p + h->Wsep0, 0, sizeof(double2) * h->Wsep_len, s));
    setup_levels(h, s, own, 0);
    setup_levels(h, s, sep, 1);
    CK(cudaStreamSynchronize(s));
  } else {
    setup_levels(h, s, sep, 2);
    setup_finish(h, s);
  }
}

ps_status check_setup_opts(ps_handle* h, const ps_setup_opts* opts) {
  if (h->setup_done) return fail(h, PS_ESTATE, "ps_setup: already set up");
  if (opts) {
    if ((opts->ordering != 0 && opts->ordering != 2) || opts->amalgamate_separators != 0)
      return fail(h, PS_EINVAL, "ps_setup: ordering must be 0 (file ND) or 2 (RCM); amalgamate_separators 0");
    if (opts->ordering == 2 && h->part_mode)
      return fail(h, PS_EINVAL, "ps_setup: ordering=2 is not supported with a row partition");
    if (!(opts->ratio_threshold > 0.0)) return fail(h, PS_EINVAL, "ps_setup: ratio_threshold must be > 0");
    h->ratio_threshold = opts->ratio_threshold;
  }
  return PS_OK;
}

}  // namespace

// ======================================================================= C ABI
extern "C" {

ps_status hm_load(const char* path, const ps_dist* dist, ps_handle** out) {
  if (!out) return fail(nullptr, PS_EINVAL, "hm_load: out is NULL");
  *out = nullptr;
  if (!path) return fail(nullptr, PS_EINVAL, "hm_load: path is NULL");
  if (dist && (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks ||
               (dist->nccl_unique_id && !dist->partition)))
    return fail(nullptr, PS_EINVAL, "hm_load: bad ps_dist (rank/nranks, or nccl_unique_id without partition)");
  std::unique_ptr<ps_handle> h(new ps_handle());
  try {
    std::vector<double2> near_arena, far_arena;
    const bool part = dist && dist->partition && dist->nranks > 1;
    h->path = path;
    read_file(h.get(), path, near_arena, far_arena, /*defer_near=*/part);
    symbolic(h.get());
    if (dist) {
      h->rank = dist->rank;
      h->nranks = dist->nranks;
      if (part) {                                    // row partition: this rank's share only
        h->part_mode = 1;
        dist_layout(h.get());
        std::vector<char> keep;
        shard_layout(h.get(), keep);
        load_near(h.get(), keep, near_arena);
      }
    }
    if (dist) {
      h->device = dist->device;
      CK(cudaSetDevice(h->device));
    } else {
      CK(cudaGetDevice(&h->device));
    }
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&h->ev0));
    CK(cudaEventCreate(&h->ev1));
    h->d_near.upload(near_arena, h->stream);
    {
      far_layout(h.get(), far_arena, h->far_host);
      far_arena.clear();
      far_arena.shrink_to_fit();
      h->Pbase = 0;
      h->Dbase = h->Plen;
      h->d_op.alloc(h->Plen + h->Dlen);
      h->d_P.p = h->d_op.p + h->Pbase;
      h->d_D.p = h->d_op.p + h->Dbase;
    }
    h->d_e2rwg.upload(h->e2rwg, h->stream);
    h->d_e2mort.upload(h->e2mort, h->stream);
    h->d_m2e.upload(h->m2e, h->stream);
    if (h->part_mode) h->d_d2rwg.upload(h->d2rwg, h->stream);
    CK(cudaStreamSynchronize(h->stream));
    if (h->part_mode && dist->nccl_unique_id) {      // collective: every rank joins
      ncclUniqueId id;
      std::memcpy(&id, dist->nccl_unique_id, sizeof(id));
      ncclComm_t comm;
      NCK(nccl_api().commInitRank(&comm, h->nranks, id, h->rank));
      h->nccl = comm;
    }
  } catch (const PsError& e) {
    return fail(nullptr, e.st, "hm_load: " + e.msg);
  } catch (const std::bad_alloc&) {
    return fail(nullptr, PS_ENOMEM, "hm_load: host allocation failed");
  }
  *out = h.release();
  return PS_OK;
}

ps_status ps_setup(ps_handle* h, const ps_setup_opts* opts) {
  if (!h) return fail(nullptr, PS_EINVAL, "ps_setup: handle is NULL");
  if (ps_status st = check_setup_opts(h, opts); st != PS_OK) return st;
  if (h->part_mode && !h->nccl)
    return fail(h, PS_ESTATE, "ps_setup: in-process row-partition handle (no NCCL id): use ps_setup_group");
  try {
    CK(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    if (h->part_mode) {
      setup_sharded(h, s, 0);
      if (h->Wsep_len > 0)                          // sum the separator rows' partial W over the ranks
        NCK(nccl_api().allReduce(h->d_W.p + h->Wsep0, h->d_W.p + h->Wsep0, 2 * h->Wsep_len, ncclDouble, ncclSum,
                                 (ncclComm_t)h->nccl, s));
      setup_sharded(h, s, 1);
    } else {
      using clk = std::chrono::steady_clock;
      const auto t0 = clk::now();
      if (opts && opts->ordering == 2) reorder_rcm(h, s);
      h->d_W.alloc(std::max<int64_t>(h->Wlen, 1));
      const auto t1 = clk::now();
      std::vector<int32_t> all(h->nl);
      std::iota(all.begin(), all.end(), 0);
      setup_levels(h, s, all, 0);
      const auto t2 = clk::now();
      setup_finish(h, s);
      static const int verbose = env_int("PS_VERBOSE", 0);
      if (verbose)
        std::fprintf(stderr, "[ps] ps_setup: %.1f ms (arenas %.1f, levels %.1f, finish %.1f)\n",
                     1e3 * std::chrono::duration<double>(clk::now() - t0).count(),
                     1e3 * std::chrono::duration<double>(t1 - t0).count(), 1e3 * std::chrono::duration<double>(t2 - t1).count(),
                     1e3 * std::chrono::duration<double>(clk::now() - t2).count());
    }
  } catch (const PsError& e) {
    h->d_W.release();
    return fail(h, e.st, "ps_setup: " + e.msg);
  } catch (const std::bad_alloc&) {
    return fail(h, PS_ENOMEM, "ps_setup: host allocation failed");
  }
  return PS_OK;
}

ps_status ps_setup_group(ps_handle* const* hs, int nranks, const ps_setup_opts* opts) {
  if (!hs || nranks < 2 || !hs[0]) return fail(nullptr, PS_EINVAL, "ps_setup_group: need nranks >= 2 handles");
  ps_handle* h = hs[0];
  for (int g = 0; g < nranks; ++g) {
    if (!hs[g] || !hs[g]->part_mode || hs[g]->nccl || hs[g]->rank != g || hs[g]->nranks != nranks ||
        hs[g]->N != h->N || hs[g]->device != h->device || hs[g]->Wsep_len != h->Wsep_len)
      return fail(h, PS_EINVAL, "ps_setup_group: handles must be ranks 0..nranks-1 of one in-process row partition");
    if (ps_status st = check_setup_opts(hs[g], opts); st != PS_OK) return st;
  }
  try {
    CK(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    for (int g = 0; g < nranks; ++g) setup_sharded(hs[g], hs[g]->stream, 0);
    if (h->Wsep_len > 0) {                          // in-process sum over the ranks, rank order
      const size_t bytes = sizeof(double2) * h->Wsep_len;
      DevBuf<double2> acc;
      acc.alloc(h->Wsep_len);
      CK(cudaMemcpyAsync(acc.p, h->d_W.p + h->Wsep0, bytes, cudaMemcpyDeviceToDevice, s));
      for (int g = 1; g < nranks; ++g)
        launch_add((double*)acc.p, (const double*)(hs[g]->d_W.p + hs[g]->Wsep0), 2 * h->Wsep_len, s);
      for (int g = 0; g < nranks; ++g)
        CK(cudaMemcpyAsync(hs[g]->d_W.p + hs[g]->Wsep0, acc.p, bytes, cudaMemcpyDeviceToDevice, s));
      CK(cudaStreamSynchronize(s));
    }
    for (int g = 0; g < nranks; ++g) setup_sharded(hs[g], hs[g]->stream, 1);
  } catch (const PsError& e) {
    for (int g = 0; g < nranks; ++g) hs[g]->d_W.release();
    return fail(h, e.st, "ps_setup_group: " + e.msg);
  } catch (const std::bad_alloc&) {
    return fail(h, PS_ENOMEM, "ps_setup_group: host allocation failed");
  }
  return PS_OK;
}

static ps_status finish_report(ps_handle* h, const double2* d_norms, int64_t R, int64_t launches, cudaStream_t s,
                                ps_report* rep);

// Every kernel of one two-term solve of sp.nrhs columns, queued on s: Bd / Xd are DEVICE
// column-major blocks (ld ldb_d / ldx_d). Returns the number of launches.
static int64_t queue_solve(ps_handle* h, SolvePlan& sp, const double2* Bd, int64_t ldb_d, double2* Xd,
                           int64_t ldx_d, cudaStream_t s) {
  const int64_t N = h->N, R = sp.nrhs;
  int64_t launches = 0;
  {
    // default: the whole solve as one dataflow launch (build_program: chain-collapsed
    // sweeps, E-order far field, producer-keyed tickets); PS_SOLVE=stages runs one
    // launch per operator (the tables ps_apply uses)
    static const bool stages_env = use_stages();
    double2* xres = sp.xt.p;   // where x ends up (elimination order)
    if (!stages_env) {
      // the whole solve as one dataflow program (build_program)
      double2* ws = sp.ws.p;
      launches += aux(h, s, [&] { launch_permute_in(N, R, h->d_e2rwg.p, Bd, ldb_d, ws + sp.oY, s); });
      if (sp.f1p) {
        launches += sp.prog.launch(0, ws, ws, h->d_op.p, ws, s, &h->prof, PC_PROG);
        launches += far1p_apply(h, sp, ws + sp.oW, ws + sp.oZ, s);
        launches += sp.prog.launch(1, ws, ws, h->d_op.p, ws, s, &h->prof, PC_PROG);
        if (h->prof.on) {
          h->prof.flops[PC_PROG] += sp.prog.alg_flops;
          h->prof.bytes[PC_PROG] += sp.prog.alg_bytes;
        }
      } else {
        launches += sp.prog.launch_all(ws, ws, h->d_op.p, ws, s, &h->prof, PC_PROG);
      }
      launches += aux(h, s, [&] {
        launch_norms2(N, R, ws + sp.oBO, ws + sp.oXT, sp.part.p, sp.rpc, s);
        launch_finalize_norms(sp.nchunks, R, sp.part.p, sp.norms.p, s);
      }) + 1;
      xres = ws + sp.oX;
    } else {
    launches += aux(h, s, [&] { launch_permute_in(N, R, h->d_e2rwg.p, Bd, ldb_d, sp.y.p, s); });  // RWG -> E
    launches += op_Rt(h, sp, sp.y.p, s);                                // b~ = R^T b     (Eq. 24)
    launches += op_Dinv(h, sp, sp.y.p, sp.bo.p, s);                     // b_o = D^-1 b~  (Eq. 32)
    launches += op_R(h, sp, sp.bo.p, sp.w.p, s);                        // w = R b_o
    launches += op_ZF(h, sp, sp.w.p, sp.y.p, s);                        // t = Z_F w
    launches += op_Rt(h, sp, sp.y.p, s);                                // z = R^T t
    launches += op_Dinv(h, sp, sp.y.p, sp.u.p, s);                      // u = D^-1 z = U b_o (Eq. 31)
    launches += aux(h, s, [&] {                                         // x~ = b_o - u (Eq. 36), norms
      launch_combine_norms(N, R, sp.bo.p, sp.u.p, sp.xt.p, sp.part.p, sp.rpc, s);
      launch_finalize_norms(sp.nchunks, R, sp.part.p, sp.norms.p, s);
    }) + 1;
    launches += op_R(h, sp, sp.xt.p, sp.xt.p, s);                       // x = R x~       (Eq. 26)
    }
    launches += aux(h, s, [&] { launch_permute_out(N, R, h->d_e2rwg.p, xres, Xd, ldx_d, s); });
  }
  return launches;
}


// ps_solve with HOST buffers and many columns: the block is solved as two column halves of equal
// width c = ceil(nrhs / 2) (one plan; an odd block's second half carries one padding column
// that is never copied out), so that the copies overlap the kernels: H2D of both halves on
// one copy stream, the halves' kernels on s in turn (each waits for its own H2D), D2H of a half
// on a second copy stream as soon as its permute_out is done (half 0's D2H and half 1's H2D run
// under the other half's kernels). Columns are independent problems (Eqs. 24-36 act column by
// column), so the result is the narrower launch's; s waits for the last D2H before the report.
static ps_status solve_host_pipelined(ps_handle* h, int64_t nrhs, const void* B, int64_t ldb, void* X, int64_t ldx,
                                      cudaStream_t s, ps_report* rep) {
  const int64_t N = h->N, c = (nrhs + 1) / 2;
  if (!h->cs_in) {
    CK(cudaStreamCreateWithFlags(&h->cs_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->cs_out, cudaStreamNonBlocking));
    for (auto& e : h->hp_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  SolvePlan& sp = get_plan(h, c);
  for (int i = 0; i < 2; ++i) {
    if (h->hp_in[i].cap < N * c) {
      h->hp_in[i].alloc(N * c);
      CK(cudaMemsetAsync(h->hp_in[i].p, 0, 16 * N * c, s));        // the padding column stays finite
    }
    h->hp_out[i].alloc(N * c);
  }
  h->hp_norms.alloc(2 * c);
  const double2* Bh = (const double2*)B;
  double2* Xh = (double2*)X;
  const int64_t w[2] = {c, nrhs - c};
  CK(cudaEventRecord(h->ev0, s));
  CK(cudaEventRecord(h->hp_ev[0], s));                 // the copy streams start after s's earlier work
  CK(cudaStreamWaitEvent(h->cs_in, h->hp_ev[0], 0));
  CK(cudaStreamWaitEvent(h->cs_out, h->hp_ev[0], 0));
  for (int i = 0; i < 2; ++i) {
    CK(cudaMemcpy2DAsync(h->hp_in[i].p, 16 * N, Bh + (int64_t)i * c * ldb, 16 * ldb, 16 * N, w[i],
                         cudaMemcpyHostToDevice, h->cs_in));
    CK(cudaEventRecord(h->hp_ev[1 + i], h->cs_in));
  }
  int64_t launches = 0;
  for (int i = 0; i < 2; ++i) {
    CK(cudaStreamWaitEvent(s, h->hp_ev[1 + i], 0));
    launches += queue_solve(h, sp, h->hp_in[i].p, N, h->hp_out[i].p, N, s);
    CK(cudaMemcpyAsync(h->hp_norms.p + (int64_t)i * c, sp.norms.p, 16 * c, cudaMemcpyDeviceToDevice, s));
    CK(cudaEventRecord(h->hp_ev[3 + i], s));
    CK(cudaStreamWaitEvent(h->cs_out, h->hp_ev[3 + i], 0));
    CK(cudaMemcpy2DAsync(Xh + (int64_t)i * c * ldx, 16 * ldx, h->hp_out[i].p, 16 * N, 16 * N, w[i],
                         cudaMemcpyDeviceToHost, h->cs_out));
  }
  CK(cudaEventRecord(h->hp_ev[5], h->cs_out));
  CK(cudaStreamWaitEvent(s, h->hp_ev[5], 0));
  CK(cudaEventRecord(h->ev1, s));
  CK(cudaGetLastError());
  sp.launches_per_solve = launches / 2;
  return finish_report(h, h->hp_norms.p, nrhs, launches, s, rep);
}

// ps_solve (defer = false) and ps_solve_async (defer = true: device buffers, no host
// synchronisation; the report is fetched later by ps_solve_report)
static ps_status solve_impl(ps_handle* h, int64_t nrhs, const void* B, int64_t ldb, void* X, int64_t ldx,
                            int on_device, void* cuda_stream, ps_report* rep, bool defer) {
  if (!h) return fail(nullptr, PS_EINVAL, "ps_solve: handle is NULL");
  if (!h->setup_done) return fail(h, PS_ESTATE, "ps_solve: ps_setup has not run");
  if (nrhs < 1 || !B || !X || ldb < h->N || ldx < h->N)
    return fail(h, PS_EINVAL, "ps_solve: bad arguments (nrhs >= 1, B/X non-NULL, ldb/ldx >= N)");
  {
    const char* b0 = (const char*)B;
    const char* b1 = b0 + 16 * (ldb * (nrhs - 1) + h->N);
    const char* x0 = (const char*)X;
    const char* x1 = x0 + 16 * (ldx * (nrhs - 1) + h->N);
    if (b0 < x1 && x0 < b1) return fail(h, PS_EINVAL, "ps_solve: X overlaps B");
  }
  if (h->part_mode) {
    if (!h->nccl)
      return fail(h, PS_ESTATE, "ps_solve: in-process row-partition handle (no NCCL id): use ps_solve_group");
    ps_handle* hs[1] = {h};
    return finish_dist(hs, 1, nrhs, B, ldb, X, ldx, on_device, cuda_stream, rep, "ps_solve");
  }
  try {
    CK(cudaSetDevice(h->device));
    cudaStream_t s = cuda_stream ? (cudaStream_t)cuda_stream : h->stream;
    static const int64_t pipe_min = env_int("PS_HOST_PIPE_MIN", 256);
    if (!on_device && !defer && nrhs >= pipe_min && nrhs >= 2) return solve_host_pipelined(h, nrhs, B, ldb, X, ldx, s, rep);
    SolvePlan& sp = get_plan(h, nrhs);
    const int64_t N = h->N, R = nrhs;
    int64_t launches = 0;
    const double2* Bd = (const double2*)B;
    int64_t ldb_d = ldb;
    if (!on_device) {
      CK(cudaMemcpy2DAsync(sp.stage.p, 16 * N, B, 16 * ldb, 16 * N, nrhs, cudaMemcpyHostToDevice, s));
      Bd = sp.stage.p;
      ldb_d = N;
    }
    CK(cudaEventRecord(h->ev0, s));
    launches += queue_solve(h, sp, Bd, ldb_d, on_device ? (double2*)X : sp.stage.p, on_device ? ldx : N, s);
    CK(cudaEventRecord(h->ev1, s));
    CK(cudaGetLastError());
    sp.launches_per_solve = launches;
    h->pend_nrhs = R;
    h->pend_stream = s;
    if (defer) return PS_OK;
    if (!on_device)
      CK(cudaMemcpy2DAsync(X, 16 * ldx, sp.stage.p, 16 * N, 16 * N, nrhs, cudaMemcpyDeviceToHost, s));
    return finish_report(h, sp.norms.p, R, launches, s, rep);
  } catch (const PsError& e) {
    return fail(h, e.st, "ps_solve: " + e.msg);
  } catch (const std::bad_alloc&) {
    return fail(h, PS_ENOMEM, "ps_solve: host allocation failed");
  }
  return PS_OK;
}

// the host half of a solve: norms of the plan's last solve read back (synchronises s), Eq. 45
// ratios, divergence status, report
static ps_status finish_report(ps_handle* h, const double2* d_norms, int64_t R, int64_t launches, cudaStream_t s,
                                ps_report* rep) {
  {
    std::vector<double2> norms(R);
    CK(cudaMemcpyAsync(norms.data(), d_norms, 16 * R, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    h->pend_nrhs = 0;
    if (h->prof.on) h->prof.collect();
    int ndiv = 0;
    for (int64_t c = 0; c < R; ++c) {
      const double r = norms[c].x > 0 ? norms[c].y / norms[c].x : 0.0;
      if (!(r < h->ratio_threshold)) ++ndiv;
    }
    if (rep) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
      rep->t_solve_ms = ms;
      rep->n_diverged = ndiv;
      rep->bytes_moved = solve_bytes(h, R);
      rep->flops = solve_flops(h, R);
      rep->kernel_launches = launches;
      const int64_t cap = std::min<int64_t>(rep->nrhs, R);
      for (int64_t c = 0; c < cap; ++c) {
        if (rep->it0_norm) rep->it0_norm[c] = norms[c].x;
        if (rep->it1_norm) rep->it1_norm[c] = norms[c].y;
        if (rep->ratio) rep->ratio[c] = norms[c].x > 0 ? norms[c].y / norms[c].x : 0.0;
      }
    }
    if (ndiv > 0)
      return fail(h, PS_EDIVERGED, "ps_solve: " + std::to_string(ndiv) + " of " + std::to_string(R) +
                                       " columns have ||it_1||/||it_0|| >= " + std::to_string(h->ratio_threshold));
  }
  return PS_OK;
}

ps_status ps_solve(ps_handle* h, int64_t nrhs, const void* B, int64_t ldb, void* X, int64_t ldx,
                   int on_device, void* cuda_stream, ps_report* rep) {
  return solve_impl(h, nrhs, B, ldb, X, ldx, on_device, cuda_stream, rep, false);
}

ps_status ps_solve_async(ps_handle* h, int64_t nrhs, const void* B, int64_t ldb, void* X, int64_t ldx,
                         void* cuda_stream) {
  if (h && h->part_mode) return fail(h, PS_ESTATE, "ps_solve_async: row-partition handles solve with ps_solve");
  return solve_impl(h, nrhs, B, ldb, X, ldx, 1, cuda_stream, nullptr, true);
}

ps_status ps_solve_report(ps_handle* h, ps_report* rep) {
  if (!h) return fail(nullptr, PS_EINVAL, "ps_solve_report: handle is NULL");
  if (h->pend_nrhs < 1) return fail(h, PS_ESTATE, "ps_solve_report: no ps_solve_async is pending");
  try {
    CK(cudaSetDevice(h->device));
    SolvePlan& sp = get_plan(h, h->pend_nrhs);
    return finish_report(h, sp.norms.p, sp.nrhs, sp.launches_per_solve, h->pend_stream, rep);
  } catch (const PsError& e) {
    return fail(h, e.st, "ps_solve_report: " + e.msg);
  } catch (const std::bad_alloc&) {
    return fail(h, PS_ENOMEM, "ps_solve_report: host allocation failed");
  }
}

ps_status ps_apply(ps_handle* h, int op, int64_t nrhs, const void* Xin, void* Yout) {
  if (!h) return fail(nullptr, PS_EINVAL, "ps_apply: handle is NULL");
  if (op < PS_OP_RT || op > PS_OP_U || nrhs < 1 || !Xin || !Yout)
    return fail(h, PS_EINVAL, "ps_apply: bad arguments");
  if (op != PS_OP_ZF && !h->setup_done) return fail(h, PS_ESTATE, "ps_apply: ps_setup has not run");
  if (h->sharded)
    return fail(h, PS_ESTATE, "ps_apply: the operator of a row-partition rank is sharded (use ps_solve)");
  try {
    CK(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    ensure_far(h, s);                                 // Z_F is legal before ps_setup
    SolvePlan& sp = get_plan(h, nrhs, true);
    const int64_t N = h->N, R = nrhs;
    launch_permute_in(N, R, h->d_e2rwg.p, (const double2*)Xin, N, sp.y.p, s);
    double2* res = sp.y.p;
    switch (op) {
      case PS_OP_RT: op_Rt(h, sp, sp.y.p, s); break;
      case PS_OP_DINV: op_Dinv(h, sp, sp.y.p, sp.bo.p, s); res = sp.bo.p; break;
      case PS_OP_R: op_R(h, sp, sp.y.p, sp.w.p, s); res = sp.w.p; break;
      case PS_OP_ZF: op_ZF(h, sp, sp.y.p, sp.w.p, s); res = sp.w.p; break;
      case PS_OP_U:
        op_R(h, sp, sp.y.p, sp.w.p, s);
        op_ZF(h, sp, sp.w.p, sp.bo.p, s);
        op_Rt(h, sp, sp.bo.p, s);
        op_Dinv(h, sp, sp.bo.p, sp.u.p, s);
        res = sp.u.p;
        break;
    }
    launch_permute_out(N, R, h->d_e2rwg.p, res, (double2*)Yout, N, s);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    if (h->prof.on) h->prof.collect();
  } catch (const PsError& e) {
    return fail(h, e.st, "ps_apply: " + e.msg);
  }
  return PS_OK;
}

// n-term series (include/ps.h ps_solve_series; Eqs. 35-36, 44-45): it_0 = D^-1 R^T b, then
// it_n = U it_{n-1} = D^-1 R^T Z_F R it_{n-1} through the per-operator tables, each term
// folded into the partial sum with its norms in one pass; with tol > 0 the per-column norms
// of the term just added are read back (one small D2H per term) to decide whether to stop.
ps_status ps_solve_series(ps_handle* h, const ps_series_opts* opts, int64_t nrhs, const void* B, int64_t ldb,
                          void* X, int64_t ldx, int on_device, void* cuda_stream, ps_series_report* rep) {
  if (!h) return fail(nullptr, PS_EINVAL, "ps_solve_series: handle is NULL");
  const int max_terms = opts ? opts->max_terms : 2;
  const double tol = opts ? opts->tol : 0.0;
  if (max_terms < 1 || max_terms > 4096 || !(tol >= 0.0))
    return fail(h, PS_EINVAL, "ps_solve_series: max_terms must be in [1, 4096] and tol >= 0");
  if (!h->setup_done) return fail(h, PS_ESTATE, "ps_solve_series: ps_setup has not run");
  if (h->part_mode || h->sharded)
    return fail(h, PS_ESTATE, "ps_solve_series: single-GPU handles only (row partition: ps_solve)");
  if (nrhs < 1 || !B || !X || ldb < h->N || ldx < h->N)
    return fail(h, PS_EINVAL, "ps_solve_series: bad arguments (nrhs >= 1, B/X non-NULL, ldb/ldx >= N)");
  {
    const char* b0 = (const char*)B;
    const char* b1 = b0 + 16 * (ldb * (nrhs - 1) + h->N);
    const char* x0 = (const char*)X;
    const char* x1 = x0 + 16 * (ldx * (nrhs - 1) + h->N);
    if (b0 < x1 && x0 < b1) return fail(h, PS_EINVAL, "ps_solve_series: X overlaps B");
  }
  int ndiv = 0, nterms = 0;
  try {
    CK(cudaSetDevice(h->device));
    cudaStream_t s = cuda_stream ? (cudaStream_t)cuda_stream : h->stream;
    ensure_far(h, s);
    SolvePlan& sp = get_plan(h, nrhs, true);
    const int64_t N = h->N, R = nrhs;
    int64_t launches = 0;
    h->series_norms.alloc((int64_t)max_terms * R);
    const double2* Bd = (const double2*)B;
    int64_t ldb_d = ldb;
    if (!on_device) {
      CK(cudaMemcpy2DAsync(sp.stage.p, 16 * N, B, 16 * ldb, 16 * N, nrhs, cudaMemcpyHostToDevice, s));
      Bd = sp.stage.p;
      ldb_d = N;
    }
    CK(cudaEventRecord(h->ev0, s));
    // it (sp.bo) = current term, acc (sp.xt) = partial sum x~, y / w scratch
    launches += aux(h, s, [&] { launch_permute_in(N, R, h->d_e2rwg.p, Bd, ldb_d, sp.y.p, s); });
    launches += op_Rt(h, sp, sp.y.p, s);                                 // b~ = R^T b  (Eq. 24)
    launches += op_Dinv(h, sp, sp.y.p, sp.bo.p, s);                      // it_0 = b_o  (Eq. 32)
    std::vector<double2> nrm(R);
    for (int n = 0; n < max_terms; ++n) {
      if (n > 0) {                                                       // it_n = U it_{n-1} (Eq. 31)
        launches += op_R(h, sp, sp.bo.p, sp.w.p, s);
        // Z_F: the one-pass far apply where the solve program uses it (narrow, large far field)
        launches += sp.f1p ? far1p_apply(h, sp, sp.w.p, sp.y.p, s) : op_ZF(h, sp, sp.w.p, sp.y.p, s);
        launches += op_Rt(h, sp, sp.y.p, s);
        launches += op_Dinv(h, sp, sp.y.p, sp.bo.p, s);
      }
      double2* nd = h->series_norms.p + (int64_t)n * R;
      launches += aux(h, s, [&] {                                        // x~ += (-1)^n it_n (Eq. 44)
        launch_series_accum(N, R, sp.bo.p, sp.xt.p, (n & 1) ? -1.0 : 1.0, n == 0, sp.part.p, sp.rpc, s);
        launch_finalize_norms(sp.nchunks, R, sp.part.p, nd, s);
      }) + 1;
      nterms = n + 1;
      if (tol > 0.0 && n >= 1 && n + 1 < max_terms) {
        CK(cudaMemcpyAsync(nrm.data(), nd, 16 * R, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        bool done = true;
        for (int64_t c = 0; c < R && done; ++c) done = nrm[c].x <= tol * nrm[c].y;
        if (done) break;
      }
    }
    launches += op_R(h, sp, sp.xt.p, sp.xt.p, s);                        // x = R x~ (Eq. 26)
    double2* Xd = on_device ? (double2*)X : sp.stage.p;
    launches += aux(h, s, [&] { launch_permute_out(N, R, h->d_e2rwg.p, sp.xt.p, Xd, on_device ? ldx : N, s); });
    CK(cudaEventRecord(h->ev1, s));
    CK(cudaGetLastError());
    if (!on_device)
      CK(cudaMemcpy2DAsync(X, 16 * ldx, sp.stage.p, 16 * N, 16 * N, nrhs, cudaMemcpyDeviceToHost, s));
    std::vector<double2> all((size_t)nterms * R);
    CK(cudaMemcpyAsync(all.data(), h->series_norms.p, 16 * all.size(), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h->prof.on) h->prof.collect();
    if (nterms >= 2)
      for (int64_t c = 0; c < R; ++c) {
        const double a = all[(size_t)(nterms - 2) * R + c].x, b = all[(size_t)(nterms - 1) * R + c].x;
        if (a > 0 && !(b < a)) ++ndiv;
      }
    if (rep) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
      rep->t_solve_ms = ms;
      rep->n_terms = nterms;
      rep->n_diverged = ndiv;
      rep->kernel_launches = launches;
      double nR = 0, nD = 0, nF = 0;
      for (int64_t p = 0; p < h->nl; ++p) {
        nR += (double)h->nsz[p] * h->S[p];
        nD += (double)h->nsz[p] * h->nsz[p];
      }
      for (int64_t b = 0; b < h->nfar; ++b)
        nF += (double)h->far_list[7 * b + 5] * (h->far_list[7 * b + 1] + h->far_list[7 * b + 3]);
      const double ex = nterms - 1;
      rep->bytes_moved = 16.0 * ((2 * nR + nD) + ex * (2 * nR + nD + nF)) + 16.0 * 6.0 * (double)N * R * nterms;
      rep->flops = 8.0 * R * ((2 * nR + nD) + ex * (2 * nR + nD + 2 * nF));
      if (rep->it_norm)
        for (int n = 0; n < nterms && n < rep->max_terms; ++n)
          for (int64_t c = 0; c < R && c < rep->nrhs; ++c) rep->it_norm[(int64_t)n * rep->nrhs + c] = all[(size_t)n * R + c].x;
    }
  } catch (const PsError& e) {
    return fail(h, e.st, "ps_solve_series: " + e.msg);
  } catch (const std::bad_alloc&) {
    return fail(h, PS_ENOMEM, "ps_solve_series: host allocation failed");
  }
  if (ndiv > 0)
    return fail(h, PS_EDIVERGED, "ps_solve_series: " + std::to_string(ndiv) + " of " + std::to_string(nrhs) +
                                     " columns have ||it_n|| / ||it_{n-1}|| >= 1 at the last term");
  return PS_OK;
}

// far field / RCS of RWG currents (include/ps.h ps_farfield; ps_rcs.cu)
ps_status ps_farfield(int64_t nnodes, const double* nodes, int64_t ntris, const int64_t* tris, int64_t N,
                      const int64_t* tp, const int64_t* tm, const int64_t* vp, const int64_t* vm, double k,
                      double eta, const void* I, int64_t ldi, int64_t nrhs, int64_t ndir, const double* rhat,
                      int mono, void* F, double* sigma, void* cuda_stream) {
  if (nnodes < 3 || ntris < 1 || N < 1 || nrhs < 1 || ndir < 0 || ldi < N || !(k >= 0.0) || !nodes || !tris ||
      !tp || !tm || !vp || !vm || !I || (ndir > 0 && (!rhat || !F)) || (mono && ndir != nrhs))
    return fail(nullptr, PS_EINVAL, "ps_farfield: bad arguments");
  if (ndir == 0) return PS_OK;
  try {
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const int64_t need = -launch_farfield(nodes, tris, N, tp, tm, vp, vm, k, eta, (const double2*)I, ldi, nrhs,
                                          ndir, rhat, mono, (double2*)F, sigma, nullptr, 0, s);
    // split partials: a grow-only workspace per device, kept across calls (calls serialise on it)
    static std::mutex mu;
    static std::map<int, DevBuf<double2>> ws;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    DevBuf<double2>& part = ws[dev];
    if (part.cap < need) part.alloc(need);
    launch_farfield(nodes, tris, N, tp, tm, vp, vm, k, eta, (const double2*)I, ldi, nrhs, ndir, rhat, mono,
                    (double2*)F, sigma, part.p, part.cap, s);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
  } catch (const PsError& e) {
    return fail(nullptr, e.st, "ps_farfield: " + e.msg);
  }
  return PS_OK;
}

int ps_analyze(const char* path, double* out, int n) { return ps_analyze_rank(path, 0, 1, out, n); }

int64_t ps_validate(const char* path, int64_t nrhs, int64_t* stats, int nstats) {
  if (!path || nrhs < 1) return -PS_EINVAL;
  ps_handle h;
  try {
    std::vector<double2> near_arena, far_arena;
    h.path = path;
    read_file(&h, path, near_arena, far_arena, /*defer_near=*/true);
    symbolic(&h);
    far_layout(&h, far_arena, h.far_host);
    h.Pbase = 0;
    h.Dbase = h.Plen;
    h.Fbase = h.Plen + h.Dlen;
    h.Tbase = h.Fbase + (int64_t)h.far_host.size();
    h.FBbase = h.Tbase + h.Tlen;
    SolvePlan sp;
    g_host_only = true;
    build_program(&h, sp, nrhs);
    g_host_only = false;
    // PS_VALIDATE_BREAK (tests of the checker itself): 1 drops one segment dependency,
    // 2 moves the last work item to the front, 3 pushes one operator offset out of its region,
    // 4 moves a far1p F1-again chunk before its unit's other chunks, 5 moves a far1p item past the FB arena
    static const int brk = env_int("PS_VALIDATE_BREAK", 0);
    Table& Pt = sp.prog;
    if (brk == 1) {
      for (GTerm& g : Pt.terms)
        if (g.dep >= 0) { g.dep = -1; break; }
    } else if (brk == 2 && Pt.work.size() > 1) {
      std::rotate(Pt.work.begin(), Pt.work.end() - 1, Pt.work.end());
    } else if (brk == 3 && !Pt.terms.empty()) {
      Pt.terms.back().oA = h.Tbase + h.Tlen + 1;
    } else if (brk == 4 && sp.f1p) {              // far1p: a big unit's first F1-again chunk moved to its front
      for (const FUnit& U : sp.f1p_unit) {
        auto b = sp.f1p_item.begin() + U.i0, e = b + U.n;
        auto it = std::find_if(b, e, [](const FItem& x) { return x.kind == 3; });
        if (it != e) { std::rotate(b, it, it + 1); break; }
      }
    } else if (brk == 5 && sp.f1p && !sp.f1p_item.empty()) {  // far1p: an item past the FB arena
      sp.f1p_item.back().off = h.FBbase + h.f1p_len;
    }
    std::vector<int64_t> st;
    std::string e = validate_program(&h, sp, st);
    if (e.empty() && sp.f1p) e = validate_far1p(&h, sp, st);
    if (!e.empty()) {
      g_err = "ps_validate: " + e;
      return -PS_ESTATE;
    }
    for (int i = 0; i < nstats && i < (int)st.size(); ++i) stats[i] = st[i];
    return (int64_t)sp.prog.work.size();
  } catch (const PsError& e) {
    g_host_only = false;
    g_err = "ps_validate: " + e.msg;
    return -(int64_t)e.st;
  } catch (const std::bad_alloc&) {
    g_host_only = false;
    g_err = "ps_validate: host allocation failed";
    return -PS_ENOMEM;
  }
}

int ps_analyze_rank(const char* path, int rank, int nranks, double* out, int n) {
  if (!path || !out || n <= 0 || nranks < 1 || rank < 0 || rank >= nranks) return -PS_EINVAL;
  ps_handle h;
  try {
    std::vector<double2> near_arena, far_arena;
    h.path = path;
    read_file(&h, path, near_arena, far_arena, /*defer_near=*/true);
    symbolic(&h);
    if (nranks > 1) {
      h.rank = rank;
      h.nranks = nranks;
      h.part_mode = 1;
      dist_layout(&h);
      std::vector<char> keep;
      shard_layout(&h, keep);
      h.near_dev_len = 0;
      for (int64_t b = 0; b < h.nnear; ++b)
        if (keep[b]) {
          const int64_t i = h.near_list[3 * b], j = h.near_list[3 * b + 1];
          h.near_dev_len += (h.leaf_off[i + 1] - h.leaf_off[i]) * (h.leaf_off[j + 1] - h.leaf_off[j]);
        }
    }
    far_layout(&h, far_arena, h.far_host);
  } catch (const PsError& e) {
    g_err = "ps_analyze: " + e.msg;
    return -(int)e.st;
  } catch (const std::bad_alloc&) {
    g_err = "ps_analyze: host allocation failed";
    return -PS_ENOMEM;
  }
  return ps_info(&h, out, n);
}

ps_status ps_profile(ps_handle* h, int enable) {
  if (!h) return fail(nullptr, PS_EINVAL, "ps_profile: handle is NULL");
  h->prof.on = enable != 0;
  h->prof.reset();
  return PS_OK;
}

int ps_profile_read(const ps_handle* h, double* out, int n) {
  if (!h || !out) return 0;
  int k = 0;
  for (int c = 0; c < PC_COUNT && k + 4 <= n; ++c) {
    out[k++] = h->prof.ms[c];
    out[k++] = (double)h->prof.n[c];
    out[k++] = h->prof.flops[c];
    out[k++] = h->prof.bytes[c];
  }
  return k;
}

// Debug: trace every work item of the next flow launches of kernel class
// `cls` (0..6; -1 disables). ps_trace_read copies the last one: 14 int64 per
// item (item, smid, t_fetch, t_ready, t_computed, t_done, t_sched0, t_sched1
// [ns, globaltimer], task, mt, nt, chunk, nchunks, klen). Returns the number of items.
ps_status ps_trace(ps_handle* h, int cls) {
  if (!h) return fail(nullptr, PS_EINVAL, "ps_trace: handle is NULL");
  h->prof.trace_on = cls >= 0;
  h->prof.trace_cls = cls;
  return PS_OK;
}

int64_t ps_trace_read(ps_handle* h, int64_t* out, int64_t cap_items) {
  if (!h || !out || !h->prof.trace_work || h->prof.trace_buf.n == 0) return 0;
  const int64_t n = std::min(cap_items, h->prof.trace_nw);
  std::vector<int64_t> raw(8 * h->prof.trace_nw);
  if (cudaMemcpy(raw.data(), h->prof.trace_buf.p, 8 * raw.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < 8; ++k) out[14 * i + k] = raw[8 * i + k];
    const GWork& w = (*h->prof.trace_work)[h->prof.trace_w0 + i];
    out[14 * i + 8] = w.task;
    out[14 * i + 9] = w.mt;
    out[14 * i + 10] = w.nt;
    out[14 * i + 11] = w.chunk;
    out[14 * i + 12] = w.nchunks;
    out[14 * i + 13] = w.kb - w.ka;
  }
  return n;
}

ps_status ps_solve_group(ps_handle* const* hs, int nranks, int64_t nrhs, const void* B, int64_t ldb, void* X,
                         int64_t ldx, void* cuda_stream, ps_report* rep) {
  if (!hs || nranks < 2 || !hs[0]) return fail(nullptr, PS_EINVAL, "ps_solve_group: need nranks >= 2 handles");
  ps_handle* h = hs[0];
  for (int g = 0; g < nranks; ++g) {
    if (!hs[g] || !hs[g]->part_mode || hs[g]->nccl || hs[g]->rank != g || hs[g]->nranks != nranks ||
        hs[g]->N != h->N || hs[g]->device != h->device)
      return fail(h, PS_EINVAL, "ps_solve_group: handles must be ranks 0..nranks-1 of one in-process row partition");
    if (!hs[g]->setup_done) return fail(h, PS_ESTATE, "ps_solve_group: ps_setup has not run on every rank");
  }
  if (nrhs < 1 || !B || !X || ldb < h->N || ldx < h->N)
    return fail(h, PS_EINVAL, "ps_solve_group: bad arguments (nrhs >= 1, B/X non-NULL, ldb/ldx >= N)");
  return finish_dist(hs, nranks, nrhs, B, ldb, X, ldx, 1, cuda_stream, rep, "ps_solve_group");
}

ps_status ps_nccl_unique_id(void* out, int64_t cap) {
  if (!out || cap < (int64_t)sizeof(ncclUniqueId)) return fail(nullptr, PS_EINVAL, "ps_nccl_unique_id: cap < 128");
  try {
    ncclUniqueId id;
    NCK(nccl_api().getUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  } catch (const PsError& e) {
    return fail(nullptr, e.st, "ps_nccl_unique_id: " + e.msg);
  }
  return PS_OK;
}

int64_t ps_partition(const char* path, int nranks, int32_t* owner, int32_t* far_owner, int64_t cap) {
  if (!path || !owner || !far_owner || nranks < 1) return -PS_EINVAL;
  ps_handle h;
  try {
    std::vector<double2> near_arena, far_arena;
    read_file(&h, path, near_arena, far_arena);
    symbolic(&h);
    if (cap < h.nl) {
      g_err = "ps_partition: cap < n_leaves";
      return -PS_EINVAL;
    }
    std::vector<int32_t> ow, fo;
    partition(&h, nranks, ow, fo);
    std::copy(ow.begin(), ow.end(), owner);
    std::copy(fo.begin(), fo.end(), far_owner);
  } catch (const PsError& e) {
    g_err = "ps_partition: " + e.msg;
    return -(int64_t)e.st;
  } catch (const std::bad_alloc&) {
    g_err = "ps_partition: host allocation failed";
    return -PS_ENOMEM;
  }
  return h.nl;
}

int64_t ps_n(const ps_handle* h) { return h ? h->N : -1; }

const char* ps_last_error(const ps_handle* h) {
  if (h) return h->err.c_str();
  return g_err.c_str();
}

void ps_free(ps_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->plan.reset();
  h->dplan.reset();
  if (h->nccl) {
    try { nccl_api().commDestroy((ncclComm_t)h->nccl); } catch (const PsError&) {}
    h->nccl = nullptr;
  }
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->cs_in) {
    cudaStreamSynchronize(h->cs_in);
    cudaStreamSynchronize(h->cs_out);
    cudaStreamDestroy(h->cs_in);
    cudaStreamDestroy(h->cs_out);
    for (auto e : h->hp_ev) cudaEventDestroy(e);
  }
  cudaStream_t s = h->stream, u = h->ustream;
  if (u) cudaStreamSynchronize(u);
  delete h;
  if (s) cudaStreamDestroy(s);
  if (u) cudaStreamDestroy(u);
}

int ps_info(const ps_handle* h, double* out, int n) {
  if (!h || !out || n <= 0) return 0;
  double v[PS_INFO_COUNT];
  double nR = 0, nD = 0, nF = 0;
  for (int64_t p = 0; p < h->nl; ++p) {
    nR += (double)h->nsz[p] * h->S[p];
    nD += (double)h->nsz[p] * h->nsz[p];
  }
  for (int64_t b = 0; b < h->nfar; ++b) nF += (double)h->far_list[7 * b + 5] * (h->far_list[7 * b + 1] + h->far_list[7 * b + 3]);
  v[PS_INFO_N] = (double)h->N;
  v[PS_INFO_NLEAVES] = (double)h->nl;
  v[PS_INFO_NNEAR] = (double)h->nnear;
  v[PS_INFO_NFAR] = (double)h->nfar;
  v[PS_INFO_ALPHA_BLOCKS] = (double)h->alpha_blocks;
  v[PS_INFO_NR] = nR;
  v[PS_INFO_ND] = nD;
  v[PS_INFO_NF] = nF;
  v[PS_INFO_HEIGHT] = h->max_height + 1;
  v[PS_INFO_DEPTH] = h->max_depth + 1;
  v[PS_INFO_SETUP_MADDS] = h->setup_madds;
  v[PS_INFO_SETUP_DONE] = h->setup_done ? 1 : 0;
  v[PS_INFO_NRANKS] = h->part_mode ? h->nranks : 1;
  v[PS_INFO_OWN_ROWS] = h->part_mode ? (double)h->own_rows : (double)h->N;
  v[PS_INFO_SEP_ROWS] = h->part_mode ? (double)h->Nsep : 0.0;
  v[PS_INFO_OP_BYTES] = 16.0 * ((double)h->Plen + (double)h->Dlen + (double)h->Tlen +
                                (double)(h->d_farbuf.p ? h->d_farbuf.n : (int64_t)h->far_host.size()));
  v[PS_INFO_SETUP_BYTES] = 16.0 * ((double)(h->part_mode ? h->near_dev_len : h->near_len) + (double)h->Wlen +
                                   (double)h->Plen + (double)h->Dlen);
  {
    double nchain = 0, tent = 0;
    for (size_t c = 0; c < h->chains.size(); ++c)
      if (h->chains[c].size() >= 2) {
        nchain += 1;
        tent += (double)h->ch_U[c] * (double)h->ch_U[c];
      }
    v[PS_INFO_CHAINS] = nchain;
    v[PS_INFO_CHAIN_HEIGHT] = h->max_ch_height + 1;
    v[PS_INFO_T_ENTRIES] = tent;
  }
  int m = std::min(n, (int)PS_INFO_COUNT);
  std::memcpy(out, v, sizeof(double) * m);
  return m;
}

int64_t ps_get_dinv(ps_handle* h, int64_t pos, void* out, int64_t cap) {
  if (!h || pos < 0 || pos >= h->nl || !h->setup_done || h->Doff[pos] < 0) return 0;   // Doff < 0: not this rank's
  const int64_t n = h->nsz[pos];
  if (!out || cap < n * n) return -(n * n);
  if (cudaMemcpy(out, h->d_D.p + h->Doff[pos], 16 * n * n, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return n;
}

int64_t ps_elim_leaf(const ps_handle* h, int64_t pos) {
  if (!h || pos < 0 || pos >= h->nl) return -1;
  return h->leaf_at[pos];
}

}  // extern "C"
