// Streaming probe for the nrhs = 1 (operator-streaming) regime: how fast can a
// persistent grid read a large operator arena in item-sized pieces with
//   (a) 16-byte cp.async.cg by 256 threads, NS-stage ring (the flow kernels' scheme),
//   (b) cp.async.bulk (TMA 1-D bulk copy) of whole stages, mbarrier completion.
// Each CTA takes "items" (ITEM bytes, random 2 MB-aligned-ish offsets) from a ticket.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe scripts/stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// (a) cp.async ring: stage = SB bytes; NS stages
template <int NS, int SB>
__global__ void __launch_bounds__(256) k_cpasync(const char* __restrict__ base, const int64_t* __restrict__ offs,
                                                  int nitems, int64_t item_bytes, int* ticket, double* sink) {
  extern __shared__ __align__(16) char sm[];
  __shared__ int s_it;
  const int tid = threadIdx.x;
  double acc = 0;
  for (;;) {
    if (tid == 0) s_it = atomicAdd(ticket, 1);
    __syncthreads();
    const int it = s_it;
    if (it >= nitems) break;
    const char* src = base + offs[it];
    const int nst = (int)(item_bytes / SB);
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) {
      if (s < nst)
        for (int e = tid; e < SB / 16; e += 256) cp_async16(sm + s * SB + 16 * e, src + (int64_t)s * SB + 16 * e);
      cp_commit();
    }
    for (int s = 0; s < nst; ++s) {
      cp_wait<NS - 2>();
      __syncthreads();
      const double* d = reinterpret_cast<const double*>(sm + (s % NS) * SB);
      acc += d[tid];
      const int sn = s + NS - 1;
      if (sn < nst)
        for (int e = tid; e < SB / 16; e += 256) cp_async16(sm + (sn % NS) * SB + 16 * e, src + (int64_t)sn * SB + 16 * e);
      cp_commit();
    }
    cp_wait<0>();
    __syncthreads();
  }
  if (acc == 12345.678) sink[0] = acc;
}

// (b) bulk copies: one elected thread issues cp.async.bulk per stage into an mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(b);
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"(a), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                   "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
               "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

template <int NS, int SB, int PIECE>
__global__ void __launch_bounds__(256) k_bulk(const char* __restrict__ base, const int64_t* __restrict__ offs,
                                               int nitems, int64_t item_bytes, int* ticket, double* sink) {
  extern __shared__ __align__(16) char sm[];
  __shared__ __align__(8) uint64_t bar[NS];
  __shared__ int s_it;
  const int tid = threadIdx.x;
  if (tid == 0)
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t phase_bits = 0;   // parity per stage
  double acc = 0;
  int gstage = 0;            // running stage counter across items (ring continues)
  for (;;) {
    if (tid == 0) s_it = atomicAdd(ticket, 1);
    __syncthreads();
    const int it = s_it;
    if (it >= nitems) break;
    const char* src = base + offs[it];
    const int nst = (int)(item_bytes / SB);
    auto issue = [&](int s) {
      const int slot = (gstage + s) % NS;
      mbar_expect_tx(&bar[slot], SB);
      for (int p = 0; p < SB / PIECE; ++p)
        bulk_g2s(sm + slot * SB + p * PIECE, src + (int64_t)s * SB + p * PIECE, PIECE, &bar[slot]);
    };
    if (tid == 0)
      for (int s = 0; s < NS - 1 && s < nst; ++s) issue(s);
    for (int s = 0; s < nst; ++s) {
      const int slot = (gstage + s) % NS;
      mbar_wait(&bar[slot], (phase_bits >> slot) & 1);
      phase_bits ^= 1u << slot;
      const double* d = reinterpret_cast<const double*>(sm + slot * SB);
      acc += d[tid];
      __syncthreads();   // everyone done with the slot refilled next
      if (tid == 0 && s + NS - 1 < nst) issue(s + NS - 1);
    }
    gstage += nst;
    __syncthreads();
  }
  if (acc == 12345.678) sink[0] = acc;
}

// (c) cp.async over an item that is a column-major block of NCOL columns x COL bytes:
// stage s reads bytes [s*RUN, (s+1)*RUN) of every column (NCOL runs of RUN bytes),
// i.e. the transposed-panel (k-major) access of the forward sweep.
template <int NS, int NCOL, int RUN>
__global__ void __launch_bounds__(256) k_runs(const char* __restrict__ base, const int64_t* __restrict__ offs,
                                               int nitems, int64_t item_bytes, int* ticket, double* sink) {
  extern __shared__ __align__(16) char sm[];
  constexpr int SB = NCOL * RUN;
  __shared__ int s_it;
  const int tid = threadIdx.x;
  const int64_t COL = item_bytes / NCOL;
  double acc = 0;
  for (;;) {
    if (tid == 0) s_it = atomicAdd(ticket, 1);
    __syncthreads();
    const int it = s_it;
    if (it >= nitems) break;
    const char* src = base + offs[it];
    const int nst = (int)(COL / RUN);
    auto issue = [&](int s, char* dst) {
      for (int e = tid; e < SB / 16; e += 256) {
        const int c = e / (RUN / 16), o = e % (RUN / 16);
        cp_async16(dst + 16 * e, src + c * COL + (int64_t)s * RUN + 16 * o);
      }
    };
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) {
      if (s < nst) issue(s, sm + s * SB);
      cp_commit();
    }
    for (int s = 0; s < nst; ++s) {
      cp_wait<NS - 2>();
      __syncthreads();
      const double* d = reinterpret_cast<const double*>(sm + (s % NS) * SB);
      acc += d[tid];
      const int sn = s + NS - 1;
      if (sn < nst) issue(sn, sm + (sn % NS) * SB);
      cp_commit();
    }
    cp_wait<0>();
    __syncthreads();
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  const int64_t arena = 6LL << 30;    // 6 GB operator
  char* d;
  CK(cudaMalloc(&d, arena));
  CK(cudaMemset(d, 1, arena));
  int* ticket; double* sink;
  CK(cudaMalloc(&ticket, 4)); CK(cudaMalloc(&sink, 8));
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  std::mt19937_64 rng(1);
  auto run = [&](const char* name, auto kern, int smem, int per_sm, int64_t item_bytes, bool contiguous) -> int {
    const int nitems = (int)(arena / item_bytes);
    std::vector<int64_t> offs(nitems);
    for (int i = 0; i < nitems; ++i) offs[i] = (int64_t)i * item_bytes;
    if (!contiguous) std::shuffle(offs.begin(), offs.end(), rng);
    int64_t* d_offs; CK(cudaMalloc(&d_offs, 8 * nitems));
    CK(cudaMemcpy(d_offs, offs.data(), 8 * nitems, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      CK(cudaMemset(ticket, 0, 4));
      cudaEventRecord(e0);
      kern<<<nsm * per_sm, 256, smem>>>(d, d_offs, nitems, item_bytes, ticket, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("%-44s item %6lld KB %s: %7.1f GB/s\n", name, (long long)(item_bytes >> 10), contiguous ? "seq " : "rand",
           (double)nitems * item_bytes / best / 1e6);
    cudaFree(d_offs);
    return 0;
  };
  // forward-sweep-like blocks: 64 columns x 112 complex (1792 B), 256 B runs per stage
  run("runs 64 x 256B (k-major, ld 112)", k_runs<3, 64, 256>, 3 * 16384, 2, 64 * 1792, false);
  run("runs 64 x 256B (k-major, ld 224)", k_runs<3, 64, 256>, 3 * 16384, 2, 64 * 3584, false);
  run("runs 16 x 1KB (k-major, ld 256)", k_runs<3, 16, 1024>, 3 * 16384, 2, 16 * 4096, false);
  run("runs 64 x 256B, 4 stages", k_runs<4, 64, 256>, 4 * 16384, 2, 64 * 1792, false);
  run("runs 32 x 512B (ld 112)", k_runs<3, 32, 512>, 3 * 16384, 2, 32 * 1792 * 2, false);
  run("runs 16 x 1KB 1 col-block contiguous 16KB", k_runs<3, 1, 16384>, 3 * 16384, 2, 160 << 10, false);
  for (int64_t ib : {160LL << 10}) {
    for (bool c : {false}) {
      run("cp.async 16B, 3 x 16KB, 2 CTA/SM", k_cpasync<3, 16384>, 3 * 16384, 2, ib, c);
      run("cp.async 16B, 4 x 16KB, 2 CTA/SM", k_cpasync<4, 16384>, 4 * 16384, 2, ib, c);
      run("cp.async 16B, 6 x 16KB, 2 CTA/SM", k_cpasync<6, 16384>, 6 * 16384, 2, ib, c);
      run("cp.async 16B, 3 x 32KB, 2 CTA/SM", k_cpasync<3, 32768>, 3 * 32768, 2, ib, c);
      run("bulk 1KB pieces, 4 x 16KB, 2 CTA/SM", k_bulk<4, 16384, 1024>, 4 * 16384, 2, ib, c);
      run("bulk 256B pieces, 4 x 16KB, 2 CTA/SM", k_bulk<4, 16384, 256>, 4 * 16384, 2, ib, c);
      run("bulk 16KB, 6 x 16KB, 2 CTA/SM", k_bulk<6, 16384, 16384>, 6 * 16384, 2, ib, c);
    }
  }
  return 0;
}
