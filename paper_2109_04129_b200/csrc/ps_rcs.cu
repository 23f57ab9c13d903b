// ps_rcs.cu — far field and RCS of RWG surface currents on the GPU (SURVEY §8(f) NEXT-4:
// the post-processing step after the solve, PAPER.md:333-341 — the bistatic and monostatic
// RCS curves the paper compares with Mie / measured data). include/ps.h ps_farfield.
//
//   F(r^, c) = sum_n I_nc  int_{T+ u T-} f_n(r') e^{+j k r^.r'} dS'          (far-field vector)
//   f_n = +l_n / (2 A+) (r' - v+) on T+,  -l_n / (2 A-) (r' - v-) on T-        (RWG)
//   sigma_p(r^, c) = (k eta)^2 / (4 pi) |F . p^|^2,  p^ = theta^ or phi^ of r^  (m^2)
//
// Each basis contributes 14 samples (the 7-point degree-5 Dunavant rule on each of its two
// triangles; the A_+- of f_n cancels against the rule's area factor, so a sample is
// (position q, real vector g = w_a (+-l_n / 2) (q - v+-))). The samples are built on the fly
// per shared-memory tile of bases; one thread per direction walks the tile: one sincos per
// (direction, sample), then FF_CB columns (bistatic) or its own column (monostatic: direction
// c paired with column c). The basis range is split over grid.z so the grid covers the SMs;
// the split partials are summed in split order by a second kernel (deterministic), which also
// projects on theta^ / phi^ and forms sigma. Bound: FP64 ALU (sincos + 10 FMA per sample and
// column); the currents and mesh are read once per block.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ps_internal.h"

namespace ps {

constexpr int FF_T = 128;           // directions per block
constexpr int FF_NB = 16;           // bases per shared-memory tile (16 x 14 = 224 samples)
constexpr int FF_NS = FF_NB * 14;

// Dunavant (1985) degree-5 7-point rule: barycentric points and weights (weights sum to 1)
__constant__ double c_qb[7][3] = {
    {1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0},
    {0.059715871789770, 0.470142064105115, 0.470142064105115},
    {0.470142064105115, 0.059715871789770, 0.470142064105115},
    {0.470142064105115, 0.470142064105115, 0.059715871789770},
    {0.797426985353087, 0.101286507323456, 0.101286507323456},
    {0.101286507323456, 0.797426985353087, 0.101286507323456},
    {0.101286507323456, 0.101286507323456, 0.797426985353087}};
__constant__ double c_qw[7] = {0.225, 0.132394152788506, 0.132394152788506, 0.132394152788506,
                               0.125939180544827, 0.125939180544827, 0.125939180544827};

struct FfArgs {
  const double* nodes;
  const int64_t* tris;
  const int64_t *tp, *tm, *vp, *vm;
  int64_t N;
  double k;
  const double2* I;
  int64_t ldi, nrhs, ncol;
  const double* rhat;
  int64_t ndir;
  int mono;
  int64_t bps;                      // bases per split
  double2* part;                    // [split][dir][ncol][3]
};

template <int CB>
__global__ void __launch_bounds__(FF_T) farfield_kernel(FfArgs a) {
  __shared__ double sp[FF_NS][3], sg[FF_NS][3];
  __shared__ double2 sI[FF_NB][CB];
  const int tid = threadIdx.x;
  const int64_t d = (int64_t)blockIdx.x * FF_T + tid;
  const int64_t c0 = a.mono ? d : (int64_t)blockIdx.y * CB;
  const int64_t nlo = (int64_t)blockIdx.z * a.bps, nhi = min(a.N, nlo + a.bps);
  const bool live = d < a.ndir;
  double rx = 0, ry = 0, rz = 0;
  if (live) { rx = a.rhat[3 * d]; ry = a.rhat[3 * d + 1]; rz = a.rhat[3 * d + 2]; }
  double2 acc[CB][3];
#pragma unroll
  for (int j = 0; j < CB; ++j)
#pragma unroll
    for (int x = 0; x < 3; ++x) acc[j][x] = make_double2(0.0, 0.0);
  for (int64_t n0 = nlo; n0 < nhi; n0 += FF_NB) {
    const int nb = (int)min((int64_t)FF_NB, nhi - n0);
    __syncthreads();
    for (int t = tid; t < nb * 14; t += FF_T) {          // the tile's samples
      const int64_t n = n0 + t / 14;
      const int s = t % 14, side = s / 7, q = s % 7;
      const int64_t tri = side ? a.tm[n] : a.tp[n];
      const int64_t v = side ? a.vm[n] : a.vp[n];
      const int64_t t0 = a.tris[3 * tri], t1 = a.tris[3 * tri + 1], t2 = a.tris[3 * tri + 2];
      // the common edge = the two vertices of T+ other than v+
      const int64_t p0 = a.tris[3 * a.tp[n]], p1 = a.tris[3 * a.tp[n] + 1], p2 = a.tris[3 * a.tp[n] + 2];
      const int64_t vpn = a.vp[n];
      const int64_t e0 = p0 == vpn ? p1 : p0, e1 = (p2 == vpn || p2 == e0) ? p1 : p2;
      const double ex = a.nodes[3 * e0] - a.nodes[3 * e1], ey = a.nodes[3 * e0 + 1] - a.nodes[3 * e1 + 1],
                   ez = a.nodes[3 * e0 + 2] - a.nodes[3 * e1 + 2];
      const double len = sqrt(ex * ex + ey * ey + ez * ez);
      double qp[3];
#pragma unroll
      for (int x = 0; x < 3; ++x)
        qp[x] = c_qb[q][0] * a.nodes[3 * t0 + x] + c_qb[q][1] * a.nodes[3 * t1 + x] + c_qb[q][2] * a.nodes[3 * t2 + x];
      const double cf = c_qw[q] * (side ? -0.5 : 0.5) * len;
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        sp[t][x] = qp[x];
        sg[t][x] = cf * (qp[x] - a.nodes[3 * v + x]);
      }
    }
    if (!a.mono)
      for (int t = tid; t < nb * CB; t += FF_T) {
        const int b = t / CB, j = t % CB;
        sI[b][j] = c0 + j < a.nrhs ? a.I[(n0 + b) + (c0 + j) * a.ldi] : make_double2(0.0, 0.0);
      }
    __syncthreads();
    if (!live) continue;
    for (int b = 0; b < nb; ++b) {
      double2 In[CB];
      if (a.mono) In[0] = a.I[(n0 + b) + c0 * a.ldi];
      else
#pragma unroll
        for (int j = 0; j < CB; ++j) In[j] = sI[b][j];
#pragma unroll 2
      for (int s = 0; s < 14; ++s) {
        const int t = b * 14 + s;
        const double ph = a.k * (rx * sp[t][0] + ry * sp[t][1] + rz * sp[t][2]);
        double sn, cs;
        sincos(ph, &sn, &cs);
        const double gx = sg[t][0], gy = sg[t][1], gz = sg[t][2];
#pragma unroll
        for (int j = 0; j < CB; ++j) {
          const double er = In[j].x * cs - In[j].y * sn, ei = In[j].x * sn + In[j].y * cs;
          acc[j][0].x = fma(gx, er, acc[j][0].x); acc[j][0].y = fma(gx, ei, acc[j][0].y);
          acc[j][1].x = fma(gy, er, acc[j][1].x); acc[j][1].y = fma(gy, ei, acc[j][1].y);
          acc[j][2].x = fma(gz, er, acc[j][2].x); acc[j][2].y = fma(gz, ei, acc[j][2].y);
        }
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    const int64_t c = a.mono ? 0 : c0 + j;
    if (c >= a.ncol) break;
    double2* o = a.part + (((int64_t)blockIdx.z * a.ndir + d) * a.ncol + c) * 3;
#pragma unroll
    for (int x = 0; x < 3; ++x) o[x] = acc[j][x];
  }
}

// F = sum over splits in order; sigma from the theta^ / phi^ projections of r^
__global__ void farfield_reduce_kernel(int64_t nsplit, int64_t ndir, int64_t ncol, const double2* __restrict__ part,
                                       const double* __restrict__ rhat, double k, double eta,
                                       double2* __restrict__ F, double* __restrict__ sigma) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ndir * ncol) return;
  const int64_t d = e / ncol;
  double2 f[3] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
  for (int64_t s = 0; s < nsplit; ++s) {
    const double2* p = part + (s * ndir * ncol + e) * 3;
#pragma unroll
    for (int x = 0; x < 3; ++x) { f[x].x += p[x].x; f[x].y += p[x].y; }
  }
#pragma unroll
  for (int x = 0; x < 3; ++x) F[e * 3 + x] = f[x];
  if (!sigma) return;
  const double rx = rhat[3 * d], ry = rhat[3 * d + 1], rz = rhat[3 * d + 2];
  const double st = sqrt(rx * rx + ry * ry);
  const double cp = st > 1e-12 ? rx / st : 1.0, sp = st > 1e-12 ? ry / st : 0.0;
  const double th[3] = {rz * cp, rz * sp, -st}, phv[3] = {-sp, cp, 0.0};
  double2 ft = make_double2(0, 0), fp = make_double2(0, 0);
#pragma unroll
  for (int x = 0; x < 3; ++x) {
    ft.x += th[x] * f[x].x; ft.y += th[x] * f[x].y;
    fp.x += phv[x] * f[x].x; fp.y += phv[x] * f[x].y;
  }
  const double c = (k * eta) * (k * eta) / (4.0 * 3.14159265358979323846);
  sigma[e * 2] = c * (ft.x * ft.x + ft.y * ft.y);
  sigma[e * 2 + 1] = c * (fp.x * fp.x + fp.y * fp.y);
}

int64_t launch_farfield(const double* nodes, const int64_t* tris, int64_t N, const int64_t* tp, const int64_t* tm,
                        const int64_t* vp, const int64_t* vm, double k, double eta, const double2* I, int64_t ldi,
                        int64_t nrhs, int64_t ndir, const double* rhat, int mono, double2* F, double* sigma,
                        double2* part, int64_t part_cap, cudaStream_t st) {
  constexpr int CB = 4;
  FfArgs a{nodes, tris, tp, tm, vp, vm, N, k, I, ldi, nrhs, mono ? 1 : nrhs, rhat, ndir, mono, 0, part};
  const int64_t gx = (ndir + FF_T - 1) / FF_T, gy = mono ? 1 : (nrhs + CB - 1) / CB;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (N + FF_NB - 1) / FF_NB;
  int64_t nsplit = (int64_t)sms * 8 / (gx * gy);
  nsplit = nsplit < 1 ? 1 : nsplit > tiles ? tiles : nsplit;
  const int64_t need = nsplit * ndir * a.ncol * 3;
  if (part == nullptr || need > part_cap) return -need;        // caller (re)allocates
  a.bps = ((tiles + nsplit - 1) / nsplit) * FF_NB;
  nsplit = (N + a.bps - 1) / a.bps;
  dim3 g((unsigned)gx, (unsigned)gy, (unsigned)nsplit);
  if (mono) farfield_kernel<1><<<g, FF_T, 0, st>>>(a);
  else farfield_kernel<CB><<<g, FF_T, 0, st>>>(a);
  const int64_t tot = ndir * a.ncol;
  farfield_reduce_kernel<<<(unsigned)((tot + 127) / 128), 128, 0, st>>>(nsplit, ndir, a.ncol, part, rhat, k, eta,
                                                                         F, sigma);
  return 2;
}

}  // namespace ps
