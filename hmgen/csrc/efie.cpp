// hmgen/csrc/efie.cpp — host-side INPUT GENERATOR for the power-series solver.
//
// This file builds the H-matrix that both the GPU path (libps) and the oracle
// consume. It is NOT part of the method under test (§III); it is the
// operator assembly of PAPER.md §II:
//   * RWG Galerkin EFIE entries, Eqs. (2)-(3), with the
//     e^{+jwt} / G = e^{-jkR}/(4 pi R) reading (reading R16):
//       Z_mn = j k eta  Int Int [ f_m.f_n - (1/k^2) div f_m div' f_n ] G dS' dS
//   * 7-point (degree-5) triangle quadrature on test and source triangles;
//     analytic extraction of the 1/R part of G on touching/self triangle
//     pairs (the potential integrals of Wilton et al. 1984 / Graglia 1993).
//   * ACA with partial pivoting, Eqs. (11)-(12), followed by
//     QR + truncated SVD recompression ([20,21]).
//
// Exposed through a tiny extern "C" API used by hmgen/build.py via ctypes.
// OpenMP parallel over blocks; every block's result is independent of the
// thread schedule (deterministic).
#include <complex>
#include <vector>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <numeric>

typedef std::complex<double> cd;
static const double PI = 3.14159265358979323846;

namespace {

struct V3 { double x, y, z; };
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }

// Dunavant degree-5, 7-point rule (barycentric coordinates, weights sum to 1).
const double QA = 0.059715871789770, QB = 0.470142064105115, QWB = 0.132394152788506;
const double QC = 0.797426985353087, QD = 0.101286507323456, QWD = 0.125939180544827;
const double QBARY[7][3] = {
    {1.0 / 3, 1.0 / 3, 1.0 / 3}, {QA, QB, QB}, {QB, QA, QB}, {QB, QB, QA},
    {QC, QD, QD}, {QD, QC, QD}, {QD, QD, QC}};
const double QW[7] = {0.225, QWB, QWB, QWB, QWD, QWD, QWD};

struct Tri {
  int v[3];
  V3 p[3];
  V3 n;         // unit normal (p1-p0)x(p2-p0)
  double area;
  V3 q[7];      // quadrature points
};

struct Ctx {
  std::vector<V3> nodes;
  std::vector<Tri> tris;
  // RWG: per basis: tri plus, tri minus, free vertex plus/minus (node ids), length
  std::vector<int> tp, tm, vp, vm;
  std::vector<double> len;
  double k, eta;
};

// Analytic potential integrals over triangle T for observation point r:
//   Js   = Int_T 1/|r-r'| dS'
//   Jvec = Int_T (r'-r)/|r-r'| dS'
void potential_integrals(const Tri& T, V3 r, double& Js, V3& Jvec) {
  V3 n = T.n;
  double d = dot(n, r - T.p[0]);
  double ad = std::fabs(d);
  double js = 0.0;
  V3 jr = {0, 0, 0};
  double scale = norm(T.p[1] - T.p[0]) + norm(T.p[2] - T.p[1]);
  double tiny = 1e-12 * scale;
  for (int e = 0; e < 3; ++e) {
    V3 a = T.p[e], b = T.p[(e + 1) % 3];
    V3 lv = b - a;
    double ll = norm(lv);
    V3 lh = (1.0 / ll) * lv;
    V3 uh = cross(lh, n);  // outward in-plane normal of the edge
    double lm = dot(a - r, lh), lp = dot(b - r, lh);
    double t0 = dot(a - r, uh);
    double R02 = t0 * t0 + d * d;
    double Rm = std::sqrt(lm * lm + R02), Rp = std::sqrt(lp * lp + R02);
    if (std::sqrt(R02) < tiny) continue;  // observation point on the edge line
    double lg;
    if (lm < 0.0 && lp < 0.0)
      lg = std::log((Rm - lm) / (Rp - lp));
    else
      lg = std::log((Rp + lp) / (Rm + lm));
    js += t0 * lg - ad * (std::atan(t0 * lp / (R02 + ad * Rp)) - std::atan(t0 * lm / (R02 + ad * Rm)));
    double c = 0.5 * (R02 * lg + lp * Rp - lm * Rm);
    jr = jr + c * uh;
  }
  Js = js;
  // r' - r = (rho' - rho) - d n
  Jvec = jr - (d * js) * n;
}

inline cd green_smooth(double k, double R) {
  // (e^{-jkR} - 1) / (4 pi R), limit -jk/(4pi) at R -> 0
  if (R < 1e-12) return cd(0.0, -k / (4 * PI));
  double s = std::sin(k * R), c = std::cos(k * R);
  return cd(c - 1.0, -s) / (4 * PI * R);
}
inline cd green_full(double k, double R) {
  double s = std::sin(k * R), c = std::cos(k * R);
  return cd(c, -s) / (4 * PI * R);
}

inline int shared_vertices(const Tri& a, const Tri& b) {
  int s = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) s += (a.v[i] == b.v[j]);
  return s;
}

// Int_{Tp} Int_{Tq} [cv (r - vm).(r' - vn) - cs] G(r,r') dS' dS
cd pair_integral(const Ctx& C, const Tri& Tp, const Tri& Tq, V3 vm, V3 vn, double cv, double cs) {
  const double k = C.k;
  cd acc(0, 0);
  bool sing = shared_vertices(Tp, Tq) > 0;
  for (int a = 0; a < 7; ++a) {
    V3 r = Tp.q[a];
    V3 rm = r - vm;
    cd inner(0, 0);
    for (int b = 0; b < 7; ++b) {
      V3 rp = Tq.q[b];
      double R = norm(r - rp);
      cd g = sing ? green_smooth(k, R) : green_full(k, R);
      double kern = cv * dot(rm, rp - vn) - cs;
      inner += (QW[b] * kern) * g;
    }
    inner *= Tq.area;
    if (sing) {
      double Js;
      V3 Jv;
      potential_integrals(Tq, r, Js, Jv);
      // Int (r'-vn)/R = Jv + (r - vn) Js
      V3 Jn = Jv + Js * (r - vn);
      double sv = cv * dot(rm, Jn) - cs * Js;
      inner += cd(sv / (4 * PI), 0.0);
    }
    acc += QW[a] * inner;
  }
  return acc * Tp.area;
}

cd efie_entry(const Ctx& C, int m, int n) {
  const double k = C.k;
  cd z(0, 0);
  for (int sm = 0; sm < 2; ++sm) {
    int tpi = sm == 0 ? C.tp[m] : C.tm[m];
    double sgm = sm == 0 ? 1.0 : -1.0;
    V3 vm = C.nodes[sm == 0 ? C.vp[m] : C.vm[m]];
    const Tri& Tp = C.tris[tpi];
    for (int sn = 0; sn < 2; ++sn) {
      int tqi = sn == 0 ? C.tp[n] : C.tm[n];
      double sgn = sn == 0 ? 1.0 : -1.0;
      V3 vn = C.nodes[sn == 0 ? C.vp[n] : C.vm[n]];
      const Tri& Tq = C.tris[tqi];
      double cv = (sgm * C.len[m] / (2 * Tp.area)) * (sgn * C.len[n] / (2 * Tq.area));
      double cs = (sgm * C.len[m] / Tp.area) * (sgn * C.len[n] / Tq.area) / (k * k);
      z += pair_integral(C, Tp, Tq, vm, vn, cv, cs);
    }
  }
  return cd(0.0, k * C.eta) * z;
}

// ---------------- small dense complex linear algebra (recompression) -------
// Thin Householder QR of A (m x r, column-major, m >= r). Returns Q (m x r), R (r x r).
void house_qr(int m, int r, std::vector<cd>& A, std::vector<cd>& Q, std::vector<cd>& R) {
  std::vector<std::vector<cd>> vs(r);
  for (int j = 0; j < r; ++j) {
    int len = m - j;
    std::vector<cd> v(len);
    double nx = 0;
    for (int i = 0; i < len; ++i) { v[i] = A[(j + i) + (size_t)j * m]; nx += std::norm(v[i]); }
    nx = std::sqrt(nx);
    if (nx == 0.0) { vs[j].assign(len, cd(0, 0)); continue; }
    cd ph = std::abs(v[0]) > 0 ? v[0] / std::abs(v[0]) : cd(1, 0);
    cd alpha = -ph * nx;
    v[0] -= alpha;
    double nv = 0;
    for (int i = 0; i < len; ++i) nv += std::norm(v[i]);
    nv = std::sqrt(nv);
    for (int i = 0; i < len; ++i) v[i] /= nv;
    for (int c = j; c < r; ++c) {
      cd s(0, 0);
      for (int i = 0; i < len; ++i) s += std::conj(v[i]) * A[(j + i) + (size_t)c * m];
      for (int i = 0; i < len; ++i) A[(j + i) + (size_t)c * m] -= 2.0 * v[i] * s;
    }
    vs[j] = v;
  }
  R.assign((size_t)r * r, cd(0, 0));
  for (int c = 0; c < r; ++c)
    for (int i = 0; i <= c; ++i) R[i + (size_t)c * r] = A[i + (size_t)c * m];
  Q.assign((size_t)m * r, cd(0, 0));
  for (int c = 0; c < r; ++c) Q[c + (size_t)c * m] = 1.0;
  for (int j = r - 1; j >= 0; --j) {
    const std::vector<cd>& v = vs[j];
    int len = m - j;
    for (int c = 0; c < r; ++c) {
      cd s(0, 0);
      for (int i = 0; i < len; ++i) s += std::conj(v[i]) * Q[(j + i) + (size_t)c * m];
      for (int i = 0; i < len; ++i) Q[(j + i) + (size_t)c * m] -= 2.0 * v[i] * s;
    }
  }
}

// One-sided Jacobi SVD of square M (r x r): M = W diag(s) X^H. Sorted descending.
void jacobi_svd(int r, std::vector<cd> M, std::vector<cd>& W, std::vector<double>& s, std::vector<cd>& X) {
  X.assign((size_t)r * r, cd(0, 0));
  for (int i = 0; i < r; ++i) X[i + (size_t)i * r] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0;
    for (int p = 0; p < r; ++p)
      for (int q = p + 1; q < r; ++q) {
        double a = 0, b = 0;
        cd g(0, 0);
        for (int i = 0; i < r; ++i) {
          a += std::norm(M[i + (size_t)p * r]);
          b += std::norm(M[i + (size_t)q * r]);
          g += std::conj(M[i + (size_t)p * r]) * M[i + (size_t)q * r];
        }
        double ag = std::abs(g);
        if (ag <= 1e-15 * std::sqrt(a * b) || ag == 0.0) continue;
        off = std::max(off, ag / std::sqrt(a * b));
        cd ph = std::conj(g / ag);  // multiply column q by e^{-i phi}
        double zeta = (b - a) / (2 * ag);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1 + zeta * zeta));
        double c = 1 / std::sqrt(1 + t * t), sn = c * t;
        for (int i = 0; i < r; ++i) {
          cd mp = M[i + (size_t)p * r], mq = M[i + (size_t)q * r] * ph;
          M[i + (size_t)p * r] = c * mp - sn * mq;
          M[i + (size_t)q * r] = sn * mp + c * mq;
          cd xp = X[i + (size_t)p * r], xq = X[i + (size_t)q * r] * ph;
          X[i + (size_t)p * r] = c * xp - sn * xq;
          X[i + (size_t)q * r] = sn * xp + c * xq;
        }
      }
    if (off < 1e-15) break;
  }
  std::vector<double> sv(r);
  for (int j = 0; j < r; ++j) {
    double t = 0;
    for (int i = 0; i < r; ++i) t += std::norm(M[i + (size_t)j * r]);
    sv[j] = std::sqrt(t);
  }
  std::vector<int> idx(r);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return sv[a] > sv[b]; });
  W.assign((size_t)r * r, cd(0, 0));
  std::vector<cd> X2((size_t)r * r);
  s.resize(r);
  for (int jj = 0; jj < r; ++jj) {
    int j = idx[jj];
    s[jj] = sv[j];
    for (int i = 0; i < r; ++i) {
      W[i + (size_t)jj * r] = sv[j] > 0 ? M[i + (size_t)j * r] / sv[j] : cd(i == jj ? 1 : 0, 0);
      X2[i + (size_t)jj * r] = X[i + (size_t)j * r];
    }
  }
  X = X2;
}

struct LowRank {
  int r = 0;
  std::vector<cd> U, V;  // U: m x r, V: n x r (block ~ U V^T)
  int capped = 0;
};

// rows/cols are global basis ids (RWG) of the block.
LowRank aca_block(const Ctx& C, const int64_t* rows, int m, const int64_t* cols, int n, double eps) {
  LowRank out;
  int cap = std::max(1, std::min(m, n) / 2);
  std::vector<std::vector<cd>> us, vs;
  std::vector<char> rowused(m, 0), colused(n, 0);
  double S2 = 0.0;
  int I = 0;
  bool converged = false;
  int zero_rows = 0;
  while ((int)us.size() < cap) {
    // residual row I
    std::vector<cd> v(n);
    for (int j = 0; j < n; ++j) v[j] = efie_entry(C, (int)rows[I], (int)cols[j]);
    for (size_t l = 0; l < us.size(); ++l) {
      cd ul = us[l][I];
      for (int j = 0; j < n; ++j) v[j] -= ul * vs[l][j];
    }
    rowused[I] = 1;
    int J = -1;
    double best = 0;
    for (int j = 0; j < n; ++j)
      if (!colused[j] && std::abs(v[j]) > best) { best = std::abs(v[j]); J = j; }
    if (J < 0 || best == 0.0) {
      // zero residual row: try another unused row
      ++zero_rows;
      int nxt = -1;
      for (int i = 0; i < m; ++i) if (!rowused[i]) { nxt = i; break; }
      if (nxt < 0 || zero_rows > 3) { converged = true; break; }
      I = nxt;
      continue;
    }
    cd piv = v[J];
    for (int j = 0; j < n; ++j) v[j] /= piv;
    colused[J] = 1;
    std::vector<cd> u(m);
    for (int i = 0; i < m; ++i) u[i] = efie_entry(C, (int)rows[i], (int)cols[J]);
    for (size_t l = 0; l < us.size(); ++l) {
      cd vl = vs[l][J];
      for (int i = 0; i < m; ++i) u[i] -= us[l][i] * vl;
    }
    double nu2 = 0, nv2 = 0;
    for (int i = 0; i < m; ++i) nu2 += std::norm(u[i]);
    for (int j = 0; j < n; ++j) nv2 += std::norm(v[j]);
    double cross_terms = 0;
    for (size_t l = 0; l < us.size(); ++l) {
      cd a(0, 0), b(0, 0);
      for (int i = 0; i < m; ++i) a += std::conj(us[l][i]) * u[i];
      for (int j = 0; j < n; ++j) b += std::conj(vs[l][j]) * v[j];
      cross_terms += 2.0 * std::real(a * b);
    }
    S2 += nu2 * nv2 + cross_terms;
    us.push_back(u);
    vs.push_back(v);
    if (std::sqrt(nu2 * nv2) <= eps * std::sqrt(std::max(S2, 0.0))) { converged = true; break; }
    // next row: max |u| among unused rows
    int nI = -1;
    double bu = -1;
    for (int i = 0; i < m; ++i)
      if (!rowused[i] && std::abs(u[i]) > bu) { bu = std::abs(u[i]); nI = i; }
    if (nI < 0) { converged = true; break; }
    I = nI;
  }
  if (!converged) {
    // rank cap reached: store the block exactly as a (full-rank) product
    out.capped = 1;
    if (n <= m) {
      out.r = n;
      out.U.resize((size_t)m * n);
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < m; ++i) out.U[i + (size_t)j * m] = efie_entry(C, (int)rows[i], (int)cols[j]);
      out.V.assign((size_t)n * n, cd(0, 0));
      for (int j = 0; j < n; ++j) out.V[j + (size_t)j * n] = 1.0;
    } else {
      out.r = m;
      out.U.assign((size_t)m * m, cd(0, 0));
      for (int i = 0; i < m; ++i) out.U[i + (size_t)i * m] = 1.0;
      out.V.resize((size_t)n * m);
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) out.V[j + (size_t)i * n] = efie_entry(C, (int)rows[i], (int)cols[j]);
    }
    return out;
  }
  int r = (int)us.size();
  if (r == 0) {
    out.r = 0;
    return out;
  }
  // recompression: U = Qu Ru, V = Qv Rv, Ru Rv^T = W S X^H
  std::vector<cd> A((size_t)m * r), B((size_t)n * r);
  for (int l = 0; l < r; ++l) {
    for (int i = 0; i < m; ++i) A[i + (size_t)l * m] = us[l][i];
    for (int j = 0; j < n; ++j) B[j + (size_t)l * n] = vs[l][j];
  }
  std::vector<cd> Qu, Ru, Qv, Rv;
  house_qr(m, r, A, Qu, Ru);
  house_qr(n, r, B, Qv, Rv);
  std::vector<cd> M((size_t)r * r, cd(0, 0));
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) {
      cd s(0, 0);
      for (int l = 0; l < r; ++l) s += Ru[i + (size_t)l * r] * Rv[j + (size_t)l * r];
      M[i + (size_t)j * r] = s;
    }
  std::vector<cd> W, X;
  std::vector<double> sv;
  jacobi_svd(r, M, W, sv, X);
  double tot = 0;
  for (double x : sv) tot += x * x;
  int kk = r;
  double tail = 0;
  while (kk > 1) {
    double t2 = tail + sv[kk - 1] * sv[kk - 1];
    if (std::sqrt(t2) <= eps * std::sqrt(tot)) { tail = t2; --kk; } else break;
  }
  out.r = kk;
  out.U.assign((size_t)m * kk, cd(0, 0));
  out.V.assign((size_t)n * kk, cd(0, 0));
  for (int c = 0; c < kk; ++c) {
    for (int i = 0; i < m; ++i) {
      cd s(0, 0);
      for (int l = 0; l < r; ++l) s += Qu[i + (size_t)l * m] * W[l + (size_t)c * r];
      out.U[i + (size_t)c * m] = s * sv[c];
    }
    for (int j = 0; j < n; ++j) {
      cd s(0, 0);
      for (int l = 0; l < r; ++l) s += Qv[j + (size_t)l * n] * std::conj(X[l + (size_t)c * r]);
      out.V[j + (size_t)c * n] = s;
    }
  }
  return out;
}

}  // namespace

extern "C" {

void* efie_create(int64_t n_nodes, const double* nodes, int64_t n_tris, const int64_t* tris,
                  int64_t N, const int64_t* tp, const int64_t* tm, const int64_t* vp,
                  const int64_t* vm, double k, double eta) {
  Ctx* C = new Ctx();
  C->k = k;
  C->eta = eta;
  C->nodes.resize(n_nodes);
  for (int64_t i = 0; i < n_nodes; ++i) C->nodes[i] = {nodes[3 * i], nodes[3 * i + 1], nodes[3 * i + 2]};
  C->tris.resize(n_tris);
  for (int64_t t = 0; t < n_tris; ++t) {
    Tri& T = C->tris[t];
    for (int a = 0; a < 3; ++a) { T.v[a] = (int)tris[3 * t + a]; T.p[a] = C->nodes[T.v[a]]; }
    V3 c = cross(T.p[1] - T.p[0], T.p[2] - T.p[0]);
    double cn = norm(c);
    T.area = 0.5 * cn;
    T.n = (1.0 / cn) * c;
    for (int q = 0; q < 7; ++q)
      T.q[q] = QBARY[q][0] * T.p[0] + QBARY[q][1] * T.p[1] + QBARY[q][2] * T.p[2];
  }
  C->tp.resize(N); C->tm.resize(N); C->vp.resize(N); C->vm.resize(N); C->len.resize(N);
  for (int64_t n = 0; n < N; ++n) {
    C->tp[n] = (int)tp[n]; C->tm[n] = (int)tm[n]; C->vp[n] = (int)vp[n]; C->vm[n] = (int)vm[n];
    // edge = the two vertices shared by T+ and T-
    const Tri& A = C->tris[tp[n]];
    int e[2], ne = 0;
    for (int a = 0; a < 3; ++a)
      if (A.v[a] != vp[n] && ne < 2) e[ne++] = A.v[a];
    C->len[n] = norm(C->nodes[e[0]] - C->nodes[e[1]]);
  }
  return C;
}

void efie_destroy(void* c) { delete (Ctx*)c; }

// Dense block: out[i + j*m] = Z(rows[i], cols[j]) (complex128 interleaved)
void efie_block(void* c, int64_t m, const int64_t* rows, int64_t n, const int64_t* cols, double* out) {
  const Ctx& C = *(Ctx*)c;
  cd* o = (cd*)out;
#pragma omp parallel for schedule(dynamic, 4) collapse(2)
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) o[i + j * m] = efie_entry(C, (int)rows[i], (int)cols[j]);
}

// Near blocks. For block b: rows = idx[roff[b] .. roff[b]+rn[b]), cols likewise.
// Writes column-major rn x cn at out + 2*ooff[b]. Diagonal blocks (sym[b]=1)
// compute the upper triangle and mirror it (exact symmetry by construction).
void efie_near(void* c, int64_t nb, const int64_t* idx, const int64_t* roff, const int64_t* rn,
               const int64_t* coff, const int64_t* cn, const int64_t* sym, const int64_t* ooff,
               double* out) {
  const Ctx& C = *(Ctx*)c;
  cd* o = (cd*)out;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t* rows = idx + roff[b];
    const int64_t* cols = idx + coff[b];
    int64_t m = rn[b], n = cn[b];
    cd* blk = o + ooff[b];
    if (sym[b]) {
      for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i <= j; ++i) {
          cd z = efie_entry(C, (int)rows[i], (int)cols[j]);
          blk[i + j * m] = z;
          blk[j + i * m] = z;
        }
    } else {
      for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) blk[i + j * m] = efie_entry(C, (int)rows[i], (int)cols[j]);
    }
  }
}

// Far blocks, two-phase. Phase 1 computes and keeps results; returns handle.
struct FarResult { std::vector<LowRank> blocks; };

void* efie_far(void* c, int64_t nb, const int64_t* idx, const int64_t* roff, const int64_t* rn,
               const int64_t* coff, const int64_t* cn, double eps, int64_t* ranks, int64_t* capped) {
  const Ctx& C = *(Ctx*)c;
  FarResult* R = new FarResult();
  R->blocks.resize(nb);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t b = 0; b < nb; ++b) {
    R->blocks[b] = aca_block(C, idx + roff[b], (int)rn[b], idx + coff[b], (int)cn[b], eps);
    ranks[b] = R->blocks[b].r;
    capped[b] = R->blocks[b].capped;
  }
  return R;
}

// Phase 2: copy U (m x r) then V (n x r) of block b to out + 2*ooff[b].
void efie_far_copy(void* h, int64_t nb, const int64_t* ooff, double* out) {
  FarResult* R = (FarResult*)h;
  cd* o = (cd*)out;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    const LowRank& L = R->blocks[b];
    cd* dst = o + ooff[b];
    std::copy(L.U.begin(), L.U.end(), dst);
    std::copy(L.V.begin(), L.V.end(), dst + L.U.size());
  }
}

void efie_far_free(void* h) { delete (FarResult*)h; }

// Analytic potential integrals (exposed for tests): tri = 3 points (9 doubles), r = 3 doubles.
void efie_potential(const double* tri, const double* r, double* Js, double* Jvec) {
  Tri T;
  for (int a = 0; a < 3; ++a) { T.p[a] = {tri[3 * a], tri[3 * a + 1], tri[3 * a + 2]}; T.v[a] = a; }
  V3 cr = cross(T.p[1] - T.p[0], T.p[2] - T.p[0]);
  T.n = (1.0 / norm(cr)) * cr;
  T.area = 0.5 * norm(cr);
  V3 jv;
  potential_integrals(T, {r[0], r[1], r[2]}, *Js, jv);
  Jvec[0] = jv.x; Jvec[1] = jv.y; Jvec[2] = jv.z;
}

// Plane-wave RHS: b_m = Int f_m . E_inc dS, E_inc = e_pol exp(-j k khat . r).
// khat/epol: nrhs x 3 (epol complex: nrhs x 3 x 2). out: column-major N x nrhs complex.
void efie_rhs(void* c, int64_t nrhs, const double* khat, const double* epol, double* out) {
  const Ctx& C = *(Ctx*)c;
  int64_t N = (int64_t)C.tp.size();
  cd* o = (cd*)out;
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t q = 0; q < nrhs; ++q)
    for (int64_t m = 0; m < N; ++m) {
      V3 kh = {khat[3 * q], khat[3 * q + 1], khat[3 * q + 2]};
      cd ex(epol[6 * q + 0], epol[6 * q + 1]), ey(epol[6 * q + 2], epol[6 * q + 3]), ez(epol[6 * q + 4], epol[6 * q + 5]);
      cd acc(0, 0);
      for (int s = 0; s < 2; ++s) {
        const Tri& T = C.tris[s == 0 ? C.tp[m] : C.tm[m]];
        double sg = s == 0 ? 1.0 : -1.0;
        V3 v = C.nodes[s == 0 ? C.vp[m] : C.vm[m]];
        double cf = sg * C.len[m] / (2 * T.area);
        cd t(0, 0);
        for (int a = 0; a < 7; ++a) {
          V3 f = T.q[a] - v;
          double ph = -C.k * dot(kh, T.q[a]);
          cd e = cd(std::cos(ph), std::sin(ph));
          t += QW[a] * (f.x * ex + f.y * ey + f.z * ez) * e;
        }
        acc += cf * T.area * t;
      }
      o[m + q * N] = acc;
    }
}

// Far-field radiation integral F(rhat) = Int J(r') exp(+j k rhat.r') dS' for
// currents I (N complex) at ndir directions; out: ndir x 3 complex.
void efie_farfield(void* c, const double* I, int64_t ndir, const double* rhat, double* out) {
  const Ctx& C = *(Ctx*)c;
  int64_t N = (int64_t)C.tp.size();
  const cd* cur = (const cd*)I;
  cd* o = (cd*)out;
#pragma omp parallel for schedule(static)
  for (int64_t d = 0; d < ndir; ++d) {
    V3 rh = {rhat[3 * d], rhat[3 * d + 1], rhat[3 * d + 2]};
    cd fx(0, 0), fy(0, 0), fz(0, 0);
    for (int64_t m = 0; m < N; ++m) {
      for (int s = 0; s < 2; ++s) {
        const Tri& T = C.tris[s == 0 ? C.tp[m] : C.tm[m]];
        double sg = s == 0 ? 1.0 : -1.0;
        V3 v = C.nodes[s == 0 ? C.vp[m] : C.vm[m]];
        double cf = sg * C.len[m] / (2 * T.area) * T.area;
        for (int a = 0; a < 7; ++a) {
          V3 f = T.q[a] - v;
          double ph = C.k * dot(rh, T.q[a]);
          cd e = cur[m] * cd(std::cos(ph), std::sin(ph)) * (QW[a] * cf);
          fx += f.x * e; fy += f.y * e; fz += f.z * e;
        }
      }
    }
    o[3 * d] = fx; o[3 * d + 1] = fy; o[3 * d + 2] = fz;
  }
}

}  // extern "C"
