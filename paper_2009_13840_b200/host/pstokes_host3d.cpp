// 3D extension of the host-side input producer (include/pstokes_host.h,
// psh_mesh_unit_cube / psh3_*): hexahedral meshes of the unit cube with
// seeded vertex jitter, tensor Gauss quadrature on the trilinear elements
// and bilinear faces, hierarchical orthonormal bases, and the HHO local
// Stokes blocks of the hybrid-pressure scheme (HHO-hp, BASELINE.json
// configs 3 and 5), plus the face-block (BSR) pattern of the condensed
// operator.
//
// The reference is 2D only (mesh.hpp:21 `using Vec2`); this is
// the 3D generalisation of its discretisation, written here and shared by
// the oracle and the GPU pipeline (SURVEY.md §0 finding 3, §7.3 H3):
//  * mesh: vertex (i,j,l) at (i/n, j/n, l/n); interior vertices moved by
//    frac*h*SplitMix64(seed).sym() in x, y, z order (l outer, j, i inner) —
//    mesh.hpp:279-288's recipe in 3D. Elements l-major, j, i inner; local
//    faces ordered x-, x+, y-, y+, z-, z+; faces numbered first-seen over
//    that loop (mesh.hpp:87-119), each stored with its vertices ordered so
//    that d/ds x cross d/dt x points out of its first (`left`) element.
//    Boundary faces: Neumann on z = 1, Dirichlet elsewhere.
//  * non-planar faces (jittered hexahedra): integrals are taken over the true
//    bilinear surface (vector area element x_s cross x_t, exact for the
//    divergence-theorem terms); the face polynomial space is P^k in the
//    coordinates of the orthogonal projection onto the face's mean plane
//    (normal = cross product of the diagonals), centred at the vertex mean
//    and scaled by the face diameter. On planar faces this is exactly
//    P^k(F) of the reference (basis.hpp:151-202).
//  * element bases: scaled monomials (x - x_T)/h_T in degree-lexicographic
//    order (z-power outer, then y), MGS with one re-orthogonalisation pass in
//    the quadrature inner product (basis.hpp:29-52, 61-147).
//  * quadrature: m^3 / m^2 tensor Gauss-Legendre rules with
//    m = (q + 2)/2 + 1 for the reference's degree q = 2(k+1)+1
//    (hho_local.hpp:28): exact for the polynomial integrands times the
//    trilinear Jacobian (degree <= q + 2 per variable).
//  * local operator: hho_local.hpp:26-318 with three velocity components:
//    reconstruction with mean-value closure, face-residual stabilisation
//    scaled by 1/h_F (h_F = face diameter), Nitsche Dirichlet terms with
//    eta = 3(k+1)^2, element pressure rows -int div u_T q, face-pressure
//    mass rows int_F (u_T - u_F).n q_F, momentum columns = transpose except
//    the face-pressure columns on Dirichlet faces. Local dof order
//    [U_T (c-major) | U_F per face (c-major) | P_T | P_F per face].
//  * data: 0 zero; 3 random modal body force (i.i.d. N(0,1) coefficients of
//    the degree-k orthonormal element modes per component, SplitMix64(seed)
//    + Box-Muller, element-major; homogeneous g_D / g_N); 4 the manufactured
//    field u = (sin pi y sin pi z, sin pi x sin pi z, sin pi x sin pi y),
//    p = sin 2pi x sin 2pi y sin 2pi z (validation).

#include "pstokes_host.h"

#include <omp.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace psh3 {

thread_local std::string g_err;

struct V3 {
  double x = 0.0, y = 0.0, z = 0.0;
};
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }

struct SplitMix64 {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double sym() { return 2.0 * double(next() >> 11) * 0x1.0p-53 - 1.0; }
  /// standard normal by Box-Muller (cosine branch; two draws per value)
  double normal() {
    const double u1 = double((next() >> 11) + 1) * 0x1.0p-53;  // (0, 1]
    const double u2 = double(next() >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
};

inline int dimP2(int d) { return d < 0 ? 0 : (d + 1) * (d + 2) / 2; }
inline int dimP3(int d) { return d < 0 ? 0 : (d + 1) * (d + 2) * (d + 3) / 6; }

// ---------------------------------------------------------------------------
// mesh
// ---------------------------------------------------------------------------

// local faces x-, x+, y-, y+, z-, z+ of the hexahedron with vertices
// v[a] at (ia, ja, la) = (a & 1, (a >> 1) & 1 ^ (a & 1)...): we use the
// explicit order v0 (0,0,0) v1 (1,0,0) v2 (1,1,0) v3 (0,1,0) and v4..v7 the
// same at l + 1; each quadruple is counter-clockwise seen from outside.
constexpr int kFaceVerts[6][4] = {{0, 4, 7, 3}, {1, 2, 6, 5}, {0, 1, 5, 4},
                                  {3, 7, 6, 2}, {0, 3, 2, 1}, {4, 5, 6, 7}};
constexpr int kHexOff[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                               {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

struct Mesh {
  int n = 0;
  std::vector<V3> v;
  std::vector<std::array<int, 8>> hex;
  std::vector<std::array<int, 4>> fv;  // oriented out of `left`
  std::vector<int> left, right, tag;   // tag: 0 interior, 1 Dirichlet, 2 Neumann
  std::vector<std::array<int, 6>> ef;  // element faces
  std::vector<std::array<int8_t, 6>> es;
  int nelem() const { return int(hex.size()); }
  int nfaces() const { return int(fv.size()); }
};

inline int vid(int i, int j, int l, int n) { return (l * (n + 1) + j) * (n + 1) + i; }

void build_unit_cube(Mesh& m, int n, double frac, uint64_t seed, bool neumann_top) {
  m.n = n;
  m.v.resize(size_t(n + 1) * (n + 1) * (n + 1));
  for (int l = 0; l <= n; ++l)
    for (int j = 0; j <= n; ++j)
      for (int i = 0; i <= n; ++i)
        m.v[vid(i, j, l, n)] = {double(i) / n, double(j) / n, double(l) / n};
  if (frac > 0.0) {
    SplitMix64 rng{seed};
    const double h = 1.0 / n;
    for (int l = 1; l < n; ++l)
      for (int j = 1; j < n; ++j)
        for (int i = 1; i < n; ++i) {
          V3& p = m.v[vid(i, j, l, n)];
          p.x += frac * h * rng.sym();
          p.y += frac * h * rng.sym();
          p.z += frac * h * rng.sym();
        }
  }
  m.hex.resize(size_t(n) * n * n);
  for (int l = 0; l < n; ++l)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        auto& h = m.hex[(size_t(l) * n + j) * n + i];
        for (int a = 0; a < 8; ++a) h[a] = vid(i + kHexOff[a][0], j + kHexOff[a][1], l + kHexOff[a][2], n);
      }
  // first-seen face numbering (mesh.hpp:87-119); key: the three smallest
  // vertex ids (three vertices of a hexahedral mesh lie on one face at most)
  const int ne = m.nelem();
  std::unordered_map<uint64_t, int> seen;
  seen.reserve(size_t(ne) * 4);
  m.ef.resize(ne);
  m.es.resize(ne);
  for (int e = 0; e < ne; ++e) {
    for (int lf = 0; lf < 6; ++lf) {
      std::array<int, 4> q;
      for (int a = 0; a < 4; ++a) q[a] = m.hex[e][kFaceVerts[lf][a]];
      std::array<int, 4> s = q;
      std::sort(s.begin(), s.end());
      const uint64_t key = (uint64_t(s[0]) << 42) | (uint64_t(s[1]) << 21) | uint64_t(s[2]);
      auto it = seen.find(key);
      if (it == seen.end()) {
        const int f = m.nfaces();
        seen.emplace(key, f);
        m.fv.push_back(q);
        m.left.push_back(e);
        m.right.push_back(-1);
        m.tag.push_back(0);
        m.ef[e][lf] = f;
        m.es[e][lf] = 1;
      } else {
        const int f = it->second;
        if (m.right[f] >= 0) throw std::runtime_error("mesh3: non-manifold face");
        m.right[f] = e;
        m.ef[e][lf] = f;
        m.es[e][lf] = -1;
      }
    }
  }
  int nneu = 0;
  for (int f = 0; f < m.nfaces(); ++f) {
    if (m.right[f] >= 0) continue;
    bool top = true;
    for (int a = 0; a < 4; ++a) top = top && m.v[m.fv[f][a]].z == 1.0;
    m.tag[f] = (neumann_top && top) ? 2 : 1;
    nneu += m.tag[f] == 2;
  }
  if (neumann_top && nneu == 0) throw std::runtime_error("mesh3: no face on z = 1");
}

// ---------------------------------------------------------------------------
// quadrature
// ---------------------------------------------------------------------------

void gauss_legendre(int m, std::vector<double>& x, std::vector<double>& w) {
  x.assign(m, 0.0);
  w.assign(m, 0.0);
  for (int i = 0; i < m; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (m + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = t;
      for (int k = 2; k <= m; ++k) {
        const double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = m * (t * p1 - p0) / (t * t - 1.0);
      const double dt = p1 / dp;
      t -= dt;
      if (std::abs(dt) < 1e-15) break;
    }
    x[i] = t;
    w[i] = 2.0 / ((1.0 - t * t) * dp * dp);
  }
}

inline int rule_points(int qdeg) { return (qdeg + 2) / 2 + 1; }

struct ElemRule {
  std::vector<V3> p;
  std::vector<double> w;
  int size() const { return int(w.size()); }
};

/// Trilinear map of element e and its m^3 Gauss rule (weights * det J).
ElemRule element_rule(const Mesh& m, int e, int qdeg) {
  std::vector<double> x, w;
  const int np = rule_points(qdeg);
  gauss_legendre(np, x, w);
  V3 X[8];
  for (int a = 0; a < 8; ++a) X[a] = m.v[m.hex[e][a]];
  ElemRule r;
  r.p.reserve(size_t(np) * np * np);
  r.w.reserve(size_t(np) * np * np);
  for (int c = 0; c < np; ++c)
    for (int b = 0; b < np; ++b)
      for (int a = 0; a < np; ++a) {
        const double xi[3] = {x[a], x[b], x[c]};
        V3 p{}, d0{}, d1{}, d2{};
        for (int v = 0; v < 8; ++v) {
          const double s[3] = {2.0 * kHexOff[v][0] - 1.0, 2.0 * kHexOff[v][1] - 1.0,
                               2.0 * kHexOff[v][2] - 1.0};
          const double f0 = 1.0 + s[0] * xi[0], f1 = 1.0 + s[1] * xi[1], f2 = 1.0 + s[2] * xi[2];
          p = p + (0.125 * f0 * f1 * f2) * X[v];
          d0 = d0 + (0.125 * s[0] * f1 * f2) * X[v];
          d1 = d1 + (0.125 * f0 * s[1] * f2) * X[v];
          d2 = d2 + (0.125 * f0 * f1 * s[2]) * X[v];
        }
        const double det = dot(d0, cross(d1, d2));
        if (!(det > 0.0))
          throw std::runtime_error("mesh3: element " + std::to_string(e) + " has a non-positive Jacobian");
        r.p.push_back(p);
        r.w.push_back(w[a] * w[b] * w[c] * det);
      }
  return r;
}

struct FaceRule {
  std::vector<V3> p, na;  // points, vector area weights (out of `left`)
  std::vector<double> w;  // scalar area weights
  int size() const { return int(w.size()); }
};

FaceRule face_rule(const Mesh& m, int f, int qdeg) {
  std::vector<double> x, w;
  const int np = rule_points(qdeg);
  gauss_legendre(np, x, w);
  const V3 a = m.v[m.fv[f][0]], b = m.v[m.fv[f][1]], c = m.v[m.fv[f][2]], d = m.v[m.fv[f][3]];
  FaceRule r;
  for (int j = 0; j < np; ++j)
    for (int i = 0; i < np; ++i) {
      const double s = x[i], t = x[j];
      const V3 p = 0.25 * ((1 - s) * (1 - t) * a + (1 + s) * (1 - t) * b + (1 + s) * (1 + t) * c +
                           (1 - s) * (1 + t) * d);
      const V3 xs = 0.25 * ((1 - t) * (b - a) + (1 + t) * (c - d));
      const V3 xt = 0.25 * ((1 - s) * (d - a) + (1 + s) * (c - b));
      const V3 nv = cross(xs, xt);
      r.p.push_back(p);
      r.na.push_back((w[i] * w[j]) * nv);
      r.w.push_back(w[i] * w[j] * norm(nv));
    }
  return r;
}

// ---------------------------------------------------------------------------
// dense helpers (column-major)
// ---------------------------------------------------------------------------

struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rr, int cc) : r(rr), c(cc), a(size_t(rr) * cc, 0.0) {}
  double& operator()(int i, int j) { return a[size_t(i) + size_t(j) * r]; }
  double operator()(int i, int j) const { return a[size_t(i) + size_t(j) * r]; }
};

void lu_solve(Mat A, Mat& B) {
  const int n = A.r;
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A(i, k)) > std::abs(A(p, k))) p = i;
    if (A(p, k) == 0.0) throw std::runtime_error("hho3: singular reconstruction system");
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
      for (int j = 0; j < B.c; ++j) std::swap(B(k, j), B(p, j));
    }
    for (int i = k + 1; i < n; ++i) {
      const double l = A(i, k) / A(k, k);
      if (l == 0.0) continue;
      for (int j = k + 1; j < n; ++j) A(i, j) -= l * A(k, j);
      for (int j = 0; j < B.c; ++j) B(i, j) -= l * B(k, j);
    }
  }
  for (int j = 0; j < B.c; ++j)
    for (int i = n - 1; i >= 0; --i) {
      double s = B(i, j);
      for (int q = i + 1; q < n; ++q) s -= A(i, q) * B(q, j);
      B(i, j) = s / A(i, i);
    }
}

/// MGS with one re-orthogonalisation pass (basis.hpp:29-52); returns the
/// lower-triangular C with phi_i = sum_j C(i,j) m_j.
Mat orthonormalize(Mat& vals, const std::vector<double>& w, const char* what) {
  const int n = vals.c, nq = vals.r;
  Mat C(n, n);
  for (int i = 0; i < n; ++i) C(i, i) = 1.0;
  auto ip = [&](int i, int j) {
    double s = 0.0;
    for (int q = 0; q < nq; ++q) s += vals(q, i) * (w[q] * vals(q, j));
    return s;
  };
  for (int i = 0; i < n; ++i) {
    for (int pass = 0; pass < 2; ++pass)
      for (int j = 0; j < i; ++j) {
        const double r = ip(i, j);
        for (int q = 0; q < nq; ++q) vals(q, i) -= r * vals(q, j);
        for (int k = 0; k <= j; ++k) C(i, k) -= r * C(j, k);
      }
    const double nrm = std::sqrt(ip(i, i));
    if (!(nrm > 1e-14)) throw std::runtime_error(std::string("orthonormalize: singular Gram matrix on ") + what);
    for (int q = 0; q < nq; ++q) vals(q, i) /= nrm;
    for (int k = 0; k <= i; ++k) C(i, k) /= nrm;
  }
  return C;
}

// ---------------------------------------------------------------------------
// bases
// ---------------------------------------------------------------------------

constexpr int kMaxMono = 56;  // dim P^5 in 3D

struct ElemBasis {
  int deg = 0, dim = 0;
  V3 c;
  double h = 1.0;
  Mat C;
  /// powers px[a] = x^a (a <= deg) of the scaled coordinates
  void powers(V3 p, double* px, double* py, double* pz) const {
    const double x = (p.x - c.x) / h, y = (p.y - c.y) / h, z = (p.z - c.z) / h;
    px[0] = py[0] = pz[0] = 1.0;
    for (int a = 1; a <= deg; ++a) {
      px[a] = px[a - 1] * x;
      py[a] = py[a - 1] * y;
      pz[a] = pz[a - 1] * z;
    }
  }
  void monos(V3 p, double* m) const {
    double px[8], py[8], pz[8];
    powers(p, px, py, pz);
    int idx = 0;
    for (int d = 0; d <= deg; ++d)
      for (int az = 0; az <= d; ++az)
        for (int ay = 0; ay <= d - az; ++ay) m[idx++] = px[d - ay - az] * py[ay] * pz[az];
  }
  void init(const ElemRule& r, V3 center, double diam, int degree) {
    deg = degree;
    dim = dimP3(degree);
    if (dim > kMaxMono) throw std::invalid_argument("hho3: degree too high");
    c = center;
    h = diam;
    Mat vals(r.size(), dim);
    double mm[kMaxMono];
    for (int q = 0; q < r.size(); ++q) {
      monos(r.p[q], mm);
      for (int i = 0; i < dim; ++i) vals(q, i) = mm[i];
    }
    C = orthonormalize(vals, r.w, "element");
  }
  void eval(V3 p, double* out) const {
    double mm[kMaxMono];
    monos(p, mm);
    for (int i = 0; i < dim; ++i) {
      double s = 0.0;
      for (int j = 0; j <= i; ++j) s += C(i, j) * mm[j];
      out[i] = s;
    }
  }
  /// gradients out[3 i + d]
  void grad(V3 p, double* out) const {
    double X[8], Y[8], Z[8];
    powers(p, X, Y, Z);
    double gx[kMaxMono], gy[kMaxMono], gz[kMaxMono];
    int idx = 0;
    for (int d = 0; d <= deg; ++d)
      for (int az = 0; az <= d; ++az)
        for (int ay = 0; ay <= d - az; ++ay) {
          const int ax = d - ay - az;
          gx[idx] = ax == 0 ? 0.0 : ax * X[ax - 1] * Y[ay] * Z[az] / h;
          gy[idx] = ay == 0 ? 0.0 : ay * X[ax] * Y[ay - 1] * Z[az] / h;
          gz[idx] = az == 0 ? 0.0 : az * X[ax] * Y[ay] * Z[az - 1] / h;
          ++idx;
        }
    for (int i = 0; i < dim; ++i) {
      double sx = 0.0, sy = 0.0, sz = 0.0;
      for (int j = 0; j <= i; ++j) {
        sx += C(i, j) * gx[j];
        sy += C(i, j) * gy[j];
        sz += C(i, j) * gz[j];
      }
      out[3 * i] = sx;
      out[3 * i + 1] = sy;
      out[3 * i + 2] = sz;
    }
  }
};

struct FaceBasis {
  int deg = 0, dim = 0;
  V3 c, t1, t2;
  double h = 1.0;
  Mat C;
  void monos(V3 p, double* m) const {
    const V3 d = p - c;
    const double x = dot(d, t1) / h, y = dot(d, t2) / h;
    double px[8], py[8];
    px[0] = py[0] = 1.0;
    for (int a = 1; a <= deg; ++a) {
      px[a] = px[a - 1] * x;
      py[a] = py[a - 1] * y;
    }
    int idx = 0;
    for (int dd = 0; dd <= deg; ++dd)
      for (int ay = 0; ay <= dd; ++ay) m[idx++] = px[dd - ay] * py[ay];
  }
  void init(const Mesh& m, int f, const FaceRule& r, int degree) {
    deg = degree;
    dim = dimP2(degree);
    const V3 a = m.v[m.fv[f][0]], b = m.v[m.fv[f][1]], cc = m.v[m.fv[f][2]], d = m.v[m.fv[f][3]];
    c = 0.25 * (a + b + cc + d);
    h = 0.0;
    const V3 P[4] = {a, b, cc, d};
    for (int i = 0; i < 4; ++i)
      for (int j = i + 1; j < 4; ++j) h = std::max(h, norm(P[i] - P[j]));
    V3 nb = cross(cc - a, d - b);
    nb = (1.0 / norm(nb)) * nb;
    V3 u = b - a;
    u = u - dot(u, nb) * nb;
    t1 = (1.0 / norm(u)) * u;
    t2 = cross(nb, t1);
    Mat vals(r.size(), dim);
    double mm[32];
    for (int q = 0; q < r.size(); ++q) {
      monos(r.p[q], mm);
      for (int i = 0; i < dim; ++i) vals(q, i) = mm[i];
    }
    C = orthonormalize(vals, r.w, "face");
  }
  void eval(V3 p, double* out) const {
    double mm[32];
    monos(p, mm);
    for (int i = 0; i < dim; ++i) {
      double s = 0.0;
      for (int j = 0; j <= i; ++j) s += C(i, j) * mm[j];
      out[i] = s;
    }
  }
};

double face_diameter(const Mesh& m, int f) {
  double h = 0.0;
  for (int i = 0; i < 4; ++i)
    for (int j = i + 1; j < 4; ++j) h = std::max(h, norm(m.v[m.fv[f][i]] - m.v[m.fv[f][j]]));
  return h;
}

// ---------------------------------------------------------------------------
// problem data
// ---------------------------------------------------------------------------

struct Data {
  int kind = 0;
  uint64_t seed = 0;
  // manufactured field (kind 4)
  static void u(V3 p, double* o) {
    const double pi = M_PI;
    o[0] = std::sin(pi * p.y) * std::sin(pi * p.z);
    o[1] = std::sin(pi * p.x) * std::sin(pi * p.z);
    o[2] = std::sin(pi * p.x) * std::sin(pi * p.y);
  }
  static double pr(V3 p) {
    return std::sin(2 * M_PI * p.x) * std::sin(2 * M_PI * p.y) * std::sin(2 * M_PI * p.z);
  }
  /// grad u: g[i][j] = d u_j / d x_i
  static void gradu(V3 p, double g[3][3]) {
    const double pi = M_PI;
    const double sx = std::sin(pi * p.x), sy = std::sin(pi * p.y), sz = std::sin(pi * p.z);
    const double cx = std::cos(pi * p.x), cy = std::cos(pi * p.y), cz = std::cos(pi * p.z);
    g[0][0] = 0.0;          g[1][0] = pi * cy * sz; g[2][0] = pi * sy * cz;
    g[0][1] = pi * cx * sz; g[1][1] = 0.0;          g[2][1] = pi * sx * cz;
    g[0][2] = pi * cx * sy; g[1][2] = pi * sx * cy; g[2][2] = 0.0;
  }
  void f_manufactured(V3 p, double* o) const {
    double uu[3];
    u(p, uu);
    const double t = 2 * M_PI;
    const double s0 = std::sin(t * p.x), s1 = std::sin(t * p.y), s2 = std::sin(t * p.z);
    const double c0 = std::cos(t * p.x), c1 = std::cos(t * p.y), c2 = std::cos(t * p.z);
    const double lap = 2.0 * M_PI * M_PI;  // -Laplacian of each component
    o[0] = lap * uu[0] + t * c0 * s1 * s2;
    o[1] = lap * uu[1] + t * s0 * c1 * s2;
    o[2] = lap * uu[2] + t * s0 * s1 * c2;
  }
  void gd(V3 p, double* o) const {
    if (kind == 4) u(p, o);
    else o[0] = o[1] = o[2] = 0.0;
  }
  /// traction -n.grad(u) + p n (stokes_data.hpp:55-60)
  void gn(V3 p, V3 n, double* o) const {
    if (kind != 4) {
      o[0] = o[1] = o[2] = 0.0;
      return;
    }
    double g[3][3];
    gradu(p, g);
    const double pp = pr(p), nn[3] = {n.x, n.y, n.z};
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int i = 0; i < 3; ++i) s += nn[i] * g[i][j];
      o[j] = -s + pp * nn[j];
    }
  }
};

// ---------------------------------------------------------------------------
// HHO-hp local blocks
// ---------------------------------------------------------------------------

struct LocalLayout {
  int ne, nf, np, nfp, nvel, n;
  int vel_elem(int c, int m) const { return c * ne + m; }
  int vel_face(int lf, int c, int m) const { return 3 * ne + lf * 3 * nf + c * nf + m; }
  int press_elem(int m) const { return nvel + m; }
  int press_face(int lf, int m) const { return nvel + np + lf * nfp + m; }
};

LocalLayout local_layout(int k) {
  LocalLayout L;
  L.ne = dimP3(k + 1);
  L.nf = dimP2(k);
  L.np = dimP3(k);
  L.nfp = L.nf;
  L.nvel = 3 * (L.ne + 6 * L.nf);
  L.n = L.nvel + L.np + 6 * L.nfp;
  return L;
}

struct Geo {
  V3 cen;
  double vol = 0.0, diam = 0.0;
};

Geo element_geo(const Mesh& m, int e, const ElemRule& r) {
  Geo g;
  V3 s{};
  for (int q = 0; q < r.size(); ++q) {
    g.vol += r.w[q];
    s = s + r.w[q] * r.p[q];
  }
  g.cen = (1.0 / g.vol) * s;
  for (int a = 0; a < 8; ++a)
    for (int b = a + 1; b < 8; ++b)
      g.diam = std::max(g.diam, norm(m.v[m.hex[e][a]] - m.v[m.hex[e][b]]));
  return g;
}

/// Local matrix (column-major n x n) and load of element e (hybrid pressure,
/// element velocity degree k+1: hho_local.hpp:193-318 in 3D).
void build_local(const Mesh& mesh, int e, int k, double eta, const Data& data, double* mat,
                 double* rhs) {
  const LocalLayout L = local_layout(k);
  const int qd = 2 * (k + 1) + 1;
  const ElemRule er = element_rule(mesh, e, qd);
  const Geo geo = element_geo(mesh, e, er);
  ElemBasis rb;
  rb.init(er, geo.cen, geo.diam, k + 1);
  const int nrec = rb.dim, ne = L.ne, nf = L.nf, ns = ne + 6 * nf;
  FaceRule fr[6];
  FaceBasis fb[6];
  int fid[6];
  double sgn[6], hf[6];
  for (int lf = 0; lf < 6; ++lf) {
    fid[lf] = mesh.ef[e][lf];
    sgn[lf] = mesh.es[e][lf];
    fr[lf] = face_rule(mesh, fid[lf], qd);
    fb[lf].init(mesh, fid[lf], fr[lf], k);
    hf[lf] = face_diameter(mesh, fid[lf]);
  }
  auto fo = [&](int lf) { return ne + lf * nf; };
  const int nq = er.size();
  // element basis values / gradients at the element points
  std::vector<double> PH(size_t(nq) * nrec), GR(size_t(nq) * nrec * 3);
  for (int q = 0; q < nq; ++q) {
    rb.eval(er.p[q], &PH[size_t(q) * nrec]);
    rb.grad(er.p[q], &GR[size_t(q) * nrec * 3]);
  }
  Mat K(nrec, nrec);
  std::vector<double> mom(nrec, 0.0);
  for (int q = 0; q < nq; ++q) {
    const double w = er.w[q];
    const double* g = &GR[size_t(q) * nrec * 3];
    for (int j = 0; j < nrec; ++j) {
      const double gj0 = w * g[3 * j], gj1 = w * g[3 * j + 1], gj2 = w * g[3 * j + 2];
      for (int i = 0; i < nrec; ++i) K(i, j) += g[3 * i] * gj0 + g[3 * i + 1] * gj1 + g[3 * i + 2] * gj2;
    }
    for (int i = 0; i < nrec; ++i) mom[i] += w * PH[size_t(q) * nrec + i];
  }
  // face tables: element values/gradients, face values, normal gradients
  struct FT {
    int nq;
    std::vector<double> phi, g, psi;  // nq x nrec, nq x nrec x 3, nq x nf
  } ft[6];
  for (int lf = 0; lf < 6; ++lf) {
    const int m = fr[lf].size();
    ft[lf].nq = m;
    ft[lf].phi.resize(size_t(m) * nrec);
    ft[lf].g.resize(size_t(m) * nrec * 3);
    ft[lf].psi.resize(size_t(m) * nf);
    for (int q = 0; q < m; ++q) {
      rb.eval(fr[lf].p[q], &ft[lf].phi[size_t(q) * nrec]);
      rb.grad(fr[lf].p[q], &ft[lf].g[size_t(q) * nrec * 3]);
      fb[lf].eval(fr[lf].p[q], &ft[lf].psi[size_t(q) * nf]);
    }
  }
  // reconstruction right-hand side and bordered solve (hho_local.hpp:130-168)
  Mat B(nrec + 1, ns);
  for (int j = 0; j < ne; ++j)
    for (int i = 0; i < nrec; ++i) B(i, j) = K(i, j);
  for (int lf = 0; lf < 6; ++lf) {
    for (int q = 0; q < ft[lf].nq; ++q) {
      const V3 na = sgn[lf] * fr[lf].na[q];
      const double* g = &ft[lf].g[size_t(q) * nrec * 3];
      const double* phi = &ft[lf].phi[size_t(q) * nrec];
      const double* psi = &ft[lf].psi[size_t(q) * nf];
      for (int i = 0; i < nrec; ++i) {
        const double gn = g[3 * i] * na.x + g[3 * i + 1] * na.y + g[3 * i + 2] * na.z;
        for (int m = 0; m < nf; ++m) B(i, fo(lf) + m) += gn * psi[m];
        for (int m = 0; m < ne; ++m) B(i, m) -= gn * phi[m];
      }
    }
  }
  for (int m = 0; m < ne; ++m) B(nrec, m) = mom[m];
  {
    Mat S(nrec + 1, nrec + 1);
    for (int j = 0; j < nrec; ++j)
      for (int i = 0; i < nrec; ++i) S(i, j) = K(i, j);
    for (int i = 0; i < nrec; ++i) {
      S(i, nrec) = mom[i];
      S(nrec, i) = mom[i];
    }
    lu_solve(S, B);
  }
  Mat P(nrec, ns);
  for (int j = 0; j < ns; ++j)
    for (int i = 0; i < nrec; ++i) P(i, j) = B(i, j);
  // viscous block A = P^T K P + sum_F 1/h_F R^T W R + Nitsche (Dirichlet)
  Mat KP(nrec, ns), A(ns, ns);
  for (int j = 0; j < ns; ++j)
    for (int i = 0; i < nrec; ++i) {
      double s = 0.0;
      for (int l = 0; l < nrec; ++l) s += K(i, l) * P(l, j);
      KP(i, j) = s;
    }
  for (int j = 0; j < ns; ++j)
    for (int i = 0; i < ns; ++i) {
      double s = 0.0;
      for (int l = 0; l < nrec; ++l) s += P(l, i) * KP(l, j);
      A(i, j) = s;
    }
  // per face: trace / weighted normal derivative of the reconstruction
  std::vector<std::vector<double>> DNW(6);  // nq x ns: (grad p(v) . n) * dA
  for (int lf = 0; lf < 6; ++lf) {
    const int m = ft[lf].nq;
    std::vector<double> rect(size_t(m) * ns), R(size_t(m) * ns);
    DNW[lf].assign(size_t(m) * ns, 0.0);
    for (int q = 0; q < m; ++q) {
      const V3 na = sgn[lf] * fr[lf].na[q];
      const double* g = &ft[lf].g[size_t(q) * nrec * 3];
      const double* phi = &ft[lf].phi[size_t(q) * nrec];
      for (int s = 0; s < ns; ++s) {
        double tr = 0.0, dn = 0.0;
        for (int i = 0; i < nrec; ++i) {
          tr += phi[i] * P(i, s);
          dn += (g[3 * i] * na.x + g[3 * i + 1] * na.y + g[3 * i + 2] * na.z) * P(i, s);
        }
        rect[size_t(q) * ns + s] = tr;
        DNW[lf][size_t(q) * ns + s] = dn;
      }
    }
    const double* psi = ft[lf].psi.data();
    const std::vector<double>& w = fr[lf].w;
    // coeff1 (nf x ns) = Psi^T W (-rec_tr) + I on this face's columns
    std::vector<double> c1(size_t(nf) * ns, 0.0);
    for (int mm = 0; mm < nf; ++mm)
      for (int s = 0; s < ns; ++s) {
        double acc = 0.0;
        for (int q = 0; q < m; ++q) acc += psi[size_t(q) * nf + mm] * w[q] * (-rect[size_t(q) * ns + s]);
        c1[size_t(mm) * ns + s] = acc;
      }
    for (int mm = 0; mm < nf; ++mm) c1[size_t(mm) * ns + fo(lf) + mm] += 1.0;
    for (int q = 0; q < m; ++q) {
      const double* phi = &ft[lf].phi[size_t(q) * nrec];
      for (int s = 0; s < ns; ++s) {
        double a1 = 0.0, a2 = 0.0;
        for (int mm = 0; mm < nf; ++mm) a1 += psi[size_t(q) * nf + mm] * c1[size_t(mm) * ns + s];
        for (int mm = 0; mm < ne; ++mm) {
          const double c2 = -P(mm, s) + (s == mm ? 1.0 : 0.0);
          a2 += phi[mm] * c2;
        }
        R[size_t(q) * ns + s] = a1 - a2;
      }
    }
    {
      // stabilisation R^T W R / h_F with q-contiguous operands (RT: ns x m)
      std::vector<double> RT(size_t(ns) * m), WRT(size_t(ns) * m);
      for (int q = 0; q < m; ++q)
        for (int i = 0; i < ns; ++i) {
          RT[size_t(i) * m + q] = R[size_t(q) * ns + i];
          WRT[size_t(i) * m + q] = w[q] * R[size_t(q) * ns + i];
        }
      const double ih = 1.0 / hf[lf];
      for (int j = 0; j < ns; ++j) {
        const double* wj = &WRT[size_t(j) * m];
        for (int i = 0; i < ns; ++i) {
          const double* ri = &RT[size_t(i) * m];
          double acc = 0.0;
          for (int q = 0; q < m; ++q) acc += ri[q] * wj[q];
          A(i, j) += acc * ih;
        }
      }
    }
    if (mesh.tag[fid[lf]] == 1) {
      const double* dnw = DNW[lf].data();
      for (int j = 0; j < ns; ++j)
        for (int i = 0; i < ns; ++i) {
          const bool jf = j >= fo(lf) && j < fo(lf) + nf;
          const bool iff = i >= fo(lf) && i < fo(lf) + nf;
          if (!jf && !iff) continue;
          double cij = 0.0, cji = 0.0, pen = 0.0;
          for (int q = 0; q < m; ++q) {
            const double vj = jf ? psi[size_t(q) * nf + (j - fo(lf))] : 0.0;
            const double vi = iff ? psi[size_t(q) * nf + (i - fo(lf))] : 0.0;
            cij += dnw[size_t(q) * ns + i] * vj;
            cji += dnw[size_t(q) * ns + j] * vi;
            pen += vi * w[q] * vj;
          }
          A(i, j) -= cij + cji;
          A(i, j) += (eta / hf[lf]) * pen;
        }
    }
  }

  // the local Stokes block
  const int n = L.n;
  std::fill(mat, mat + size_t(n) * n, 0.0);
  std::fill(rhs, rhs + n, 0.0);
  auto M = [&](int i, int j) -> double& { return mat[size_t(i) + size_t(j) * n]; };
  auto vel_index = [&](int s, int c) {
    return s < ne ? L.vel_elem(c, s) : L.vel_face((s - ne) / nf, c, (s - ne) % nf);
  };
  for (int c = 0; c < 3; ++c)
    for (int j = 0; j < ns; ++j)
      for (int i = 0; i < ns; ++i) M(vel_index(i, c), vel_index(j, c)) += A(i, j);
  const int np = L.np;
  // random modal body force: coefficients of the degree-k modes
  double coef[3][kMaxMono] = {};
  if (data.kind == 3) {
    SplitMix64 rng{data.seed + uint64_t(e) * uint64_t(6 * np) * 0x9e3779b97f4a7c15ULL};
    for (int c = 0; c < 3; ++c)
      for (int m = 0; m < np; ++m) coef[c][m] = rng.normal();
  }
  for (int q = 0; q < nq; ++q) {
    const double w = er.w[q];
    const double* phi = &PH[size_t(q) * nrec];
    const double* g = &GR[size_t(q) * nrec * 3];
    for (int c = 0; c < 3; ++c)
      for (int m = 0; m < ne; ++m) {
        const double dv = g[3 * m + c];
        for (int i = 0; i < np; ++i) M(L.press_elem(i), L.vel_elem(c, m)) -= w * dv * phi[i];
      }
    double fv[3] = {0.0, 0.0, 0.0};
    if (data.kind == 3) {
      for (int c = 0; c < 3; ++c)
        for (int m = 0; m < np; ++m) fv[c] += coef[c][m] * phi[m];
    } else if (data.kind == 4) {
      data.f_manufactured(er.p[q], fv);
    }
    if (data.kind != 0)
      for (int c = 0; c < 3; ++c)
        for (int m = 0; m < ne; ++m) rhs[L.vel_elem(c, m)] += w * fv[c] * phi[m];
  }
  for (int lf = 0; lf < 6; ++lf) {
    const int tag = mesh.tag[fid[lf]];
    const int m = ft[lf].nq;
    for (int q = 0; q < m; ++q) {
      const double w = fr[lf].w[q];
      const V3 na = sgn[lf] * fr[lf].na[q];
      const double ncomp[3] = {na.x, na.y, na.z};
      const double* phi = &ft[lf].phi[size_t(q) * nrec];
      const double* psi = &ft[lf].psi[size_t(q) * nf];
      // hybrid face-pressure mass rows: int_F (u_T - u_F).n q_F
      for (int i = 0; i < L.nfp; ++i)
        for (int c = 0; c < 3; ++c) {
          for (int mm = 0; mm < ne; ++mm) M(L.press_face(lf, i), L.vel_elem(c, mm)) += psi[i] * phi[mm] * ncomp[c];
          for (int mm = 0; mm < nf; ++mm) M(L.press_face(lf, i), L.vel_face(lf, c, mm)) -= psi[i] * psi[mm] * ncomp[c];
        }
      if (tag == 1) {
        double gdv[3];
        data.gd(fr[lf].p[q], gdv);
        if (gdv[0] != 0.0 || gdv[1] != 0.0 || gdv[2] != 0.0)
          for (int c = 0; c < 3; ++c) {
            for (int s = 0; s < ns; ++s) rhs[vel_index(s, c)] -= gdv[c] * DNW[lf][size_t(q) * ns + s];
            for (int mm = 0; mm < nf; ++mm) rhs[L.vel_face(lf, c, mm)] += w * (eta / hf[lf]) * gdv[c] * psi[mm];
          }
      } else if (tag == 2) {
        const double an = norm(na);
        const V3 nu = (1.0 / an) * na;
        double gnv[3];
        data.gn(fr[lf].p[q], nu, gnv);
        for (int c = 0; c < 3; ++c)
          for (int mm = 0; mm < nf; ++mm) rhs[L.vel_face(lf, c, mm)] -= w * gnv[c] * psi[mm];
      }
    }
  }
  // momentum pressure columns = transpose of the mass rows, without the
  // face-pressure / face-velocity coupling on Dirichlet faces
  const int npress = n - L.nvel;
  for (int i = 0; i < npress; ++i)
    for (int j = 0; j < L.nvel; ++j) M(j, L.nvel + i) = M(L.nvel + i, j);
  for (int lf = 0; lf < 6; ++lf) {
    if (mesh.tag[fid[lf]] != 1) continue;
    for (int i = 0; i < L.nfp; ++i)
      for (int c = 0; c < 3; ++c)
        for (int mm = 0; mm < nf; ++mm) M(L.vel_face(lf, c, mm), L.press_face(lf, i)) = 0.0;
  }
}

// ---------------------------------------------------------------------------
// DG (BR2) local terms in 3D — BASELINE.json config 4 (equal-order DG, 80 x 80
// element blocks at k = 3). The reference's DG is BR2 in 2D
// (assemble.hpp:177-346, dg_local.hpp); this is the same scheme with three
// velocity components (SURVEY.md §0 finding 7: the reference DG, not SIP).
//  * element basis: orthonormal P^k (ElemBasis), quadrature degree 2(k+1)+1;
//    local order [u_x | u_y | u_z | p], ne = dim P^k(3D) modes each.
//  * volume: grad-grad per component, +int div(u) q rows, -int p div v
//    columns (assemble.hpp:219-231); loads int f_c v.
//  * faces (assemble.hpp:238-345): BR2 penalty eta = (max faces of the
//    adjacent elements) + 1 = 7 on hexahedra (dg_penalty_bound); Dirichlet:
//    4 eta <L,L> - cons - cons^T, momentum pressure flux with the trace;
//    interior: the jump/average tables; pressure-jump stabilisation scaled by
//    h_F = face diameter. Normals are taken per quadrature point from the
//    vector area element (exact on the bilinear face), so n_c x (table)
//    becomes the table with weights na_c: identical on planar faces.
//  * face loads (Dirichlet consistency + penalty, Neumann traction) are
//    formed as local vectors and added once per face.
//  * assembly order (the reference's scatter_block sequence): every entry is
//    0.0 + volume term, then + each face term in face-id order.
// ---------------------------------------------------------------------------

inline int dg_ne(int k) { return dimP3(k); }

struct DgElem {
  ElemRule er;
  ElemBasis b;
  Geo geo;
};

void dg_elem_init(const Mesh& mesh, int e, int k, DgElem& d) {
  const int qd = 2 * (k + 1) + 1;
  d.er = element_rule(mesh, e, qd);
  d.geo = element_geo(mesh, e, d.er);
  d.b.init(d.er, d.geo.cen, d.geo.diam, k);
}

/// Volume block (nloc x nloc column-major, nloc = 4 ne) and load of element e.
void dg_volume(const Mesh& mesh, int e, int k, const Data& data, const DgElem& d, double* mat,
               double* rhs) {
  const int ne = dg_ne(k), nloc = 4 * ne;
  const int nq = d.er.size();
  std::vector<double> st(size_t(ne) * ne, 0.0), dv[3];
  for (int c = 0; c < 3; ++c) dv[c].assign(size_t(ne) * ne, 0.0);
  double v[kMaxMono], g[3 * kMaxMono];
  double coef[3][kMaxMono] = {};
  if (data.kind == 3) {
    SplitMix64 rng{data.seed + uint64_t(e) * uint64_t(6 * ne) * 0x9e3779b97f4a7c15ULL};
    for (int c = 0; c < 3; ++c)
      for (int m = 0; m < ne; ++m) coef[c][m] = rng.normal();
  }
  std::fill(rhs, rhs + nloc, 0.0);
  for (int q = 0; q < nq; ++q) {
    const double w = d.er.w[q];
    d.b.eval(d.er.p[q], v);
    d.b.grad(d.er.p[q], g);
    // m_stiff += w g g^T ; m_div_c += w v g_c^T (dg_local.hpp:67-71)
    for (int j = 0; j < ne; ++j)
      for (int i = 0; i < ne; ++i) {
        double s = 0.0;
        for (int a = 0; a < 3; ++a) s += (w * g[3 * i + a]) * g[3 * j + a];
        st[size_t(i) + size_t(j) * ne] += s;
        for (int c = 0; c < 3; ++c) dv[c][size_t(i) + size_t(j) * ne] += (w * v[i]) * g[3 * j + c];
      }
    double fv[3] = {0.0, 0.0, 0.0};
    if (data.kind == 3) {
      for (int c = 0; c < 3; ++c)
        for (int m = 0; m < ne; ++m) fv[c] += coef[c][m] * v[m];
    } else if (data.kind == 4) {
      data.f_manufactured(d.er.p[q], fv);
    }
    if (data.kind != 0)
      for (int c = 0; c < 3; ++c)
        for (int i = 0; i < ne; ++i) rhs[c * ne + i] += (w * fv[c]) * v[i];
  }
  std::fill(mat, mat + size_t(nloc) * nloc, 0.0);
  auto M = [&](int i, int j) -> double& { return mat[size_t(i) + size_t(j) * nloc]; };
  for (int c = 0; c < 3; ++c)
    for (int j = 0; j < ne; ++j)
      for (int i = 0; i < ne; ++i) {
        M(c * ne + i, c * ne + j) += st[size_t(i) + size_t(j) * ne];
        M(3 * ne + i, c * ne + j) += dv[c][size_t(i) + size_t(j) * ne];
        M(c * ne + i, 3 * ne + j) -= dv[c][size_t(j) + size_t(i) * ne];
      }
}

/// Scalar face tables of face f over the stacked element dofs [left | right]
/// (side count ns = 1 on boundary faces): visc, vmom_c, mass_c, pjump, all
/// (ns ne) x (ns ne) column-major, plus the per-side loads (3 x ns ne).
struct DgFace {
  int ns = 0, tag = 0, m = 0;
  std::vector<double> visc, vmom[3], mass[3], pjump, load;
};

double dg_penalty_bound3(const Mesh&, int) { return 6.0; }  // hexahedra: 6 faces per element

void dg_face(const Mesh& mesh, int f, int k, const Data& data, double eta_override,
             const DgElem& dl, const DgElem* dr, DgFace& out) {
  const int ne = dg_ne(k), qd = 2 * (k + 1) + 1;
  const FaceRule fr = face_rule(mesh, f, qd);
  const int nq = fr.size();
  const double hF = face_diameter(mesh, f);
  const double bound = dg_penalty_bound3(mesh, f);
  const double eta = eta_override > 0.0 ? eta_override : bound + 1.0;
  out.tag = mesh.tag[f];
  out.ns = (mesh.right[f] >= 0) ? 2 : 1;
  const int ns = out.ns, m = ns * ne;
  out.m = m;
  // per point: values, normal derivatives, unit normal, weights
  std::vector<double> psi(size_t(nq) * m), dn(size_t(nq) * m), nu(size_t(nq) * 3);
  double v[kMaxMono], g[3 * kMaxMono];
  for (int q = 0; q < nq; ++q) {
    const double an = norm(fr.na[q]);
    const V3 n = (1.0 / an) * fr.na[q];
    nu[3 * q] = n.x;
    nu[3 * q + 1] = n.y;
    nu[3 * q + 2] = n.z;
    for (int s = 0; s < ns; ++s) {
      const ElemBasis& b = s == 0 ? dl.b : dr->b;
      b.eval(fr.p[q], v);
      b.grad(fr.p[q], g);
      for (int i = 0; i < ne; ++i) {
        psi[size_t(q) * m + s * ne + i] = v[i];
        dn[size_t(q) * m + s * ne + i] = g[3 * i] * n.x + g[3 * i + 1] * n.y + g[3 * i + 2] * n.z;
      }
    }
  }
  const std::vector<double>& w = fr.w;
  auto T = [&](std::vector<double>& t) { t.assign(size_t(m) * m, 0.0); };
  T(out.visc);
  T(out.pjump);
  for (int c = 0; c < 3; ++c) {
    T(out.vmom[c]);
    T(out.mass[c]);
  }
  out.load.assign(size_t(3) * m, 0.0);
  // lifting moments m_s = 0.5 Psi_s^T W (ne x nq per side)
  std::vector<double> mom(size_t(ns) * ne * nq);
  for (int s = 0; s < ns; ++s)
    for (int l = 0; l < ne; ++l)
      for (int q = 0; q < nq; ++q)
        mom[(size_t(s) * ne + l) * nq + q] = (0.5 * psi[size_t(q) * m + s * ne + l]) * w[q];
  if (ns == 1) {
    if (out.tag == 2) {
      // Neumann: traction load -int g_N . v (assemble.hpp:255-264)
      for (int q = 0; q < nq; ++q) {
        double gn[3];
        data.gn(fr.p[q], V3{nu[3 * q], nu[3 * q + 1], nu[3 * q + 2]}, gn);
        for (int c = 0; c < 3; ++c)
          for (int i = 0; i < ne; ++i) out.load[c * m + i] -= (w[q] * gn[c]) * psi[size_t(q) * m + i];
      }
      return;
    }
    // Dirichlet (assemble.hpp:266-290): lifted jump 2(u_T - g)
    std::vector<double> cons(size_t(ne) * ne), lift(size_t(ne) * ne);
    for (int j = 0; j < ne; ++j)
      for (int i = 0; i < ne; ++i) {
        double a = 0.0, b = 0.0;
        for (int q = 0; q < nq; ++q) {
          a += (psi[size_t(q) * m + i] * w[q]) * dn[size_t(q) * m + j];
          b += mom[size_t(i) * nq + q] * psi[size_t(q) * m + j];
        }
        cons[i + size_t(j) * ne] = a;
        lift[i + size_t(j) * ne] = b;
      }
    for (int j = 0; j < ne; ++j)
      for (int i = 0; i < ne; ++i) {
        double pen = 0.0;
        for (int l = 0; l < ne; ++l) pen += ((4.0 * eta) * lift[l + size_t(i) * ne]) * lift[l + size_t(j) * ne];
        out.visc[i + size_t(j) * m] = (pen - cons[i + size_t(j) * ne]) - cons[j + size_t(i) * ne];
        for (int c = 0; c < 3; ++c) {
          double pf = 0.0;
          for (int q = 0; q < nq; ++q)
            pf += (psi[size_t(q) * m + i] * (w[q] * nu[3 * q + c])) * psi[size_t(q) * m + j];
          out.vmom[c][i + size_t(j) * m] = pf;
        }
      }
    // loads: -int (n.grad v) g + 4 eta <L(g), L(v)>
    double gq[3];
    std::vector<double> gv(size_t(3) * nq);
    bool nz = false;
    for (int q = 0; q < nq; ++q) {
      data.gd(fr.p[q], gq);
      for (int c = 0; c < 3; ++c) {
        gv[size_t(c) * nq + q] = gq[c];
        nz = nz || gq[c] != 0.0;
      }
    }
    if (nz)
      for (int c = 0; c < 3; ++c) {
        std::vector<double> mg(ne, 0.0);
        for (int l = 0; l < ne; ++l)
          for (int q = 0; q < nq; ++q) mg[l] += mom[size_t(l) * nq + q] * gv[size_t(c) * nq + q];
        for (int i = 0; i < ne; ++i) {
          double a = 0.0, b = 0.0;
          for (int q = 0; q < nq; ++q) a += (dn[size_t(q) * m + i] * w[q]) * gv[size_t(c) * nq + q];
          for (int l = 0; l < ne; ++l) b += ((4.0 * eta) * lift[l + size_t(i) * ne]) * mg[l];
          out.load[c * m + i] = (-a) + b;
        }
      }
    return;
  }
  // interior face (assemble.hpp:292-345)
  std::vector<double> jmp(size_t(nq) * m), avg(size_t(nq) * m), adn(size_t(nq) * m),
      plain(size_t(nq) * m);
  for (int q = 0; q < nq; ++q)
    for (int a = 0; a < m; ++a) {
      const double p = psi[size_t(q) * m + a];
      jmp[size_t(q) * m + a] = a < ne ? p : -p;
      avg[size_t(q) * m + a] = 0.5 * p;
      adn[size_t(q) * m + a] = 0.5 * dn[size_t(q) * m + a];
      plain[size_t(q) * m + a] = p;
    }
  // (m_s jmp): ne x m per side
  std::vector<double> mj(size_t(2) * ne * m, 0.0);
  for (int s = 0; s < 2; ++s)
    for (int b = 0; b < m; ++b)
      for (int l = 0; l < ne; ++l) {
        double acc = 0.0;
        for (int q = 0; q < nq; ++q) acc += mom[(size_t(s) * ne + l) * nq + q] * jmp[size_t(q) * m + b];
        mj[(size_t(s) * ne + l) + size_t(b) * 2 * ne] = acc;
      }
  std::vector<double> cons(size_t(m) * m);
  for (int b = 0; b < m; ++b)
    for (int a = 0; a < m; ++a) {
      double acc = 0.0;
      for (int q = 0; q < nq; ++q) acc += (jmp[size_t(q) * m + a] * w[q]) * adn[size_t(q) * m + b];
      cons[a + size_t(b) * m] = acc;
    }
  for (int b = 0; b < m; ++b)
    for (int a = 0; a < m; ++a) {
      double p1 = 0.0, p2 = 0.0;
      for (int l = 0; l < ne; ++l) {
        p1 += mj[size_t(l) + size_t(a) * 2 * ne] * mj[size_t(l) + size_t(b) * 2 * ne];
        p2 += mj[size_t(ne + l) + size_t(a) * 2 * ne] * mj[size_t(ne + l) + size_t(b) * 2 * ne];
      }
      const double pen = eta * (p1 + p2);
      out.visc[a + size_t(b) * m] = (pen - cons[a + size_t(b) * m]) - cons[b + size_t(a) * m];
      double pj = 0.0;
      for (int q = 0; q < nq; ++q) pj += (jmp[size_t(q) * m + a] * w[q]) * jmp[size_t(q) * m + b];
      out.pjump[a + size_t(b) * m] = hF * pj;
      for (int c = 0; c < 3; ++c) {
        double vm = 0.0, ms = 0.0;
        for (int q = 0; q < nq; ++q) {
          const double wn = w[q] * nu[3 * q + c];
          vm += (jmp[size_t(q) * m + a] * wn) * avg[size_t(q) * m + b];
          ms += ((0.5 * plain[size_t(q) * m + a]) * wn) * jmp[size_t(q) * m + b];
        }
        out.vmom[c][a + size_t(b) * m] = vm;
        out.mass[c][a + size_t(b) * m] = ms;
      }
    }
}

/// The face's local matrix over [left | right] element dofs (ns nloc square,
/// column-major; assemble.hpp:324-339's placement; Dirichlet: the left block).
void dg_face_matrix(const DgFace& t, int ne, double* mat) {
  const int nloc = 4 * ne, ns = t.ns, N = ns * nloc, m = t.m;
  std::fill(mat, mat + size_t(N) * N, 0.0);
  if (t.tag == 2) return;
  auto M = [&](int i, int j) -> double& { return mat[size_t(i) + size_t(j) * N]; };
  auto sdof = [&](int s, int c, int i) { return s * nloc + c * ne + i; };
  auto spr = [&](int s, int i) { return s * nloc + 3 * ne + i; };
  for (int s1 = 0; s1 < ns; ++s1)
    for (int i = 0; i < ne; ++i)
      for (int s2 = 0; s2 < ns; ++s2)
        for (int j = 0; j < ne; ++j) {
          const int a = s1 * ne + i, b = s2 * ne + j;
          const size_t ab = size_t(a) + size_t(b) * m;
          for (int c = 0; c < 3; ++c) {
            M(sdof(s1, c, i), sdof(s2, c, j)) += t.visc[ab];
            M(sdof(s1, c, i), spr(s2, j)) += t.vmom[c][ab];
            if (ns == 2) M(spr(s1, i), sdof(s2, c, j)) -= t.mass[c][ab];
          }
          if (ns == 2) M(spr(s1, i), spr(s2, j)) += t.pjump[ab];
        }
}

/// Panel layout of one element block of the DG operator ("DG block
/// storage", csrc/dgb.cu): velocity panel c (ne x 2ne, column-major:
/// columns [u_c modes | p modes]) at c 2ne^2, pressure panel (ne x 4ne:
/// [u_x | u_y | u_z | p]) at 6 ne^2; 10 ne^2 structural entries per block.
inline size_t dgb_index(int ne, int r, int col) {
  // r, col: rows / columns of the dense 4ne block; caller guarantees coupling
  const int rc = r / ne, ri = r % ne;
  if (rc < 3) {
    const int cc = col / ne, cj = col % ne;
    const int pc = cc == 3 ? ne + cj : cj;
    return size_t(rc) * 2 * ne * ne + size_t(pc) * ne + ri;
  }
  return size_t(6) * ne * ne + size_t(col) * ne + ri;
}
inline bool dg_coupled(int ne, int r, int col) {
  const int rc = r / ne, cc = col / ne;
  return rc == 3 || cc == 3 || rc == cc;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

} // namespace psh3

using namespace psh3;

struct psh_mesh3 {
  Mesh m;
};

extern "C" {

const char* psh3_last_error(void) { return psh3::g_err.c_str(); }

int psh_mesh_unit_cube(int n, double frac, uint64_t seed, int neumann_top, psh_mesh3** out) {
  return guard([&] {
    if (n < 1) throw std::invalid_argument("unit cube: n must be >= 1");
    if (n > 127) throw std::invalid_argument("unit cube: n must be <= 127");
    auto pm = std::make_unique<psh_mesh3>();
    build_unit_cube(pm->m, n, frac, seed, neumann_top != 0);
    *out = pm.release();
  });
}

void psh_mesh3_destroy(psh_mesh3* m) { delete m; }

void psh_mesh3_counts(const psh_mesh3* m, int64_t* out) {
  out[0] = int64_t(m->m.v.size());
  out[1] = m->m.nelem();
  out[2] = m->m.nfaces();
}

void psh_mesh3_faces(const psh_mesh3* pm, int32_t* faces) {
  const Mesh& m = pm->m;
  for (int f = 0; f < m.nfaces(); ++f) {
    for (int a = 0; a < 4; ++a) faces[7 * f + a] = m.fv[f][a];
    faces[7 * f + 4] = m.left[f];
    faces[7 * f + 5] = m.right[f];
    faces[7 * f + 6] = m.tag[f];
  }
}

void psh_mesh3_element_faces(const psh_mesh3* pm, int32_t* ef) {
  const Mesh& m = pm->m;
  for (int e = 0; e < m.nelem(); ++e)
    for (int lf = 0; lf < 6; ++lf) ef[6 * e + lf] = m.ef[e][lf];
}

void psh_mesh3_vertices(const psh_mesh3* pm, double* xyz) {
  const Mesh& m = pm->m;
  for (size_t i = 0; i < m.v.size(); ++i) {
    xyz[3 * i] = m.v[i].x;
    xyz[3 * i + 1] = m.v[i].y;
    xyz[3 * i + 2] = m.v[i].z;
  }
}

int psh3_hp_info(int k, int32_t* info) {
  return guard([&] {
    if (k < 0 || k > 4) throw std::invalid_argument("hho3: k must be in [0, 4]");
    const LocalLayout L = local_layout(k);
    const int nelim = 3 * L.ne + L.np;
    const int32_t v[8] = {L.n, nelim, L.n - nelim, L.nf, L.nfp, 3 * L.nf + L.nfp, 6, L.ne};
    std::memcpy(info, v, sizeof v);
  });
}

/// eliminated_dofs (condense.hpp:44-55) for hho-hp vp-cond: every element
/// velocity mode (c-major), then every element pressure mode.
int psh3_hp_elim(int k, int32_t* elim) {
  return guard([&] {
    const LocalLayout L = local_layout(k);
    int t = 0;
    for (int c = 0; c < 3; ++c)
      for (int m = 0; m < L.ne; ++m) elim[t++] = L.vel_elem(c, m);
    for (int m = 0; m < L.np; ++m) elim[t++] = L.press_elem(m);
  });
}

/// (local face, offset in the global face block [vx | vy | vz | p]) of
/// every retained local dof, in local keep order (assemble.hpp:72-96).
int psh3_hp_keep_pos(int k, int32_t* pos) {
  return guard([&] {
    const LocalLayout L = local_layout(k);
    std::vector<int> lf_of(L.n, -1), off_of(L.n, -1);
    for (int lf = 0; lf < 6; ++lf) {
      for (int c = 0; c < 3; ++c)
        for (int m = 0; m < L.nf; ++m) {
          lf_of[L.vel_face(lf, c, m)] = lf;
          off_of[L.vel_face(lf, c, m)] = c * L.nf + m;
        }
      for (int m = 0; m < L.nfp; ++m) {
        lf_of[L.press_face(lf, m)] = lf;
        off_of[L.press_face(lf, m)] = 3 * L.nf + m;
      }
    }
    int t = 0;
    for (int i = 0; i < L.n; ++i)
      if (lf_of[i] >= 0) {
        pos[2 * t] = lf_of[i];
        pos[2 * t + 1] = off_of[i];
        ++t;
      }
  });
}

int psh3_local_blocks(const psh_mesh3* pm, int k, int data, uint64_t seed, double eta, int e0,
                      int e1, int nthreads, double* mats, double* rhs) {
  return guard([&] {
    const Mesh& mesh = pm->m;
    if (k < 0 || k > 4) throw std::invalid_argument("hho3: k must be in [0, 4]");
    if (e0 < 0 || e1 > mesh.nelem() || e0 > e1) throw std::invalid_argument("hho3: element range");
    if (data != 0 && data != 3 && data != 4) throw std::invalid_argument("hho3: unknown data kind");
    const LocalLayout L = local_layout(k);
    const double eta_v = eta > 0.0 ? eta : 3.0 * (k + 1) * (k + 1);
    Data dd{data, seed};
    if (nthreads > 0) omp_set_num_threads(nthreads);
    std::string err;
#pragma omp parallel for schedule(dynamic, 16)
    for (int e = e0; e < e1; ++e) {
      try {
        build_local(mesh, e, k, eta_v, dd, mats + size_t(e - e0) * L.n * L.n,
                    rhs + size_t(e - e0) * L.n);
      } catch (const std::exception& ex) {
#pragma omp critical
        err = ex.what();
      }
    }
    if (!err.empty()) throw std::runtime_error(err);
  });
}

/// Inputs of the device local-block producer (pscu_local_blocks3) for
/// elements [e0, e1): hexahedron vertex ids (8 per element), element faces
/// and orientation signs (6 each), the face table {4 vertex ids, tag}
/// (all faces), the Gauss-Legendre rule of the degree-2(k+1)+1 tensor rules
/// (points then weights, rule_points entries each) and, for data 3, the
/// per-element random modal coefficients (3 x dim P_k(3D), SplitMix64 /
/// Box-Muller on the host's libm, as build_local draws them). Null outputs
/// are skipped; returns the rule size.
int psh3_device_inputs(const psh_mesh3* pm, int k, int data, uint64_t seed, int e0, int e1,
                       int32_t* hex, int32_t* ef, int32_t* es, int32_t* ftab, double* gl,
                       double* coef) {
  int npts = 0;
  const int rc = guard([&] {
    const Mesh& m = pm->m;
    if (k < 0 || k > 4) throw std::invalid_argument("hho3: k must be in [0, 4]");
    if (e0 < 0 || e1 > m.nelem() || e0 > e1) throw std::invalid_argument("hho3: element range");
    const int qd = 2 * (k + 1) + 1;
    npts = rule_points(qd);
    for (int e = e0; e < e1; ++e) {
      const size_t i = size_t(e - e0);
      if (hex)
        for (int a = 0; a < 8; ++a) hex[8 * i + a] = m.hex[e][a];
      for (int lf = 0; lf < 6; ++lf) {
        if (ef) ef[6 * i + lf] = m.ef[e][lf];
        if (es) es[6 * i + lf] = m.es[e][lf];
      }
    }
    if (ftab)
      for (int f = 0; f < m.nfaces(); ++f) {
        for (int a = 0; a < 4; ++a) ftab[5 * f + a] = m.fv[f][a];
        ftab[5 * f + 4] = m.tag[f];
      }
    if (gl) {
      std::vector<double> x, w;
      gauss_legendre(npts, x, w);
      for (int i = 0; i < npts; ++i) {
        gl[i] = x[i];
        gl[npts + i] = w[i];
      }
    }
    if (coef && data == 3) {
      const int np = dimP3(k);
      for (int e = e0; e < e1; ++e) {
        SplitMix64 rng{seed + uint64_t(e) * uint64_t(6 * np) * 0x9e3779b97f4a7c15ULL};
        double* c = coef + size_t(e - e0) * 3 * np;
        for (int t = 0; t < 3 * np; ++t) c[t] = rng.normal();
      }
    }
  });
  return rc ? -rc : npts;
}

/// Face-block pattern of the condensed hho-hp vp-cond operator: block row f
/// couples every face of the (<= 2) elements holding f, columns ascending.
/// Returns the block count; brow_ptr (n_faces + 1) / bcols may be null.
int64_t psh3_block_pattern(const psh_mesh3* pm, int64_t* brow_ptr, int32_t* bcols) {
  const Mesh& m = pm->m;
  const int nf = m.nfaces();
  std::vector<int64_t> rp(size_t(nf) + 1, 0);
  std::vector<std::array<int32_t, 11>> cols(nf);
  std::vector<int> cnt(nf, 0);
#pragma omp parallel for schedule(static)
  for (int f = 0; f < nf; ++f) {
    int32_t c[12];
    int t = 0;
    for (int side = 0; side < 2; ++side) {
      const int e = side ? m.right[f] : m.left[f];
      if (e < 0) continue;
      for (int lf = 0; lf < 6; ++lf) c[t++] = m.ef[e][lf];
    }
    std::sort(c, c + t);
    t = int(std::unique(c, c + t) - c);
    cnt[f] = t;
    for (int i = 0; i < t; ++i) cols[f][i] = c[i];
  }
  for (int f = 0; f < nf; ++f) rp[f + 1] = rp[f] + cnt[f];
  if (brow_ptr) std::memcpy(brow_ptr, rp.data(), sizeof(int64_t) * rp.size());
  if (bcols)
    for (int f = 0; f < nf; ++f) std::memcpy(bcols + rp[f], cols[f].data(), sizeof(int32_t) * cnt[f]);
  return rp[nf];
}

/// L2 projections of the manufactured solution (data kind 4) onto every
/// face's basis, in the global face-block layout [ux | uy | uz | p]
/// (n_faces x (3 nf + nf)): the exact counterpart of the face unknowns.
int psh3_face_projection(const psh_mesh3* pm, int k, double* out) {
  return guard([&] {
    const Mesh& m = pm->m;
    const int qd = 2 * (k + 1) + 1, nf = dimP2(k), fbk = 4 * nf;
#pragma omp parallel for schedule(dynamic, 64)
    for (int f = 0; f < m.nfaces(); ++f) {
      const FaceRule r = face_rule(m, f, qd);
      FaceBasis b;
      b.init(m, f, r, k);
      double* o = out + size_t(f) * fbk;
      std::fill(o, o + fbk, 0.0);
      double psi[32], u[3];
      for (int q = 0; q < r.size(); ++q) {
        b.eval(r.p[q], psi);
        Data::u(r.p[q], u);
        const double p = Data::pr(r.p[q]);
        for (int i = 0; i < nf; ++i) {
          for (int c = 0; c < 3; ++c) o[c * nf + i] += r.w[q] * u[c] * psi[i];
          o[3 * nf + i] += r.w[q] * p * psi[i];
        }
      }
    }
  });
}

/// Geometry checks: element volumes and the closure sum_F int_F n dA per
/// element (out: nelem volumes, then nelem closure norms).
int psh3_geometry(const psh_mesh3* pm, double* out) {
  return guard([&] {
    const Mesh& m = pm->m;
    const int ne = m.nelem();
#pragma omp parallel for schedule(static)
    for (int e = 0; e < ne; ++e) {
      const ElemRule r = element_rule(m, e, 3);
      double vol = 0.0;
      for (int q = 0; q < r.size(); ++q) vol += r.w[q];
      V3 s{};
      for (int lf = 0; lf < 6; ++lf) {
        const FaceRule fr = face_rule(m, m.ef[e][lf], 3);
        for (int q = 0; q < fr.size(); ++q) s = s + double(m.es[e][lf]) * fr.na[q];
      }
      out[e] = vol;
      out[ne + e] = norm(s);
    }
  });
}

} // extern "C"

// ---------------------------------------------------------------------------
// DG (BR2) in 3D: BASELINE.json config 4 (see the DG section above)
// ---------------------------------------------------------------------------

extern "C" {

/* info[0..1] = modes per component ne (dim P^k), element block 4 ne */
int psh3_dg_info(int k, int32_t* info) {
  return guard([&] {
    if (k < 1 || k > 4) throw std::invalid_argument("dg: polynomial degree must be in [1, 4]");
    info[0] = dg_ne(k);
    info[1] = 4 * dg_ne(k);
  });
}

/* Element-block pattern of the DG operator: block row e couples e and the
 * elements across its interior faces, ascending. Returns the block count. */
int64_t psh3_dg_block_pattern(const psh_mesh3* pm, int64_t* brow_ptr, int32_t* bcols) {
  const Mesh& m = pm->m;
  const int ne = m.nelem();
  std::vector<int64_t> rp(size_t(ne) + 1, 0);
  std::vector<std::array<int32_t, 7>> cols(ne);
  std::vector<int> cnt(ne, 0);
#pragma omp parallel for schedule(static)
  for (int e = 0; e < ne; ++e) {
    int32_t c[7];
    int t = 0;
    c[t++] = e;
    for (int lf = 0; lf < 6; ++lf) {
      const int f = m.ef[e][lf];
      if (m.right[f] < 0) continue;
      c[t++] = m.left[f] == e ? m.right[f] : m.left[f];
    }
    std::sort(c, c + t);
    cnt[e] = t;
    for (int i = 0; i < t; ++i) cols[e][i] = c[i];
  }
  for (int e = 0; e < ne; ++e) rp[e + 1] = rp[e] + cnt[e];
  if (brow_ptr) std::memcpy(brow_ptr, rp.data(), sizeof(int64_t) * rp.size());
  if (bcols)
    for (int e = 0; e < ne; ++e) std::memcpy(bcols + rp[e], cols[e].data(), sizeof(int32_t) * cnt[e]);
  return rp[ne];
}

/* The DG local terms for the oracle's reference-order scatter (small
 * meshes): per element the volume block (nloc^2, column-major) and load
 * (nloc); per face the face matrix over [left | right] dofs ((2 nloc)^2,
 * column-major, leading dimension 2 nloc; boundary faces fill the left
 * nloc block only) and the face load (2 nloc). Null outputs skipped. */
int psh3_dg_local(const psh_mesh3* pm, int k, int data, uint64_t seed, double eta, int nthreads,
                  double* vol, double* vrhs, double* fmat, double* frhs) {
  return guard([&] {
    const Mesh& mesh = pm->m;
    if (k < 1 || k > 4) throw std::invalid_argument("dg: polynomial degree must be in [1, 4]");
    if (data != 0 && data != 3 && data != 4) throw std::invalid_argument("dg: unknown data kind");
    const int ne = dg_ne(k), nloc = 4 * ne, N2 = 2 * nloc;
    Data dd{data, seed};
    if (nthreads > 0) omp_set_num_threads(nthreads);
    std::vector<DgElem> el(mesh.nelem());
#pragma omp parallel for schedule(dynamic, 8)
    for (int e = 0; e < mesh.nelem(); ++e) {
      dg_elem_init(mesh, e, k, el[e]);
      std::vector<double> m(size_t(nloc) * nloc), r(nloc);
      dg_volume(mesh, e, k, dd, el[e], m.data(), r.data());
      if (vol) std::memcpy(vol + size_t(e) * nloc * nloc, m.data(), sizeof(double) * m.size());
      if (vrhs) std::memcpy(vrhs + size_t(e) * nloc, r.data(), sizeof(double) * nloc);
    }
#pragma omp parallel for schedule(dynamic, 8)
    for (int f = 0; f < mesh.nfaces(); ++f) {
      DgFace t;
      const int r = mesh.right[f];
      dg_face(mesh, f, k, dd, eta, el[mesh.left[f]], r >= 0 ? &el[r] : nullptr, t);
      std::vector<double> fm(size_t(t.ns * nloc) * (t.ns * nloc));
      dg_face_matrix(t, ne, fm.data());
      if (fmat) {
        double* o = fmat + size_t(f) * N2 * N2;
        std::fill(o, o + size_t(N2) * N2, 0.0);
        const int n = t.ns * nloc;
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i) o[size_t(i) + size_t(j) * N2] = fm[size_t(i) + size_t(j) * n];
      }
      if (frhs) {
        double* o = frhs + size_t(f) * N2;
        std::fill(o, o + N2, 0.0);
        for (int s = 0; s < t.ns; ++s)
          for (int c = 0; c < 3; ++c)
            for (int i = 0; i < ne; ++i) o[s * nloc + c * ne + i] = t.load[c * t.m + s * ne + i];
      }
    }
  });
}

/* Block rows [e0, e1) of the assembled DG operator in DG block storage
 * (csrc/dgb.cu panels, 10 ne^2 values per block, blocks in pattern order:
 * vals receives blocks brow_ptr[e0] .. brow_ptr[e1] - 1) and their loads
 * (rhs: rows of e0 .. e1 - 1). Entry sums follow the reference's scatter
 * order: 0.0 + volume, then + each face term in face-id order; the loads
 * likewise (volume load, then face loads in face-id order). */
int psh3_dg_rows(const psh_mesh3* pm, int k, int data, uint64_t seed, double eta, int e0, int e1,
                 const int64_t* brow_ptr, const int32_t* bcols, int nthreads, double* vals,
                 double* rhs) {
  return guard([&] {
    const Mesh& mesh = pm->m;
    if (k < 1 || k > 4) throw std::invalid_argument("dg: polynomial degree must be in [1, 4]");
    if (e0 < 0 || e1 > mesh.nelem() || e0 > e1) throw std::invalid_argument("dg: element range");
    if (data != 0 && data != 3 && data != 4) throw std::invalid_argument("dg: unknown data kind");
    const int ne = dg_ne(k), nloc = 4 * ne;
    const size_t bsz = size_t(10) * ne * ne;
    Data dd{data, seed};
    if (nthreads > 0) omp_set_num_threads(nthreads);
    const int64_t q00 = brow_ptr[e0];
    std::string err;
#pragma omp parallel for schedule(dynamic, 4)
    for (int e = e0; e < e1; ++e) {
      try {
        DgElem de;
        dg_elem_init(mesh, e, k, de);
        std::vector<double> vm(size_t(nloc) * nloc), vr(nloc);
        dg_volume(mesh, e, k, dd, de, vm.data(), vr.data());
        const int64_t q0 = brow_ptr[e], q1 = brow_ptr[e + 1];
        double* out = vals + size_t(q0 - q00) * bsz;
        std::fill(out, out + size_t(q1 - q0) * bsz, 0.0);
        auto blk = [&](int col_elem) -> double* {
          for (int64_t q = q0; q < q1; ++q)
            if (bcols[q] == col_elem) return out + size_t(q - q0) * bsz;
          throw std::runtime_error("dg: block outside the pattern");
        };
        double* dgl = blk(e);
        for (int j = 0; j < nloc; ++j)
          for (int i = 0; i < nloc; ++i)
            if (dg_coupled(ne, i, j)) dgl[dgb_index(ne, i, j)] += vm[size_t(i) + size_t(j) * nloc];
        double* r = rhs + size_t(e - e0) * nloc;
        for (int i = 0; i < nloc; ++i) r[i] = 0.0 + vr[i];
        // faces of e in face-id order
        int fs[6];
        for (int lf = 0; lf < 6; ++lf) fs[lf] = mesh.ef[e][lf];
        std::sort(fs, fs + 6);
        std::vector<double> fm;
        for (int t6 = 0; t6 < 6; ++t6) {
          const int f = fs[t6];
          const int L = mesh.left[f], R = mesh.right[f];
          DgElem other;
          const bool interior = R >= 0;
          const int se = L == e ? 0 : 1;
          if (interior) dg_elem_init(mesh, se == 0 ? R : L, k, other);
          DgFace t;
          dg_face(mesh, f, k, dd, eta, se == 0 ? de : other, interior ? (se == 0 ? &other : &de) : nullptr, t);
          for (int c = 0; c < 3; ++c)
            for (int i = 0; i < ne; ++i) r[c * ne + i] += t.load[c * t.m + se * ne + i];
          if (t.tag == 2) continue;
          const int n = t.ns * nloc;
          fm.resize(size_t(n) * n);
          dg_face_matrix(t, ne, fm.data());
          for (int s2 = 0; s2 < t.ns; ++s2) {
            double* b = s2 == se ? dgl : blk(s2 == 0 ? L : R);
            for (int j = 0; j < nloc; ++j)
              for (int i = 0; i < nloc; ++i)
                if (dg_coupled(ne, i, j))
                  b[dgb_index(ne, i, j)] += fm[size_t(se * nloc + i) + size_t(s2 * nloc + j) * n];
          }
        }
      } catch (const std::exception& ex) {
#pragma omp critical
        err = ex.what();
      }
    }
    if (!err.empty()) throw std::runtime_error(err);
  });
}

} // extern "C"

extern "C" {
/* L2 errors of a DG solution x (element blocks [ux | uy | uz | p]) against
 * the manufactured field of data 4: out[0] = ||u_h - u||, out[1] =
 * ||p_h - p|| (validation of the 3D DG discretisation). */
int psh3_dg_l2_errors(const psh_mesh3* pm, int k, const double* x, double* out) {
  return guard([&] {
    const Mesh& mesh = pm->m;
    const int ne = dg_ne(k), nloc = 4 * ne;
    double eu = 0.0, ep = 0.0;
#pragma omp parallel for schedule(dynamic, 8) reduction(+ : eu, ep)
    for (int e = 0; e < mesh.nelem(); ++e) {
      DgElem d;
      dg_elem_init(mesh, e, k, d);
      const ElemRule r = element_rule(mesh, e, 2 * (k + 2) + 3);
      double v[kMaxMono], u[3];
      const double* xe = x + size_t(e) * nloc;
      for (int q = 0; q < r.size(); ++q) {
        d.b.eval(r.p[q], v);
        Data::u(r.p[q], u);
        for (int c = 0; c < 4; ++c) {
          double s = 0.0;
          for (int i = 0; i < ne; ++i) s += xe[c * ne + i] * v[i];
          const double ex = c < 3 ? u[c] : Data::pr(r.p[q]);
          (c < 3 ? eu : ep) += r.w[q] * (s - ex) * (s - ex);
        }
      }
    }
    out[0] = std::sqrt(eu);
    out[1] = std::sqrt(ep);
  });
}
} // extern "C"
