// Host-side input producer (include/pstokes_host.h): 2D meshes with the
// reference's first-seen face numbering, quadrature, hierarchical
// orthonormal bases, HHO local Stokes blocks, eliminated-dof lists,
// retained global ids and the structural CSR pattern.
//
// This is the front end the reference runs inside assemble_hho
// (assemble.hpp:136-172) before condensation; it is restated here from the
// discretisation in PAPER.md / hho_local.hpp with plain arrays (no Eigen) and
// OpenMP over elements. Values agree with the reference to rounding (the
// parity tests compare the assembled condensed operator at 1e-12 relative
// and the pattern / numbering exactly).
#include "pstokes_host.h"

#include <omp.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace psh {

thread_local std::string g_err;

struct P2 {
  double x = 0.0, y = 0.0;
};

// ---------------------------------------------------------------------------
// mesh
// ---------------------------------------------------------------------------

struct FaceRec {
  int a, b, left, right, tag;  // tag: 0 interior, 1 Dirichlet, 2 Neumann
};

struct Mesh {
  std::vector<P2> v;
  std::vector<int> eoff{0}, loop;  // CCW vertex loops
  std::vector<FaceRec> faces;
  std::vector<int> efac, esgn;     // parallel to loop: face id and sign of each element edge
  std::vector<double> area, diam, hF;
  std::vector<P2> cen;

  int nelem() const { return int(eoff.size()) - 1; }
  int nfaces() const { return int(faces.size()); }
  int nv_of(int e) const { return eoff[e + 1] - eoff[e]; }

  P2 tangent(int f) const {
    const P2 a = v[faces[f].a], b = v[faces[f].b];
    return {(b.x - a.x) / hF[f], (b.y - a.y) / hF[f]};
  }
  P2 normal(int f) const {  // unit normal out of `left`
    const P2 t = tangent(f);
    return {t.y, -t.x};
  }
  P2 mid(int f) const {
    const P2 a = v[faces[f].a], b = v[faces[f].b];
    return {0.5 * (a.x + b.x), 0.5 * (a.y + b.y)};
  }

  /// Faces in first-seen order over the element loops (mesh.hpp:87-119).
  void finalize() {
    faces.clear();
    std::unordered_map<uint64_t, int> seen;
    seen.reserve(loop.size());
    efac.assign(loop.size(), -1);
    esgn.assign(loop.size(), 0);
    for (int e = 0; e < nelem(); ++e) {
      const int n = nv_of(e);
      if (n < 3) throw std::runtime_error("mesh: element with fewer than 3 vertices");
      for (int i = 0; i < n; ++i) {
        const int a = loop[eoff[e] + i], b = loop[eoff[e] + (i + 1) % n];
        const uint64_t key = (uint64_t(uint32_t(std::min(a, b))) << 32) | uint32_t(std::max(a, b));
        auto it = seen.find(key);
        if (it == seen.end()) {
          seen.emplace(key, nfaces());
          efac[eoff[e] + i] = nfaces();
          esgn[eoff[e] + i] = 1;
          faces.push_back({a, b, e, -1, 0});
        } else {
          FaceRec& f = faces[it->second];
          if (f.right >= 0) throw std::runtime_error("mesh: non-manifold edge");
          if (f.a != b || f.b != a)
            throw std::runtime_error("mesh: inconsistent edge orientation between elements");
          f.right = e;
          efac[eoff[e] + i] = it->second;
          esgn[eoff[e] + i] = -1;
        }
      }
    }
    for (auto& f : faces)
      if (f.right < 0) f.tag = 1;
    measures();
  }

  /// Element-face links of an explicit face list (mesh.hpp:121-142; the
  /// reader's finalize_with_faces), then the measures.
  void finalize_with_faces() {
    std::unordered_map<uint64_t, int> byedge;
    byedge.reserve(faces.size() * 2);
    for (int f = 0; f < nfaces(); ++f) {
      const int a = faces[f].a, b = faces[f].b;
      byedge.emplace((uint64_t(uint32_t(std::min(a, b))) << 32) | uint32_t(std::max(a, b)), f);
    }
    efac.assign(loop.size(), -1);
    esgn.assign(loop.size(), 0);
    for (int e = 0; e < nelem(); ++e) {
      const int n = nv_of(e);
      for (int i = 0; i < n; ++i) {
        const int a = loop[eoff[e] + i], b = loop[eoff[e] + (i + 1) % n];
        auto it = byedge.find((uint64_t(uint32_t(std::min(a, b))) << 32) | uint32_t(std::max(a, b)));
        if (it == byedge.end()) throw std::runtime_error("mesh: element edge without a face record");
        const FaceRec& f = faces[it->second];
        const int sign = f.left == e ? 1 : -1;
        if (sign < 0 && f.right != e)
          throw std::runtime_error("mesh: face incidence does not match element loop");
        efac[eoff[e] + i] = it->second;
        esgn[eoff[e] + i] = sign;
      }
    }
    measures();
  }

  void measures() {
    // measures (mesh.hpp:144-173)
    const int ne = nelem();
    area.assign(ne, 0.0);
    diam.assign(ne, 0.0);
    cen.assign(ne, P2{});
    for (int e = 0; e < ne; ++e) {
      const int n = nv_of(e);
      double a2 = 0.0, cx = 0.0, cy = 0.0;
      for (int i = 0; i < n; ++i) {
        const P2 p = v[loop[eoff[e] + i]], q = v[loop[eoff[e] + (i + 1) % n]];
        const double cr = p.x * q.y - q.x * p.y;
        a2 += cr;
        cx += cr * (p.x + q.x);
        cy += cr * (p.y + q.y);
      }
      area[e] = 0.5 * a2;
      if (area[e] <= 0.0)
        throw std::runtime_error("mesh: element " + std::to_string(e) +
                                 " has non-positive signed area");
      cen[e] = {cx / (6.0 * area[e]), cy / (6.0 * area[e])};
      for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
          const P2 p = v[loop[eoff[e] + i]], q = v[loop[eoff[e] + j]];
          diam[e] = std::max(diam[e], std::sqrt((p.x - q.x) * (p.x - q.x) + (p.y - q.y) * (p.y - q.y)));
        }
    }
    hF.assign(nfaces(), 0.0);
    for (int f = 0; f < nfaces(); ++f) {
      const P2 a = v[faces[f].a], b = v[faces[f].b];
      hF[f] = std::sqrt((b.x - a.x) * (b.x - a.x) + (b.y - a.y) * (b.y - a.y));
    }
  }

  /// classify_boundary (mesh.hpp:510-531): midpoint on the chosen side is
  /// Neumann, every other boundary face Dirichlet.
  void classify(int side, double lo, double hi) {
    int nneu = 0;
    for (int f = 0; f < nfaces(); ++f) {
      if (faces[f].right >= 0) {
        faces[f].tag = 0;
        continue;
      }
      const P2 m = mid(f);
      const double tol = 1e-12;
      bool neu = false;
      switch (side) {
        case PSH_SIDE_LEFT: neu = std::abs(m.x - lo) < tol; break;
        case PSH_SIDE_RIGHT: neu = std::abs(m.x - hi) < tol; break;
        case PSH_SIDE_TOP: neu = std::abs(m.y - hi) < tol; break;
        case PSH_SIDE_BOTTOM: neu = std::abs(m.y - lo) < tol; break;
        default: throw std::invalid_argument("unknown Neumann side");
      }
      faces[f].tag = neu ? 2 : 1;
      nneu += neu;
    }
    if (nneu == 0)
      throw std::runtime_error("classify_boundary: no face found on the requested Neumann side");
  }
};

struct SplitMix64 {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double sym() { return 2.0 * double(next() >> 11) * 0x1.0p-53 - 1.0; }
};

inline int gv(int i, int j, int n) { return j * (n + 1) + i; }

void grid_elements(Mesh& m, int n, bool tri) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const int v00 = gv(i, j, n), v10 = gv(i + 1, j, n), v11 = gv(i + 1, j + 1, n),
                v01 = gv(i, j + 1, n);
      if (tri) {
        for (int x : {v00, v10, v11}) m.loop.push_back(x);
        m.eoff.push_back(int(m.loop.size()));
        for (int x : {v00, v11, v01}) m.loop.push_back(x);
        m.eoff.push_back(int(m.loop.size()));
      } else {
        for (int x : {v00, v10, v11, v01}) m.loop.push_back(x);
        m.eoff.push_back(int(m.loop.size()));
      }
    }
}

// ---------------------------------------------------------------------------
// quadrature (quadrature.hpp)
// ---------------------------------------------------------------------------

/// Gauss-Legendre nodes/weights on [-1,1] by Newton iteration on the
/// three-term recurrence, started from cos(pi (i + 3/4) / (m + 1/2)).
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

struct Rule {
  std::vector<P2> p;
  std::vector<double> w;
  int size() const { return int(w.size()); }
};

/// Collapsed (Duffy) rule on triangle (a,b,c), exact to total degree deg.
void triangle_rule(P2 a, P2 b, P2 c, int deg, Rule& r) {
  const int mu = (deg + 2) / 2 + 1, mv = deg / 2 + 1;
  std::vector<double> xu, wu, xv, wv;
  gauss_legendre(mu, xu, wu);
  gauss_legendre(mv, xv, wv);
  const double area2 = (b.x - a.x) * (c.y - a.y) - (c.x - a.x) * (b.y - a.y);
  for (int i = 0; i < mu; ++i) {
    const double u = 0.5 * (xu[i] + 1.0);
    for (int j = 0; j < mv; ++j) {
      const double s = 0.5 * (xv[j] + 1.0) * (1.0 - u);
      r.p.push_back({a.x + u * (b.x - a.x) + s * (c.x - a.x), a.y + u * (b.y - a.y) + s * (c.y - a.y)});
      r.w.push_back(0.25 * wu[i] * wv[j] * (1.0 - u) * area2);
    }
  }
}

Rule element_rule(const Mesh& m, int e, int deg) {
  Rule r;
  const int n = m.nv_of(e);
  const int* L = &m.loop[m.eoff[e]];
  if (n == 3) {
    triangle_rule(m.v[L[0]], m.v[L[1]], m.v[L[2]], deg, r);
    return r;
  }
  const P2 c = m.cen[e];
  for (int i = 0; i < n; ++i) {
    const P2 a = m.v[L[i]], b = m.v[L[(i + 1) % n]];
    if ((a.x - c.x) * (b.y - c.y) - (b.x - c.x) * (a.y - c.y) <= 0.0)
      throw std::runtime_error("element " + std::to_string(e) +
                               " is not star-shaped w.r.t. its centroid");
    triangle_rule(c, a, b, deg, r);
  }
  return r;
}

Rule face_rule(const Mesh& m, int f, int deg) {
  const int npts = deg / 2 + 1;
  std::vector<double> x, w;
  gauss_legendre(npts, x, w);
  const P2 a = m.v[m.faces[f].a], b = m.v[m.faces[f].b];
  Rule r;
  const double half = 0.5 * m.hF[f];
  for (int i = 0; i < npts; ++i) {
    r.p.push_back({0.5 * (a.x + b.x) + 0.5 * x[i] * (b.x - a.x),
                   0.5 * (a.y + b.y) + 0.5 * x[i] * (b.y - a.y)});
    r.w.push_back(half * w[i]);
  }
  return r;
}

// ---------------------------------------------------------------------------
// small dense helpers (column-major)
// ---------------------------------------------------------------------------

struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rr, int cc) : r(rr), c(cc), a(size_t(rr) * cc, 0.0) {}
  double& operator()(int i, int j) { return a[size_t(i) + size_t(j) * r]; }
  double operator()(int i, int j) const { return a[size_t(i) + size_t(j) * r]; }
};

/// Solves A X = B in place (partial pivoting); A is n x n, B is n x m.
void lu_solve(Mat A, Mat& B) {
  const int n = A.r;
  std::vector<int> piv(n);
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A(i, k)) > std::abs(A(p, k))) p = i;
    if (A(p, k) == 0.0) throw std::runtime_error("singular local system");
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

// ---------------------------------------------------------------------------
// hierarchical orthonormal bases (basis.hpp)
// ---------------------------------------------------------------------------

inline int dimP2(int d) { return (d + 1) * (d + 2) / 2; }

/// Modified Gram-Schmidt with one re-orthogonalisation pass in the
/// weighted quadrature inner product; returns lower-triangular C with
/// phi_i = sum_j C(i,j) m_j. vals (nq x n) is overwritten.
Mat orthonormalize(Mat& vals, const std::vector<double>& w, const char* what) {
  const int n = vals.c, nq = vals.r;
  Mat C(n, n);
  for (int i = 0; i < n; ++i) C(i, i) = 1.0;
  // dot(col i, w .* col j) with the Eigen subset's fixed-shape reduction
  // (include/eigen_subset/Eigen/Dense repro_dot: T = pow2 >= ceil(nq/16)
  // strided lane partials in index order, then an adjacent-pair tree), the
  // arithmetic the reference's mgs_coefficients (basis.hpp:29-52) runs with
  auto ip = [&](int i, int j) {
    int T = 1;
    while (T < (nq + 15) / 16 && T < (1 << 18)) T <<= 1;
    if (T == 1) {
      double s = 0.0;
      for (int q = 0; q < nq; ++q) s = s + vals(q, i) * (w[q] * vals(q, j));
      return s;
    }
    std::vector<double> part(T, 0.0);
    for (int q = 0; q < nq; ++q) part[q % T] = part[q % T] + vals(q, i) * (w[q] * vals(q, j));
    for (int width = T; width > 1; width >>= 1)
      for (int k = 0; k < width / 2; ++k) part[k] = part[2 * k] + part[2 * k + 1];
    return part[0];
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

struct ElemBasis {
  int deg = 0, dim = 0;
  P2 c;
  double h = 1.0;
  Mat C;  // dim x dim
  Rule rule;

  void monos(P2 p, double* m) const {
    const double x = (p.x - c.x) / h, y = (p.y - c.y) / h;
    int idx = 0;
    for (int d = 0; d <= deg; ++d)
      for (int ay = 0; ay <= d; ++ay) m[idx++] = std::pow(x, d - ay) * std::pow(y, ay);
  }
  void init(const Mesh& m, int e, int degree, int qdeg) {
    deg = degree;
    dim = dimP2(degree);
    c = m.cen[e];
    h = m.diam[e];
    rule = element_rule(m, e, qdeg);
    Mat vals(rule.size(), dim);
    std::vector<double> mm(dim);
    for (int q = 0; q < rule.size(); ++q) {
      monos(rule.p[q], mm.data());
      for (int i = 0; i < dim; ++i) vals(q, i) = mm[i];
    }
    C = orthonormalize(vals, rule.w, "element");
  }
  /// values of the first nd functions
  void eval(P2 p, int nd, double* out) const {
    double mm[64];
    monos(p, mm);
    for (int i = 0; i < nd; ++i) {
      double s = 0.0;
      for (int j = 0; j <= i; ++j) s += C(i, j) * mm[j];
      out[i] = s;
    }
  }
  /// gradients of all functions: out[2*i + d]
  void grad(P2 p, double* out) const {
    const double x = (p.x - c.x) / h, y = (p.y - c.y) / h;
    double gx[64], gy[64];
    int idx = 0;
    for (int d = 0; d <= deg; ++d)
      for (int ay = 0; ay <= d; ++ay) {
        const int ax = d - ay;
        gx[idx] = ax == 0 ? 0.0 : ax * std::pow(x, ax - 1) * std::pow(y, ay) / h;
        gy[idx] = ay == 0 ? 0.0 : ay * std::pow(x, ax) * std::pow(y, ay - 1) / h;
        ++idx;
      }
    for (int i = 0; i < dim; ++i) {
      double sx = 0.0, sy = 0.0;
      for (int j = 0; j <= i; ++j) {
        sx += C(i, j) * gx[j];
        sy += C(i, j) * gy[j];
      }
      out[2 * i] = sx;
      out[2 * i + 1] = sy;
    }
  }
};

struct FaceBasis {
  int dim = 0;
  P2 mid, t;
  double h = 1.0;
  Mat C;
  Rule rule;
  void init(const Mesh& m, int f, int degree, int qdeg) {
    dim = degree + 1;
    mid = m.mid(f);
    t = m.tangent(f);
    h = m.hF[f];
    rule = face_rule(m, f, qdeg);
    Mat vals(rule.size(), dim);
    for (int q = 0; q < rule.size(); ++q) {
      const double s = param(rule.p[q]);
      double pw = 1.0;
      for (int d = 0; d < dim; ++d, pw *= s) vals(q, d) = pw;
    }
    C = orthonormalize(vals, rule.w, "face");
  }
  double param(P2 p) const { return 2.0 * ((p.x - mid.x) * t.x + (p.y - mid.y) * t.y) / h; }
  void eval(P2 p, double* out) const {
    const double s = param(p);
    double mm[16];
    double pw = 1.0;
    for (int d = 0; d < dim; ++d, pw *= s) mm[d] = pw;
    for (int i = 0; i < dim; ++i) {
      double acc = 0.0;
      for (int j = 0; j <= i; ++j) acc += C(i, j) * mm[j];
      out[i] = acc;
    }
  }
};

// ---------------------------------------------------------------------------
// problem data (stokes_data.hpp; BASELINE.json sin/cos field)
// ---------------------------------------------------------------------------

struct Data {
  int kind = 0;
  void grad_u(P2 p, double g[2][2]) const {  // g[i][j] = d u_j / d x_i
    if (kind == PSH_DATA_EXP) {
      const double ex = std::exp(p.x), sy = std::sin(p.y), cy = std::cos(p.y);
      g[0][0] = -ex * (p.y * cy + sy);
      g[1][0] = -ex * (2.0 * cy - p.y * sy);
      g[0][1] = ex * p.y * sy;
      g[1][1] = ex * (sy + p.y * cy);
    } else {
      const double pi = M_PI;
      g[0][0] = pi * std::cos(pi * p.x) * std::cos(pi * p.y);
      g[1][0] = -pi * std::sin(pi * p.x) * std::sin(pi * p.y);
      g[0][1] = pi * std::sin(pi * p.x) * std::sin(pi * p.y);
      g[1][1] = -pi * std::cos(pi * p.x) * std::cos(pi * p.y);
    }
  }
  double pressure(P2 p) const {
    if (kind == PSH_DATA_EXP) return 2.0 * std::exp(p.x) * std::sin(p.y);
    return std::sin(2.0 * M_PI * p.x) * std::sin(2.0 * M_PI * p.y);
  }
  void f(P2 p, double out[2]) const {
    if (kind != PSH_DATA_SINCOS) {
      out[0] = out[1] = 0.0;
      return;
    }
    const double pi = M_PI, x = p.x, y = p.y;
    out[0] = 2.0 * pi * pi * std::sin(pi * x) * std::cos(pi * y) +
             2.0 * pi * std::cos(2.0 * pi * x) * std::sin(2.0 * pi * y);
    out[1] = -2.0 * pi * pi * std::cos(pi * x) * std::sin(pi * y) +
             2.0 * pi * std::sin(2.0 * pi * x) * std::cos(2.0 * pi * y);
  }
  void gd(P2 p, double out[2]) const {
    if (kind == PSH_DATA_ZERO) {
      out[0] = out[1] = 0.0;
    } else if (kind == PSH_DATA_EXP) {
      const double ex = std::exp(p.x);
      out[0] = -ex * (p.y * std::cos(p.y) + std::sin(p.y));
      out[1] = ex * p.y * std::sin(p.y);
    } else {
      out[0] = std::sin(M_PI * p.x) * std::cos(M_PI * p.y);
      out[1] = -std::cos(M_PI * p.x) * std::sin(M_PI * p.y);
    }
  }
  void gn(P2 p, P2 n, double out[2]) const {  // -n.grad(u) + p n
    if (kind == PSH_DATA_ZERO) {
      out[0] = out[1] = 0.0;
      return;
    }
    double g[2][2];
    grad_u(p, g);
    const double pr = pressure(p);
    out[0] = -(n.x * g[0][0] + n.y * g[1][0]) + pr * n.x;
    out[1] = -(n.x * g[0][1] + n.y * g[1][1]) + pr * n.y;
  }
};

// ---------------------------------------------------------------------------
// HHO local blocks (hho_local.hpp restated)
// ---------------------------------------------------------------------------

struct LocalLayout {
  int ne, nf, np, nfp, nfaces, nvel, n;
  int vel_elem(int c, int m) const { return c * ne + m; }
  int vel_face(int lf, int c, int m) const { return 2 * ne + lf * 2 * nf + c * nf + m; }
  int press_elem(int m) const { return nvel + m; }
  int press_face(int lf, int m) const { return nvel + np + lf * nfp + m; }
};

LocalLayout local_layout(int k, bool hybrid, int nfaces) {
  LocalLayout L;
  const int ke = hybrid ? k + 1 : k;
  L.ne = dimP2(ke);
  L.nf = k + 1;
  L.np = dimP2(k);
  L.nfp = hybrid ? k + 1 : 0;
  L.nfaces = nfaces;
  L.nvel = 2 * (L.ne + nfaces * L.nf);
  L.n = L.nvel + L.np + nfaces * L.nfp;
  return L;
}

/// Builds the local matrix (column-major, n x n) and load of element e.
/// With P_out set, stops after the reconstruction and stores it there
/// (nrec x ns, column-major) instead of building the blocks.
void build_local(const Mesh& mesh, int e, int k, bool hybrid, double eta, const Data& data,
                 double* mat, double* rhs, double* P_out = nullptr) {
  const int nfc = mesh.nv_of(e);
  const LocalLayout L = local_layout(k, hybrid, nfc);
  const int qd = 2 * (k + 1) + 1;
  ElemBasis rb;
  rb.init(mesh, e, k + 1, qd);
  const int nrec = rb.dim, ne = L.ne, nf = L.nf, ns = ne + nfc * nf;
  std::vector<FaceBasis> fb(nfc);
  std::vector<int> fid(nfc);
  std::vector<P2> nout(nfc);
  for (int lf = 0; lf < nfc; ++lf) {
    fid[lf] = mesh.efac[mesh.eoff[e] + lf];
    fb[lf].init(mesh, fid[lf], k, qd);
    const P2 nn = mesh.normal(fid[lf]);
    const int s = mesh.esgn[mesh.eoff[e] + lf];
    nout[lf] = {s * nn.x, s * nn.y};
  }
  auto fo = [&](int lf) { return ne + lf * nf; };

  // reconstruction: stiffness, mean moments, bordered Neumann solve
  Mat K(nrec, nrec);
  std::vector<double> mom(nrec, 0.0), phi(64), g(128), fv(16);
  for (int q = 0; q < rb.rule.size(); ++q) {
    const double w = rb.rule.w[q];
    rb.grad(rb.rule.p[q], g.data());
    rb.eval(rb.rule.p[q], nrec, phi.data());
    // m_stiff += w * g * g^T (hho_local.hpp:136): (w g_id) g_jd summed over d from 0
    for (int j = 0; j < nrec; ++j)
      for (int i = 0; i < nrec; ++i)
        K(i, j) += (w * g[2 * i]) * g[2 * j] + (w * g[2 * i + 1]) * g[2 * j + 1];
    for (int i = 0; i < nrec; ++i) mom[i] += w * phi[i];
  }
  Mat B(nrec + 1, ns);
  for (int j = 0; j < ne; ++j)
    for (int i = 0; i < nrec; ++i) B(i, j) = K(i, j);
  for (int lf = 0; lf < nfc; ++lf) {
    const Rule& fr = fb[lf].rule;
    for (int q = 0; q < fr.size(); ++q) {
      const double w = fr.w[q];
      rb.grad(fr.p[q], g.data());
      rb.eval(fr.p[q], nrec, phi.data());
      fb[lf].eval(fr.p[q], fv.data());
      for (int i = 0; i < nrec; ++i) {
        const double gn = g[2 * i] * nout[lf].x + g[2 * i + 1] * nout[lf].y;
        for (int m = 0; m < nf; ++m) B(i, fo(lf) + m) += w * gn * fv[m];
        for (int m = 0; m < ne; ++m) B(i, m) -= w * gn * phi[m];
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
  Mat P(nrec, ns);  // reconstruction operator
  for (int j = 0; j < ns; ++j)
    for (int i = 0; i < nrec; ++i) P(i, j) = B(i, j);
  if (P_out) {
    std::copy(P.a.begin(), P.a.end(), P_out);
    return;
  }

  // viscous block A = P^T K P + stabilisation + Nitsche
  // a = P^T K P evaluated left to right like the reference (hho_local.hpp:78)
  Mat PK(ns, nrec), A(ns, ns);
  for (int j = 0; j < nrec; ++j)
    for (int i = 0; i < ns; ++i) {
      double s = 0.0;
      for (int l = 0; l < nrec; ++l) s = s + P(l, i) * K(l, j);
      PK(i, j) = s;
    }
  for (int j = 0; j < ns; ++j)
    for (int i = 0; i < ns; ++i) {
      double s = 0.0;
      for (int l = 0; l < nrec; ++l) s = s + PK(i, l) * P(l, j);
      A(i, j) = s;
    }
  std::vector<double> R, DN;
  for (int lf = 0; lf < nfc; ++lf) {
    const Rule& fr = fb[lf].rule;
    const int nq = fr.size();
    const double hf = mesh.hF[fid[lf]];
    // residual R (nq x ns): pi_F(v_F - p(v)) - pi_T(v_T - p(v)) at the face points
    std::vector<double> psi(size_t(nq) * nf), rect(size_t(nq) * ns), ev(size_t(nq) * ne);
    R.assign(size_t(nq) * ns, 0.0);
    DN.assign(size_t(nq) * ns, 0.0);
    for (int q = 0; q < nq; ++q) {
      fb[lf].eval(fr.p[q], &psi[size_t(q) * nf]);
      rb.eval(fr.p[q], nrec, phi.data());
      rb.grad(fr.p[q], g.data());
      for (int m = 0; m < ne; ++m) ev[size_t(q) * ne + m] = phi[m];
      for (int s = 0; s < ns; ++s) {
        double tr = 0.0, dn = 0.0;
        for (int i = 0; i < nrec; ++i) {
          tr += phi[i] * P(i, s);
          dn += (g[2 * i] * nout[lf].x + g[2 * i + 1] * nout[lf].y) * P(i, s);
        }
        rect[size_t(q) * ns + s] = tr;
        DN[size_t(q) * ns + s] = dn;
      }
    }
    // coeff1 (nf x ns) = Psi^T W (-rec_tr) + I on this face's columns
    std::vector<double> c1(size_t(nf) * ns, 0.0);
    for (int m = 0; m < nf; ++m)
      for (int s = 0; s < ns; ++s) {
        double acc = 0.0;
        for (int q = 0; q < nq; ++q) acc += psi[size_t(q) * nf + m] * fr.w[q] * (-rect[size_t(q) * ns + s]);
        c1[size_t(m) * ns + s] = acc;
      }
    for (int m = 0; m < nf; ++m) c1[size_t(m) * ns + fo(lf) + m] += 1.0;
    // coeff2 (ne x ns) = -P[0:ne] + I on the element columns
    for (int q = 0; q < nq; ++q)
      for (int s = 0; s < ns; ++s) {
        double a1 = 0.0, a2 = 0.0;
        for (int m = 0; m < nf; ++m) a1 += psi[size_t(q) * nf + m] * c1[size_t(m) * ns + s];
        for (int m = 0; m < ne; ++m) {
          const double c2 = -P(m, s) + (s == m ? 1.0 : 0.0);
          a2 += ev[size_t(q) * ne + m] * c2;
        }
        R[size_t(q) * ns + s] = a1 - a2;
      }
    // a += (1/hF) r^T diag(w) r (hho_local.hpp:86): ((1/hF) r_qi) w_q r_qj over q from 0
    const double ih = 1.0 / hf;
    for (int j = 0; j < ns; ++j)
      for (int i = 0; i < ns; ++i) {
        double acc = 0.0;
        for (int q = 0; q < nq; ++q)
          acc = acc + ((ih * R[size_t(q) * ns + i]) * fr.w[q]) * R[size_t(q) * ns + j];
        A(i, j) += acc;
      }
    if (mesh.faces[fid[lf]].tag == 1) {
      for (int j = 0; j < ns; ++j)
        for (int i = 0; i < ns; ++i) {
          // cross(i,j) = sum_q DN(q,i) w V(q,j), V = face values on face cols
          double cij = 0.0, cji = 0.0, pen = 0.0;
          const bool jf = j >= fo(lf) && j < fo(lf) + nf;
          const bool iff = i >= fo(lf) && i < fo(lf) + nf;
          const double eh = eta / hf;
          for (int q = 0; q < nq; ++q) {
            const double vj = jf ? psi[size_t(q) * nf + (j - fo(lf))] : 0.0;
            const double vi = iff ? psi[size_t(q) * nf + (i - fo(lf))] : 0.0;
            cij = cij + (DN[size_t(q) * ns + i] * fr.w[q]) * vj;
            cji = cji + (DN[size_t(q) * ns + j] * fr.w[q]) * vi;
            // a += (eta/hF) vf^T diag(w) vf (hho_local.hpp:92)
            pen = pen + ((eh * vi) * fr.w[q]) * vj;
          }
          A(i, j) -= cij + cji;
          A(i, j) += pen;
        }
    }
  }

  // assemble the local Stokes block
  const int n = L.n;
  std::fill(mat, mat + size_t(n) * n, 0.0);
  std::fill(rhs, rhs + n, 0.0);
  auto M = [&](int i, int j) -> double& { return mat[size_t(i) + size_t(j) * n]; };
  auto vel_index = [&](int s, int c) {
    return s < ne ? L.vel_elem(c, s) : L.vel_face((s - ne) / nf, c, (s - ne) % nf);
  };
  for (int c = 0; c < 2; ++c)
    for (int j = 0; j < ns; ++j)
      for (int i = 0; i < ns; ++i) M(vel_index(i, c), vel_index(j, c)) += A(i, j);
  const int np = L.np;
  for (int q = 0; q < rb.rule.size(); ++q) {
    const double w = rb.rule.w[q];
    rb.eval(rb.rule.p[q], nrec, phi.data());
    rb.grad(rb.rule.p[q], g.data());
    for (int c = 0; c < 2; ++c)
      for (int m = 0; m < ne; ++m) {
        const double dv = g[2 * m + c];
        for (int i = 0; i < np; ++i) M(L.press_elem(i), L.vel_elem(c, m)) -= w * dv * phi[i];
      }
    double fvv[2];
    data.f(rb.rule.p[q], fvv);
    for (int c = 0; c < 2; ++c)
      for (int m = 0; m < ne; ++m) rhs[L.vel_elem(c, m)] += w * fvv[c] * phi[m];
  }
  for (int lf = 0; lf < nfc; ++lf) {
    const int f = fid[lf];
    const int tag = mesh.faces[f].tag;
    const Rule& fr = fb[lf].rule;
    const P2 nn = nout[lf];
    const double hf = mesh.hF[f];
    const double ncomp[2] = {nn.x, nn.y};
    for (int q = 0; q < fr.size(); ++q) {
      const double w = fr.w[q];
      rb.eval(fr.p[q], nrec, phi.data());
      rb.grad(fr.p[q], g.data());
      fb[lf].eval(fr.p[q], fv.data());
      if (!hybrid) {
        for (int i = 0; i < np; ++i)
          for (int c = 0; c < 2; ++c) {
            for (int m = 0; m < ne; ++m) M(L.press_elem(i), L.vel_elem(c, m)) += w * phi[i] * phi[m] * ncomp[c];
            if (tag != 1)
              for (int m = 0; m < nf; ++m) M(L.press_elem(i), L.vel_face(lf, c, m)) -= w * phi[i] * fv[m] * ncomp[c];
          }
      } else {
        for (int i = 0; i < L.nfp; ++i)
          for (int c = 0; c < 2; ++c) {
            for (int m = 0; m < ne; ++m) M(L.press_face(lf, i), L.vel_elem(c, m)) += w * fv[i] * phi[m] * ncomp[c];
            for (int m = 0; m < nf; ++m) M(L.press_face(lf, i), L.vel_face(lf, c, m)) -= w * fv[i] * fv[m] * ncomp[c];
          }
      }
      if (tag == 1) {
        double gdv[2];
        data.gd(fr.p[q], gdv);
        for (int c = 0; c < 2; ++c) {
          for (int s = 0; s < ns; ++s) {
            double dn = 0.0;
            for (int i = 0; i < nrec; ++i) dn += (g[2 * i] * nn.x + g[2 * i + 1] * nn.y) * P(i, s);
            rhs[vel_index(s, c)] -= w * gdv[c] * dn;
          }
          for (int m = 0; m < nf; ++m) rhs[L.vel_face(lf, c, m)] += w * (eta / hf) * gdv[c] * fv[m];
        }
        if (!hybrid)
          for (int i = 0; i < np; ++i) rhs[L.press_elem(i)] += w * (gdv[0] * nn.x + gdv[1] * nn.y) * phi[i];
      } else if (tag == 2) {
        double gnv[2];
        data.gn(fr.p[q], nn, gnv);
        for (int c = 0; c < 2; ++c)
          for (int m = 0; m < nf; ++m) rhs[L.vel_face(lf, c, m)] -= w * gnv[c] * fv[m];
      }
    }
  }
  // momentum pressure columns = transpose of the mass rows
  const int npress = n - L.nvel;
  for (int i = 0; i < npress; ++i)
    for (int j = 0; j < L.nvel; ++j) M(j, L.nvel + i) = M(L.nvel + i, j);
  if (hybrid)
    for (int lf = 0; lf < nfc; ++lf) {
      if (mesh.faces[fid[lf]].tag != 1) continue;
      for (int i = 0; i < L.nfp; ++i)
        for (int c = 0; c < 2; ++c)
          for (int m = 0; m < nf; ++m) M(L.vel_face(lf, c, m), L.press_face(lf, i)) = 0.0;
    }
}

// ---------------------------------------------------------------------------
// layout, retained ids, pattern (dof_layout.hpp, assemble.hpp)
// ---------------------------------------------------------------------------

struct System {
  int scheme = 0, strategy = 0, k = 0, nelem = 0, nloc = 0;
  int face_vel = 0, face_press = 0, elem_vel = 0, elem_press = 0, n_faces = 0;
  int64_t dim = 0;
  std::vector<double> mats, rhs;
  std::vector<int32_t> elim;
  int nkeep = 0;
  std::vector<int64_t> kept, row_ptr;
  std::vector<int32_t> cols;
  double seconds = 0.0;

  int fb() const { return 2 * face_vel + face_press; }
  int eb() const { return 2 * elem_vel + elem_press; }
  int kind(int64_t g) const {  // 0 vx, 1 vy, 2 p (assemble.hpp:25-39)
    const int64_t fsz = int64_t(n_faces) * fb();
    int within, nv;
    if (g < fsz) {
      within = int(g % fb());
      nv = face_vel;
    } else {
      within = int((g - fsz) % eb());
      nv = elem_vel;
    }
    return within < nv ? 0 : (within < 2 * nv ? 1 : 2);
  }
  bool coupled(int ka, int kb) const {  // assemble.hpp:41-46
    const bool av = ka != 2, bv = kb != 2;
    if (av && bv && ka != kb) return strategy == 2;
    if (!av && !bv) return strategy != 0;
    return true;
  }
};

} // namespace psh

using namespace psh;

struct psh_mesh {
  Mesh m;
};
struct psh_system {
  System s;
};

namespace {
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
} // namespace

extern "C" {

const char* psh_last_error(void) { return g_err.c_str(); }

int psh_mesh_unit_square(int n, int tri, double frac, uint64_t seed, int side, psh_mesh** out) {
  return guard([&] {
    if (n < 1) throw std::invalid_argument("unit square: n must be >= 1");
    auto pm = std::make_unique<psh_mesh>();
    Mesh& m = pm->m;
    m.v.resize(size_t(n + 1) * (n + 1));
    for (int j = 0; j <= n; ++j)
      for (int i = 0; i <= n; ++i) m.v[gv(i, j, n)] = {double(i) / double(n), double(j) / double(n)};
    if (frac > 0.0) {
      SplitMix64 rng{seed};
      const double h = 1.0 / double(n);
      for (int j = 1; j < n; ++j)
        for (int i = 1; i < n; ++i) {
          P2& p = m.v[gv(i, j, n)];
          p.x += frac * h * rng.sym();
          p.y += frac * h * rng.sym();
        }
    }
    grid_elements(m, n, tri != 0);
    m.finalize();
    m.classify(side, 0.0, 1.0);
    *out = pm.release();
  });
}

int psh_mesh_family(const char* family, int n, int side, psh_mesh** out) {
  return guard([&] {
    if (n < 1) throw std::invalid_argument("family mesh: n must be >= 1");
    const std::string fam = family;
    auto pm = std::make_unique<psh_mesh>();
    Mesh& m = pm->m;
    m.v.resize(size_t(n + 1) * (n + 1));
    for (int j = 0; j <= n; ++j)
      for (int i = 0; i <= n; ++i)
        m.v[gv(i, j, n)] = {-1.0 + 2.0 * i / n, -1.0 + 2.0 * j / n};
    if (fam == "trapz") {
      const double dy = 2.0 / n;
      for (int j = 1; j < n; ++j)
        for (int i = 0; i <= n; ++i) m.v[gv(i, j, n)].y += (i % 2 == 0 ? 1.0 : -1.0) * 0.1 * dy;
      grid_elements(m, n, false);
    } else if (fam == "quad") {
      grid_elements(m, n, false);
    } else if (fam == "tri") {
      grid_elements(m, n, true);
    } else {
      throw std::invalid_argument("unknown mesh family '" + fam + "'");
    }
    m.finalize();
    m.classify(side, -1.0, 1.0);
    *out = pm.release();
  });
}

void psh_mesh_destroy(psh_mesh* m) { delete m; }

void psh_mesh_counts(const psh_mesh* m, int64_t* out) {
  out[0] = int64_t(m->m.v.size());
  out[1] = m->m.nelem();
  out[2] = m->m.nfaces();
}

void psh_mesh_faces(const psh_mesh* m, int32_t* faces) {
  for (int f = 0; f < m->m.nfaces(); ++f) {
    const FaceRec& r = m->m.faces[f];
    faces[5 * f] = r.a;
    faces[5 * f + 1] = r.b;
    faces[5 * f + 2] = r.left;
    faces[5 * f + 3] = r.right;
    faces[5 * f + 4] = r.tag;
  }
}

// ---------------------------------------------------------------------------
// wire formats: MatrixMarket coordinate export (csr.hpp:98-111) and the
// pmesh2 v1 mesh file (mesh.hpp:535-645), byte-compatible with the
// reference's writers (same iostream formatting, precision 17)
// ---------------------------------------------------------------------------

int psh_write_matrix_market(int64_t n, const int64_t* row_ptr, const int32_t* cols,
                            const double* vals, const char* path) {
  return guard([&] {
    std::ofstream os(path);
    if (!os) throw std::runtime_error(std::string("write_matrix_market: cannot open '") + path + "'");
    os << "%%MatrixMarket matrix coordinate real general\n";
    os << n << ' ' << n << ' ' << row_ptr[n] << '\n';
    os.precision(17);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p)
        os << i + 1 << ' ' << cols[p] + 1 << ' ' << vals[p] << '\n';
    if (!os) throw std::runtime_error("write_matrix_market: write failed");
  });
}

int psh_mesh_write(const psh_mesh* pm, const char* path) {
  return guard([&] {
    const Mesh& m = pm->m;
    std::ofstream os(path);
    if (!os) throw std::runtime_error(std::string("write_mesh: cannot open '") + path + "'");
    os.precision(17);
    os << "pmesh2 v1 " << m.v.size() << ' ' << m.nelem() << ' ' << m.nfaces() << '\n';
    for (const P2& p : m.v) os << "v " << p.x << ' ' << p.y << '\n';
    for (int e = 0; e < m.nelem(); ++e) {
      os << 'e';
      for (int i = m.eoff[e]; i < m.eoff[e + 1]; ++i) os << ' ' << m.loop[i];
      os << '\n';
    }
    for (const FaceRec& f : m.faces)
      os << "f " << f.a << ' ' << f.b << ' ' << f.left << ' ' << f.right << ' '
         << (f.tag == 0 ? 'i' : (f.tag == 1 ? 'd' : 'n')) << '\n';
  });
}

int psh_mesh_read(const char* path, psh_mesh** out) {
  return guard([&] {
    std::ifstream is(path);
    if (!is) throw std::runtime_error(std::string("read_mesh: cannot open '") + path + "'");
    auto fail = [](int line, const std::string& what) {
      throw std::runtime_error("read_mesh: line " + std::to_string(line) + ": " + what);
    };
    std::string line;
    int lineno = 0;
    if (!std::getline(is, line)) fail(1, "empty file");
    ++lineno;
    std::istringstream hs(line);
    std::string magic, version;
    int nv = 0, ne = 0, nf = 0;
    if (!(hs >> magic >> version >> nv >> ne >> nf) || magic != "pmesh2" || version != "v1")
      fail(lineno, "malformed header, expected 'pmesh2 v1 <nv> <ne> <nf>'");
    if (ne == 0) fail(lineno, "no elements");
    auto next_record = [&](char want) -> std::istringstream {
      while (std::getline(is, line)) {
        ++lineno;
        if (line.empty() || line[0] == '#') continue;
        std::istringstream ls(line);
        std::string kind;
        ls >> kind;
        if (kind.size() != 1 || kind[0] != want)
          fail(lineno, std::string("expected a '") + want + "' record");
        return ls;
      }
      fail(lineno + 1, std::string("unexpected end of file, wanted a '") + want + "' record");
      return std::istringstream();
    };
    auto pm = std::make_unique<psh_mesh>();
    Mesh& m = pm->m;
    for (int i = 0; i < nv; ++i) {
      auto ls = next_record('v');
      double x, y;
      if (!(ls >> x >> y)) fail(lineno, "malformed vertex");
      m.v.push_back({x, y});
    }
    for (int i = 0; i < ne; ++i) {
      auto ls = next_record('e');
      int v, cnt = 0;
      while (ls >> v) {
        if (v < 0 || v >= nv) fail(lineno, "vertex index " + std::to_string(v) + " out of range");
        m.loop.push_back(v);
        ++cnt;
      }
      if (cnt < 3) fail(lineno, "element with fewer than 3 vertices");
      m.eoff.push_back(int(m.loop.size()));
    }
    if (nf == 0) {
      m.finalize();
      *out = pm.release();
      return;
    }
    for (int i = 0; i < nf; ++i) {
      auto ls = next_record('f');
      FaceRec f{};
      std::string tag;
      if (!(ls >> f.a >> f.b >> f.left >> f.right >> tag)) fail(lineno, "malformed face");
      if (f.a < 0 || f.a >= nv || f.b < 0 || f.b >= nv) fail(lineno, "face vertex out of range");
      if (f.left < 0 || f.left >= ne)
        fail(lineno, "face references element " + std::to_string(f.left) + " of " + std::to_string(ne));
      if (f.right >= ne)
        fail(lineno, "face references element " + std::to_string(f.right) + " of " + std::to_string(ne));
      if (tag == "i") f.tag = 0;
      else if (tag == "d") f.tag = 1;
      else if (tag == "n") f.tag = 2;
      else fail(lineno, "unknown face tag '" + tag + "'");
      if (f.right < 0 && f.tag == 0) fail(lineno, "boundary face tagged interior");
      if (f.right >= 0 && f.tag != 0) fail(lineno, "interior face carries a boundary tag");
      m.faces.push_back(f);
    }
    m.finalize_with_faces();
    *out = pm.release();
  });
}

void psh_mesh_vertices(const psh_mesh* m, double* xy) {
  for (size_t i = 0; i < m->m.v.size(); ++i) {
    xy[2 * i] = m->m.v[i].x;
    xy[2 * i + 1] = m->m.v[i].y;
  }
}

int psh_build(const psh_mesh* pm, int scheme, int strategy, int k, int data, double eta,
              int nthreads, psh_system** out) {
  return guard([&] {
    const auto t0 = std::chrono::steady_clock::now();
    const Mesh& mesh = pm->m;
    if (scheme != 0 && scheme != 1)
      throw std::invalid_argument("host producer: HHO schemes only (hho-dp, hho-hp)");
    if (k < 0) throw std::invalid_argument("layout: k must be >= 0");
    if (scheme == 1 && strategy == 1)
      throw std::invalid_argument("hho-hp: supported strategies are uncond and vp-cond");
    const int ne_el = mesh.nelem();
    const int nfc = mesh.nv_of(0);
    for (int e = 1; e < ne_el; ++e)
      if (mesh.nv_of(e) != nfc)
        throw std::invalid_argument("host producer: meshes must have one element type");
    auto ps = std::make_unique<psh_system>();
    System& S = ps->s;
    const bool hybrid = scheme == 1;
    const LocalLayout L = local_layout(k, hybrid, nfc);
    S.scheme = scheme;
    S.strategy = strategy;
    S.k = k;
    S.nelem = ne_el;
    S.nloc = L.n;
    S.n_faces = mesh.nfaces();
    // make_layout (dof_layout.hpp:87-126)
    S.face_vel = k + 1;
    S.face_press = hybrid ? k + 1 : 0;
    if (strategy == 0) {
      S.elem_vel = L.ne;
      S.elem_press = L.np;
    } else if (!hybrid) {
      S.elem_press = strategy == 1 ? L.np : 1;
    }
    S.dim = int64_t(S.n_faces) * S.fb() + int64_t(ne_el) * S.eb();
    // eliminated_dofs (condense.hpp:44-55)
    if (strategy != 0) {
      for (int c = 0; c < 2; ++c)
        for (int m = 0; m < L.ne; ++m) S.elim.push_back(L.vel_elem(c, m));
      if (strategy == 2)
        for (int m = hybrid ? 0 : 1; m < L.np; ++m) S.elim.push_back(L.press_elem(m));
    }
    std::vector<char> is_elim(L.n, 0);
    for (int i : S.elim) is_elim[i] = 1;
    std::vector<int> keep;
    for (int i = 0; i < L.n; ++i)
      if (!is_elim[i]) keep.push_back(i);
    S.nkeep = int(keep.size());

    const double eta_v = eta > 0.0 ? eta : 3.0 * (k + 1) * (k + 1);
    Data dd{data};
    S.mats.resize(size_t(ne_el) * L.n * L.n);
    S.rhs.resize(size_t(ne_el) * L.n);
    S.kept.resize(size_t(ne_el) * S.nkeep);
    if (nthreads > 0) omp_set_num_threads(nthreads);
    std::string err;
#pragma omp parallel for schedule(dynamic, 64)
    for (int e = 0; e < ne_el; ++e) {
      try {
        build_local(mesh, e, k, hybrid, eta_v, dd, &S.mats[size_t(e) * L.n * L.n],
                    &S.rhs[size_t(e) * L.n]);
      } catch (const std::exception& ex) {
#pragma omp critical
        err = ex.what();
      }
      // retained global ids in local keep order (assemble.hpp:72-96)
      std::vector<int64_t> full(L.n, -1);
      for (int lf = 0; lf < nfc; ++lf) {
        const int64_t base = int64_t(mesh.efac[mesh.eoff[e] + lf]) * S.fb();
        for (int c = 0; c < 2; ++c)
          for (int m = 0; m < L.nf; ++m) full[L.vel_face(lf, c, m)] = base + c * S.face_vel + m;
        for (int m = 0; m < L.nfp; ++m) full[L.press_face(lf, m)] = base + 2 * S.face_vel + m;
      }
      const int64_t eb = int64_t(S.n_faces) * S.fb() + int64_t(e) * S.eb();
      for (int c = 0; c < 2; ++c)
        for (int m = 0; m < S.elem_vel; ++m) full[L.vel_elem(c, m)] = eb + c * S.elem_vel + m;
      for (int m = 0; m < S.elem_press; ++m) full[L.press_elem(m)] = eb + 2 * S.elem_vel + m;
      for (int i = 0; i < S.nkeep; ++i) S.kept[size_t(e) * S.nkeep + i] = full[keep[i]];
    }
    if (!err.empty()) throw std::runtime_error(err);

    // structural pattern, row-centric: the union over the (<= 2) elements
    // holding a dof of their coupled retained dofs, plus the diagonal
    std::vector<std::vector<int>> face_elems(S.n_faces);
    for (int f = 0; f < S.n_faces; ++f) {
      face_elems[f].push_back(mesh.faces[f].left);
      if (mesh.faces[f].right >= 0) face_elems[f].push_back(mesh.faces[f].right);
    }
    const int fbk = S.fb(), ebk = S.eb();
    const int64_t nface_rows = int64_t(S.n_faces) * fbk;
    std::vector<int64_t> rowlen(S.dim, 0);
    auto row_cols = [&](int64_t g, const std::vector<int64_t>& uni, std::vector<int32_t>& outc) {
      outc.clear();
      const int kg = S.kind(g);
      for (int64_t h : uni)
        if (h == g || S.coupled(kg, S.kind(h))) outc.push_back(int32_t(h));
    };
    auto union_of = [&](const std::vector<int>& els, std::vector<int64_t>& uni) {
      uni.clear();
      for (int e : els)
        for (int i = 0; i < S.nkeep; ++i) uni.push_back(S.kept[size_t(e) * S.nkeep + i]);
      std::sort(uni.begin(), uni.end());
      uni.erase(std::unique(uni.begin(), uni.end()), uni.end());
    };
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1) {
        S.row_ptr.assign(S.dim + 1, 0);
        for (int64_t i = 0; i < S.dim; ++i) S.row_ptr[i + 1] = S.row_ptr[i] + rowlen[i];
        S.cols.resize(S.row_ptr[S.dim]);
      }
#pragma omp parallel
      {
        std::vector<int64_t> uni;
        std::vector<int32_t> rc;
#pragma omp for schedule(dynamic, 256)
        for (int f = 0; f < S.n_faces; ++f) {
          union_of(face_elems[f], uni);
          for (int r = 0; r < fbk; ++r) {
            const int64_t g = int64_t(f) * fbk + r;
            row_cols(g, uni, rc);
            if (pass == 0) rowlen[g] = int64_t(rc.size());
            else std::copy(rc.begin(), rc.end(), S.cols.begin() + S.row_ptr[g]);
          }
        }
#pragma omp for schedule(dynamic, 256)
        for (int e = 0; e < ne_el; ++e) {
          if (ebk == 0) continue;
          union_of(std::vector<int>{e}, uni);
          for (int r = 0; r < ebk; ++r) {
            const int64_t g = nface_rows + int64_t(e) * ebk + r;
            row_cols(g, uni, rc);
            if (pass == 0) rowlen[g] = int64_t(rc.size());
            else std::copy(rc.begin(), rc.end(), S.cols.begin() + S.row_ptr[g]);
          }
        }
      }
    }
    S.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = ps.release();
  });
}

/// Point tables for error_norms (errors.hpp:32-117), element-major from e0:
/// per element the velocity reconstruction P (nrec x ns, column-major), then
/// per point of the degree-2(k+2)+3 element rule {w, phi[nrec], dphi/dx[nrec],
/// dphi/dy[nrec], u(2), grad u (d u_j/d x_i at 2*j+i), p} of the degree-(k+1)
/// reconstruction basis (the basis the error loop rebuilds) and the
/// closed-form field. dims = {nrec, ns, nq, qstride, per_elem, ne, nf, np,
/// nloc, nfc, hybrid}.
int psh_error_tables(const psh_mesh* pm, int scheme, int k, int data, int e0, int nelem,
                     int nthreads, double* out, int32_t* dims) {
  return guard([&] {
    const Mesh& mesh = pm->m;
    if (scheme != 0 && scheme != 1)
      throw std::invalid_argument("error tables: HHO schemes only (hho-dp, hho-hp)");
    if (data != PSH_DATA_EXP && data != PSH_DATA_SINCOS)
      throw std::invalid_argument("error tables: data must have a closed form (exp or sincos)");
    if (k < 0) throw std::invalid_argument("layout: k must be >= 0");
    if (e0 < 0 || nelem < 0 || e0 + nelem > mesh.nelem())
      throw std::invalid_argument("error tables: element range out of bounds");
    const bool hybrid = scheme == 1;
    const int nfc = mesh.nv_of(0);
    const LocalLayout L = local_layout(k, hybrid, nfc);
    const int nrec = dimP2(k + 1), ns = L.ne + nfc * L.nf;
    const int eq = 2 * (k + 2) + 3;
    const int nq = element_rule(mesh, 0, eq).size();
    const int qstride = 3 * nrec + 8;
    const int64_t per = int64_t(nrec) * ns + int64_t(nq) * qstride;
    const int32_t d[11] = {nrec, ns, nq, qstride, int32_t(per), L.ne, L.nf, L.np, L.n, nfc, hybrid};
    std::copy(d, d + 11, dims);
    if (!out) return;
    const Data dd{data};
    if (nthreads > 0) omp_set_num_threads(nthreads);
    std::string err;
#pragma omp parallel for schedule(dynamic, 64)
    for (int i = 0; i < nelem; ++i) {
      try {
        const int e = e0 + i;
        if (mesh.nv_of(e) != nfc)
          throw std::invalid_argument("error tables: meshes must have one element type");
        double* t = out + size_t(i) * per;
        build_local(mesh, e, k, hybrid, 0.0, dd, nullptr, nullptr, t);
        t += size_t(nrec) * ns;
        ElemBasis rb;
        rb.init(mesh, e, k + 1, 2 * (k + 1) + 1);
        const Rule q = element_rule(mesh, e, eq);
        if (q.size() != nq) throw std::runtime_error("error tables: ragged element rules");
        std::vector<double> g(2 * nrec);
        for (int iq = 0; iq < nq; ++iq, t += qstride) {
          const P2 p = q.p[iq];
          t[0] = q.w[iq];
          rb.eval(p, nrec, t + 1);
          rb.grad(p, g.data());
          for (int j = 0; j < nrec; ++j) {
            t[1 + nrec + j] = g[2 * j];
            t[1 + 2 * nrec + j] = g[2 * j + 1];
          }
          double* x = t + 1 + 3 * nrec;
          dd.gd(p, x);
          double gu[2][2];
          dd.grad_u(p, gu);
          x[2] = gu[0][0];
          x[3] = gu[1][0];
          x[4] = gu[0][1];
          x[5] = gu[1][1];
          x[6] = dd.pressure(p);
        }
      } catch (const std::exception& ex) {
#pragma omp critical
        err = ex.what();
      }
    }
    if (!err.empty()) throw std::runtime_error(err);
  });
}

void psh_system_destroy(psh_system* s) { delete s; }

void psh_system_info(const psh_system* ps, int64_t* info) {
  const System& s = ps->s;
  const int64_t v[14] = {s.nelem,   s.nloc,     int64_t(s.elim.size()), s.nkeep,   s.dim,
                         int64_t(s.cols.size()), s.scheme, s.strategy,  s.k,         s.n_faces,
                         s.face_vel, s.face_press, s.elem_vel,          s.elem_press};
  std::memcpy(info, v, sizeof v);
}

const double* psh_local_mats(const psh_system* s) { return s->s.mats.data(); }
const double* psh_local_rhs(const psh_system* s) { return s->s.rhs.data(); }
const int32_t* psh_elim(const psh_system* s) { return s->s.elim.data(); }
const int64_t* psh_kept_global(const psh_system* s) { return s->s.kept.data(); }
const int64_t* psh_row_ptr(const psh_system* s) { return s->s.row_ptr.data(); }
const int32_t* psh_cols(const psh_system* s) { return s->s.cols.data(); }
double psh_build_seconds(const psh_system* s) { return s->s.seconds; }

} // extern "C"
