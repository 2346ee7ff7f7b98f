// HHO-hp 3D local element blocks on the device: the
// element geometry, quadrature, orthonormal bases, velocity reconstruction,
// stabilisation, Nitsche terms, pressure couplings and the random modal load
// of build_local (repo:paper_2009_13840_b200/host/pstokes_host3d.cpp, the 3D
// generalisation of hho_local.hpp:26-318 / basis.hpp / quadrature.hpp),
// evaluated with every sum in the host producer's order (--fmad=false, one
// rounding per operation), so the blocks are bit-identical to the host's.
//
// One CTA per element; each output entry's accumulation chain runs in one
// thread, the chains of an element in parallel. The Gram-Schmidt
// orthonormalisations are warp-cooperative (lane 0 forms each inner product
// in quadrature order, the lanes update the columns): warp 0 the element
// basis, warps 1-6 the six face bases, concurrently. Per-element work
// arrays live in a per-CTA global scratch slot (L2-resident); the 214 x 214
// block is written once, column-major, into the batch output the
// condensation kernel consumes.
//
// The host supplies what depends on its libm: the Gauss-Legendre rule
// (cos-seeded Newton) and the data-3 random modal coefficients (Box-Muller);
// data 4 (closed-form field) stays on the host producer.
#include "internal.cuh"

namespace pscu {

namespace {

struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 operator+(D3 a, D3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ D3 operator-(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ D3 operator*(double s, D3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ double dot(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ D3 cross(D3 a, D3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double norm(D3 a) { return sqrt(dot(a, a)); }

__host__ __device__ inline int dim2(int d) { return d < 0 ? 0 : (d + 1) * (d + 2) / 2; }
__host__ __device__ inline int dim3(int d) { return d < 0 ? 0 : (d + 1) * (d + 2) * (d + 3) / 6; }

constexpr int kL3Threads = 256;
constexpr int kMaxMono3 = 56;  // dim P^5 (k <= 4)

__constant__ int c_hex_off[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                    {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

/// Sizes and scratch offsets (doubles) of one element's work arrays.
struct L3Shape {
  int k, nq1, nq, fq, nrec, ne, nf, np, nfp, ns, n, nvel;
  // scratch offsets
  int64_t ep, ew, fp, fna, fw, vals, c, fvals, fc, ph, gr, kk, mom, fphi, fg, fpsi, b, s, p, kp,
      a, rect, dnw, r, c1, rt, wrt, per;
};

struct L3Args {
  L3Shape S;
  int data;
  double eta;
  int e0, nelem;
  const double* xyz;
  const int32_t* hex;
  const int32_t* ef;
  const int32_t* es;
  const int32_t* ftab;  // per face: 4 vertex ids, tag
  const double* glx;
  const double* glw;
  const double* coef;  // data 3: per element 3 x np
  double* mats;
  double* rhs;
  double* scratch;
  int* err;  // first failing element (code in the high bits)
};

__device__ __forceinline__ void fail(int* err, int e, int code) {
  atomicMin(err, (code << 28) | (e & 0x0fffffff));
}

/// Modified Gram-Schmidt with one re-orthogonalisation pass (basis.hpp:29-52
/// as the host producer restates it) by one warp: vals (nq x n, column
/// major) is overwritten, C (n x n, column major) receives the
/// lower-triangular coefficients. Returns false on a singular Gram matrix.
__device__ bool warp_orthonormalize(double* vals, const double* w, int nq, int n, double* C) {
  const int lane = threadIdx.x & 31;
  for (int t = lane; t < n * n; t += 32) C[t] = (t % n == t / n) ? 1.0 : 0.0;
  __syncwarp();
  auto ip = [&](int i, int j) {
    double s = 0.0;
    if (lane == 0)
      for (int q = 0; q < nq; ++q) s += vals[q + size_t(i) * nq] * (w[q] * vals[q + size_t(j) * nq]);
    return __shfl_sync(0xffffffffu, s, 0);
  };
  for (int i = 0; i < n; ++i) {
    for (int pass = 0; pass < 2; ++pass)
      for (int j = 0; j < i; ++j) {
        const double r = ip(i, j);
        for (int q = lane; q < nq; q += 32) vals[q + size_t(i) * nq] -= r * vals[q + size_t(j) * nq];
        for (int kk = lane; kk <= j; kk += 32) C[i + kk * n] -= r * C[j + kk * n];
        __syncwarp();
      }
    const double nrm = sqrt(ip(i, i));
    if (!(nrm > 1e-14)) return false;
    for (int q = lane; q < nq; q += 32) vals[q + size_t(i) * nq] /= nrm;
    for (int kk = lane; kk <= i; kk += 32) C[i + kk * n] /= nrm;
    __syncwarp();
  }
  return true;
}

/// Element basis monomials at p (ElemBasis::monos): scaled powers, graded order.
__device__ void elem_monos(D3 p, D3 c, double h, int deg, double* m) {
  const double x = (p.x - c.x) / h, y = (p.y - c.y) / h, z = (p.z - c.z) / h;
  double px[8], py[8], pz[8];
  px[0] = py[0] = pz[0] = 1.0;
  for (int a = 1; a <= deg; ++a) {
    px[a] = px[a - 1] * x;
    py[a] = py[a - 1] * y;
    pz[a] = pz[a - 1] * z;
  }
  int idx = 0;
  for (int d = 0; d <= deg; ++d)
    for (int az = 0; az <= d; ++az)
      for (int ay = 0; ay <= d - az; ++ay) m[idx++] = px[d - ay - az] * py[ay] * pz[az];
}

/// Values (out[i]) and gradients (og[3 i + d]) of the element basis at p.
__device__ void elem_eval(D3 p, D3 c, double h, int deg, int dim, const double* C, double* out,
                          double* og) {
  const double x = (p.x - c.x) / h, y = (p.y - c.y) / h, z = (p.z - c.z) / h;
  double X[8], Y[8], Z[8];
  X[0] = Y[0] = Z[0] = 1.0;
  for (int a = 1; a <= deg; ++a) {
    X[a] = X[a - 1] * x;
    Y[a] = Y[a - 1] * y;
    Z[a] = Z[a - 1] * z;
  }
  double mm[kMaxMono3], gx[kMaxMono3], gy[kMaxMono3], gz[kMaxMono3];
  int idx = 0;
  for (int d = 0; d <= deg; ++d)
    for (int az = 0; az <= d; ++az)
      for (int ay = 0; ay <= d - az; ++ay) {
        const int ax = d - ay - az;
        mm[idx] = X[ax] * Y[ay] * Z[az];
        gx[idx] = ax == 0 ? 0.0 : ax * X[ax - 1] * Y[ay] * Z[az] / h;
        gy[idx] = ay == 0 ? 0.0 : ay * X[ax] * Y[ay - 1] * Z[az] / h;
        gz[idx] = az == 0 ? 0.0 : az * X[ax] * Y[ay] * Z[az - 1] / h;
        ++idx;
      }
  for (int i = 0; i < dim; ++i) {
    double s = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
    for (int j = 0; j <= i; ++j) {
      const double cij = C[i + j * dim];
      s += cij * mm[j];
      sx += cij * gx[j];
      sy += cij * gy[j];
      sz += cij * gz[j];
    }
    if (out) out[i] = s;
    if (og) {
      og[3 * i] = sx;
      og[3 * i + 1] = sy;
      og[3 * i + 2] = sz;
    }
  }
}

struct FaceFrame {
  D3 c, t1, t2;
  double h;
};

__device__ void face_monos(D3 p, const FaceFrame& F, int deg, double* m) {
  const D3 d = p - F.c;
  const double x = dot(d, F.t1) / F.h, y = dot(d, F.t2) / F.h;
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

__global__ void __launch_bounds__(kL3Threads)
    local3_kernel(L3Args A) {
  const L3Shape& S = A.S;
  __shared__ D3 X[8];
  __shared__ D3 FV[6][4];
  __shared__ int fid[6], ftag[6];
  __shared__ double sgn[6], hf[6];
  __shared__ FaceFrame FF[6];
  __shared__ D3 cen;
  __shared__ double diam, rpiv;
  __shared__ int piv, bad;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nrec = S.nrec, ne = S.ne, nf = S.nf, ns = S.ns, nq = S.nq, fq = S.fq, nq1 = S.nq1;
  double* W = A.scratch + size_t(blockIdx.x) * S.per;
  double* EP = W + S.ep;      // nq x 3
  double* EW = W + S.ew;      // nq
  double* FPt = W + S.fp;     // 6 x fq x 3
  double* FNA = W + S.fna;    // 6 x fq x 3
  double* FW = W + S.fw;      // 6 x fq
  double* VALS = W + S.vals;  // nq x nrec
  double* CE = W + S.c;       // nrec x nrec
  double* FVALS = W + S.fvals;  // 6 x fq x nf
  double* FC = W + S.fc;      // 6 x nf x nf
  double* PH = W + S.ph;      // nq x nrec
  double* GR = W + S.gr;      // nq x nrec x 3
  double* K = W + S.kk;       // nrec x nrec
  double* MOM = W + S.mom;    // nrec
  double* FPHI = W + S.fphi;  // 6 x fq x nrec
  double* FG = W + S.fg;      // 6 x fq x nrec x 3
  double* FPSI = W + S.fpsi;  // 6 x fq x nf
  double* B = W + S.b;        // (nrec+1) x ns
  double* SM = W + S.s;       // (nrec+1) x (nrec+1)
  double* P = W + S.p;        // nrec x ns
  double* KP = W + S.kp;      // nrec x ns
  double* AV = W + S.a;       // ns x ns
  double* RECT = W + S.rect;  // fq x ns
  double* DNW = W + S.dnw;    // fq x ns
  double* R = W + S.r;        // fq x ns
  double* C1 = W + S.c1;      // nf x ns
  double* RT = W + S.rt;      // ns x fq
  double* WRT = W + S.wrt;    // ns x fq
  const int nb = nrec + 1;
  for (int el = blockIdx.x; el < A.nelem; el += gridDim.x) {
    const int e = A.e0 + el;
    if (tid == 0) bad = 0;
    if (tid < 8) {
      const int v = A.hex[size_t(el) * 8 + tid];
      X[tid] = {A.xyz[3 * size_t(v)], A.xyz[3 * size_t(v) + 1], A.xyz[3 * size_t(v) + 2]};
    }
    if (tid < 24) {
      const int lf = tid / 4, a = tid % 4;
      const int f = A.ef[size_t(el) * 6 + lf];
      const int v = A.ftab[5 * size_t(f) + a];
      FV[lf][a] = {A.xyz[3 * size_t(v)], A.xyz[3 * size_t(v) + 1], A.xyz[3 * size_t(v) + 2]};
      if (a == 0) {
        fid[lf] = f;
        ftag[lf] = A.ftab[5 * size_t(f) + 4];
        sgn[lf] = double(A.es[size_t(el) * 6 + lf]);
      }
    }
    __syncthreads();
    // element rule (element_rule): tensor Gauss points through the trilinear map
    for (int q = tid; q < nq; q += blockDim.x) {
      const int a = q % nq1, b = (q / nq1) % nq1, c = q / (nq1 * nq1);
      const double xi[3] = {A.glx[a], A.glx[b], A.glx[c]};
      D3 p{0.0, 0.0, 0.0}, d0{0.0, 0.0, 0.0}, d1{0.0, 0.0, 0.0}, d2{0.0, 0.0, 0.0};
      for (int v = 0; v < 8; ++v) {
        const double s0 = 2.0 * c_hex_off[v][0] - 1.0, s1 = 2.0 * c_hex_off[v][1] - 1.0,
                     s2 = 2.0 * c_hex_off[v][2] - 1.0;
        const double f0 = 1.0 + s0 * xi[0], f1 = 1.0 + s1 * xi[1], f2 = 1.0 + s2 * xi[2];
        p = p + (0.125 * f0 * f1 * f2) * X[v];
        d0 = d0 + (0.125 * s0 * f1 * f2) * X[v];
        d1 = d1 + (0.125 * f0 * s1 * f2) * X[v];
        d2 = d2 + (0.125 * f0 * f1 * s2) * X[v];
      }
      const double det = dot(d0, cross(d1, d2));
      if (!(det > 0.0)) bad = 1;
      EP[3 * q] = p.x;
      EP[3 * q + 1] = p.y;
      EP[3 * q + 2] = p.z;
      EW[q] = A.glw[a] * A.glw[b] * A.glw[c] * det;
    }
    // face rules (face_rule) of the six faces, points in the face's own orientation
    for (int t = tid; t < 6 * fq; t += blockDim.x) {
      const int lf = t / fq, q = t % fq;
      const int i = q % nq1, j = q / nq1;
      const double s = A.glx[i], u = A.glx[j];
      const D3 a = FV[lf][0], b = FV[lf][1], c = FV[lf][2], d = FV[lf][3];
      const D3 p = 0.25 * ((1 - s) * (1 - u) * a + (1 + s) * (1 - u) * b + (1 + s) * (1 + u) * c +
                           (1 - s) * (1 + u) * d);
      const D3 xs = 0.25 * ((1 - u) * (b - a) + (1 + u) * (c - d));
      const D3 xt = 0.25 * ((1 - s) * (d - a) + (1 + s) * (c - b));
      const D3 nv = cross(xs, xt);
      const D3 na = (A.glw[i] * A.glw[j]) * nv;
      double* fp = FPt + 3 * size_t(t);
      fp[0] = p.x;
      fp[1] = p.y;
      fp[2] = p.z;
      double* fn = FNA + 3 * size_t(t);
      fn[0] = na.x;
      fn[1] = na.y;
      fn[2] = na.z;
      FW[t] = A.glw[i] * A.glw[j] * norm(nv);
    }
    // face frames (FaceBasis::init) and diameters (face_diameter)
    if (tid < 6) {
      const int lf = tid;
      const D3 a = FV[lf][0], b = FV[lf][1], cc = FV[lf][2], d = FV[lf][3];
      FaceFrame F;
      F.c = 0.25 * (a + b + cc + d);
      double h = 0.0;
      const D3 Pv[4] = {a, b, cc, d};
      for (int i = 0; i < 4; ++i)
        for (int j = i + 1; j < 4; ++j) h = fmax(h, norm(Pv[i] - Pv[j]));
      F.h = h;
      D3 nb = cross(cc - a, d - b);
      nb = (1.0 / norm(nb)) * nb;
      D3 u = b - a;
      u = u - dot(u, nb) * nb;
      F.t1 = (1.0 / norm(u)) * u;
      F.t2 = cross(nb, F.t1);
      FF[lf] = F;
      hf[lf] = h;
    }
    __syncthreads();
    // element geometry (element_geo): volume-weighted centroid, vertex diameter
    if (tid == 0) {
      double vol = 0.0;
      D3 s{0.0, 0.0, 0.0};
      for (int q = 0; q < nq; ++q) {
        vol += EW[q];
        const D3 p{EP[3 * q], EP[3 * q + 1], EP[3 * q + 2]};
        s = s + EW[q] * p;
      }
      cen = (1.0 / vol) * s;
      double dm = 0.0;
      for (int a = 0; a < 8; ++a)
        for (int b = a + 1; b < 8; ++b) dm = fmax(dm, norm(X[a] - X[b]));
      diam = dm;
    }
    __syncthreads();
    // monomial tables of the element basis and of the face bases
    const int kdeg = S.k;
    for (int q = tid; q < nq; q += blockDim.x) {
      double mm[kMaxMono3];
      elem_monos({EP[3 * q], EP[3 * q + 1], EP[3 * q + 2]}, cen, diam, kdeg + 1, mm);
      for (int i = 0; i < nrec; ++i) VALS[q + size_t(i) * nq] = mm[i];
    }
    for (int t = tid; t < 6 * fq; t += blockDim.x) {
      const int lf = t / fq, q = t % fq;
      double mm[32];
      face_monos({FPt[3 * t], FPt[3 * t + 1], FPt[3 * t + 2]}, FF[lf], kdeg, mm);
      for (int i = 0; i < nf; ++i) FVALS[size_t(lf) * fq * nf + q + size_t(i) * fq] = mm[i];
    }
    __syncthreads();
    // orthonormalisation: warp 0 the element basis, warps 1-6 the faces
    if (wid == 0) {
      if (!warp_orthonormalize(VALS, EW, nq, nrec, CE) && lane == 0) bad = 2;
    } else if (wid <= 6) {
      const int lf = wid - 1;
      if (!warp_orthonormalize(FVALS + size_t(lf) * fq * nf, FW + size_t(lf) * fq, fq, nf,
                               FC + size_t(lf) * nf * nf) &&
          lane == 0)
        bad = 3;
    }
    __syncthreads();
    if (bad) {
      if (tid == 0) fail(A.err, e, bad);
      __syncthreads();
      continue;
    }
    // basis tables: element values / gradients at the element points, and at
    // the face points with the face basis values
    for (int q = tid; q < nq; q += blockDim.x)
      elem_eval({EP[3 * q], EP[3 * q + 1], EP[3 * q + 2]}, cen, diam, kdeg + 1, nrec, CE,
                PH + size_t(q) * nrec, GR + size_t(q) * nrec * 3);
    for (int t = tid; t < 6 * fq; t += blockDim.x) {
      const int lf = t / fq;
      const D3 p{FPt[3 * t], FPt[3 * t + 1], FPt[3 * t + 2]};
      elem_eval(p, cen, diam, kdeg + 1, nrec, CE, FPHI + size_t(t) * nrec, FG + size_t(t) * nrec * 3);
      double mm[32];
      face_monos(p, FF[lf], kdeg, mm);
      const double* Cf = FC + size_t(lf) * nf * nf;
      for (int i = 0; i < nf; ++i) {
        double s = 0.0;
        for (int j = 0; j <= i; ++j) s += Cf[i + j * nf] * mm[j];
        FPSI[size_t(t) * nf + i] = s;
      }
    }
    __syncthreads();
    // stiffness K and mean moments (quadrature order)
    for (int t = tid; t < nrec * nrec; t += blockDim.x) {
      const int i = t % nrec, j = t / nrec;
      double kij = 0.0;
      for (int q = 0; q < nq; ++q) {
        const double w = EW[q];
        const double* g = GR + size_t(q) * nrec * 3;
        const double gj0 = w * g[3 * j], gj1 = w * g[3 * j + 1], gj2 = w * g[3 * j + 2];
        kij += g[3 * i] * gj0 + g[3 * i + 1] * gj1 + g[3 * i + 2] * gj2;
      }
      K[t] = kij;
    }
    for (int i = tid; i < nrec; i += blockDim.x) {
      double m = 0.0;
      for (int q = 0; q < nq; ++q) m += EW[q] * PH[size_t(q) * nrec + i];
      MOM[i] = m;
    }
    __syncthreads();
    // reconstruction right-hand side B ((nrec+1) x ns) and the bordered matrix
    for (int t = tid; t < nb * ns; t += blockDim.x) {
      const int i = t % nb, col = t / nb;
      double v = 0.0;
      if (i == nrec) {
        v = col < ne ? MOM[col] : 0.0;
      } else {
        if (col < ne) v = K[i + col * nrec];
        const int cf = col < ne ? -1 : (col - ne) / nf, m = col < ne ? col : (col - ne) % nf;
        for (int lf = 0; lf < 6; ++lf) {
          if (cf >= 0 && lf != cf) continue;
          for (int q = 0; q < fq; ++q) {
            const size_t t2 = size_t(lf) * fq + q;
            const D3 na = sgn[lf] * D3{FNA[3 * t2], FNA[3 * t2 + 1], FNA[3 * t2 + 2]};
            const double* g = FG + t2 * nrec * 3;
            const double gn = g[3 * i] * na.x + g[3 * i + 1] * na.y + g[3 * i + 2] * na.z;
            if (cf >= 0) v += gn * FPSI[t2 * nf + m];
            else v -= gn * FPHI[t2 * nrec + m];
          }
        }
      }
      B[t] = v;
    }
    for (int t = tid; t < nb * nb; t += blockDim.x) {
      const int i = t % nb, j = t / nb;
      SM[t] = i < nrec && j < nrec ? K[i + j * nrec] : (i == nrec && j == nrec ? 0.0 : MOM[i == nrec ? j : i]);
    }
    __syncthreads();
    // lu_solve(S, B): partial pivoting (first largest |a|), rows swapped
    for (int kk = 0; kk < nb; ++kk) {
      if (tid == 0) {
        int p = kk;
        for (int i = kk + 1; i < nb; ++i)
          if (fabs(SM[i + kk * nb]) > fabs(SM[p + kk * nb])) p = i;
        piv = p;
        if (SM[p + kk * nb] == 0.0) bad = 4;
      }
      __syncthreads();
      if (bad) break;
      const int p = piv;
      if (p != kk) {
        for (int j = tid; j < nb; j += blockDim.x) {
          const double t = SM[kk + j * nb];
          SM[kk + j * nb] = SM[p + j * nb];
          SM[p + j * nb] = t;
        }
        for (int j = tid; j < ns; j += blockDim.x) {
          const double t = B[kk + j * nb];
          B[kk + j * nb] = B[p + j * nb];
          B[p + j * nb] = t;
        }
      }
      __syncthreads();
      if (tid == 0) rpiv = SM[kk + kk * nb];
      __syncthreads();
      const int rows = nb - kk - 1, cols = (nb - kk - 1) + ns;
      for (int t = tid; t < rows * cols; t += blockDim.x) {
        const int i = kk + 1 + t % rows, c = t / rows;
        const double l = SM[i + kk * nb] / rpiv;
        if (l == 0.0) continue;
        if (c < nb - kk - 1) {
          const int j = kk + 1 + c;
          SM[i + j * nb] -= l * SM[kk + j * nb];
        } else {
          const int j = c - (nb - kk - 1);
          B[i + j * nb] -= l * B[kk + j * nb];
        }
      }
      __syncthreads();
    }
    if (bad) {
      if (tid == 0) fail(A.err, e, bad);
      __syncthreads();
      continue;
    }
    for (int j = tid; j < ns; j += blockDim.x)
      for (int i = nb - 1; i >= 0; --i) {
        double s = B[i + j * nb];
        for (int q = i + 1; q < nb; ++q) s -= SM[i + q * nb] * B[q + j * nb];
        B[i + j * nb] = s / SM[i + i * nb];
      }
    __syncthreads();
    for (int t = tid; t < nrec * ns; t += blockDim.x) P[t] = B[t % nrec + (t / nrec) * nb];
    __syncthreads();
    // A = P^T (K P)
    for (int t = tid; t < nrec * ns; t += blockDim.x) {
      const int i = t % nrec, j = t / nrec;
      double s = 0.0;
      for (int l = 0; l < nrec; ++l) s += K[i + l * nrec] * P[l + j * nrec];
      KP[t] = s;
    }
    __syncthreads();
    for (int t = tid; t < ns * ns; t += blockDim.x) {
      const int i = t % ns, j = t / ns;
      double s = 0.0;
      for (int l = 0; l < nrec; ++l) s += P[l + i * nrec] * KP[l + j * nrec];
      AV[t] = s;
    }
    __syncthreads();
    // per face: reconstruction trace / weighted normal derivative, the
    // stabilisation R^T W R / h_F and, on Dirichlet faces, Nitsche
    auto fo = [&](int lf) { return ne + lf * nf; };
    for (int lf = 0; lf < 6; ++lf) {
      const double* fw = FW + size_t(lf) * fq;
      const double* psi = FPSI + size_t(lf) * fq * nf;
      for (int t = tid; t < fq * ns; t += blockDim.x) {
        const int q = t / ns, s = t % ns;
        const size_t t2 = size_t(lf) * fq + q;
        const D3 na = sgn[lf] * D3{FNA[3 * t2], FNA[3 * t2 + 1], FNA[3 * t2 + 2]};
        const double* g = FG + t2 * nrec * 3;
        const double* phi = FPHI + t2 * nrec;
        double tr = 0.0, dn = 0.0;
        for (int i = 0; i < nrec; ++i) {
          tr += phi[i] * P[i + s * nrec];
          dn += (g[3 * i] * na.x + g[3 * i + 1] * na.y + g[3 * i + 2] * na.z) * P[i + s * nrec];
        }
        RECT[t] = tr;
        DNW[t] = dn;
      }
      __syncthreads();
      for (int t = tid; t < nf * ns; t += blockDim.x) {
        const int mm = t / ns, s = t % ns;
        double acc = 0.0;
        for (int q = 0; q < fq; ++q) acc += psi[size_t(q) * nf + mm] * fw[q] * (-RECT[size_t(q) * ns + s]);
        if (s == fo(lf) + mm) acc += 1.0;
        C1[t] = acc;
      }
      __syncthreads();
      for (int t = tid; t < fq * ns; t += blockDim.x) {
        const int q = t / ns, s = t % ns;
        const double* phi = FPHI + (size_t(lf) * fq + q) * nrec;
        double a1 = 0.0, a2 = 0.0;
        for (int mm = 0; mm < nf; ++mm) a1 += psi[size_t(q) * nf + mm] * C1[size_t(mm) * ns + s];
        for (int mm = 0; mm < ne; ++mm) {
          const double c2 = -P[mm + s * nrec] + (s == mm ? 1.0 : 0.0);
          a2 += phi[mm] * c2;
        }
        R[t] = a1 - a2;
      }
      __syncthreads();
      for (int t = tid; t < fq * ns; t += blockDim.x) {
        const int q = t / ns, i = t % ns;
        RT[size_t(i) * fq + q] = R[t];
        WRT[size_t(i) * fq + q] = fw[q] * R[t];
      }
      __syncthreads();
      const double ih = 1.0 / hf[lf];
      const bool dir = ftag[lf] == 1;
      const double pen_s = A.eta / hf[lf];
      for (int t = tid; t < ns * ns; t += blockDim.x) {
        const int i = t % ns, j = t / ns;
        const double* ri = RT + size_t(i) * fq;
        const double* wj = WRT + size_t(j) * fq;
        double acc = 0.0;
        for (int q = 0; q < fq; ++q) acc += ri[q] * wj[q];
        double a = AV[t] + acc * ih;
        if (dir) {
          const bool jf = j >= fo(lf) && j < fo(lf) + nf;
          const bool iff = i >= fo(lf) && i < fo(lf) + nf;
          if (jf || iff) {
            double cij = 0.0, cji = 0.0, pen = 0.0;
            for (int q = 0; q < fq; ++q) {
              const double vj = jf ? psi[size_t(q) * nf + (j - fo(lf))] : 0.0;
              const double vi = iff ? psi[size_t(q) * nf + (i - fo(lf))] : 0.0;
              cij += DNW[size_t(q) * ns + i] * vj;
              cji += DNW[size_t(q) * ns + j] * vi;
              pen += vi * fw[q] * vj;
            }
            a -= cij + cji;
            a += pen_s * pen;
          }
        }
        AV[t] = a;
      }
      __syncthreads();
    }
    // the local Stokes block (column-major n x n) and load
    const int n = S.n, nvel = S.nvel, npr = S.np, nfp = S.nfp;
    double* M = A.mats + size_t(el) * n * n;
    double* rh = A.rhs + size_t(el) * n;
    // row -> (kind, lf / c, offset): velocity element (c, m), velocity face
    // (lf, c, m), pressure element m, pressure face (lf, m)
    for (int t = tid; t < n * n; t += blockDim.x) {
      const int i = t % n, j = t / n;
      double v = 0.0;
      if (i < nvel && j < nvel) {
        // viscous block: component-diagonal copies of A
        const int ci = i < 3 * ne ? i / ne : ((i - 3 * ne) % (3 * nf)) / nf;
        const int cj = j < 3 * ne ? j / ne : ((j - 3 * ne) % (3 * nf)) / nf;
        if (ci == cj) {
          const int si = i < 3 * ne ? i % ne : ne + ((i - 3 * ne) / (3 * nf)) * nf + (i - 3 * ne) % nf;
          const int sj = j < 3 * ne ? j % ne : ne + ((j - 3 * ne) / (3 * nf)) * nf + (j - 3 * ne) % nf;
          v = 0.0 + AV[si + sj * ns];
        }
      } else {
        // pressure rows (i >= nvel, j < nvel) and their transposes
        int pr = i, vc = j;
        bool zero_dir = false;
        if (i < nvel) {
          pr = j;
          vc = i;
        }
        if (pr >= nvel && vc < nvel) {
          const int pi = pr - nvel;
          if (pi < npr) {
            // element pressure row: -sum_q w dv phi_i over the element velocity
            if (vc < 3 * ne) {
              const int c = vc / ne, m = vc % ne;
              double acc = 0.0;
              for (int q = 0; q < nq; ++q) {
                const double w = EW[q];
                const double dv = GR[(size_t(q) * nrec + m) * 3 + c];
                acc -= w * dv * PH[size_t(q) * nrec + pi];
              }
              v = acc;
            }
          } else {
            const int lf = (pi - npr) / nfp, ii = (pi - npr) % nfp;
            // face pressure row: int_F (u_T - u_F).n q_F on this face's columns
            double acc = 0.0;
            bool hit = false;
            int c = -1, mm = -1;
            bool elem = false;
            if (vc < 3 * ne) {
              c = vc / ne;
              mm = vc % ne;
              elem = true;
              hit = true;
            } else {
              const int lfv = (vc - 3 * ne) / (3 * nf);
              if (lfv == lf) {
                c = ((vc - 3 * ne) % (3 * nf)) / nf;
                mm = (vc - 3 * ne) % nf;
                hit = true;
              }
            }
            if (hit) {
              for (int q = 0; q < fq; ++q) {
                const size_t t2 = size_t(lf) * fq + q;
                const D3 na = sgn[lf] * D3{FNA[3 * t2], FNA[3 * t2 + 1], FNA[3 * t2 + 2]};
                const double ncomp = c == 0 ? na.x : (c == 1 ? na.y : na.z);
                const double ps = FPSI[t2 * nf + ii];
                if (elem) acc += ps * FPHI[t2 * nrec + mm] * ncomp;
                else acc -= ps * FPSI[t2 * nf + mm] * ncomp;
              }
              v = acc;
              // Dirichlet faces: no face-pressure / face-velocity coupling in
              // the momentum rows (the transposed copy only)
              zero_dir = i < nvel && !elem && ftag[lf] == 1;
            }
          }
        }
        if (zero_dir) v = 0.0;
      }
      M[t] = v;
    }
    for (int t = tid; t < n; t += blockDim.x) {
      double v = 0.0;
      if (A.data == 3 && t < 3 * ne) {
        const int c = t / ne, m = t % ne;
        const double* cf = A.coef + size_t(el) * 3 * npr + size_t(c) * npr;
        for (int q = 0; q < nq; ++q) {
          const double* phi = PH + size_t(q) * nrec;
          double fv = 0.0;
          for (int mm = 0; mm < npr; ++mm) fv += cf[mm] * phi[mm];
          v += EW[q] * fv * phi[m];
        }
      }
      rh[t] = v;
    }
    __syncthreads();
  }
}

} // namespace

/// pscu_local_blocks3 on device buffers: S sizes from k, elements [e0, e0+nelem)
/// of the batch inputs (hex/ef/es/coef batch-relative, xyz/ftab whole mesh).
void local_blocks3(Context& c, int k, int data, double eta, int nq1, const double* glx,
                   const double* glw, const double* xyz, const int32_t* hex, const int32_t* ef,
                   const int32_t* es, const int32_t* ftab, const double* coef, int e0, int nelem,
                   double* mats, double* rhs) {
  if (k < 0 || k > 4) throw Error(PSCU_EINVAL, "hho3: k must be in [0, 4]");
  if (data != 0 && data != 3)
    throw Error(PSCU_EINVAL, "local_blocks3: device data kinds are 0 (zero) and 3 (random modal)");
  if (nelem <= 0) return;
  L3Shape S{};
  S.k = k;
  S.nq1 = nq1;
  S.nq = nq1 * nq1 * nq1;
  S.fq = nq1 * nq1;
  S.nrec = dim3(k + 1);
  S.ne = dim3(k + 1);
  S.nf = dim2(k);
  S.np = dim3(k);
  S.nfp = S.nf;
  S.ns = S.ne + 6 * S.nf;
  S.nvel = 3 * (S.ne + 6 * S.nf);
  S.n = S.nvel + S.np + 6 * S.nfp;
  const int64_t nq = S.nq, fq = S.fq, nrec = S.nrec, nf = S.nf, ns = S.ns, nb = nrec + 1;
  int64_t o = 0;
  auto take = [&](int64_t cnt) {
    const int64_t at = o;
    o += (cnt + 1) & ~int64_t(1);
    return at;
  };
  S.ep = take(3 * nq);
  S.ew = take(nq);
  S.fp = take(6 * fq * 3);
  S.fna = take(6 * fq * 3);
  S.fw = take(6 * fq);
  S.vals = take(nq * nrec);
  S.c = take(nrec * nrec);
  S.fvals = take(6 * fq * nf);
  S.fc = take(6 * nf * nf);
  S.ph = take(nq * nrec);
  S.gr = take(nq * nrec * 3);
  S.kk = take(nrec * nrec);
  S.mom = take(nrec);
  S.fphi = take(6 * fq * nrec);
  S.fg = take(6 * fq * nrec * 3);
  S.fpsi = take(6 * fq * nf);
  S.b = take(nb * ns);
  S.s = take(nb * nb);
  S.p = take(nrec * ns);
  S.kp = take(nrec * ns);
  S.a = take(ns * ns);
  S.rect = take(fq * ns);
  S.dnw = take(fq * ns);
  S.r = take(fq * ns);
  S.c1 = take(nf * ns);
  S.rt = take(ns * fq);
  S.wrt = take(ns * fq);
  S.per = o;
  const int grid = int(std::min<int64_t>(nelem, 148 * 4));
  if (c.l3_scratch.n < size_t(grid) * S.per) c.l3_scratch.alloc(size_t(grid) * S.per);
  const int big = 0x7fffffff;
  PSCU_CUDA(cudaMemcpyAsync(c.err_flag.p, &big, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  L3Args A{S, data, eta, e0, nelem, xyz, hex, ef, es, ftab, glx, glw, coef, mats, rhs,
           c.l3_scratch.p, c.err_flag.p};
  local3_kernel<<<grid, kL3Threads, 0, c.stream>>>(A);
  PSCU_LAUNCHED(&c);
  int bad = big;
  PSCU_CUDA(cudaMemcpyAsync(&bad, c.err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  PSCU_CUDA(cudaStreamSynchronize(c.stream));
  if (bad != big) {
    const int code = bad >> 28, e = bad & 0x0fffffff;
    const char* what = code == 1   ? "has a non-positive Jacobian"
                       : code == 2 ? "orthonormalize: singular Gram matrix on element"
                       : code == 3 ? "orthonormalize: singular Gram matrix on face"
                                   : "hho3: singular reconstruction system";
    throw Error(PSCU_ESINGULAR, std::string("local_blocks3: element ") + std::to_string(e) + " " + what);
  }
}

} // namespace pscu
