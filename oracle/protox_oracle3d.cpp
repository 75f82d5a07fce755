/*
 * protox_oracle3d.cpp -- CPU ORACLE for the 3D point-Jacobi relaxation of the
 * Poisson equation.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py may load this library
 * (it is linked into oracle/liborc.so next to protox_oracle.cpp).  The
 * product library never links, loads or calls it and shares no code with it.
 *
 * The paper states its model problem in 2D but defines every abstraction for
 * a general dimension D: Point and Box live in Z^D, the
 * Jacobi step size is λ = h²/(4D) and the Laplacian is the
 * (2D+1)-point stencil (Eq.1, written for D = 2 as
 * [0,1,0;1,-4,1;0,1,0]).  For D = 3 this file writes out the
 * UNFUSED Proto semantics of figure `Proto` exactly as the
 * 2D oracle does:
 *
 *     for iter < maxiter:
 *        exchange ghosts
 *        for each box: temp = laplace(phiPatch, wgt)
 *                      forallInPlace(jacobiUpdate, ...)    (Eq.3)
 *        residual max / L2 of the iterate                  (Eq.7)
 *
 * Readings (R-3D1..R-3D3):
 *  R-3D1 stencil: taps W,E,S,N,B,T (offsets -x,+x,-y,+y,-z,+z) weight 1 and
 *        C weight -6, in that order; L is the left fold of the taps starting
 *        from the first product; Δ_h = scale·L, scale = 1/h² (R2 in 3D).
 *  R-3D2 boundary rules as in 2D (R5): PERIODIC wrap, DIRICHLET_CC odd
 *        reflection per dimension (a ghost outside Ω in several dimensions
 *        gets the product of the signs), FIXED_GHOSTS (ghosts outside Ω are
 *        the caller's and never change).
 *  R-3D4 27-point compact Mehrstellen variant (the 3D counterpart of
 *        BASELINE config 5): faces 14, edges 3, corners 1, centre -128,
 *        scale 1/(30h²); fourth order with f = ρ + (1/12)·S7(ρ).
 *  R-3D3 layout: a global ghosted array of (n0+2g)(n1+2g)(n2+2g) doubles,
 *        dimension 0 fastest, then 1, then 2; the domain is split into
 *        b0 x b1 x b2 boxes, each with its own ghost ring (BoxData).
 * Norm schedule, NaN propagation and the Neumaier Σr² are the 2D oracle's
 * (R4, R7, R26).  Single thread, IEEE double, -ffp-contract=off.
 *
 * Parity pins: tests/test_oracle_pins3d.py.
 */
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

namespace orc3 {

static thread_local std::string g_err3;

/* Point in Z^3. */
struct P3 {
  int64_t c[3];
};
static P3 p3(int64_t x, int64_t y, int64_t z) {
  P3 p;
  p.c[0] = x;
  p.c[1] = y;
  p.c[2] = z;
  return p;
}

/* Box [lo, hi], inclusive corners. */
struct Box3 {
  P3 lo, hi;
  int64_t extent(int d) const { return hi.c[d] - lo.c[d] + 1; }
  bool contains(P3 p) const {
    for (int d = 0; d < 3; ++d)
      if (p.c[d] < lo.c[d] || p.c[d] > hi.c[d]) return false;
    return true;
  }
  Box3 grow(int64_t r) const {
    return Box3{p3(lo.c[0] - r, lo.c[1] - r, lo.c[2] - r), p3(hi.c[0] + r, hi.c[1] + r, hi.c[2] + r)};
  }
  /* dimension-0-fastest ordinal */
  int64_t ordinal(P3 p) const {
    return (p.c[0] - lo.c[0]) + extent(0) * ((p.c[1] - lo.c[1]) + extent(1) * (p.c[2] - lo.c[2]));
  }
};

/* one double per point of a (ghosted) box */
struct BoxData3 {
  Box3 box;
  std::vector<double> v;
  explicit BoxData3(Box3 b) : box(b), v((size_t)(b.extent(0) * b.extent(1) * b.extent(2)), 0.0) {}
  double& at(P3 p) { return v[(size_t)box.ordinal(p)]; }
  double at(P3 p) const { return v[(size_t)box.ordinal(p)]; }
};

struct Tap3 {
  P3 off;
  double alpha;
};

/* 7-point Laplacian (reading R-3D1) */
static std::vector<Tap3> laplace7() {
  return {{p3(-1, 0, 0), 1.0}, {p3(1, 0, 0), 1.0}, {p3(0, -1, 0), 1.0}, {p3(0, 1, 0), 1.0},
          {p3(0, 0, -1), 1.0}, {p3(0, 0, 1), 1.0}, {p3(0, 0, 0), -6.0}};
}

/* 27-point compact fourth-order Mehrstellen operator (reading R-3D4; the 3D
 * counterpart of the BASELINE config-5 9-point stencil, not in the paper):
 * scale 1/(30h²), faces 14, edges 3, corners 1, centre -128, in the order
 * faces W,E,S,N,B,T; edges xy (-1,-1),(1,-1),(-1,1),(1,1), xz (-1,·,-1),
 * (1,·,-1),(-1,·,1),(1,·,1), yz (·,-1,-1),(·,1,-1),(·,-1,1),(·,1,1);
 * corners z-major then y then x; centre. */
static std::vector<Tap3> mehrstellen27() {
  std::vector<Tap3> t = {{p3(-1, 0, 0), 14.0}, {p3(1, 0, 0), 14.0}, {p3(0, -1, 0), 14.0},
                         {p3(0, 1, 0), 14.0},  {p3(0, 0, -1), 14.0}, {p3(0, 0, 1), 14.0}};
  const int e2[4][2] = {{-1, -1}, {1, -1}, {-1, 1}, {1, 1}};
  for (auto& e : e2) t.push_back({p3(e[0], e[1], 0), 3.0});
  for (auto& e : e2) t.push_back({p3(e[0], 0, e[1]), 3.0});
  for (auto& e : e2) t.push_back({p3(0, e[0], e[1]), 3.0});
  for (int z = -1; z <= 1; z += 2)
    for (int y = -1; y <= 1; y += 2)
      for (int x = -1; x <= 1; x += 2) t.push_back({p3(x, y, z), 1.0});
  t.push_back({p3(0, 0, 0), -128.0});
  return t;
}

static double tap_sum3(const std::vector<Tap3>& taps, const BoxData3& src, P3 i) {
  double acc = 0.0;
  for (size_t t = 0; t < taps.size(); ++t) {
    P3 q = p3(i.c[0] + taps[t].off.c[0], i.c[1] + taps[t].off.c[1], i.c[2] + taps[t].off.c[2]);
    double term = taps[t].alpha * src.at(q);
    acc = (t == 0) ? term : acc + term;
  }
  return acc;
}

enum { BC_PERIODIC = 0, BC_DIRICHLET_CC = 1, BC_FIXED = 2 };

struct Layout3 {
  int64_t n[3], b[3], nb[3];
  int64_t g;
  int bc;
  std::vector<Box3> boxes;
  int64_t owner(P3 p) const {
    return (p.c[0] / b[0]) + nb[0] * ((p.c[1] / b[1]) + nb[1] * (p.c[2] / b[2]));
  }
  bool in_domain(P3 p) const {
    for (int d = 0; d < 3; ++d)
      if (p.c[d] < 0 || p.c[d] >= n[d]) return false;
    return true;
  }
};

static bool make_layout3(const int64_t n[3], const int64_t b[3], int64_t g, int bc, Layout3& L) {
  for (int d = 0; d < 3; ++d)
    if (n[d] < 1 || b[d] < 1 || n[d] % b[d] || g < 0 || g > b[d]) {
      g_err3 = "bad 3D layout: need n % b == 0 and 0 <= g <= b";
      return false;
    }
  for (int d = 0; d < 3; ++d) {
    L.n[d] = n[d];
    L.b[d] = b[d];
    L.nb[d] = n[d] / b[d];
  }
  L.g = g;
  L.bc = bc;
  L.boxes.clear();
  for (int64_t bz = 0; bz < L.nb[2]; ++bz)
    for (int64_t by = 0; by < L.nb[1]; ++by)
      for (int64_t bx = 0; bx < L.nb[0]; ++bx)
        L.boxes.push_back(Box3{p3(bx * b[0], by * b[1], bz * b[2]),
                               p3(bx * b[0] + b[0] - 1, by * b[1] + b[1] - 1, bz * b[2] + b[2] - 1)});
  return true;
}

struct Level3 {
  const Layout3* L;
  std::vector<BoxData3> data;
  explicit Level3(const Layout3& lay) : L(&lay) {
    for (const Box3& b : lay.boxes) data.emplace_back(b.grow(lay.g));
  }
};

/* Ghost exchange, every ghost point of every box gets the value
 * of the interior point it images (reading R-3D2). */
static void exchange3(Level3& lev) {
  const Layout3& L = *lev.L;
  for (size_t ib = 0; ib < L.boxes.size(); ++ib) {
    const Box3& B = L.boxes[ib];
    const Box3 G = B.grow(L.g);
    for (int64_t z = G.lo.c[2]; z <= G.hi.c[2]; ++z)
      for (int64_t y = G.lo.c[1]; y <= G.hi.c[1]; ++y)
        for (int64_t x = G.lo.c[0]; x <= G.hi.c[0]; ++x) {
          const P3 p = p3(x, y, z);
          if (B.contains(p)) continue;
          double sign = 1.0;
          bool skip = false;
          P3 q = p;
          for (int d = 0; d < 3; ++d) {
            const int64_t c = p.c[d], n = L.n[d];
            if (c >= 0 && c < n) continue;
            if (L.bc == BC_PERIODIC) {
              q.c[d] = ((c % n) + n) % n;
            } else if (L.bc == BC_DIRICHLET_CC) {
              q.c[d] = (c < 0) ? (-c - 1) : (2 * n - 1 - c);
              sign = -sign;
            } else {
              skip = true;
            }
          }
          if (skip) continue;
          lev.data[ib].at(p) = sign * lev.data[(size_t)L.owner(q)].at(q);
        }
  }
}

static int64_t gidx(const Layout3& L, int64_t x, int64_t y, int64_t z) {
  const int64_t W0 = L.n[0] + 2 * L.g, W1 = L.n[1] + 2 * L.g;
  return (x + L.g) + W0 * ((y + L.g) + W1 * (z + L.g));
}

static void scatter3(const double* glob, Level3& lev) {
  const Layout3& L = *lev.L;
  for (BoxData3& bd : lev.data)
    for (int64_t z = bd.box.lo.c[2]; z <= bd.box.hi.c[2]; ++z)
      for (int64_t y = bd.box.lo.c[1]; y <= bd.box.hi.c[1]; ++y)
        for (int64_t x = bd.box.lo.c[0]; x <= bd.box.hi.c[0]; ++x)
          bd.at(p3(x, y, z)) = glob[gidx(L, x, y, z)];
}

static void gather3(const Level3& lev, double* glob) {
  const Layout3& L = *lev.L;
  for (const BoxData3& bd : lev.data)  // ghosts outside Ω first
    for (int64_t z = bd.box.lo.c[2]; z <= bd.box.hi.c[2]; ++z)
      for (int64_t y = bd.box.lo.c[1]; y <= bd.box.hi.c[1]; ++y)
        for (int64_t x = bd.box.lo.c[0]; x <= bd.box.hi.c[0]; ++x)
          if (!L.in_domain(p3(x, y, z))) glob[gidx(L, x, y, z)] = bd.at(p3(x, y, z));
  for (size_t ib = 0; ib < L.boxes.size(); ++ib) {
    const Box3& B = L.boxes[ib];
    for (int64_t z = B.lo.c[2]; z <= B.hi.c[2]; ++z)
      for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
        for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x)
          glob[gidx(L, x, y, z)] = lev.data[ib].at(p3(x, y, z));
  }
}

struct Neumaier3 {
  double s = 0.0, c = 0.0;
  void add(double x) {
    const double t = s + x;
    if (std::fabs(s) >= std::fabs(x))
      c += (s - t) + x;
    else
      c += (x - t) + s;
    s = t;
  }
  // The compensation only refines a finite sum.  With an infinite term the
  // plain running sum is +inf (every term r*r >= 0) or NaN (a NaN term), and
  // that is the value of the sum (reading R6: Σr² is the plain sum of the
  // squares); (s - t) would turn inf into a spurious NaN in c.
  double value() const { return std::isfinite(s) ? s + c : s; }
};

/* Eq.7: exchange, r = scale*S(φ) − ρ over every interior point, max |r|
 * (NaN-propagating) and Σr² (Neumaier). */
static void residual3(const std::vector<Tap3>& taps, double scale, Level3& phi, const Level3& rho,
                      double out[2]) {
  exchange3(phi);
  double m = 0.0;
  bool nan = false;
  Neumaier3 sum;
  for (size_t ib = 0; ib < phi.L->boxes.size(); ++ib) {
    const Box3& B = phi.L->boxes[ib];
    for (int64_t z = B.lo.c[2]; z <= B.hi.c[2]; ++z)
      for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
        for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x) {
          const P3 p = p3(x, y, z);
          const double L = tap_sum3(taps, phi.data[ib], p);
          const double d = scale * L;
          const double r = d - rho.data[ib].at(p);
          const double a = std::fabs(r);
          if (a != a) nan = true;
          if (a > m) m = a;
          sum.add(r * r);
        }
  }
  out[0] = nan ? std::nan("") : m;
  out[1] = sum.value();
}

/* One Jacobi iteration in the order of figure `Proto`: exchange; per box
 * temp = laplace(phi, wgt); then φ = φ + λ(temp − ρ) in place (Eq.3). */
static void jacobi3(const std::vector<Tap3>& taps, double scale, Level3& phi, const Level3& rho,
                    double lambda) {
  exchange3(phi);
  for (size_t ib = 0; ib < phi.L->boxes.size(); ++ib) {
    const Box3& B = phi.L->boxes[ib];
    BoxData3 temp(B);
    for (int64_t z = B.lo.c[2]; z <= B.hi.c[2]; ++z)
      for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
        for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x) {
          const P3 p = p3(x, y, z);
          temp.at(p) = scale * tap_sum3(taps, phi.data[ib], p);
        }
    for (int64_t z = B.lo.c[2]; z <= B.hi.c[2]; ++z)
      for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
        for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x) {
          const P3 p = p3(x, y, z);
          double& v = phi.data[ib].at(p);
          v = v + lambda * (temp.at(p) - rho.data[ib].at(p));
        }
  }
}

}  // namespace orc3

using namespace orc3;

extern "C" {

typedef struct {
  int64_t n[3];   /* domain cells per dimension */
  int64_t b[3];   /* box size per dimension (must divide n) */
  int32_t ghost;  /* ghost width g >= 1 */
  int32_t bc;     /* 0 periodic, 1 dirichlet-cc, 2 fixed ghosts */
  int32_t stencil;         /* 0 = 7-point, 1 = 27-point Mehrstellen */
  int32_t rhs_correction;  /* 27-point only: f = rho + (1/12) S7(rho) */
  double h, lambda;
  int64_t nsweeps, norm_every;
} orc3_problem;

static bool setup3(const orc3_problem* p, std::vector<Tap3>& taps, double& scale) {
  if (p->stencil == 0) {
    taps = laplace7();
    scale = 1.0 / (p->h * p->h);
  } else if (p->stencil == 1) {
    taps = mehrstellen27();
    scale = 1.0 / (30.0 * p->h * p->h);
  } else {
    g_err3 = "stencil must be 0 (7-point) or 1 (27-point Mehrstellen)";
    return false;
  }
  return true;
}

/* f = ρ on the interior; with the 27-point stencil and rhs_correction,
 * f = ρ + (1/12)·S7(ρ) with ρ's ghosts filled by the boundary rule (R-3D4). */
static void make_rhs3(const orc3_problem* p, const double* rho_g, Level3& f) {
  scatter3(rho_g, f);
  if (p->stencil != 1 || !p->rhs_correction) return;
  exchange3(f);
  const std::vector<Tap3> s7 = laplace7();
  const double c12 = 1.0 / 12.0;
  for (size_t ib = 0; ib < f.L->boxes.size(); ++ib) {
    const Box3& B = f.L->boxes[ib];
    BoxData3 corr(B);
    for (int64_t z = B.lo.c[2]; z <= B.hi.c[2]; ++z)
      for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
        for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x) corr.at(p3(x, y, z)) = tap_sum3(s7, f.data[ib], p3(x, y, z));
    for (int64_t z = B.lo.c[2]; z <= B.hi.c[2]; ++z)
      for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
        for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x) {
          const P3 q = p3(x, y, z);
          f.data[ib].at(q) = f.data[ib].at(q) + c12 * corr.at(q);
        }
  }
}

const char* orc3_last_error(void) { return g_err3.c_str(); }

/* N iterations of figure `Proto` in 3D.  phi0, rho, phi_out: global ghosted
 * arrays (reading R-3D3).  norms[2j], [2j+1] = (max|r|, Σr²) of φ^(jE) for
 * jE < N, then of φ^N (E = norm_every; E = 0: final only; E < 0: none). */
int orc3_solve(const orc3_problem* p, const double* phi0, const double* rho, double* phi_out,
               double* norms, int64_t cap, int64_t* nwritten) {
  if (!p || !phi0 || !rho) {
    g_err3 = "null argument";
    return 1;
  }
  if (p->ghost < 1) {
    g_err3 = "ghost width must be >= 1";
    return 1;
  }
  Layout3 L;
  if (!make_layout3(p->n, p->b, p->ghost, p->bc, L)) return 1;
  std::vector<Tap3> taps;
  double scale;
  if (!setup3(p, taps, scale)) return 1;
  Level3 phi(L), f(L);
  scatter3(phi0, phi);
  make_rhs3(p, rho, f);
  int64_t nw = 0;
  auto record = [&]() {
    double r[2];
    residual3(taps, scale, phi, f, r);
    if (nw < cap && norms) {
      norms[2 * nw] = r[0];
      norms[2 * nw + 1] = r[1];
    }
    ++nw;
  };
  for (int64_t it = 0; it < p->nsweeps; ++it) {
    if (p->norm_every > 0 && it % p->norm_every == 0) record();
    jacobi3(taps, scale, phi, f, p->lambda);
  }
  if (p->norm_every >= 0) record();
  exchange3(phi);
  if (phi_out) gather3(phi, phi_out);
  if (nwritten) *nwritten = nw;
  return 0;
}

/* Δ_h φ = scale·S(φ) on the interior after the exchange; out: n2 x n1 x n0. */
int orc3_apply_laplacian(const orc3_problem* p, const double* phi_g, double* out) {
  Layout3 L;
  if (!make_layout3(p->n, p->b, p->ghost, p->bc, L)) return 1;
  std::vector<Tap3> taps;
  double scale;
  if (!setup3(p, taps, scale)) return 1;
  Level3 phi(L);
  scatter3(phi_g, phi);
  exchange3(phi);
  for (size_t ib = 0; ib < L.boxes.size(); ++ib) {
    const Box3& B = L.boxes[ib];
    for (int64_t z = B.lo.c[2]; z <= B.hi.c[2]; ++z)
      for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
        for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x)
          out[x + L.n[0] * (y + L.n[1] * z)] = scale * tap_sum3(taps, phi.data[ib], p3(x, y, z));
  }
  return 0;
}

/* the right-hand side the solve uses (f = ρ, or ρ + S7(ρ)/12), interior n2 x n1 x n0 */
int orc3_rhs(const orc3_problem* p, const double* rho_g, double* out) {
  Layout3 L;
  if (!make_layout3(p->n, p->b, p->ghost, p->bc, L)) return 1;
  Level3 f(L);
  make_rhs3(p, rho_g, f);
  for (size_t ib = 0; ib < L.boxes.size(); ++ib) {
    const Box3& B = L.boxes[ib];
    for (int64_t z = B.lo.c[2]; z <= B.hi.c[2]; ++z)
      for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
        for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x) out[x + L.n[0] * (y + L.n[1] * z)] = f.data[ib].at(p3(x, y, z));
  }
  return 0;
}

/* the exchange alone, on a global ghosted array in place */
int orc3_exchange(const orc3_problem* p, double* glob) {
  Layout3 L;
  if (!make_layout3(p->n, p->b, p->ghost, p->bc, L)) return 1;
  Level3 lev(L);
  scatter3(glob, lev);
  exchange3(lev);
  gather3(lev, glob);
  return 0;
}

}  // extern "C"
