/*
 * protox_oracle.cpp -- CPU ORACLE for the ProtoX 2D Poisson point-Jacobi
 * relaxation.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product library
 * (paper_2307_07931_b200/libprotox.so) never links, loads or calls it, and this
 * file shares no code, header, table or constant generator with it.
 *
 * What it computes: the UNFUSED Proto semantics of figure `Proto` of
 * /root/reference/PAPER.md (lines 154-180):
 *
 *     for iter < maxiter:
 *        exchange ghosts ("information is exchanged
 *                         between the boxes")
 *        for each box:
 *           temp = laplace(phiPatch, wgt)                   (Eq.1)
 *           forallInPlace(jacobiUpdate, phi, temp, rho, λ)  (Eq.3)
 *        resmax = computeMaxResidualAcrossProcs(phi,rho,dx) (Eq.7)
 *
 * written plainly: Point / Box / BoxData per box, a generic
 * tap-list Stencil (Eq.1), per-box ghost rings filled by an exchange, a
 * per-box temporary, an in-place pointwise update, and a separate residual
 * pass.  Single thread, IEEE double, compiled with -ffp-contract=off so every
 * `*` and `+` below is one rounded IEEE operation (reading R10).
 *
 * Readings of the paper taken here (all listed in DESIGN.md §3):
 *  R1  λ is an explicit input (paper: λ = h²/4D).
 *  R2  Δ_h = (1/h²)·S  (the `wgt` of PAPER.md:166; Fig. ProtoX divides by
 *      a_h1² in the residual).
 *  R4  the residual of an iterate φ is r = Δ_hφ − ρ (Eq.7);
 *      the oracle records it for φ^m, m = 0, E, 2E, ... < N, and φ^N.
 *  R5  boundary conditions: PERIODIC (Proto), DIRICHLET_CC
 *      (cell-centred homogeneous Dirichlet by odd reflection), FIXED_GHOSTS
 *      (domain ghost ring supplied by the caller and never changed).
 *  R7  max-norm propagates NaN.
 *  R18 Mehrstellen 9-point variant (not in the paper; BASELINE.json config 5):
 *      taps W,E,S,N:4  SW,SE,NW,NE:1  C:-20, scale 1/(6h²), optional
 *      right-hand side f = ρ + (1/12)·S5(ρ).
 *  R26 Σr² is accumulated with Neumaier compensation.
 *
 * Parity pins: tests/test_oracle_pins.py (closed-form spectra, 8x8 dense
 * brute force, spectral N-sweep closed form, exact trajectories, truncation
 * and discretisation order ladders, exchange vs flat periodic array).
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace orc {

static thread_local std::string g_err;

/* Point: a lattice point / offset in Z^2. */
struct Point {
  int64_t c[2];
};

static Point pt(int64_t x, int64_t y) {
  Point p;
  p.c[0] = x;
  p.c[1] = y;
  return p;
}

/* Box B = [lo, hi], inclusive corners. */
struct Box {
  Point lo, hi;
  bool empty() const { return lo.c[0] > hi.c[0] || lo.c[1] > hi.c[1]; }
  int64_t extent(int d) const { return empty() ? 0 : hi.c[d] - lo.c[d] + 1; }
  int64_t size() const { return extent(0) * extent(1); }
  Box grow(int64_t r) const {
    Box b;
    b.lo = pt(lo.c[0] - r, lo.c[1] - r);
    b.hi = pt(hi.c[0] + r, hi.c[1] + r);
    return b;
  }
  bool contains(Point p) const {
    return !empty() && p.c[0] >= lo.c[0] && p.c[0] <= hi.c[0] && p.c[1] >= lo.c[1] &&
           p.c[1] <= hi.c[1];
  }
  /* dimension-0-fastest ordinal (Fig. ProtoX index arithmetic) */
  int64_t ordinal(Point p) const {
    return (p.c[0] - lo.c[0]) + (p.c[1] - lo.c[1]) * extent(0);
  }
};

static Box mkbox(int64_t x0, int64_t y0, int64_t x1, int64_t y1) {
  Box b;
  b.lo = pt(x0, y0);
  b.hi = pt(x1, y1);
  return b;
}

/* BoxData<double,1,1,1>: one double per point of a box. */
struct BoxData {
  Box box;
  std::vector<double> v;
  explicit BoxData(Box b) : box(b), v((size_t)b.size(), 0.0) {}
  double& at(Point p) { return v[(size_t)box.ordinal(p)]; }
  double at(Point p) const { return v[(size_t)box.ordinal(p)]; }
};

/* Stencil (Eq.1): S(x)_i = Σ_j α_j x_{i+j}, taps kept in a
 * fixed order; `scale` is the wgt passed to laplace(...). */
struct Tap {
  Point off;
  double alpha;
};
struct Stencil {
  std::vector<Tap> taps;
  double scale;
  int64_t span;  // max |offset| over taps
};

/* 5-point Laplacian, taps [0,1,0;1,-4,1;0,1,0],
 * order W, E, S, N, C.  scale = 1/h² (reading R2). */
static Stencil laplace5(double h) {
  Stencil s;
  s.taps = {{pt(-1, 0), 1.0}, {pt(1, 0), 1.0}, {pt(0, -1), 1.0}, {pt(0, 1), 1.0},
            {pt(0, 0), -4.0}};
  s.scale = 1.0 / (h * h);
  s.span = 1;
  return s;
}

/* Mehrstellen 9-point (reading R18), order W,E,S,N (4), SW,SE,NW,NE (1), C (-20). */
static Stencil mehrstellen9(double h) {
  Stencil s;
  s.taps = {{pt(-1, 0), 4.0},  {pt(1, 0), 4.0},  {pt(0, -1), 4.0}, {pt(0, 1), 4.0},
            {pt(-1, -1), 1.0}, {pt(1, -1), 1.0}, {pt(-1, 1), 1.0}, {pt(1, 1), 1.0},
            {pt(0, 0), -20.0}};
  s.scale = 1.0 / (6.0 * h * h);
  s.span = 1;
  return s;
}

/* Undivided stencil value at point i: left fold over the taps in order,
 * starting from the first term (Eq.1). */
static double tap_sum(const Stencil& s, const BoxData& src, Point i) {
  double acc = 0.0;
  for (size_t t = 0; t < s.taps.size(); ++t) {
    Point q = pt(i.c[0] + s.taps[t].off.c[0], i.c[1] + s.taps[t].off.c[1]);
    double term = s.taps[t].alpha * src.at(q);
    acc = (t == 0) ? term : acc + term;
  }
  return acc;
}

/* stencil apply with a domain check naming the first violation. */
static bool stencil_apply(const Stencil& s, const BoxData& src, Box dest, BoxData& out,
                          double scale) {
  for (int64_t y = dest.lo.c[1]; y <= dest.hi.c[1]; ++y)
    for (int64_t x = dest.lo.c[0]; x <= dest.hi.c[0]; ++x)
      for (const Tap& t : s.taps) {
        Point q = pt(x + t.off.c[0], y + t.off.c[1]);
        if (!src.box.contains(q)) {
          char buf[160];
          snprintf(buf, sizeof buf,
                   "stencil domain violation at i=(%lld,%lld) tap=(%lld,%lld)", (long long)x,
                   (long long)y, (long long)t.off.c[0], (long long)t.off.c[1]);
          g_err = buf;
          return false;
        }
      }
  for (int64_t y = dest.lo.c[1]; y <= dest.hi.c[1]; ++y)
    for (int64_t x = dest.lo.c[0]; x <= dest.hi.c[0]; ++x) {
      double L = tap_sum(s, src, pt(x, y));
      out.at(pt(x, y)) = scale * L;
    }
  return true;
}

enum { BC_PERIODIC = 0, BC_DIRICHLET_CC = 1, BC_FIXED = 2 };

/* Domain Ω split into boxes B_j of b0 x b1 cells; the domain
 * is [0,n0-1]x[0,n1-1]; box index = bx + by*nb0. */
struct Layout {
  int64_t n[2], b[2], nb[2];
  int64_t g;
  int bc;
  std::vector<Box> boxes;
  Box domain() const { return mkbox(0, 0, n[0] - 1, n[1] - 1); }
  int64_t owner(Point p) const { return (p.c[0] / b[0]) + (p.c[1] / b[1]) * nb[0]; }
};

static bool make_layout(int64_t n0, int64_t n1, int64_t b0, int64_t b1, int64_t g, int bc,
                        Layout& L) {
  if (n0 < 1 || n1 < 1 || b0 < 1 || b1 < 1 || n0 % b0 || n1 % b1 || g < 0 || g > b0 ||
      g > b1) {
    g_err = "bad layout: need n % b == 0 and 0 <= g <= b";
    return false;
  }
  L.n[0] = n0;
  L.n[1] = n1;
  L.b[0] = b0;
  L.b[1] = b1;
  L.nb[0] = n0 / b0;
  L.nb[1] = n1 / b1;
  L.g = g;
  L.bc = bc;
  L.boxes.clear();
  for (int64_t by = 0; by < L.nb[1]; ++by)
    for (int64_t bx = 0; bx < L.nb[0]; ++bx)
      L.boxes.push_back(mkbox(bx * b0, by * b1, bx * b0 + b0 - 1, by * b1 + b1 - 1));
  return true;
}

/* LevelBoxData: one ghosted BoxData per box. */
struct Level {
  const Layout* L;
  std::vector<BoxData> data;
  explicit Level(const Layout& lay) : L(&lay) {
    for (const Box& b : lay.boxes) data.emplace_back(b.grow(lay.g));
  }
};

/* Ghost exchange: every ghost point of every box gets the
 * value of the interior point it images.  Periodic: wrap.
 * Dirichlet-CC: odd reflection per dimension outside Ω (x=-t <- -(t-1),
 * x=n-1+t <- -(n-t)), so a corner gets the product of the signs.
 * Fixed: ghost points outside Ω are left untouched; inter-box ghosts are copied. */
static void exchange(Level& lev) {
  const Layout& L = *lev.L;
  for (size_t ib = 0; ib < L.boxes.size(); ++ib) {
    const Box& B = L.boxes[ib];
    Box G = B.grow(L.g);
    for (int64_t y = G.lo.c[1]; y <= G.hi.c[1]; ++y)
      for (int64_t x = G.lo.c[0]; x <= G.hi.c[0]; ++x) {
        Point p = pt(x, y);
        if (B.contains(p)) continue;
        double sign = 1.0;
        bool skip = false;
        Point q = p;
        for (int d = 0; d < 2; ++d) {
          int64_t c = p.c[d], n = L.n[d];
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
        const BoxData& src = lev.data[(size_t)L.owner(q)];
        lev.data[ib].at(p) = sign * src.at(q);
      }
  }
}

/* Copy a global ghosted array (n0+2g) x (n1+2g), dim-0 fastest, into the
 * per-box storage (interior and every ghost point each box has). */
static void scatter_global(const double* glob, Level& lev) {
  const Layout& L = *lev.L;
  int64_t W = L.n[0] + 2 * L.g;
  for (size_t ib = 0; ib < L.boxes.size(); ++ib) {
    BoxData& bd = lev.data[ib];
    for (int64_t y = bd.box.lo.c[1]; y <= bd.box.hi.c[1]; ++y)
      for (int64_t x = bd.box.lo.c[0]; x <= bd.box.hi.c[0]; ++x) {
        /* ghost points that fall inside Ω belong to another box: take its value;
         * points outside Ω take the global ghost ring value. */
        bd.at(pt(x, y)) = glob[(x + L.g) + (y + L.g) * W];
      }
  }
}

static void gather_global(const Level& lev, double* glob) {
  const Layout& L = *lev.L;
  int64_t W = L.n[0] + 2 * L.g;
  /* ghosts first, interiors last so interior values win */
  for (size_t ib = 0; ib < L.boxes.size(); ++ib) {
    const BoxData& bd = lev.data[ib];
    for (int64_t y = bd.box.lo.c[1]; y <= bd.box.hi.c[1]; ++y)
      for (int64_t x = bd.box.lo.c[0]; x <= bd.box.hi.c[0]; ++x) {
        Point p = pt(x, y);
        if (L.domain().contains(p)) continue;
        glob[(x + L.g) + (y + L.g) * W] = bd.at(p);
      }
  }
  for (size_t ib = 0; ib < L.boxes.size(); ++ib) {
    const Box& B = L.boxes[ib];
    for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
      for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x)
        glob[(x + L.g) + (y + L.g) * W] = lev.data[ib].at(pt(x, y));
  }
}

/* Neumaier-compensated sum accumulator (reading R26; non-finite sums: R6). */
struct Neumaier {
  double s = 0.0, c = 0.0;
  void add(double x) {
    double t = s + x;
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

/* computeMaxResidualAcrossProcs and Eq.7:
 * exchange, then r = scale*S(φ) − f on every interior point of every box;
 * max |r| (NaN-propagating, reading R7) and Σ r². */
static void residual(const Stencil& st, Level& phi, const Level& f, double out[2]) {
  exchange(phi);
  double m = 0.0;
  bool nan = false;
  Neumaier sum;
  for (size_t ib = 0; ib < phi.L->boxes.size(); ++ib) {
    const Box& B = phi.L->boxes[ib];
    for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
      for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x) {
        Point p = pt(x, y);
        double L = tap_sum(st, phi.data[ib], p);
        double d = st.scale * L;
        double r = d - f.data[ib].at(p);
        double a = std::fabs(r);
        if (a != a) nan = true;
        if (a > m) m = a;
        sum.add(r * r);
      }
  }
  out[0] = nan ? std::nan("") : m;
  out[1] = sum.value();
}

/* One Jacobi iteration in the order of figure `Proto`:
 * exchange; per box: temp = laplace(phiPatch, wgt); forallInPlace update
 * φ = φ + λ(temp − f) (Eq.3). */
static void jacobi_iteration(const Stencil& st, Level& phi, const Level& f, double lambda) {
  exchange(phi);
  for (size_t ib = 0; ib < phi.L->boxes.size(); ++ib) {
    const Box& B = phi.L->boxes[ib];
    BoxData temp(B);
    stencil_apply(st, phi.data[ib], B, temp, st.scale);
    for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
      for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x) {
        Point p = pt(x, y);
        double r = temp.at(p) - f.data[ib].at(p);
        phi.data[ib].at(p) = phi.data[ib].at(p) + lambda * r;
      }
  }
}

/* ------------------------------------------------------------------------
 * Multigrid V-cycle with the Jacobi sweep as smoother (SURVEY §8(f) NEXT
 * rank 2; the paper names multigrid as a Proto use of stencils, PAPER.md:25,
 * and as future work for ProtoX, without defining one).  The
 * definition written out here is DESIGN.md readings R-MG1..R-MG6:
 *   levels ℓ = 0..L-1, n_ℓ = n/2^ℓ cells, h_ℓ = 2^ℓ h, same stencil and
 *   boundary rule on every level (homogeneous on ℓ >= 1), λ_ℓ = 4^ℓ λ;
 *   V(ℓ): ℓ = L-1: ν_c Jacobi iterations; else ν1 iterations,
 *         f_{ℓ+1} = −R d_ℓ  with d_ℓ = scale_ℓ·S(φ_ℓ) − f_ℓ (Eq.7),
 *         φ_{ℓ+1} = 0, V(ℓ+1), φ_ℓ += P φ_{ℓ+1}, ν2 iterations;
 *   R: average of the 2x2 children, summed in the order (0,0),(1,0),(0,1),(1,1);
 *   P: cell-centred bilinear, fine cell (2I+a, 2J+b) gets
 *      (9·e(I,J) + 3·e(I±1,J) + 3·e(I,J±1) + e(I±1,J±1)) / 16, the ± towards
 *      the fine cell, summed left to right, coarse ghosts by the level's rule.
 * ---------------------------------------------------------------------- */
struct MGLevel {
  Layout L;
  Stencil st;
  double lambda = 0.0;
  std::vector<Level> phi, f;  // one element each (Level holds a pointer to L)
};

static double level_at(const Level& lev, Point p) {
  return lev.data[(size_t)lev.L->owner(p)].at(p);
}
static double& level_ref(Level& lev, Point p) { return lev.data[(size_t)lev.L->owner(p)].at(p); }

/* f_{ℓ+1} = −R d_ℓ */
static void restrict_defect(MGLevel& fine, MGLevel& coarse) {
  Level& phi = fine.phi[0];
  exchange(phi);
  const int64_t n0 = fine.L.n[0], n1 = fine.L.n[1];
  std::vector<double> d((size_t)(n0 * n1));
  for (size_t ib = 0; ib < fine.L.boxes.size(); ++ib) {
    const Box& B = fine.L.boxes[ib];
    for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
      for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x) {
        Point q = pt(x, y);
        double L = tap_sum(fine.st, phi.data[ib], q);
        d[(size_t)(x + y * n0)] = fine.st.scale * L - fine.f[0].data[ib].at(q);
      }
  }
  Level& fc = coarse.f[0];
  for (int64_t J = 0; J < coarse.L.n[1]; ++J)
    for (int64_t I = 0; I < coarse.L.n[0]; ++I) {
      const double* r0 = &d[(size_t)(2 * I + 2 * J * n0)];
      double t = r0[0] + r0[1];
      t = t + r0[n0];
      t = t + r0[n0 + 1];
      level_ref(fc, pt(I, J)) = -0.25 * t;
    }
}

/* φ_ℓ += P φ_{ℓ+1} */
static void prolong_correct(MGLevel& coarse, MGLevel& fine) {
  Level& e = coarse.phi[0];
  exchange(e);
  const BoxData& E = e.data[0];  // coarse levels are one box
  for (size_t ib = 0; ib < fine.L.boxes.size(); ++ib) {
    const Box& B = fine.L.boxes[ib];
    for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
      for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x) {
        const int64_t I = x / 2, J = y / 2;
        const int64_t xn = (x % 2) ? I + 1 : I - 1, yn = (y % 2) ? J + 1 : J - 1;
        double t = 9.0 * E.at(pt(I, J));
        t = t + 3.0 * E.at(pt(xn, J));
        t = t + 3.0 * E.at(pt(I, yn));
        t = t + E.at(pt(xn, yn));
        double v = 0.0625 * t;
        Point q = pt(x, y);
        fine.phi[0].data[ib].at(q) = fine.phi[0].data[ib].at(q) + v;
      }
  }
}

struct MGOpts {
  int64_t levels, nu1, nu2, nu_coarse, ncycles;
};

static void vcycle(std::vector<MGLevel>& lv, size_t l, const MGOpts& m) {
  MGLevel& F = lv[l];
  if (l + 1 == lv.size()) {
    for (int64_t k = 0; k < m.nu_coarse; ++k) jacobi_iteration(F.st, F.phi[0], F.f[0], F.lambda);
    return;
  }
  for (int64_t k = 0; k < m.nu1; ++k) jacobi_iteration(F.st, F.phi[0], F.f[0], F.lambda);
  MGLevel& C = lv[l + 1];
  restrict_defect(F, C);
  for (BoxData& bd : C.phi[0].data) std::fill(bd.v.begin(), bd.v.end(), 0.0);
  vcycle(lv, l + 1, m);
  prolong_correct(C, F);
  for (int64_t k = 0; k < m.nu2; ++k) jacobi_iteration(F.st, F.phi[0], F.f[0], F.lambda);
}

}  // namespace orc

using namespace orc;

extern "C" {

typedef struct {
  int64_t n0, n1;          /* domain cells per dimension */
  int64_t b0, b1;          /* box size (must divide n) */
  int32_t ghost;           /* ghost width g (>= 1) */
  int32_t bc;              /* 0 periodic, 1 dirichlet-cc, 2 fixed ghosts */
  int32_t stencil;         /* 0 = 5-point, 1 = Mehrstellen 9-point */
  int32_t rhs_correction;  /* 9-point only: f = rho + (1/12) S5(rho) */
  double h, lambda;
  int64_t nsweeps, norm_every;
} orc_problem;

const char* orc_last_error(void) { return g_err.c_str(); }

static bool build(const orc_problem* p, Layout& L, Stencil& st) {
  if (!p) {
    g_err = "null problem";
    return false;
  }
  if (!make_layout(p->n0, p->n1, p->b0, p->b1, p->ghost, p->bc, L)) return false;
  if (p->ghost < 1) {
    g_err = "ghost must be >= 1";
    return false;
  }
  st = (p->stencil == 1) ? mehrstellen9(p->h) : laplace5(p->h);
  return true;
}

/* Right-hand side f of the update: ρ, or for the Mehrstellen variant with
 * rhs_correction, f = ρ + (1/12)·S5(ρ) evaluated after filling ρ's ghosts
 * by the same boundary rule (reading R18). */
static void make_rhs(const orc_problem* p, const Layout& L, const double* rho_g, Level& f) {
  scatter_global(rho_g, f);
  if (p->stencil == 1 && p->rhs_correction) {
    exchange(f);
    Stencil s5 = laplace5(1.0);
    const double c12 = 1.0 / 12.0;
    for (size_t ib = 0; ib < L.boxes.size(); ++ib) {
      const Box& B = L.boxes[ib];
      BoxData corr(B);
      for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
        for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x)
          corr.at(pt(x, y)) = tap_sum(s5, f.data[ib], pt(x, y));
      for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
        for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x) {
          Point q = pt(x, y);
          f.data[ib].at(q) = f.data[ib].at(q) + c12 * corr.at(q);
        }
    }
  }
}

/* Full solve: N Jacobi iterations of figure `Proto`.  Arrays are global
 * ghosted (n0+2g) x (n1+2g), dim-0 fastest.  norms[2j], norms[2j+1] =
 * (max|r|, Σr²) of φ^(jE) for jE < N, then of φ^N.  Returns 0 or an error. */
int orc_solve(const orc_problem* p, const double* phi0, const double* rho, double* phi_out,
              double* norms, int64_t cap, int64_t* nwritten) {
  Layout L;
  Stencil st;
  if (!build(p, L, st)) return 1;
  Level phi(L), f(L);
  scatter_global(phi0, phi);
  make_rhs(p, L, rho, f);
  int64_t nw = 0;
  auto record = [&]() {
    double r[2];
    residual(st, phi, f, r);
    if (nw < cap && norms) {
      norms[2 * nw] = r[0];
      norms[2 * nw + 1] = r[1];
    }
    ++nw;
  };
  for (int64_t it = 0; it < p->nsweeps; ++it) {
    if (p->norm_every > 0 && it % p->norm_every == 0) record();
    jacobi_iteration(st, phi, f, p->lambda);
  }
  if (p->norm_every >= 0) record();
  exchange(phi);
  if (phi_out) gather_global(phi, phi_out);
  if (nwritten) *nwritten = nw;
  return 0;
}

/* Δ_h φ on the interior after an exchange (for the spectral pins). */
int orc_apply_laplacian(const orc_problem* p, const double* phi_g, double* out_interior) {
  Layout L;
  Stencil st;
  if (!build(p, L, st)) return 1;
  Level phi(L);
  scatter_global(phi_g, phi);
  exchange(phi);
  for (size_t ib = 0; ib < L.boxes.size(); ++ib) {
    const Box& B = L.boxes[ib];
    BoxData out(B);
    stencil_apply(st, phi.data[ib], B, out, st.scale);
    for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
      for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x)
        out_interior[x + y * L.n[0]] = out.at(pt(x, y));
  }
  return 0;
}

/* Residual norms of φ as given (PAPER.md:173 semantics). */
int orc_residual(const orc_problem* p, const double* phi_g, const double* rho_g,
                 double out[2]) {
  Layout L;
  Stencil st;
  if (!build(p, L, st)) return 1;
  Level phi(L), f(L);
  scatter_global(phi_g, phi);
  make_rhs(p, L, rho_g, f);
  residual(st, phi, f, out);
  return 0;
}

/* The right-hand side f the iteration uses (interior only). */
int orc_rhs(const orc_problem* p, const double* rho_g, double* f_interior) {
  Layout L;
  Stencil st;
  if (!build(p, L, st)) return 1;
  Level f(L);
  make_rhs(p, L, rho_g, f);
  for (size_t ib = 0; ib < L.boxes.size(); ++ib) {
    const Box& B = L.boxes[ib];
    for (int64_t y = B.lo.c[1]; y <= B.hi.c[1]; ++y)
      for (int64_t x = B.lo.c[0]; x <= B.hi.c[0]; ++x)
        f_interior[x + y * L.n[0]] = f.data[ib].at(pt(x, y));
  }
  return 0;
}

/* Exchange a global ghosted array through the per-box storage; the result
 * holds, at every ghost point, the exchanged value of the box owning it
 * (for inter-box points inside Ω, the interior value). */
int orc_exchange(const orc_problem* p, double* glob) {
  Layout L;
  Stencil st;
  if (!build(p, L, st)) return 1;
  Level lev(L);
  scatter_global(glob, lev);
  exchange(lev);
  gather_global(lev, glob);
  return 0;
}

/* Per-box exchange, exported per box for the decomposition pins: writes
 * box ib's full ghosted BoxData (dim-0 fastest over grow(B_ib, g)). */
int orc_exchange_box(const orc_problem* p, const double* glob, int64_t ib, double* out) {
  Layout L;
  Stencil st;
  if (!build(p, L, st)) return 1;
  if (ib < 0 || ib >= (int64_t)L.boxes.size()) {
    g_err = "box index out of range";
    return 2;
  }
  Level lev(L);
  scatter_global(glob, lev);
  exchange(lev);
  const BoxData& bd = lev.data[(size_t)ib];
  std::memcpy(out, bd.v.data(), bd.v.size() * sizeof(double));
  return 0;
}

/* Generic tap stencil apply on one BoxData (Eq.1): src over box
 * [s0,s1]x.., dest box [d0..]; out = scale * Σ α_j src(i+j), dest-box
 * ordered.  Returns 3 on a domain violation (message in orc_last_error). */
int orc_apply_taps(int64_t ntaps, const int64_t* offs, const double* alpha, double scale,
                   const double* src, int64_t s_lo0, int64_t s_lo1, int64_t s_hi0,
                   int64_t s_hi1, int64_t d_lo0, int64_t d_lo1, int64_t d_hi0, int64_t d_hi1,
                   double* out) {
  if (ntaps < 1) {
    g_err = "stencil needs at least one tap";
    return 1;
  }
  Stencil st;
  st.scale = scale;
  st.span = 0;
  for (int64_t t = 0; t < ntaps; ++t) st.taps.push_back({pt(offs[2 * t], offs[2 * t + 1]), alpha[t]});
  BoxData s(mkbox(s_lo0, s_lo1, s_hi0, s_hi1));
  std::memcpy(s.v.data(), src, s.v.size() * sizeof(double));
  Box d = mkbox(d_lo0, d_lo1, d_hi0, d_hi1);
  BoxData o(d);
  if (!stencil_apply(st, s, d, o, scale)) return 3;
  std::memcpy(out, o.v.data(), o.v.size() * sizeof(double));
  return 0;
}

/* The oracle's canonical tap lists (for the pins). */
int64_t orc_stencil_taps(int32_t kind, double h, int64_t* offs, double* alpha, double* scale) {
  Stencil st = (kind == 1) ? mehrstellen9(h) : laplace5(h);
  for (size_t t = 0; t < st.taps.size(); ++t) {
    if (offs) {
      offs[2 * t] = st.taps[t].off.c[0];
      offs[2 * t + 1] = st.taps[t].off.c[1];
    }
    if (alpha) alpha[t] = st.taps[t].alpha;
  }
  if (scale) *scale = st.scale;
  return (int64_t)st.taps.size();
}

/* Box helpers (Fig. ProtoX layout pins). */
int64_t orc_box_ordinal(int64_t lo0, int64_t lo1, int64_t hi0, int64_t hi1, int64_t p0,
                        int64_t p1) {
  Box b = mkbox(lo0, lo1, hi0, hi1);
  if (!b.contains(pt(p0, p1))) return -1;
  return b.ordinal(pt(p0, p1));
}

/* ---- multigrid (readings R-MG1..R-MG6) ---- */
typedef struct {
  int64_t levels, nu1, nu2, nu_coarse, ncycles;
} orc_mg;

/* V-cycles on the problem p (bc PERIODIC or DIRICHLET_CC; n0, n1 divisible
 * by 2^(levels-1)).  phi0 / rho / phi_out as orc_solve; norms[2k], [2k+1] =
 * (max|r|, Σr²) of the finest iterate after k cycles, k = 0..ncycles. */
int orc_mg_solve(const orc_problem* p, const orc_mg* m, const double* phi0, const double* rho,
                 double* phi_out, double* norms, int64_t cap, int64_t* nwritten) {
  if (!p || !m) {
    g_err = "null argument";
    return 1;
  }
  if (m->levels < 1 || m->nu1 < 0 || m->nu2 < 0 || m->nu_coarse < 0 || m->ncycles < 0) {
    g_err = "bad multigrid options";
    return 1;
  }
  if (p->bc == BC_FIXED) {
    g_err = "multigrid needs PERIODIC or DIRICHLET_CC";
    return 1;
  }
  const int64_t div = (int64_t)1 << (m->levels - 1);
  if (p->n0 % div || p->n1 % div) {
    g_err = "n must be divisible by 2^(levels-1)";
    return 1;
  }
  MGOpts o{m->levels, m->nu1, m->nu2, m->nu_coarse, m->ncycles};
  std::vector<MGLevel> lv((size_t)m->levels);
  for (int64_t l = 0; l < m->levels; ++l) {
    MGLevel& M = lv[(size_t)l];
    const int64_t s = (int64_t)1 << l;
    const double h = p->h * (double)s;
    bool ok = (l == 0) ? make_layout(p->n0, p->n1, p->b0, p->b1, p->ghost, p->bc, M.L)
                       : make_layout(p->n0 / s, p->n1 / s, p->n0 / s, p->n1 / s, 1, p->bc, M.L);
    if (!ok) return 1;
    M.st = (p->stencil == 1) ? mehrstellen9(h) : laplace5(h);
    M.lambda = p->lambda * (double)(s * s);
  }
  for (MGLevel& M : lv) {  // after the vector is final: Level keeps &M.L
    M.phi.emplace_back(M.L);
    M.f.emplace_back(M.L);
  }
  orc_problem p0 = *p;
  Layout L0;
  Stencil st0;
  if (!build(&p0, L0, st0)) return 1;
  scatter_global(phi0, lv[0].phi[0]);
  make_rhs(p, lv[0].L, rho, lv[0].f[0]);
  int64_t nw = 0;
  auto record = [&]() {
    double r[2];
    residual(lv[0].st, lv[0].phi[0], lv[0].f[0], r);
    if (nw < cap && norms) {
      norms[2 * nw] = r[0];
      norms[2 * nw + 1] = r[1];
    }
    ++nw;
  };
  record();
  for (int64_t k = 0; k < m->ncycles; ++k) {
    vcycle(lv, 0, o);
    record();
  }
  exchange(lv[0].phi[0]);
  if (phi_out) gather_global(lv[0].phi[0], phi_out);
  if (nwritten) *nwritten = nw;
  return 0;
}

/* Components, for the pins: coarse (n0/2 x n1/2) = −R d of a fine interior
 * array d (n0 x n1); fine (2nc0 x 2nc1 interior) += P e for a coarse
 * interior array e with the boundary rule bc. */
int orc_mg_restrict(int64_t n0, int64_t n1, const double* d, double* coarse) {
  if (n0 % 2 || n1 % 2) {
    g_err = "odd extent";
    return 1;
  }
  MGLevel F, C;
  make_layout(n0, n1, n0, n1, 1, BC_PERIODIC, F.L);
  make_layout(n0 / 2, n1 / 2, n0 / 2, n1 / 2, 1, BC_PERIODIC, C.L);
  /* restrict_defect takes d = scale·S(φ) − f: with φ = 0 and f = −d it is d */
  F.st = laplace5(1.0);
  F.phi.emplace_back(F.L);
  F.f.emplace_back(F.L);
  C.phi.emplace_back(C.L);
  C.f.emplace_back(C.L);
  for (int64_t y = 0; y < n1; ++y)
    for (int64_t x = 0; x < n0; ++x) F.f[0].data[0].at(pt(x, y)) = -d[x + y * n0];
  restrict_defect(F, C);
  for (int64_t y = 0; y < n1 / 2; ++y)
    for (int64_t x = 0; x < n0 / 2; ++x) coarse[x + y * (n0 / 2)] = C.f[0].data[0].at(pt(x, y));
  return 0;
}

int orc_mg_prolong(int64_t nc0, int64_t nc1, int32_t bc, const double* e, double* fine) {
  if (bc == BC_FIXED) {
    g_err = "prolongation needs PERIODIC or DIRICHLET_CC";
    return 1;
  }
  MGLevel F, C;
  make_layout(2 * nc0, 2 * nc1, 2 * nc0, 2 * nc1, 1, bc, F.L);
  make_layout(nc0, nc1, nc0, nc1, 1, bc, C.L);
  F.phi.emplace_back(F.L);
  C.phi.emplace_back(C.L);
  for (int64_t y = 0; y < nc1; ++y)
    for (int64_t x = 0; x < nc0; ++x) C.phi[0].data[0].at(pt(x, y)) = e[x + y * nc0];
  for (int64_t y = 0; y < 2 * nc1; ++y)
    for (int64_t x = 0; x < 2 * nc0; ++x) F.phi[0].data[0].at(pt(x, y)) = fine[x + y * 2 * nc0];
  prolong_correct(C, F);
  for (int64_t y = 0; y < 2 * nc1; ++y)
    for (int64_t x = 0; x < 2 * nc0; ++x) fine[x + y * 2 * nc0] = F.phi[0].data[0].at(pt(x, y));
  return 0;
}

double orc_neumaier_sum(const double* x, int64_t n) {
  Neumaier s;
  for (int64_t i = 0; i < n; ++i) s.add(x[i]);
  return s.value();
}

}  // extern "C"
