/*
 * protox_cpu.cpp -- the paper's own CPU experiment, re-run on this host as
 * CONTEXT.  Not the product (the product is the
 * CUDA library paper_2307_07931_b200/libprotox.so) and not the oracle
 * (oracle/ is the plain reference the GPU path is checked against).
 *
 * PAPER.md:212 / 320-325 (figure `runtime`): Proto (separate abstractions per
 * kernel, figure `Proto`) against ProtoX (the SPIRAL-fused single
 * loop, figure `ProtoX`; OpenMP variant figure `ProtoXomp`,
 * P:244-283) on a periodic 2D Poisson problem, 4 x 4 boxes of 64², 128² and
 * 256² cells, a fixed 100 Jacobi iterations; "ProtoX performs up to 2x faster
 * than the base Proto code" on a 2.3 GHz quad-core i7.  Both variants here use
 * the same data structures (one ghosted array per box, as Proto's BoxData)
 * and the same compiler flags, so the ratio measures the fusion:
 *
 *   variant 0  Proto, unfused: per iteration exchange; per box
 *              temp = laplace(φ, wgt) (pass 1), forallInPlace update
 *              φ += λ(temp − ρ) (pass 2); then computeMaxResidualAcrossProcs
 *              (exchange + pass 3: max|wgt·S(φ) − ρ| of the updated φ).
 *   variant 1  ProtoX, fused (Fig. ProtoX transcribed): per iteration
 *              exchange; per box ONE loop: s20 = φ_c,
 *              s21 = (((φ_S − 4 s20) + φ_W) + φ_E) + φ_N, s22 = ρ,
 *              Y = (s20 + weight1·s21) − λ·s22 with weight1 = λ/h² (R3),
 *              retval = max(retval, |s21/h² − s22|) (the PRE-update residual,
 *              P:233-237, R4); then swap X/Y.
 * threads > 1: OpenMP over (box, row) with a max reduction (Fig. ProtoXomp;
 * its racy shared retval, is replaced by a reduction, R12).
 *
 * Compiled with -O3 -march=native -fopenmp -ffp-contract=off: variant 0 is
 * bit-identical to the oracle (same expression tree); variant 1 uses the
 * figure's tree and is checked against the oracle to rounding
 * (tests/test_hostref_cpu.py).
 */
#include <omp.h>

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

struct Boxes {
  int b, nb, w;                    // box size, boxes per dimension, ghosted width b+2
  std::vector<std::vector<double>> phi, tmp, rho;  // per box: (b+2)^2 ghosted, rho b^2
  double& at(std::vector<double>& v, int x, int y) { return v[(size_t)(x + 1) + (size_t)(y + 1) * w]; }
};

// ghost ring of every box from its periodic neighbours (edges and corners)
void exchange(Boxes& B, std::vector<std::vector<double>>& f) {
  const int b = B.b, nb = B.nb, w = B.w;
  for (int by = 0; by < nb; ++by)
    for (int bx = 0; bx < nb; ++bx) {
      std::vector<double>& d = f[(size_t)(bx + by * nb)];
      auto src = [&](int dx, int dy) -> const std::vector<double>& {
        return f[(size_t)(((bx + dx + nb) % nb) + ((by + dy + nb) % nb) * nb)];
      };
      const std::vector<double>&S = src(0, -1), &N = src(0, 1), &W = src(-1, 0), &E = src(1, 0);
      for (int x = 0; x < b; ++x) {
        d[(size_t)(x + 1)] = S[(size_t)(x + 1) + (size_t)b * w];              // row -1 <- S's row b-1
        d[(size_t)(x + 1) + (size_t)(b + 1) * w] = N[(size_t)(x + 1) + (size_t)w];  // row b <- N's row 0
      }
      for (int y = 0; y < b; ++y) {
        d[(size_t)(y + 1) * w] = W[(size_t)b + (size_t)(y + 1) * w];            // col -1 <- W's col b-1
        d[(size_t)(b + 1) + (size_t)(y + 1) * w] = E[1 + (size_t)(y + 1) * w];  // col b <- E's col 0
      }
      d[0] = src(-1, -1)[(size_t)b + (size_t)b * w];
      d[(size_t)(b + 1)] = src(1, -1)[1 + (size_t)b * w];
      d[(size_t)(b + 1) * w] = src(-1, 1)[(size_t)b + (size_t)w];
      d[(size_t)(b + 1) + (size_t)(b + 1) * w] = src(1, 1)[1 + (size_t)w];
    }
}

inline double lap(const double* c, int w) {  // canonical order W, E, S, N, C(-4) (oracle R10)
  return (((c[-1] + c[1]) + c[-w]) + c[w]) + (-4.0 * c[0]);
}

}  // namespace

extern "C" {

/* Run `iters` iterations of variant 0 (Proto, unfused) or 1 (ProtoX, fused)
 * on nb x nb periodic boxes of b x b cells, φ0 = 0, ρ = rho (n x n, n = nb·b,
 * x fastest).  Writes φ^iters to phi_out (n x n), the seconds of the
 * iteration loop and the max-norm history (iters entries: Proto's post-update
 * residual for variant 0, the fused pre-update residual for variant 1).
 * Returns 0, or 1 on bad arguments. */
int cpu_run(int variant, int b, int nb, int iters, int threads, double h, double lambda, const double* rho,
            double* phi_out, double* seconds, double* maxnorm) {
  if (b < 1 || nb < 1 || iters < 0 || threads < 1 || (variant != 0 && variant != 1)) return 1;
  Boxes B;
  B.b = b;
  B.nb = nb;
  B.w = b + 2;
  const int n = nb * b, w = B.w, nbox = nb * nb;
  B.phi.assign((size_t)nbox, std::vector<double>((size_t)w * w, 0.0));
  B.tmp.assign((size_t)nbox, std::vector<double>((size_t)w * w, 0.0));
  B.rho.assign((size_t)nbox, std::vector<double>((size_t)b * b, 0.0));
  for (int k = 0; k < nbox; ++k) {
    const int bx = k % nb, by = k / nb;
    for (int y = 0; y < b; ++y)
      for (int x = 0; x < b; ++x) B.rho[(size_t)k][(size_t)(x + y * b)] = rho[(size_t)(bx * b + x) + (size_t)(by * b + y) * n];
  }
  const double wgt = 1.0 / (h * h);
  const double weight1 = lambda / (h * h);
  omp_set_num_threads(threads);
  const auto t0 = std::chrono::steady_clock::now();
  for (int it = 0; it < iters; ++it) {
    double m = 0.0;
    if (variant == 0) {
      exchange(B, B.phi);
#pragma omp parallel for collapse(2) schedule(static)
      for (int k = 0; k < nbox; ++k)
        for (int y = 0; y < b; ++y) {
          const double* p = B.phi[(size_t)k].data() + (size_t)(y + 1) * w + 1;
          double* t = B.tmp[(size_t)k].data() + (size_t)(y + 1) * w + 1;
          for (int x = 0; x < b; ++x) t[x] = wgt * lap(p + x, w);  // temp = laplace(phi, wgt)
        }
#pragma omp parallel for collapse(2) schedule(static)
      for (int k = 0; k < nbox; ++k)
        for (int y = 0; y < b; ++y) {
          double* p = B.phi[(size_t)k].data() + (size_t)(y + 1) * w + 1;
          const double* t = B.tmp[(size_t)k].data() + (size_t)(y + 1) * w + 1;
          const double* f = B.rho[(size_t)k].data() + (size_t)y * b;
          for (int x = 0; x < b; ++x) p[x] = p[x] + lambda * (t[x] - f[x]);  // forallInPlace
        }
      exchange(B, B.phi);  // computeMaxResidualAcrossProcs
#pragma omp parallel for collapse(2) schedule(static) reduction(max : m)
      for (int k = 0; k < nbox; ++k)
        for (int y = 0; y < b; ++y) {
          const double* p = B.phi[(size_t)k].data() + (size_t)(y + 1) * w + 1;
          const double* f = B.rho[(size_t)k].data() + (size_t)y * b;
          for (int x = 0; x < b; ++x) {
            const double r = std::fabs(wgt * lap(p + x, w) - f[x]);
            m = r > m ? r : m;
          }
        }
    } else {
      exchange(B, B.phi);
#pragma omp parallel for collapse(2) schedule(static) reduction(max : m)
      for (int k = 0; k < nbox; ++k)
        for (int y = 0; y < b; ++y) {
          const double* X = B.phi[(size_t)k].data() + (size_t)(y + 1) * w + 1;
          double* Y = B.tmp[(size_t)k].data() + (size_t)(y + 1) * w + 1;
          const double* f = B.rho[(size_t)k].data() + (size_t)y * b;
          for (int x = 0; x < b; ++x) {
            const double s20 = X[x];
            const double s21 = (((X[x - w] - 4.0 * s20) + X[x - 1]) + X[x + 1]) + X[x + w];
            const double s22 = f[x];
            Y[x] = (s20 + weight1 * s21) - lambda * s22;
            const double r = std::fabs((1.0 / (h * h)) * s21 - s22);
            m = m >= r ? m : r;
          }
        }
      std::swap(B.phi, B.tmp);
    }
    if (maxnorm) maxnorm[it] = m;
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  for (int k = 0; k < nbox; ++k) {
    const int bx = k % nb, by = k / nb;
    for (int y = 0; y < b; ++y)
      for (int x = 0; x < b; ++x)
        phi_out[(size_t)(bx * b + x) + (size_t)(by * b + y) * n] = B.phi[(size_t)k][(size_t)(x + 1) + (size_t)(y + 1) * w];
  }
  return 0;
}

}  // extern "C"
