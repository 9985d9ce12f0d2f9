// Seeded synthetic input generator: FIM compositional Jacobians with the block
// structure of PAPER.md Eq. 17/18 on a 7-point TPFA grid (Eq. 13,
// P:150-155), as specified in SURVEY.md §8(d).
//
// This module is shared by the oracle side and the CUDA side ONLY as an input
// source.  It holds none of the method's arithmetic (no decoupling, coloring,
// aggregation, smoothing, Krylov).  The only linear-algebra it does is the
// manufactured right-hand side b = A x* (SURVEY §8(d) "RHS"), which is input
// generation, not a step of the solve path.
//
// Layout of the output (the C-ABI input layout of include/msp.h):
//   cells are numbered c = i + nx*(j + ny*k)  (x fastest, z slowest, so a
//   z-slab is a contiguous cell range); block size b = nc+1, unknown 0 is the
//   pressure P and unknowns 1..nc are N_1..N_nc (Eq. 20 order);
//   BSR row_ptr[n+1], col[nnzb] ascending per row, val[nnzb*b*b] with each
//   b x b block stored ROW-major.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>

namespace {

struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed, uint64_t tag) {
    s = seed * 0xD1342543DE82EF95ull + tag * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  }
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }   // [0,1)
  double uniform(double a, double b) { return a + (b - a) * uniform(); }
  double normal() {                                                  // Box-Muller
    double u1 = 1.0 - uniform();                                     // (0,1]
    double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
};

// stream tags (one independent stream per purpose)
enum : uint64_t { T_FIELD = 1, T_CHAN = 2, T_COEF = 3, T_POT = 4, T_XSTAR = 5, T_DRIFT = 100 };

}  // namespace

extern "C" {

typedef struct {
  int32_t nx, ny, nz, nc;
  double dx, dy, dz;
  int32_t perm_kind;   // 0 homogeneous kappa=1, 1 log-normal ln k = sigma*G, 2 SPE10-like channelized
  double sigma;        // for perm_kind 1
  double acc;          // accumulation ratio ACC; dt = 1/(ACC*mean_c sum_s T_s)
  uint64_t seed;
  int32_t newton_step; // 0: base Jacobian; iota>=1: coefficients drifted iota times (C4 sequence)
  double drift;        // relative drift magnitude per step (default 1e-2)
  int32_t kz_ratio_x10;// kappa_z = (kz_ratio_x10/10)*kappa_x ; 10 = isotropic
} gen_params;

int64_t gen_nnzb(int32_t nx, int32_t ny, int32_t nz) {
  int64_t n = (int64_t)nx * ny * nz;
  int64_t faces = (int64_t)(nx - 1) * ny * nz + (int64_t)nx * (ny - 1) * nz + (int64_t)nx * ny * (nz - 1);
  return n + 2 * faces;
}

// Correlated standard Gaussian field: iid N(0,1), two passes of a box filter
// (3x3x3, or 3x3x1 in layers with flat2d[k] != 0), renormalised to mean 0, var 1.
static void gaussian_field(int nx, int ny, int nz, SplitMix64& rng, const std::vector<char>& flat2d,
                           std::vector<double>& g) {
  const int64_t n = (int64_t)nx * ny * nz;
  g.resize(n);
  for (int64_t c = 0; c < n; ++c) g[c] = rng.normal();
  std::vector<double> t(n);
  for (int pass = 0; pass < 2; ++pass) {
    for (int k = 0; k < nz; ++k)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
          double s = 0.0;
          int cnt = 0;
          int kr = flat2d[k] ? 0 : 1;
          for (int dk = -kr; dk <= kr; ++dk) {
            int kk = k + dk;
            if (kk < 0 || kk >= nz || flat2d[kk] != flat2d[k]) continue;
            for (int dj = -1; dj <= 1; ++dj) {
              int jj = j + dj;
              if (jj < 0 || jj >= ny) continue;
              for (int di = -1; di <= 1; ++di) {
                int ii = i + di;
                if (ii < 0 || ii >= nx) continue;
                s += g[ii + (int64_t)nx * (jj + (int64_t)ny * kk)];
                ++cnt;
              }
            }
          }
          t[i + (int64_t)nx * (j + (int64_t)ny * k)] = s / cnt;
        }
    g.swap(t);
  }
  double mean = 0.0, var = 0.0;
  for (int64_t c = 0; c < n; ++c) mean += g[c];
  mean /= (double)n;
  for (int64_t c = 0; c < n; ++c) var += (g[c] - mean) * (g[c] - mean);
  var /= (double)n;
  double sd = var > 0 ? std::sqrt(var) : 1.0;
  for (int64_t c = 0; c < n; ++c) g[c] = (g[c] - mean) / sd;
}

// Fills kappa_x (horizontal) per cell.
static void permeability(const gen_params* p, std::vector<double>& kx) {
  const int nx = p->nx, ny = p->ny, nz = p->nz;
  const int64_t n = (int64_t)nx * ny * nz;
  kx.assign(n, 1.0);
  if (p->perm_kind == 0) return;
  SplitMix64 rng(p->seed, T_FIELD);
  if (p->perm_kind == 1) {
    std::vector<char> flat(nz, 0);
    std::vector<double> g;
    gaussian_field(nx, ny, nz, rng, flat, g);
    for (int64_t c = 0; c < n; ++c) kx[c] = std::exp(p->sigma * g[c]);
    return;
  }
  // SPE10-like: upper Tarbert-like layers (35 of 85), lower Ness-like layers
  // with sinusoidal high-permeability channels along y.
  int ntar = (int)std::lround(nz * 35.0 / 85.0);
  if (ntar < 1) ntar = 1;
  std::vector<char> flat(nz, 0);
  for (int k = ntar; k < nz; ++k) flat[k] = 1;
  std::vector<double> g;
  gaussian_field(nx, ny, nz, rng, flat, g);
  SplitMix64 ch(p->seed, T_CHAN);
  for (int k = 0; k < nz; ++k) {
    if (k < ntar) {
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
          int64_t c = i + (int64_t)nx * (j + (int64_t)ny * k);
          kx[c] = std::pow(10.0, 1.0 + g[c]);
        }
      continue;
    }
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int64_t c = i + (int64_t)nx * (j + (int64_t)ny * k);
        kx[c] = std::pow(10.0, -1.0 + 0.5 * g[c]);
      }
    for (int q = 0; q < 6; ++q) {
      double x0 = ch.uniform(0.0, (double)nx);
      double amp = ch.uniform(5.0, 15.0);
      double lam = ch.uniform(60.0, 200.0);
      double th = ch.uniform(0.0, 6.283185307179586);
      double wid = ch.uniform(2.0, 6.0);
      for (int j = 0; j < ny; ++j) {
        double xc = x0 + amp * std::sin(6.283185307179586 * j / lam + th);
        for (int i = 0; i < nx; ++i) {
          if (std::fabs(i + 0.5 - xc) <= 0.5 * wid) {
            int64_t c = i + (int64_t)nx * (j + (int64_t)ny * k);
            kx[c] = std::pow(10.0, 3.0 + 0.3 * ch.normal());
          }
        }
      }
    }
  }
}

// Main generator.  alpha_out (optional): n*(nc+1) doubles [alpha_P, alpha_1..alpha_nc]
// per cell, exported for the decoupling closed-form pin.
int gen_jacobian(const gen_params* p, int32_t* row_ptr, int32_t* col, double* val, double* xstar,
                 double* rhs, double* alpha_out, double* dt_out) {
  const int nx = p->nx, ny = p->ny, nz = p->nz, nc = p->nc, b = nc + 1;
  if (nx < 1 || ny < 1 || nz < 1 || nc < 0) return 1;
  const int64_t n = (int64_t)nx * ny * nz;
  const int64_t bb = (int64_t)b * b;

  std::vector<double> kx;
  permeability(p, kx);
  const double kzr = p->kz_ratio_x10 / 10.0;

  // per-cell coefficients of the Eq. 17/18 rows
  std::vector<double> aP(n), al((size_t)n * nc), lam((size_t)n * nc), gam((size_t)n * nc * nc);
  {
    SplitMix64 r(p->seed, T_COEF);
    for (int64_t c = 0; c < n; ++c) {
      aP[c] = r.uniform(0.5, 1.5);
      for (int i = 0; i < nc; ++i) al[c * nc + i] = r.uniform(0.5, 1.5);
      for (int i = 0; i < nc; ++i) lam[c * nc + i] = r.uniform(0.2, 1.0);
      for (int i = 0; i < nc; ++i)
        for (int k = 0; k < nc; ++k)
          gam[(c * nc + i) * nc + k] = (i == k) ? r.uniform(0.5, 1.0) : r.uniform(0.0, 0.1);
    }
  }
  // Newton-sequence drift: coefficients multiplied by (1 + drift*U(-1,1)) per
  // cell per step, then the Jacobian is re-assembled (keeps conservation).
  for (int st = 1; st <= p->newton_step; ++st) {
    SplitMix64 r(p->seed, T_DRIFT + (uint64_t)(40 + st));
    const double d = p->drift;
    for (int64_t c = 0; c < n; ++c) {
      aP[c] *= 1.0 + d * r.uniform(-1.0, 1.0);
      for (int i = 0; i < nc; ++i) al[c * nc + i] *= 1.0 + d * r.uniform(-1.0, 1.0);
      for (int i = 0; i < nc; ++i) lam[c * nc + i] *= 1.0 + d * r.uniform(-1.0, 1.0);
      for (int i = 0; i < nc * nc; ++i) gam[c * nc * nc + i] *= 1.0 + d * r.uniform(-1.0, 1.0);
    }
  }
  // potential for upstream weighting ("upstream weighted value")
  std::vector<double> phi(n);
  {
    SplitMix64 r(p->seed, T_POT);
    for (int k = 0; k < nz; ++k)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
          int64_t c = i + (int64_t)nx * (j + (int64_t)ny * k);
          phi[c] = (double)i + 0.1 * r.normal();
        }
  }
  // transmissibility T_s = L*kappa_harm/d (Eq. 13)
  auto harm = [](double a, double c) { return 2.0 * a * c / (a + c); };
  auto trans = [&](int64_t c, int64_t d, int dir) -> double {
    double L, dist, k1 = kx[c], k2 = kx[d];
    if (dir == 0) { L = p->dy * p->dz; dist = p->dx; }
    else if (dir == 1) { L = p->dx * p->dz; dist = p->dy; }
    else { L = p->dx * p->dy; dist = p->dz; k1 *= kzr; k2 *= kzr; }
    return L * harm(k1, k2) / dist;
  };
  // dt from ACC
  double tsum = 0.0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        int64_t c = i + (int64_t)nx * (j + (int64_t)ny * k);
        if (i + 1 < nx) tsum += 2.0 * trans(c, c + 1, 0);
        if (j + 1 < ny) tsum += 2.0 * trans(c, c + nx, 1);
        if (k + 1 < nz) tsum += 2.0 * trans(c, c + (int64_t)nx * ny, 2);
      }
  const double dt = (tsum > 0.0) ? 1.0 / (p->acc * (tsum / (double)n)) : 1.0;  // no faces: dt = 1
  if (dt_out) *dt_out = dt;

  // assemble
  int64_t pos = 0;
  row_ptr[0] = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int64_t c = i + (int64_t)nx * (j + (int64_t)ny * k);
        int64_t nb[6];
        int dirs[6];
        int cnt = 0;
        if (k > 0) { nb[cnt] = c - (int64_t)nx * ny; dirs[cnt++] = 2; }
        if (j > 0) { nb[cnt] = c - nx; dirs[cnt++] = 1; }
        if (i > 0) { nb[cnt] = c - 1; dirs[cnt++] = 0; }
        int before = cnt;
        if (i + 1 < nx) { nb[cnt] = c + 1; dirs[cnt++] = 0; }
        if (j + 1 < ny) { nb[cnt] = c + nx; dirs[cnt++] = 1; }
        if (k + 1 < nz) { nb[cnt] = c + (int64_t)nx * ny; dirs[cnt++] = 2; }
        int64_t diagpos = pos + before;
        // column indices ascending: lower neighbours, diagonal, upper neighbours
        int64_t q = pos;
        for (int t = 0; t < before; ++t) col[q++] = (int32_t)nb[t];
        col[q++] = (int32_t)c;
        for (int t = before; t < cnt; ++t) col[q++] = (int32_t)nb[t];
        for (int64_t e = pos; e < q; ++e) std::memset(val + e * bb, 0, sizeof(double) * bb);
        double* D = val + diagpos * bb;
        // diagonal block row 0: [alpha_P/dt, -alpha_i/dt]   (Eq. 17)
        D[0] = aP[c] / dt;
        for (int ii = 0; ii < nc; ++ii) D[1 + ii] = -al[c * nc + ii] / dt;
        // accumulation of N rows (Eq. 18): delta_ik/dt
        for (int ii = 0; ii < nc; ++ii) D[(1 + ii) * b + (1 + ii)] += 1.0 / dt;
        for (int t = 0; t < cnt; ++t) {
          const int64_t d = nb[t];
          const double T = trans(c, d, dirs[t]);
          const int64_t up = (phi[c] > phi[d] || (phi[c] == phi[d] && c < d)) ? c : d;  // upstream u(s)
          int64_t e = (t < before) ? pos + t : pos + t + 1;
          double* O = val + e * bb;
          for (int ii = 0; ii < nc; ++ii) {
            const double tl = T * lam[up * nc + ii];
            D[(1 + ii) * b + 0] += tl;            // row i, col 0 of diagonal block
            O[(1 + ii) * b + 0] = -tl;            // row i, col 0 of off-diagonal block
            for (int kk = 0; kk < nc; ++kk) {
              const double tg = T * gam[(up * nc + ii) * nc + kk];
              if (up == c) D[(1 + ii) * b + (1 + kk)] += tg;
              else O[(1 + ii) * b + (1 + kk)] = -tg;
            }
          }
        }
        pos = q;
        row_ptr[c + 1] = (int32_t)pos;
      }
  // manufactured solution and RHS
  {
    SplitMix64 r(p->seed, T_XSTAR);
    for (int64_t t = 0; t < n * b; ++t) xstar[t] = r.uniform(-1.0, 1.0);
  }
  for (int64_t c = 0; c < n; ++c) {
    for (int ii = 0; ii < b; ++ii) {
      double s = 0.0;
      for (int64_t e = row_ptr[c]; e < row_ptr[c + 1]; ++e) {
        const double* B = val + e * bb;
        const int64_t d = col[e];
        for (int kk = 0; kk < b; ++kk) s += B[ii * b + kk] * xstar[d * b + kk];
      }
      rhs[c * b + ii] = s;
    }
  }
  if (alpha_out) {
    for (int64_t c = 0; c < n; ++c) {
      alpha_out[c * b] = aP[c];
      for (int ii = 0; ii < nc; ++ii) alpha_out[c * b + 1 + ii] = al[c * nc + ii];
    }
  }
  return 0;
}

}  // extern "C"
