/*
 * fv2d_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of the first-order
 * finite-volume scheme of Essadki, Jung, Larat, Pelletier & Perrier,
 * "A task-driven implementation of a simple numerical solver for hyperbolic
 * conservation laws" (arXiv:1701.05431).  It is the parity oracle for the
 * CUDA library (paper_1701_05431_b200/csrc): only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares
 * no code, header, table or constant with the CUDA path.
 *
 * Citations: "P:L" = /root/reference/PAPER.md line L, "S:L" = SPEC.md line L,
 * "R<n>" = the reading numbered n in DESIGN.md §3 (taken from SURVEY.md §8c).
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC
 *        (every + - * / sqrt is a separately rounded IEEE binary64 op, so the
 *        result is the "canonical evaluation order" (CEO) of DESIGN.md §3.1.)
 *
 * Layout: the paper's Cell array-of-structures, W[(j*nx + i)*nvar + v],
 * x fastest, variable innermost (R11).
 *
 * Parity status per function (pins live in tests/test_oracle_*.py):
 *   or_phys_flux / or_lf_flux   pinned (consistency, A1 values, upwind special case)
 *   or_transport_step           pinned (3x3 exact, 3x3 50-digit, CFL=1 translation,
 *                               conservation, constant state, mirror symmetry)
 *   or_smax                     pinned (brute-force max on known states, bell s=2)
 *   or_reconstruct              pinned (uniform NDF, closed-form lambda=(0,1,0,0))
 *   or_source_step              pinned (uniform NDF closed form, drag-only ODE)
 *   or_gl24                     pinned (polynomial exactness to degree 47)
 *   or_spray_guard              pinned (closed-form boundary dt = 0.1*min(m3/m1)/K)
 *   ghosts (get_state)          pinned (Dirichlet: exact rationals, 50-digit,
 *                               constant-state; wall: closed forms, 50-digit,
 *                               conservation) -- tests/test_oracle_boundaries.py
 *   spray phys_flux / speed     pinned (uniform velocity == per-moment upwind
 *                               bitwise; 50-digit primitive-notation step)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Status codes (same numbers as the library's, defined independently). */
enum { OR_OK = 0, OR_E_ARG = 1, OR_E_CFL = 2, OR_E_NONFINITE = 3, OR_E_RECON = 4 };
enum { OR_ADVECTION = 0, OR_EULER = 1, OR_SPRAY = 2 };
enum { OR_BC_PERIODIC = 0, OR_BC_DIRICHLET = 1, OR_BC_WALL = 2 };

typedef struct {
  int32_t nx, ny, nvar, system;
  int32_t bc_x, bc_y;
  double x0, x1, y0, y1;
  double param[8];     /* advection: ax, ay | euler: gamma | spray: K, theta */
  double dirichlet[6]; /* constant ghost state for FV2D_BC_DIRICHLET */
} or_cfg;

typedef struct {
  int32_t code;        /* OR_* */
  int64_t cell;        /* j*nx+i of the offending cell, -1 if none */
  double value;        /* offending speed / moment residual */
} or_err;

static int nvar_of(int system) {
  return system == OR_ADVECTION ? 1 : system == OR_EULER ? 4 : system == OR_SPRAY ? 6 : -1;
}

static double dmax(double a, double b) { return a > b ? a : b; }

/* ------------------------------------------------------------------------ */
/* Gauss-Legendre, 24 nodes, mapped to [0,1] ("fixed-order
 * Gauss-Legendre quadrature (order 24) in the variable t = sqrt(S)").
 * Nodes by Newton's method on the three-term recurrence of P_24.          */
static double gl_t[24], gl_w[24];
static int gl_ready = 0;

static void gl_init(void) {
  const int n = 24;
  for (int k = 0; k < n; ++k) {
    double x = cos(M_PI * (k + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int l = 2; l <= n; ++l) {
        double p2 = ((2.0 * l - 1.0) * x * p1 - (l - 1.0) * p0) / l;
        p0 = p1; p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      double dx = p1 / dp;
      x -= dx;
      if (fabs(dx) < 1e-17) break;
    }
    {
      double p0 = 1.0, p1 = x;
      for (int l = 2; l <= n; ++l) {
        double p2 = ((2.0 * l - 1.0) * x * p1 - (l - 1.0) * p0) / l;
        p0 = p1; p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
    }
    double w = 2.0 / ((1.0 - x * x) * dp * dp);
    /* ascending order on [0,1]: x decreasing in k, so store at n-1-k */
    gl_t[n - 1 - k] = (x + 1.0) / 2.0;
    gl_w[n - 1 - k] = w / 2.0;
  }
  gl_ready = 1;
}

void or_gl24(double* t, double* w) {
  if (!gl_ready) gl_init();
  for (int q = 0; q < 24; ++q) { t[q] = gl_t[q]; w[q] = gl_w[q]; }
}

/* ------------------------------------------------------------------------ */
/* Physical flux F(W).n and directional spectral radius max_p |lambda_p(W,n)|
 * for an axis normal n = e_x (dir 0) or e_y (dir 1) (R2).
 * Returns 0 if the state is admissible, OR_E_NONFINITE otherwise.          */
int or_phys_flux(const or_cfg* c, const double* W, int dir, double* F, double* s) {
  if (c->system == OR_ADVECTION) {
    /* F = (a_x u, a_y u); lambda = a.n  (BASELINE.json configs[0]) */
    double a = dir == 0 ? c->param[0] : c->param[1];
    F[0] = a * W[0];
    *s = fabs(a);
    return isfinite(F[0]) ? OR_OK : OR_E_NONFINITE;
  }
  if (c->system == OR_EULER) {
    /* eq:Euler, conserved E := rho*E (R7), gm1 = fl(gamma-1) (R8) */
    const double gamma = c->param[0];
    const double gm1 = gamma - 1.0;
    const double rho = W[0], mx = W[1], my = W[2], E = W[3];
    const double inv = 1.0 / rho;
    const double u = mx * inv;
    const double v = my * inv;
    const double ke = 0.5 * ((mx * u) + (my * v));
    const double p = gm1 * (E - ke);
    const double cs = sqrt((gamma * p) * inv);
    if (dir == 0) {
      F[0] = mx;                 /* rho u.n with the conserved momentum (R9) */
      F[1] = (mx * u) + p;       /* rho u u.n + p n_x */
      F[2] = my * u;             /* rho v u.n */
      F[3] = (E + p) * u;        /* rho u.n H, H = E + p/rho */
      *s = fabs(u) + cs;         /* max(|u.n - c|, |u.n|, |u.n + c|) */
    } else {
      F[0] = my;
      F[1] = mx * v;
      F[2] = (my * v) + p;
      F[3] = (E + p) * v;
      *s = fabs(v) + cs;
    }
    if (!(rho > 0.0) || !(p > 0.0) || !isfinite(*s)) return OR_E_NONFINITE;
    for (int k = 0; k < 4; ++k) if (!isfinite(F[k])) return OR_E_NONFINITE;
    return OR_OK;
  }
  if (c->system == OR_SPRAY) {
    /* eq:Essadki left-hand side: pressureless transport at u = m2u/m2 */
    const double m0 = W[0], m1 = W[1], m2 = W[2], m3 = W[3], m2u = W[4], m2v = W[5];
    const double inv = 1.0 / m2;
    const double u = m2u * inv;
    const double v = m2v * inv;
    if (dir == 0) {
      F[0] = m0 * u; F[1] = m1 * u; F[2] = m2u; F[3] = m3 * u;
      F[4] = m2u * u; F[5] = m2v * u;
      *s = fabs(u);
    } else {
      F[0] = m0 * v; F[1] = m1 * v; F[2] = m2v; F[3] = m3 * v;
      F[4] = m2u * v; F[5] = m2v * v;
      *s = fabs(v);
    }
    if (!(m2 > 0.0) || !isfinite(*s)) return OR_E_NONFINITE;
    for (int k = 0; k < 6; ++k) if (!isfinite(F[k])) return OR_E_NONFINITE;
    return OR_OK;
  }
  return OR_E_ARG;
}

/* Lax-Friedrichs flux:
 *   F~(L,R,n) = (F(L).n + F(R).n)/2 - sigma/2 (R - L),
 *   sigma = max_p max(|lambda_p(L)|, |lambda_p(R)|)   (R2: directional).
 * CEO: hs = 0.5*max(sL,sR); F_k = (0.5*(FL_k+FR_k)) - (hs*(R_k-L_k)).      */
int or_lf_flux(const or_cfg* c, const double* L, const double* R, int dir, double* F) {
  double FL[6], FR[6], sL, sR;
  int e1 = or_phys_flux(c, L, dir, FL, &sL);
  int e2 = or_phys_flux(c, R, dir, FR, &sR);
  const double hs = 0.5 * dmax(sL, sR);
  for (int k = 0; k < c->nvar; ++k)
    F[k] = (0.5 * (FL[k] + FR[k])) - (hs * (R[k] - L[k]));
  return e1 ? e1 : e2;
}

/* ------------------------------------------------------------------------ */
/* Ghost states (R13).  Periodic: wrap.  Dirichlet: constant state.
 * Wall: mirror of the adjacent interior cell with the normal momentum negated
 * (Euler: index 1 for x, 2 for y; spray: 4 for x, 5 for y).                 */
static void get_state(const or_cfg* c, const double* W, int i, int j, double* out) {
  const int nx = c->nx, ny = c->ny, nv = c->nvar;
  int ii = i, jj = j;
  int mirror_dir = -1;
  if (i < 0 || i >= nx) {
    if (c->bc_x == OR_BC_PERIODIC) ii = ((i % nx) + nx) % nx;
    else if (c->bc_x == OR_BC_DIRICHLET) { for (int k = 0; k < nv; ++k) out[k] = c->dirichlet[k]; return; }
    else { ii = i < 0 ? 0 : nx - 1; mirror_dir = 0; }
  }
  if (j < 0 || j >= ny) {
    if (c->bc_y == OR_BC_PERIODIC) jj = ((j % ny) + ny) % ny;
    else if (c->bc_y == OR_BC_DIRICHLET) { for (int k = 0; k < nv; ++k) out[k] = c->dirichlet[k]; return; }
    else { jj = j < 0 ? 0 : ny - 1; mirror_dir = 1; }
  }
  const double* src = W + ((size_t)jj * nx + ii) * nv;
  for (int k = 0; k < nv; ++k) out[k] = src[k];
  if (mirror_dir >= 0) {
    if (c->system == OR_EULER) out[1 + mirror_dir] = -out[1 + mirror_dir];
    else if (c->system == OR_SPRAY) out[4 + mirror_dir] = -out[4 + mirror_dir];
  }
}

/* ------------------------------------------------------------------------ */
/* CFL reduction (eq:CFL_cond; R3): smax = max_ij max(s_x, s_y);
 * argmax = lowest j*nx+i among maxima.                                      */
int or_smax(const or_cfg* c, const double* W, double* smax, int64_t* argmax, or_err* err) {
  double best = -1.0;
  int64_t arg = -1;
  double F[6], sx, sy;
  for (int j = 0; j < c->ny; ++j)
    for (int i = 0; i < c->nx; ++i) {
      const double* w = W + ((size_t)j * c->nx + i) * c->nvar;
      int e1 = or_phys_flux(c, w, 0, F, &sx);
      int e2 = or_phys_flux(c, w, 1, F, &sy);
      if (e1 || e2) {
        if (err) { err->code = OR_E_NONFINITE; err->cell = (int64_t)j * c->nx + i; err->value = w[0]; }
        return OR_E_NONFINITE;
      }
      const double s = dmax(sx, sy);
      if (s > best) { best = s; arg = (int64_t)j * c->nx + i; }
    }
  *smax = best;
  if (argmax) *argmax = arg;
  return OR_OK;
}

/* Per-cell directional speeds (for tests and diagnostics). */
int or_speeds(const or_cfg* c, const double* W, double* sx, double* sy) {
  double F[6];
  for (size_t n = 0; n < (size_t)c->nx * c->ny; ++n) {
    int e1 = or_phys_flux(c, W + n * c->nvar, 0, F, &sx[n]);
    int e2 = or_phys_flux(c, W + n * c->nvar, 1, F, &sy[n]);
    if (e1 || e2) return OR_E_NONFINITE;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Transport step, eq:VF_scheme with the minus sign (R1):
 *   W* = W - dt/dx (F~(W_ij,W_i+1j,x) - F~(W_i-1j,W_ij,x))
 *          - dt/dy (F~(W_ij,W_ij+1,y) - F~(W_ij-1,W_ij,y)).
 * CEO: W*_k = W_k + (-((lx*(Fe_k-Fw_k)) + (ly*(Fn_k-Fs_k)))), lx = dt/dx.
 * Each face flux is (re)computed per cell -- "face twice", which gives the
 * same bits as "face once" since a face's value depends only on (L,R,dir). */
int or_transport_step(const or_cfg* c, const double* W, double* Wout, double dt, or_err* err) {
  const int nx = c->nx, ny = c->ny, nv = c->nvar;
  const double dx = (c->x1 - c->x0) / nx;
  const double dy = (c->y1 - c->y0) / ny;
  const double lx = dt / dx;
  const double ly = dt / dy;
  double C[6], E[6], Wn[6], N[6], S[6];
  double Fe[6], Fw[6], Fn[6], Fs[6];
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      get_state(c, W, i, j, C);
      get_state(c, W, i + 1, j, E);
      get_state(c, W, i - 1, j, Wn);
      get_state(c, W, i, j + 1, N);
      get_state(c, W, i, j - 1, S);
      int e = 0;
      e |= or_lf_flux(c, C, E, 0, Fe);
      e |= or_lf_flux(c, Wn, C, 0, Fw);
      e |= or_lf_flux(c, C, N, 1, Fn);
      e |= or_lf_flux(c, S, C, 1, Fs);
      if (e) {
        if (err) { err->code = OR_E_NONFINITE; err->cell = (int64_t)j * nx + i; err->value = C[0]; }
        return OR_E_NONFINITE;
      }
      double* out = Wout + ((size_t)j * nx + i) * nv;
      for (int k = 0; k < nv; ++k)
        out[k] = C[k] + (-((lx * (Fe[k] - Fw[k])) + (ly * (Fn[k] - Fs[k]))));
    }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Spray NDF reconstruction ("entropy maximization procedure";
 * concrete algorithm, R19):
 *   n(S) = exp(-(l0 + l1 S^1/2 + l2 S + l3 S^3/2)), t = sqrt(S), P(t) = l0+t(l1+t(l2+t l3))
 *   mu_j = 2 sum_q w_q t_q^j exp(-P(t_q)), j = 0..7;  m_k = mu_{k+1}, m_-1/2 = mu_0
 *   Newton on mu_{k+1}(l) = m_k with J_kl = -mu_{k+l+1}; init l = (-ln m0,0,0,0);
 *   backtracking alpha in {1, 1/2, ..., 2^-30} until the max relative residual
 *   decreases; stop at residual <= 1e-10 (<= 50 iterations), then ONE undamped
 *   polishing Newton step (R19).  Returns n(0) = exp(-l0) and m_-1/2.        */
static void moments8(const double* lam, double* mu) {
  if (!gl_ready) gl_init();
  for (int k = 0; k < 8; ++k) mu[k] = 0.0;
  for (int q = 0; q < 24; ++q) {
    const double t = gl_t[q];
    const double P = lam[0] + t * (lam[1] + t * (lam[2] + t * lam[3]));
    const double e = exp(-P);
    double tp = 1.0; /* t^k */
    for (int k = 0; k < 8; ++k) {
      mu[k] = mu[k] + (gl_w[q] * tp) * e;
      tp = tp * t;
    }
  }
  for (int k = 0; k < 8; ++k) mu[k] = 2.0 * mu[k];
}

static double max_rel_residual(const double* mu, const double* m) {
  double r = 0.0;
  for (int k = 0; k < 4; ++k) {
    const double rk = fabs(mu[k + 1] - m[k]) / m[k];
    if (!(rk <= r)) r = rk; /* NaN-propagating max */
  }
  return r;
}

/* Solve H d = r with H_kl = mu_{k+l+1} (symmetric positive definite Hankel
 * matrix of the positive measure) by an unpivoted Cholesky factorisation.  */
static int hankel_solve(const double* mu, const double* r, double* d) {
  double A[4][4], L[4][4], y[4];
  for (int k = 0; k < 4; ++k)
    for (int l = 0; l < 4; ++l) { A[k][l] = mu[k + l + 1]; L[k][l] = 0.0; }
  for (int k = 0; k < 4; ++k) {
    double s = A[k][k];
    for (int p = 0; p < k; ++p) s = s - L[k][p] * L[k][p];
    if (!(s > 0.0)) return -1;
    L[k][k] = sqrt(s);
    for (int l = k + 1; l < 4; ++l) {
      double t = A[l][k];
      for (int p = 0; p < k; ++p) t = t - L[l][p] * L[k][p];
      L[l][k] = t / L[k][k];
    }
  }
  for (int k = 0; k < 4; ++k) {
    double s = r[k];
    for (int p = 0; p < k; ++p) s = s - L[k][p] * y[p];
    y[k] = s / L[k][k];
  }
  for (int k = 3; k >= 0; --k) {
    double s = y[k];
    for (int p = k + 1; p < 4; ++p) s = s - L[p][k] * d[p];
    d[k] = s / L[k][k];
  }
  return 0;
}

int or_reconstruct(const double* m, double* lam, double* n0, double* mmh, int32_t* iters) {
  double mu[8], mut[8], lt[4], r[4], d[4];
  for (int k = 0; k < 4; ++k)
    if (!(m[k] > 0.0) || !isfinite(m[k])) return OR_E_RECON;
  lam[0] = -log(m[0]); lam[1] = 0.0; lam[2] = 0.0; lam[3] = 0.0;
  moments8(lam, mu);
  double res = max_rel_residual(mu, m);
  int it = 0;
  while (!(res <= 1e-10)) {
    if (it >= 50 || !isfinite(res)) { if (iters) *iters = it; return OR_E_RECON; }
    for (int k = 0; k < 4; ++k) r[k] = mu[k + 1] - m[k];
    if (hankel_solve(mu, r, d)) { if (iters) *iters = it; return OR_E_RECON; }
    double alpha = 1.0;
    int accepted = 0;
    for (int b = 0; b <= 30; ++b) {
      for (int k = 0; k < 4; ++k) lt[k] = lam[k] + alpha * d[k];
      moments8(lt, mut);
      const double rt = max_rel_residual(mut, m);
      if (rt < res) {
        for (int k = 0; k < 4; ++k) lam[k] = lt[k];
        for (int k = 0; k < 8; ++k) mu[k] = mut[k];
        res = rt;
        accepted = 1;
        break;
      }
      alpha = 0.5 * alpha;
    }
    ++it;
    if (!accepted) { if (iters) *iters = it; return OR_E_RECON; }
  }
  /* one undamped polishing Newton step (R19) */
  for (int k = 0; k < 4; ++k) r[k] = mu[k + 1] - m[k];
  if (hankel_solve(mu, r, d)) { if (iters) *iters = it; return OR_E_RECON; }
  for (int k = 0; k < 4; ++k) lam[k] = lam[k] + d[k];
  moments8(lam, mu);
  *n0 = exp(-lam[0]);
  *mmh = mu[0];
  if (iters) *iters = it;
  if (!isfinite(*n0) || !isfinite(*mmh)) return OR_E_RECON;
  return OR_OK;
}

/* Taylor-Green gas velocity (P:1016 names it; S:421-429 fixes the form, R20). */
static void taylor_green(double x, double y, double* ugx, double* ugy) {
  const double tp = 2.0 * M_PI;
  *ugx = sin(tp * x) * cos(tp * y);
  *ugy = -(cos(tp * x) * sin(tp * y));
}

/* Spray source by first-order splitting, eq:SourceTerm:
 *   W^{n+1} = W* + dt S(W*), with S from eq:Essadki:
 *   S = (-K n0, -(K/2) m_-1/2, -K m0, -(3K/2) m1,
 *        -K m0 u + m0 (ugx - u)/theta, -K m0 v + m0 (ugy - v)/theta).
 * In place on W (AoS).  iters_sum (optional) accumulates Newton iterations. */
int or_source_step(const or_cfg* c, double* W, double dt, int64_t* iters_sum, or_err* err) {
  if (c->system != OR_SPRAY) return OR_OK; /* S = 0 ("The source term is set to zero") */
  const double K = c->param[0], theta = c->param[1];
  const double dx = (c->x1 - c->x0) / c->nx;
  const double dy = (c->y1 - c->y0) / c->ny;
  for (int j = 0; j < c->ny; ++j) {
    const double y = c->y0 + (j + 0.5) * dy; /* cell centre (R24) */
    for (int i = 0; i < c->nx; ++i) {
      const double x = c->x0 + (i + 0.5) * dx;
      double* w = W + ((size_t)j * c->nx + i) * 6;
      double lam[4], n0, mmh;
      int32_t it = 0;
      int e = or_reconstruct(w, lam, &n0, &mmh, &it);
      if (iters_sum) *iters_sum += it;
      if (e) {
        if (err) { err->code = OR_E_RECON; err->cell = (int64_t)j * c->nx + i; err->value = w[0]; }
        return OR_E_RECON;
      }
      double ugx, ugy;
      taylor_green(x, y, &ugx, &ugy);
      const double m0 = w[0], m1 = w[1];
      const double inv = 1.0 / w[2];
      const double u = w[4] * inv;
      const double v = w[5] * inv;
      double S[6];
      S[0] = -(K * n0);
      S[1] = -((0.5 * K) * mmh);
      S[2] = -(K * m0);
      S[3] = -((1.5 * K) * m1);
      S[4] = (-((K * m0) * u)) + ((m0 * (ugx - u)) / theta);
      S[5] = (-((K * m0) * v)) + ((m0 * (ugy - v)) / theta);
      for (int k = 0; k < 6; ++k) w[k] = w[k] + dt * S[k];
      for (int k = 0; k < 6; ++k)
        if (!isfinite(w[k])) {
          if (err) { err->code = OR_E_NONFINITE; err->cell = (int64_t)j * c->nx + i; err->value = w[k]; }
          return OR_E_NONFINITE;
        }
    }
  }
  return OR_OK;
}

/* Source-step realizability guard (SPEC "Design decisions"): reject
 * a run whose first dt has dt*K > 0.1*min_cells(m3/m1), erroring at startup
 * (forward Euler, eq:SourceTerm, could destroy positivity).  CEO:
 * r = m3/m1 per cell, rmin by `<` (lowest index on ties), reject iff
 * (dt*K) > (0.1*rmin).  Returns OR_E_ARG with the argmin cell and rmin.     */
int or_spray_guard(const or_cfg* c, const double* W, double dt, or_err* err) {
  if (c->system != OR_SPRAY) return OR_OK;
  const double K = c->param[0];
  double rmin = INFINITY;
  int64_t arg = -1;
  for (size_t n = 0; n < (size_t)c->nx * c->ny; ++n) {
    const double r = W[n * 6 + 3] / W[n * 6 + 1];
    if (r < rmin) { rmin = r; arg = (int64_t)n; }
  }
  if ((dt * K) > (0.1 * rmin)) {
    if (err) { err->code = OR_E_ARG; err->cell = arg; err->value = rmin; }
    return OR_E_ARG;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Full time loop (DESIGN.md §3.1 steps 1-8).
 *   mode 0 = fixed dt (value = dt): check dt*smax <= min(dx,dy) at the
 *            beginning of every iteration (R14); on violation the
 *            state is left at W^k and OR_E_CFL is returned.
 *   mode 1 = adaptive: dt_n = (value*hmin)/smax(W^n), value = C (R4/R5).
 * Spray: the first step's dt must pass or_spray_guard, else OR_E_ARG
 * with W untouched.
 * W (AoS) is advanced in place by nsteps.  dt_log (nsteps, may be NULL)
 * receives every dt used.  dump_steps (sorted, ndump) / dumps: W^k copies
 * for k in dump_steps (k = 0 means the input).  steps_done: completed steps. */
int or_run(const or_cfg* c, double* W, int32_t nsteps, int32_t mode, double value,
           double* dt_log, const int32_t* dump_steps, int32_t ndump, double* dumps,
           int32_t* steps_done, int64_t* newton_iters, or_err* err) {
  if (nvar_of(c->system) != c->nvar || c->nx < 1 || c->ny < 1) return OR_E_ARG;
  const size_t n = (size_t)c->nx * c->ny * c->nvar;
  const double dx = (c->x1 - c->x0) / c->nx;
  const double dy = (c->y1 - c->y0) / c->ny;
  const double hmin = dx < dy ? dx : dy;
  double* tmp = (double*)malloc(n * sizeof(double));
  if (!tmp) return OR_E_ARG;
  int di = 0;
  int rc = OR_OK;
  if (steps_done) *steps_done = 0;
  for (int32_t s = 0; s <= nsteps; ++s) {
    while (di < ndump && dump_steps[di] == s) { memcpy(dumps + (size_t)di * n, W, n * sizeof(double)); ++di; }
    if (s == nsteps) break;
    double smax; int64_t arg;
    rc = or_smax(c, W, &smax, &arg, err);
    if (rc) break;
    double dt;
    if (mode == 0) {
      dt = value;
      if (dt * smax > hmin) {
        rc = OR_E_CFL;
        if (err) { err->code = OR_E_CFL; err->cell = arg; err->value = smax; }
        break;
      }
    } else {
      dt = (value * hmin) / smax;
    }
    if (s == 0 && c->system == OR_SPRAY) {
      rc = or_spray_guard(c, W, dt, err);
      if (rc) break;
    }
    if (dt_log) dt_log[s] = dt;
    rc = or_transport_step(c, W, tmp, dt, err);
    if (rc) break;
    rc = or_source_step(c, tmp, dt, newton_iters, err);
    if (rc) break;
    memcpy(W, tmp, n * sizeof(double));
    if (steps_done) *steps_done = s + 1;
  }
  free(tmp);
  return rc;
}
