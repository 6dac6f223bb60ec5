/* A plain C client of libfv2d (include/fv2d.h): no Python, no torch.
 *
 *   gcc -O2 -I include examples/c_client.c -L paper_1701_05431_b200/lib -lfv2d \
 *       -Wl,-rpath,$PWD/paper_1701_05431_b200/lib -o c_client && ./c_client
 *
 * Checks, through the ABI only: a constant Euler state is preserved exactly
 * (consistency of eq:VF_scheme); sum(W) is conserved to round-off on a
 * periodic random state; a fixed dt above the CFL bound is rejected
 * with FV2D_E_CFL and the state is left at W^k; the host-resident
 * step fv2d_step_host (pipelined over row bands) gives the same bits as
 * set_state + step + get_state.  Exit code 0 = ok. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fv2d.h"

#define CHECK(x)                                                              \
  do {                                                                        \
    fv2d_status s_ = (x);                                                     \
    if (s_ != FV2D_OK) {                                                      \
      fprintf(stderr, "%s:%d: %s -> %d\n", __FILE__, __LINE__, #x, (int)s_); \
      return 1;                                                               \
    }                                                                         \
  } while (0)

static double lcg(uint64_t* s) { /* uniform [0,1) */
  *s = *s * 6364136223846793005ull + 1442695040888963407ull;
  return (double)(*s >> 11) / 9007199254740992.0;
}

int main(void) {
  const int nx = 300, ny = 200, nv = 4;
  const double gamma = 1.4;
  fv2d_config cfg;
  CHECK(fv2d_config_default(&cfg, nx, ny, FV2D_EULER));
  fv2d_ctx* ctx = NULL;
  CHECK(fv2d_create(&cfg, NULL, NULL, &ctx));
  double* W = malloc(sizeof(double) * nx * ny * nv);
  double* out = malloc(sizeof(double) * nx * ny * nv);

  /* 1. constant state: bitwise preserved */
  for (int c = 0; c < nx * ny; ++c) {
    const double rho = 1.3, u = 0.4, v = -0.2, p = 0.9;
    W[c * nv + 0] = rho;
    W[c * nv + 1] = rho * u;
    W[c * nv + 2] = rho * v;
    W[c * nv + 3] = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v);
  }
  CHECK(fv2d_set_state(ctx, W, FV2D_AOS));
  double dt, smax;
  CHECK(fv2d_compute_dt(ctx, 0.45, &dt, &smax));
  CHECK(fv2d_step(ctx, dt, 10));
  CHECK(fv2d_get_state(ctx, out, FV2D_AOS));
  if (memcmp(W, out, sizeof(double) * nx * ny * nv) != 0) {
    fprintf(stderr, "constant state not preserved\n");
    return 1;
  }

  /* 2. random admissible state: conservation of sum(W) (periodic, S = 0) */
  uint64_t seed = 12345;
  double s0[4] = {0, 0, 0, 0}, a0[4] = {0, 0, 0, 0};
  for (int c = 0; c < nx * ny; ++c) {
    const double rho = 0.5 + 1.5 * lcg(&seed), p = 0.5 + 1.5 * lcg(&seed);
    const double u = -1.0 + 2.0 * lcg(&seed), v = -1.0 + 2.0 * lcg(&seed);
    W[c * nv + 0] = rho;
    W[c * nv + 1] = rho * u;
    W[c * nv + 2] = rho * v;
    W[c * nv + 3] = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v);
    for (int k = 0; k < 4; ++k) {
      s0[k] += W[c * nv + k];
      a0[k] += fabs(W[c * nv + k]);
    }
  }
  CHECK(fv2d_set_state(ctx, W, FV2D_AOS));
  double dtlog[20];
  CHECK(fv2d_step_adaptive(ctx, 0.45, 20, dtlog));
  CHECK(fv2d_get_state(ctx, out, FV2D_AOS));
  for (int k = 0; k < 4; ++k) {
    double s1 = 0;
    for (int c = 0; c < nx * ny; ++c) s1 += out[c * nv + k];
    if (fabs(s1 - s0[k]) > 1e-12 * a0[k] * 20) {
      fprintf(stderr, "sum of variable %d changed: %.17g -> %.17g\n", k, s0[k], s1);
      return 1;
    }
  }

  /* 3. fixed dt above the CFL bound: FV2D_E_CFL at step 0, state unchanged */
  CHECK(fv2d_set_state(ctx, W, FV2D_AOS));
  CHECK(fv2d_compute_dt(ctx, 1.0, &dt, &smax));
  CHECK(fv2d_step(ctx, dt * 1.000001, 5));
  if (fv2d_synchronize(ctx) != FV2D_E_CFL) {
    fprintf(stderr, "expected FV2D_E_CFL\n");
    return 1;
  }
  char msg[256];
  int64_t step, cell;
  double val;
  fv2d_last_error(ctx, msg, sizeof msg, &step, &cell, &val);
  if (fv2d_get_state(ctx, out, FV2D_AOS) != FV2D_E_CFL || step != 0 ||
      memcmp(W, out, sizeof(double) * nx * ny * nv) != 0) {
    fprintf(stderr, "CFL error did not leave W^0 (step %lld)\n", (long long)step);
    return 1;
  }
  /* 4. fv2d_step_host (host -> 3 steps -> host, in place) == set_state + step + get_state */
  CHECK(fv2d_set_state(ctx, W, FV2D_AOS));
  CHECK(fv2d_compute_dt(ctx, 0.45, &dt, &smax));
  CHECK(fv2d_step(ctx, dt, 3));
  CHECK(fv2d_get_state(ctx, out, FV2D_AOS));
  double* hs = malloc(sizeof(double) * nx * ny * nv);
  memcpy(hs, W, sizeof(double) * nx * ny * nv);
  CHECK(fv2d_step_host(ctx, hs, hs, FV2D_AOS, dt, 3));
  if (memcmp(hs, out, sizeof(double) * nx * ny * nv) != 0) {
    fprintf(stderr, "fv2d_step_host differs from set_state + step + get_state\n");
    return 1;
  }
  free(hs);
  printf("c_client ok: dt0=%.6g smax=%.6g, CFL error '%s' at cell %lld\n", dtlog[0], smax, msg, (long long)cell);
  fv2d_destroy(ctx);
  free(W);
  free(out);
  return 0;
}
