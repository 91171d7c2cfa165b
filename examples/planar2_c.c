/* planar2_c.c -- the C ABI (include/rd.h) from plain C, no CUDA headers, no Python.
 *
 * Builds BASELINE config C1's robot (the 2-link planar arm of SURVEY 8(c):
 * M_1 = I, M_2 = Trans(l1, 0, 0), S_1 = S_2 = (0,0,0, 0,0,1), link i with mass
 * m_i, centre of mass (r_i, 0, 0), rotational inertia I_i about it; gravity
 * (0, -g, 0)) with rd_model_create, runs inverse dynamics (Eq. 1-2)
 * and forward dynamics (Eq. 4) on HOST arrays through
 * rd_inverse_dynamics_host_f64 / rd_forward_dynamics_host_f64, and checks
 *   - tau against the textbook closed form tau = M(q) qdd + C(q, qd) + G(q),
 *   - FD(q, qd, ID(q, qd, qdd)) = qdd (the round trip),
 * both at 1e-10 relative to max |tau| (max |qdd|).  Exit status 0 = pass.
 *
 *   gcc -O2 -std=c99 -Iinclude examples/planar2_c.c -Lpaper_1609_04493_b200 -lrd \
 *       -Wl,-rpath,$PWD/paper_1609_04493_b200 -lm -o planar2_c && ./planar2_c
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include "rd.h"

enum { N = 2, B = 4096 };
static const double kPi = 3.14159265358979323846;
static const double l1 = 1.1, r1 = 0.45, r2 = 0.6, m1 = 1.3, m2 = 0.9, I1 = 0.12, I2 = 0.07, g = 9.81;

/* J = [[m 1, -m [c]], [m [c], I_c + m([c]^T [c])]] for c = (cx, 0, 0), I_c = Ic 1 ((v, w) ordering) */
static void inertia(double m, double cx, double Ic, double* J) {
  memset(J, 0, 36 * sizeof(double));
  for (int k = 0; k < 3; ++k) J[6 * k + k] = m;
  /* m [c] for c = (cx, 0, 0): [[0, 0, 0], [0, 0, -cx], [0, cx, 0]] * m */
  J[6 * 4 + 2] = -m * cx; J[6 * 5 + 1] = m * cx;          /* lower-left  m [c]  */
  J[6 * 2 + 4] = -m * cx; J[6 * 1 + 5] = m * cx;          /* upper-right -m [c] */
  J[6 * 3 + 3] = Ic;                                      /* I_o = I_c + m (|c|^2 1 - c c^T) */
  J[6 * 4 + 4] = Ic + m * cx * cx;
  J[6 * 5 + 5] = Ic + m * cx * cx;
}

/* splitmix64 -> uniform in [lo, hi) (a plain seeded generator for the example's states) */
static uint64_t sm_state = 0x1234567ull;
static double uniform(double lo, double hi) {
  uint64_t z = (sm_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return lo + (hi - lo) * (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

int main(void) {
  double M[N * 16] = {0}, S[N * 6] = {0}, J[N * 36];
  for (int i = 0; i < N; ++i) {
    for (int k = 0; k < 4; ++k) M[16 * i + 5 * k] = 1.0;
    S[6 * i + 5] = 1.0;                                  /* revolute about the local z axis */
  }
  M[16 * 1 + 3] = l1;                                    /* M_2 = Trans(l1, 0, 0) */
  inertia(m1, r1, I1, J);
  inertia(m2, r2, I2, J + 36);
  const double gravity[3] = {0.0, -g, 0.0};
  rd_model_t model = NULL;
  if (rd_model_create(N, M, S, J, gravity, &model) != RD_OK) {
    fprintf(stderr, "rd_model_create: %s\n", rd_last_error());
    return 2;
  }
  double *q = malloc(sizeof(double) * N * B), *qd = malloc(sizeof(double) * N * B),
         *qdd = malloc(sizeof(double) * N * B), *tau = malloc(sizeof(double) * N * B),
         *back = malloc(sizeof(double) * N * B);
  for (int b = 0; b < B; ++b)                            /* [n][B] link-major, the C1 state ranges */
    for (int i = 0; i < N; ++i) {
      q[i * B + b] = uniform(-kPi, kPi);
      qd[i * B + b] = uniform(-2.0, 2.0);
      qdd[i * B + b] = uniform(-5.0, 5.0);
    }
  if (rd_inverse_dynamics_host_f64(model, B, q, qd, qdd, tau) != RD_OK ||
      rd_forward_dynamics_host_f64(model, B, q, qd, tau, back) != RD_OK) {
    fprintf(stderr, "rd call failed: %s\n", rd_last_error());
    return 2;
  }
  double err_id = 0, max_tau = 0, err_fd = 0, max_qdd = 0;
  for (int b = 0; b < B; ++b) {
    const double q1 = q[b], q2 = q[B + b], w1 = qd[b], w2 = qd[B + b], a1 = qdd[b], a2 = qdd[B + b];
    const double c2 = cos(q2), h = m2 * l1 * r2 * sin(q2);
    const double M11 = I1 + I2 + m1 * r1 * r1 + m2 * (l1 * l1 + r2 * r2 + 2 * l1 * r2 * c2);
    const double M12 = I2 + m2 * (r2 * r2 + l1 * r2 * c2), M22 = I2 + m2 * r2 * r2;
    const double t1 = M11 * a1 + M12 * a2 - h * w2 * (2 * w1 + w2) + (m1 * r1 + m2 * l1) * g * cos(q1) +
                      m2 * r2 * g * cos(q1 + q2);
    const double t2 = M12 * a1 + M22 * a2 + h * w1 * w1 + m2 * r2 * g * cos(q1 + q2);
    err_id = fmax(err_id, fmax(fabs(tau[b] - t1), fabs(tau[B + b] - t2)));
    max_tau = fmax(max_tau, fmax(fabs(t1), fabs(t2)));
    err_fd = fmax(err_fd, fmax(fabs(back[b] - a1), fabs(back[B + b] - a2)));
    max_qdd = fmax(max_qdd, fmax(fabs(a1), fabs(a2)));
  }
  const double rel_id = err_id / max_tau, rel_fd = err_fd / max_qdd;
  printf("planar2_c: %d states, ID vs closed form %.3e, FD round trip %.3e (relative)\n", B, rel_id, rel_fd);
  rd_model_destroy(model);
  free(q); free(qd); free(qdd); free(tau); free(back);
  if (!(rel_id <= 1e-10 && rel_fd <= 1e-10)) {
    printf("planar2_c: FAIL\n");
    return 1;
  }
  printf("planar2_c: ok\n");
  return 0;
}
