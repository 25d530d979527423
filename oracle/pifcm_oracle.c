/*
 * pifcm_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, fp64 CPU implementation of what the 3DPIFCM hot path computes
 * (arXiv 2002.01981).  It exists so that tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py can check the CUDA path against the paper.  The
 * product library (paper_2002_01981_b200/) never links, imports or calls this
 * file, and this file shares no code, header, table or constant generator
 * with it.
 *
 * Citation shorthand: PAPER:N = /root/reference/PAPER.md line N (plus the
 * equation / algorithm it falls in).  Where the paper is silent or garbled the
 * reading taken is named "Rk" and listed in DESIGN.md ("Readings").
 *
 * Layouts (all fp64 unless stated):
 *   x  [nz][ny][nx]       normalized intensities, x fastest (voxel i = (Z*ny+Y)*nx+X)
 *   U  [N][C]             membership rows ("membership matrix U")
 *   c  [C]                cluster centres (Eq. 3)
 *
 * Pins: every function here is checked by tests/test_oracle_*.py against
 * values the paper or mathematics fixes (worked examples, closed forms,
 * special cases, brute force).  Functions without such a pin say
 * "parity unpinned" below.
 *
 * Threading: OpenMP over z-planes; every reduction is accumulated per plane and
 * the planes are summed in increasing z afterwards, so results do not depend on
 * the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_AFLOOR 1e-9   /* R4: floor of the Eq. 4 attraction factor */
#define ORC_DEN_EPS 1e-12 /* R9: keep c_j when sum_i u_ij^m < 1e-12 */

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------------- */
/* Eq. 10: W_i = e^{-i/h} / sum_{r=1..v} e^{-r/h}, i = 1..v.        */
/* W[0] holds W_1.                                                            */
void orc_shell_weights(int v, double h, double *W) {
    double s = 0.0;
    for (int r = 1; r <= v; ++r) s += exp(-(double)r / h);
    for (int i = 1; i <= v; ++i) W[i - 1] = exp(-(double)i / h) / s;
}

/* Eq. 8: q_ik = dX^2 + dY^2 + dZ^2.
 * Eq. 7 uses q_ik^2.  R1: q_mode 0 (LITERAL) squares Eq. 8's
 * value as printed; q_mode 1 (SQEUCLID) reads Eq. 8's value as q^2 itself. */
static double q2_of(int dx, int dy, int dz, int q_mode) {
    double q = (double)(dx * dx + dy * dy + dz * dz);
    return q_mode == 0 ? q * q : q;
}

/* Neighbourhood of voxel i (Eq. 9) partitioned into shells.
 * R2: shell r = in-bounds voxels at Chebyshev distance exactly r, r = 1..v
 * (for v = 1 this is exactly Eq. 9 with L = 3: 0 < dX^2+dY^2+dZ^2 < 4, the
 * 26-neighbourhood; tests/bruteforce.py checks the equality pairwise).
 * Out-of-bounds voxels are excluded (no padding).                  */

/* Per-voxel IFCM evaluation: Eqs. 4-9 and the Eq. 2 membership for one voxel.
 *   outputs u_new[C], d2[C] (Eq. 4 distances), H[C], F[C].                   */
static void ifcm_voxel(const double *x, int nx, int ny, int nz, int C, double m,
                       double lam, double xi, int q_mode, int v, const double *W,
                       const double *U, const double *c, int X, int Y, int Z,
                       double *u_new, double *d2, double *H, double *F) {
    const long i = ((long)Z * ny + Y) * nx + X;
    const double xi_val = x[i];
    /* per-shell sums (v <= 8 supported by the oracle) */
    double Gs[8], Qs[8], Hn[8][8], Fn[8][8];
    for (int r = 0; r < v; ++r) {
        Gs[r] = 0.0; Qs[r] = 0.0;
        for (int j = 0; j < C; ++j) { Hn[r][j] = 0.0; Fn[r][j] = 0.0; }
    }
    for (int dz = -v; dz <= v; ++dz)
        for (int dy = -v; dy <= v; ++dy)
            for (int dx = -v; dx <= v; ++dx) {
                if (dx == 0 && dy == 0 && dz == 0) continue;          /* Eq. 9: 0 < ... */
                const int Xk = X + dx, Yk = Y + dy, Zk = Z + dz;
                if (Xk < 0 || Xk >= nx || Yk < 0 || Yk >= ny || Zk < 0 || Zk >= nz) continue;
                int r = abs(dx);
                if (abs(dy) > r) r = abs(dy);
                if (abs(dz) > r) r = abs(dz);
                const long k = ((long)Zk * ny + Yk) * nx + Xk;
                const double g = fabs(xi_val - x[k]);                 /* Eq. 6 */
                const double q2 = q2_of(dx, dy, dz, q_mode);          /* Eq. 8, R1 */
                Gs[r - 1] += g;
                Qs[r - 1] += q2;
                for (int j = 0; j < C; ++j) {
                    const double ukj = U[k * C + j];
                    Hn[r - 1][j] += ukj * g;                           /* Eq. 5 numerator */
                    Fn[r - 1][j] += ukj * ukj * q2;                    /* Eq. 7 numerator */
                }
            }
    for (int j = 0; j < C; ++j) {
        double h = 0.0, f = 0.0;
        for (int r = 0; r < v; ++r) {
            /* R3: a shell whose g's are all zero contributes 0 to H (0/0 guard) */
            if (Gs[r] > 0.0) h += W[r] * Hn[r][j] / Gs[r];             /* Eq. 5 */
            if (Qs[r] > 0.0) f += W[r] * Fn[r][j] / Qs[r];             /* Eq. 7 */
        }
        H[j] = h; F[j] = f;
        double a = 1.0 - lam * h - xi * f;                             /* Eq. 4 factor */
        if (a < ORC_AFLOOR) a = ORC_AFLOOR;                            /* R4 */
        const double diff = xi_val - c[j];
        d2[j] = diff * diff * a;                                       /* Eq. 4 */
    }
    /* Eq. 2 in the squared form (d_ij/d_ik)^{2/(m-1)} =
     * (d2_ij/d2_ik)^{1/(m-1)}.  R5: a zero distance makes the row crisp at the
     * lowest such cluster. */
    int zero_j = -1;
    for (int j = 0; j < C; ++j)
        if (d2[j] == 0.0) { zero_j = j; break; }
    if (zero_j >= 0) {
        for (int j = 0; j < C; ++j) u_new[j] = (j == zero_j) ? 1.0 : 0.0;
        return;
    }
    const double e = 1.0 / (m - 1.0);
    for (int j = 0; j < C; ++j) {
        double s = 0.0;
        for (int k = 0; k < C; ++k) s += pow(d2[j] / d2[k], e);
        u_new[j] = 1.0 / s;
    }
}

/* One IFCM step ("The step function runs a single iteration";
 * Alg. 2 steps 6-8): Jacobi update of every membership row from
 * the previous U (R7), then Eq. 3 centres from the new U (R6), then Eq. 1 cost
 * with the same Eq. 4 distances (R8), and max |u_new - u_old|.
 * Only the rows of the target planes [zt0, zt1) are updated and summed; the
 * other planes' rows are copied (they are neighbours only -- the literal slice
 * mode, R25).  orc_ifcm_step = all planes.
 * If c_new is NULL the centres are not updated. */
void orc_ifcm_step_planes(const double *x, int nx, int ny, int nz, int zt0, int zt1, int C, double m,
                          double lam, double xi, int q_mode, int v, double h,
                          const double *U_old, const double *c_old,
                          double *U_new, double *c_new, double *J_out, double *maxdu_out) {
    double W[8];
    orc_shell_weights(v, h, W);
    double *pnum = (double *)calloc((size_t)nz * C, sizeof(double));
    double *pden = (double *)calloc((size_t)nz * C, sizeof(double));
    double *pJ = (double *)calloc((size_t)nz, sizeof(double));
    double *pdu = (double *)calloc((size_t)nz, sizeof(double));
#pragma omp parallel for schedule(dynamic, 1)
    for (int Z = 0; Z < nz; ++Z) {
        double u[8], d2[8], H[8], F[8];
        const int target = Z >= zt0 && Z < zt1;
        for (int Y = 0; Y < ny; ++Y)
            for (int X = 0; X < nx; ++X) {
                const long i = ((long)Z * ny + Y) * nx + X;
                if (!target) {
                    for (int j = 0; j < C; ++j) U_new[i * C + j] = U_old[i * C + j];
                    continue;
                }
                ifcm_voxel(x, nx, ny, nz, C, m, lam, xi, q_mode, v, W, U_old, c_old,
                           X, Y, Z, u, d2, H, F);
                for (int j = 0; j < C; ++j) {
                    U_new[i * C + j] = u[j];
                    const double um = pow(u[j], m);
                    pnum[(long)Z * C + j] += um * x[i];                /* Eq. 3 numerator */
                    pden[(long)Z * C + j] += um;                       /* Eq. 3 denominator */
                    pJ[Z] += um * d2[j];                               /* Eq. 1 */
                    const double du = fabs(u[j] - U_old[i * C + j]);
                    if (du > pdu[Z]) pdu[Z] = du;
                }
            }
    }
    double J = 0.0, mdu = 0.0;
    for (int j = 0; j < C; ++j) {
        double num = 0.0, den = 0.0;
        for (int Z = 0; Z < nz; ++Z) { num += pnum[(long)Z * C + j]; den += pden[(long)Z * C + j]; }
        if (c_new) c_new[j] = (den < ORC_DEN_EPS) ? c_old[j] : num / den;   /* Eq. 3, R9 */
    }
    for (int Z = 0; Z < nz; ++Z) { J += pJ[Z]; if (pdu[Z] > mdu) mdu = pdu[Z]; }
    if (J_out) *J_out = J;
    if (maxdu_out) *maxdu_out = mdu;
    free(pnum); free(pden); free(pJ); free(pdu);
}

void orc_ifcm_step(const double *x, int nx, int ny, int nz, int C, double m,
                   double lam, double xi, int q_mode, int v, double h,
                   const double *U_old, const double *c_old,
                   double *U_new, double *c_new, double *J_out, double *maxdu_out) {
    orc_ifcm_step_planes(x, nx, ny, nz, 0, nz, C, m, lam, xi, q_mode, v, h, U_old, c_old, U_new, c_new, J_out,
                         maxdu_out);
}

/* Per-voxel evaluation at a list of voxels (for sampled parity at full size):
 * returns u_new, d2, H, F rows ([n][C] each) for the given voxel indices. */
void orc_ifcm_voxels(const double *x, int nx, int ny, int nz, int C, double m,
                     double lam, double xi, int q_mode, int v, double h,
                     const double *U_old, const double *c_old,
                     const int64_t *idx, long n,
                     double *u_out, double *d2_out, double *H_out, double *F_out) {
    double W[8];
    orc_shell_weights(v, h, W);
#pragma omp parallel for schedule(static)
    for (long t = 0; t < n; ++t) {
        const long i = (long)idx[t];
        const int X = (int)(i % nx), Y = (int)((i / nx) % ny), Z = (int)(i / ((long)nx * ny));
        ifcm_voxel(x, nx, ny, nz, C, m, lam, xi, q_mode, v, W, U_old, c_old, X, Y, Z,
                   u_out + t * C, d2_out + t * C, H_out + t * C, F_out + t * C);
    }
}

/* ------------------------------------------------------------------------- */
/* Standard FCM (Bezdek, PAPER:51-57 with d^2 = (x_i - c_j)^2): membership   */
/* from centres (Eq. 2), then centres from the new memberships (Eq. 3).       */
/* Written independently of orc_ifcm_step so the lambda = xi = 0 reduction    */
/* (PAPER:61 with lambda = xi = 0) can be checked against it.                 */
void orc_fcm_step(const double *x, long N, int C, double m, const double *c_old,
                  const double *U_old /* nullable */, double *U_new, double *c_new,
                  double *J_out, double *maxdu_out) {
    const double e = 1.0 / (m - 1.0);
    double J = 0.0, mdu = 0.0;
    double num[8] = {0}, den[8] = {0};
    for (long i = 0; i < N; ++i) {
        double d2[8];
        int zero_j = -1;
        for (int j = 0; j < C; ++j) {
            d2[j] = (x[i] - c_old[j]) * (x[i] - c_old[j]);
            if (d2[j] == 0.0 && zero_j < 0) zero_j = j;
        }
        for (int j = 0; j < C; ++j) {
            double u;
            if (zero_j >= 0) {
                u = (j == zero_j) ? 1.0 : 0.0;
            } else {
                double s = 0.0;
                for (int k = 0; k < C; ++k) s += pow(d2[j] / d2[k], e);
                u = 1.0 / s;
            }
            U_new[i * C + j] = u;
            const double um = pow(u, m);
            num[j] += um * x[i];
            den[j] += um;
            J += um * d2[j];
            if (U_old) {
                const double du = fabs(u - U_old[i * C + j]);
                if (du > mdu) mdu = du;
            }
        }
    }
    for (int j = 0; j < C; ++j) c_new[j] = (den[j] < ORC_DEN_EPS) ? c_old[j] : num[j] / den[j];
    if (J_out) *J_out = J;
    if (maxdu_out) *maxdu_out = mdu;
}

/* Eq. 3 alone over a given U. */
void orc_centers(const double *x, long N, int C, double m, const double *U,
                 const double *c_old, double *c_new) {
    for (int j = 0; j < C; ++j) {
        double num = 0.0, den = 0.0;
        for (long i = 0; i < N; ++i) {
            const double um = pow(U[i * C + j], m);
            num += um * x[i];
            den += um;
        }
        c_new[j] = (den < ORC_DEN_EPS) ? c_old[j] : num / den;
    }
}

/* Defuzzification ("Display membership result"):
 * label = argmax_j u_ij, ties -> lowest j (R13). */
void orc_argmax(const double *U, long N, int C, uint8_t *labels) {
    for (long i = 0; i < N; ++i) {
        int best = 0;
        for (int j = 1; j < C; ++j)
            if (U[i * C + j] > U[i * C + best]) best = j;
        labels[i] = (uint8_t)best;
    }
}

/* ------------------------------------------------------------------------- */
/* Alg. 2 step 1: min-max normalisation over the whole volume */
/* into [0,1]; R16: a constant volume maps to 0.                              */
void orc_normalize_u8(const uint8_t *vol, long N, double *x) {
    int mn = 255, mx = 0;
    for (long i = 0; i < N; ++i) {
        if (vol[i] < mn) mn = vol[i];
        if (vol[i] > mx) mx = vol[i];
    }
    for (long i = 0; i < N; ++i)
        x[i] = (mx > mn) ? (double)(vol[i] - mn) / (double)(mx - mn) : 0.0;
}

/* R15: 256-bin histogram of the normalised volume, computed in integers:
 * bin = floor(((v - min) * 255 + (max - min) / 2) / (max - min)), i.e. the
 * nearest of 256 evenly spaced levels b/255.  Constant volume -> all in bin 0. */
void orc_histogram_u8_range(const uint8_t *vol, long N, int mn, int mx, int64_t *hist);
void orc_histogram_u8(const uint8_t *vol, long N, int64_t *hist) {
    int mn = 255, mx = 0;
    for (long i = 0; i < N; ++i) {
        if (vol[i] < mn) mn = vol[i];
        if (vol[i] > mx) mx = vol[i];
    }
    orc_histogram_u8_range(vol, N, mn, mx, hist);
}
/* The same bins for values vol[0..N) of a volume whose range is [mn, mx]
 * (the slice of R25 binned on the whole volume's levels). */
void orc_histogram_u8_range(const uint8_t *vol, long N, int mn, int mx, int64_t *hist) {
    for (int b = 0; b < 256; ++b) hist[b] = 0;
    const int rng = mx - mn;
    for (long i = 0; i < N; ++i) {
        int b = 0;
        if (rng > 0) b = ((vol[i] - mn) * 255 + rng / 2) / rng;
        hist[b] += 1;
    }
}

/* Alg. 2 step 1 for 16-bit and fp32 volumes (u8 / u16 /
 * f32 inputs): the same global min-max normalisation (R16) and the R15
 * histogram of the same levels b/255 -- u16 in integers like u8; f32 in fp64:
 * bin = floor((v - min) * 255 / (max - min) + 0.5). */
void orc_normalize_u16(const uint16_t *vol, long N, double *x) {
    int mn = 65535, mx = 0;
    for (long i = 0; i < N; ++i) {
        if (vol[i] < mn) mn = vol[i];
        if (vol[i] > mx) mx = vol[i];
    }
    for (long i = 0; i < N; ++i)
        x[i] = (mx > mn) ? (double)(vol[i] - mn) / (double)(mx - mn) : 0.0;
}
void orc_histogram_u16(const uint16_t *vol, long N, int64_t *hist) {
    int64_t mn = 65535, mx = 0;
    for (long i = 0; i < N; ++i) {
        if (vol[i] < mn) mn = vol[i];
        if (vol[i] > mx) mx = vol[i];
    }
    for (int b = 0; b < 256; ++b) hist[b] = 0;
    const int64_t rng = mx - mn;
    for (long i = 0; i < N; ++i) {
        int64_t b = 0;
        if (rng > 0) b = (((int64_t)vol[i] - mn) * 255 + rng / 2) / rng;
        hist[b] += 1;
    }
}
void orc_normalize_f32(const float *vol, long N, double *x) {
    double mn = INFINITY, mx = -INFINITY;
    for (long i = 0; i < N; ++i) {
        if ((double)vol[i] < mn) mn = vol[i];
        if ((double)vol[i] > mx) mx = vol[i];
    }
    for (long i = 0; i < N; ++i) x[i] = (mx > mn) ? ((double)vol[i] - mn) / (mx - mn) : 0.0;
}
void orc_histogram_f32(const float *vol, long N, int64_t *hist) {
    double mn = INFINITY, mx = -INFINITY;
    for (long i = 0; i < N; ++i) {
        if ((double)vol[i] < mn) mn = vol[i];
        if ((double)vol[i] > mx) mx = vol[i];
    }
    for (int b = 0; b < 256; ++b) hist[b] = 0;
    for (long i = 0; i < N; ++i) {
        int b = 0;
        if (mx > mn) {
            b = (int)floor(((double)vol[i] - mn) * 255.0 / (mx - mn) + 0.5);
            if (b < 0) b = 0;
            if (b > 255) b = 255;
        }
        hist[b] += 1;
    }
}

/* R15: "Modified_FCM with Gaussian mixture model" is read as a
 * 1-D EM fit of a C-component Gaussian mixture on the 256-bin histogram
 * (bin b at level y_b = b/255), evenly spaced initialisation, <= max_iter EM
 * iterations, component means (sorted ascending) -> initial centres.
 * Degenerate fits fall back to evenly spaced centres c_j = j/(C-1).
 * Pins: the two-mode fixed point (-> the modes), a hand-worked one-iteration
 * case, and every EM iteration against scikit-learn's GaussianMixture from the
 * same start (tests/test_oracle_pso.py, tests/test_oracle_pins_init.py); the
 * R15 reading itself (what the paper's undefined step is) stays a reading. */
void orc_gmm_init(const int64_t *hist, int C, int max_iter, double *c0) {
    double y[256], n[256], Ntot = 0.0;
    int distinct = 0;
    for (int b = 0; b < 256; ++b) {
        y[b] = (double)b / 255.0;
        n[b] = (double)hist[b];
        Ntot += n[b];
        if (hist[b] > 0) distinct++;
    }
    if (Ntot <= 0.0 || distinct < C) {
        for (int j = 0; j < C; ++j) c0[j] = (double)j / (double)(C - 1);
        return;
    }
    double mu[8], s2[8], w[8];
    /* R15: evenly spaced initialisation over the normalised range,
     * mu_j = (j + 0.5) / C, sigma_j = 1 / (2C), w_j = 1 / C.  (A k-quantile
     * start collapses two components onto the dominant background mode of the
     * nested phantoms, so the spread start is taken.) */
    for (int j = 0; j < C; ++j) {
        mu[j] = ((double)j + 0.5) / (double)C;
        s2[j] = 1.0 / (4.0 * (double)C * (double)C);
        w[j] = 1.0 / (double)C;
    }
    const double two_pi = 6.283185307179586476925286766559;
    for (int it = 0; it < max_iter; ++it) {
        double Nj[8] = {0}, Sy[8] = {0}, Syy[8] = {0};
        /* E step + accumulation of sufficient statistics */
        for (int b = 0; b < 256; ++b) {
            if (n[b] <= 0.0) continue;
            double p[8], s = 0.0;
            for (int j = 0; j < C; ++j) {
                const double d = y[b] - mu[j];
                p[j] = w[j] * exp(-d * d / (2.0 * s2[j])) / sqrt(two_pi * s2[j]);
                s += p[j];
            }
            if (!(s > 0.0)) {
                /* all responsibilities underflowed: give the bin to the nearest mean */
                int jb = 0;
                for (int j = 1; j < C; ++j)
                    if (fabs(y[b] - mu[j]) < fabs(y[b] - mu[jb])) jb = j;
                for (int j = 0; j < C; ++j) p[j] = (j == jb) ? 1.0 : 0.0;
                s = 1.0;
            }
            for (int j = 0; j < C; ++j) {
                const double r = p[j] / s;
                Nj[j] += n[b] * r;
                Sy[j] += n[b] * r * y[b];
            }
        }
        double new_mu[8];
        for (int j = 0; j < C; ++j) new_mu[j] = (Nj[j] > 1e-12) ? Sy[j] / Nj[j] : mu[j];
        for (int b = 0; b < 256; ++b) {
            if (n[b] <= 0.0) continue;
            double p[8], s = 0.0;
            for (int j = 0; j < C; ++j) {
                const double d = y[b] - mu[j];
                p[j] = w[j] * exp(-d * d / (2.0 * s2[j])) / sqrt(two_pi * s2[j]);
                s += p[j];
            }
            if (!(s > 0.0)) {
                int jb = 0;
                for (int j = 1; j < C; ++j)
                    if (fabs(y[b] - mu[j]) < fabs(y[b] - mu[jb])) jb = j;
                for (int j = 0; j < C; ++j) p[j] = (j == jb) ? 1.0 : 0.0;
                s = 1.0;
            }
            for (int j = 0; j < C; ++j) {
                const double d = y[b] - new_mu[j];
                Syy[j] += n[b] * (p[j] / s) * d * d;
            }
        }
        double shift = 0.0;
        for (int j = 0; j < C; ++j) {
            if (Nj[j] > 1e-12) {
                w[j] = Nj[j] / Ntot;
                s2[j] = Syy[j] / Nj[j];
                if (s2[j] < 1e-6) s2[j] = 1e-6;
            }
            const double dm = fabs(new_mu[j] - mu[j]);
            if (dm > shift) shift = dm;
            mu[j] = new_mu[j];
        }
        if (shift < 1e-9) break;
    }
    /* sort ascending (insertion sort) */
    for (int a = 1; a < C; ++a) {
        const double t = mu[a];
        int b = a - 1;
        while (b >= 0 && mu[b] > t) { mu[b + 1] = mu[b]; --b; }
        mu[b + 1] = t;
    }
    int degenerate = 0;
    for (int j = 1; j < C; ++j)
        if (mu[j] - mu[j - 1] < 1e-6) degenerate = 1;
    for (int j = 0; j < C; ++j) c0[j] = degenerate ? (double)j / (double)(C - 1) : mu[j];
}

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as    */
/* 1, 2, 3"): counter-based generator used for every PSO draw so that the GPU */
/* path and this oracle see identical particle trajectories (north_star).      */
/* Pin: Random123 known-answer vectors (tests/test_oracle_pso.py).             */
static uint32_t mulhi32(uint32_t a, uint32_t b) {
    return (uint32_t)(((uint64_t)a * (uint64_t)b) >> 32);
}

void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = mulhi32(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = mulhi32(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n1 = lo1;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        const uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Two 32-bit words -> a double in [0,1) with 53 random bits (R12). */
static double u01_from(uint32_t w_lo, uint32_t w_hi) {
    const uint64_t a = ((uint64_t)w_hi << 32) | (uint64_t)w_lo;
    return (double)(a >> 11) * (1.0 / 9007199254740992.0);
}

/* Draw two doubles for counter (c0, c1, c2, c3) under key = seed. */
void orc_philox_pair(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                     double *a, double *b) {
    const uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    const uint32_t ctr[4] = {c0, c1, c2, c3};
    uint32_t o[4];
    orc_philox4x32_10(ctr, key, o);
    *a = u01_from(o[0], o[1]);
    *b = u01_from(o[2], o[3]);
}

/* Alg. 1 step 3 / Alg. 2 step 3: random swarm in
 * [0,1]^2 (D = 2: lambda, xi).  R12: x ~ U[0,1]^2 from counter
 * (0xFFFFFFFF, p, 1, 0); v ~ U[-v0, v0]^2 from counter (0xFFFFFFFF, p, 2, 0). */
void orc_pso_init(int P, uint64_t seed, double v0, double *pos /*[P][2]*/, double *vel /*[P][2]*/) {
    for (int p = 0; p < P; ++p) {
        double a, b;
        orc_philox_pair(seed, 0xFFFFFFFFu, (uint32_t)p, 1u, 0u, &a, &b);
        pos[2 * p] = a;
        pos[2 * p + 1] = b;
        orc_philox_pair(seed, 0xFFFFFFFFu, (uint32_t)p, 2u, 0u, &a, &b);
        vel[2 * p] = (2.0 * a - 1.0) * v0;
        vel[2 * p + 1] = (2.0 * b - 1.0) * v0;
    }
}

/* Alg. 1 steps 7-8 with explicit draws p1[p], p2[p] and
 * lbest indices lb[p]: v = clamp(v + p1 (x_pbest - x) + p2 (x_lbest - x), +-vmax)
 * (R12), x = clamp(x + v, 0, 1). */
void orc_pso_move(int P, double vmax, const double *p1, const double *p2, const int *lb,
                  const double *pbest_x, double *pos, double *vel) {
    for (int p = 0; p < P; ++p) {
        for (int d = 0; d < 2; ++d) {
            double vv = vel[2 * p + d] + p1[p] * (pbest_x[2 * p + d] - pos[2 * p + d]) +
                        p2[p] * (pbest_x[2 * lb[p] + d] - pos[2 * p + d]);
            if (vv > vmax) vv = vmax;
            if (vv < -vmax) vv = -vmax;
            vel[2 * p + d] = vv;
            double xx = pos[2 * p + d] + vv;
            if (xx < 0.0) xx = 0.0;
            if (xx > 1.0) xx = 1.0;
            pos[2 * p + d] = xx;
        }
    }
}

/* One PSO bookkeeping + move after the fitnesses f[P] of generation `gen`
 * have been evaluated at positions pos (Alg. 1 steps 5-8):
 *   step 5: pbest (strict <)
 *   step 6: lbest over the ring {p-k..p+k} mod P of the pbests (R12; ties ->
 *           lowest particle index)
 *   step 7: v = v + p1 (x_pbest - x) + p2 (x_lbest - x), p1, p2 in [0,1) from
 *           Philox counter (gen, p, 0, 0); R12: |v| clamped to vmax
 *   step 8: x = clamp(x + v, 0, 1)
 * gbest (lowest index on ties, except that the incumbent keeps it on an exact
 * tie, R13) is returned in *gbest; *improved is 1 when the
 * global best fitness strictly decreased this generation.                    */
void orc_pso_update(int P, int ring_k, uint32_t gen, uint64_t seed, double vmax,
                    const double *f, double *pos, double *vel, double *pbest_f,
                    double *pbest_x, int *gbest, int *improved) {
    const int g_old = *gbest;
    const double gf_old = (g_old >= 0) ? pbest_f[g_old] : INFINITY;
    for (int p = 0; p < P; ++p) {
        if (f[p] < pbest_f[p]) {
            pbest_f[p] = f[p];
            pbest_x[2 * p] = pos[2 * p];
            pbest_x[2 * p + 1] = pos[2 * p + 1];
        }
    }
    int g = 0;
    for (int p = 1; p < P; ++p)
        if (pbest_f[p] < pbest_f[g]) g = p;
    /* R13: the incumbent gbest keeps the title on an exact tie (its state is
     * the pinned snapshot; a tied lower index did not improve on it) */
    if (g_old >= 0 && !(pbest_f[g] < pbest_f[g_old])) g = g_old;
    *gbest = g;
    *improved = (pbest_f[g] < gf_old) ? 1 : 0;
    int *lb = (int *)malloc(sizeof(int) * (size_t)P);
    for (int p = 0; p < P; ++p) {
        int best = -1;
        for (int d = -ring_k; d <= ring_k; ++d) {
            const int q = ((p + d) % P + P) % P;
            if (best < 0 || pbest_f[q] < pbest_f[best] ||
                (pbest_f[q] == pbest_f[best] && q < best))
                best = q;
        }
        lb[p] = best;
    }
    double *r1 = (double *)malloc(sizeof(double) * (size_t)P);
    double *r2 = (double *)malloc(sizeof(double) * (size_t)P);
    for (int p = 0; p < P; ++p) orc_philox_pair(seed, gen, (uint32_t)p, 0u, 0u, &r1[p], &r2[p]);
    orc_pso_move(P, vmax, r1, r2, lb, pbest_x, pos, vel);
    free(r1); free(r2);
    free(lb);
}

/* ------------------------------------------------------------------------- */
/* PSO over (lambda, xi) (Alg. 1 steps 3-10).  Fitness modes     */
/* (R11):                                                 */
/*  0 CHAINED  particle p owns a state (U_p, c_p) that starts at (U0, c0); each*/
/*             generation advances it by one IFCM step at the particle's       */
/*             current position, and the fitness is that step's J.            */
/*  1 ANCHORED every evaluation is one IFCM step from the shared start         */
/*             (U0, c0) at the particle's position; fitness = its J.          */
/*  2 LEADER   every evaluation is one step from the shared state S_t (S_0 =   */
/*             (U0, c0)); after the generation's PSO update, S_{t+1} = the     */
/*             state the gbest particle's evaluation produced (R22).          */
/* In every mode the gbest snapshot is the (U, c) produced by the evaluation   */
/* that improved the gbest (Alg. 1 step 10).                        */
/* Stop (R12, Alg. 1 step 9 "until convergence (i.e small changes to J)"):    */
/* relative change of the gbest fitness < tol for `patience` consecutive       */
/* generations, or max_gen.  patience <= 0 disables the early stop.            */
/* Outputs: the gbest snapshot (Alg. 1 step 10): lambda, xi, J, and */
/* the (U, c) its evaluation produced; per-generation traces for testing.      */
/* Pin: partial (PSO invariants and worked example); end-to-end trajectory     */
/* parity unpinned (only oracle-vs-GPU agreement).                             */
static int pso_core(const double *x, int nx, int ny, int nz, int zt0, int zt1, int C, double m, int q_mode,
                    int v, double h, const double *U0, const double *c0,
                    int P, int ring_k, int max_gen, int patience, double tol, double v0,
                    double vmax, uint64_t seed, double *best_lx, double *best_J, double *best_U,
                    double *best_c, double *trace_pos, double *trace_f, int *trace_gbest, int fitness_mode);

int orc_pso_run(const double *x, int nx, int ny, int nz, int C, double m, int q_mode,
                int v, double h, const double *U0, const double *c0,
                int P, int ring_k, int max_gen, int patience, double tol, double v0,
                double vmax, uint64_t seed,
                double *best_lx /*[2]*/, double *best_J, double *best_U /*[N][C]*/,
                double *best_c /*[C]*/,
                double *trace_pos /*[max_gen][P][2] nullable*/,
                double *trace_f /*[max_gen][P] nullable*/,
                int *trace_gbest /*[max_gen] nullable*/, int fitness_mode) {
    return pso_core(x, nx, ny, nz, 0, nz, C, m, q_mode, v, h, U0, c0, P, ring_k, max_gen, patience, tol, v0,
                    vmax, seed, best_lx, best_J, best_U, best_c, trace_pos, trace_f, trace_gbest, fitness_mode);
}

/* The PSO of orc_pso_run over the target planes [zt0, zt1) (R25). */
static int pso_core(const double *x, int nx, int ny, int nz, int zt0, int zt1, int C, double m, int q_mode,
                    int v, double h, const double *U0, const double *c0,
                    int P, int ring_k, int max_gen, int patience, double tol, double v0,
                    double vmax, uint64_t seed, double *best_lx, double *best_J, double *best_U,
                    double *best_c, double *trace_pos, double *trace_f, int *trace_gbest, int fitness_mode) {
    const long N = (long)nx * ny * nz;
    const int shared = (fitness_mode == 1 || fitness_mode == 2);
    double *pos = (double *)malloc(sizeof(double) * 2 * P);
    double *vel = (double *)malloc(sizeof(double) * 2 * P);
    double *pbf = (double *)malloc(sizeof(double) * P);
    double *pbx = (double *)malloc(sizeof(double) * 2 * P);
    double *f = (double *)malloc(sizeof(double) * P);
    /* CHAINED: one state per particle; ANCHORED / LEADER: one shared state */
    const int nst = shared ? 1 : P;
    double *Us = (double *)malloc(sizeof(double) * (size_t)N * C * nst);
    double *Ut = (double *)malloc(sizeof(double) * (size_t)N * C);
    double *cs = (double *)malloc(sizeof(double) * C * nst);
    double *eval_pos = (double *)malloc(sizeof(double) * 2 * P);
    orc_pso_init(P, seed, v0, pos, vel);
    for (int p = 0; p < P; ++p) {
        pbf[p] = INFINITY;
        pbx[2 * p] = pos[2 * p];
        pbx[2 * p + 1] = pos[2 * p + 1];
        if (p < nst) {
            memcpy(Us + (size_t)p * N * C, U0, sizeof(double) * (size_t)N * C);
            memcpy(cs + (size_t)p * C, c0, sizeof(double) * C);
        }
    }
    int gbest = -1, improved = 0, gen = 0, calm = 0;
    double prev_gf = INFINITY;
    for (gen = 0; gen < max_gen; ++gen) {
        for (int p = 0; p < P; ++p) {
            double cn[8], J, du;
            const int sp = shared ? 0 : p;
            orc_ifcm_step_planes(x, nx, ny, nz, zt0, zt1, C, m, pos[2 * p], pos[2 * p + 1], q_mode, v, h,
                          Us + (size_t)sp * N * C, cs + (size_t)sp * C, Ut, cn, &J, &du);
            if (!shared) {
                memcpy(Us + (size_t)p * N * C, Ut, sizeof(double) * (size_t)N * C);
                memcpy(cs + (size_t)p * C, cn, sizeof(double) * C);
            }
            f[p] = J;
            if (trace_pos) { trace_pos[((size_t)gen * P + p) * 2] = pos[2 * p];
                             trace_pos[((size_t)gen * P + p) * 2 + 1] = pos[2 * p + 1]; }
            if (trace_f) trace_f[(size_t)gen * P + p] = J;
        }
        /* positions at which this generation was evaluated (for the snapshot) */
        memcpy(eval_pos, pos, sizeof(double) * 2 * P);
        orc_pso_update(P, ring_k, (uint32_t)gen, seed, vmax, f, pos, vel, pbf, pbx, &gbest, &improved);
        if (trace_gbest) trace_gbest[gen] = gbest;
        double cg[8];
        if (shared && (improved || fitness_mode == 2)) {
            /* the state the gbest's evaluation produced this generation (the
             * evaluation is deterministic, so it is recomputed rather than kept) */
            double J, du;
            orc_ifcm_step_planes(x, nx, ny, nz, zt0, zt1, C, m, eval_pos[2 * gbest], eval_pos[2 * gbest + 1], q_mode, v, h,
                          Us, cs, Ut, cg, &J, &du);
        }
        if (improved) {
            best_lx[0] = eval_pos[2 * gbest];
            best_lx[1] = eval_pos[2 * gbest + 1];
            *best_J = pbf[gbest];
            if (shared) {
                memcpy(best_U, Ut, sizeof(double) * (size_t)N * C);
                memcpy(best_c, cg, sizeof(double) * C);
            } else {
                memcpy(best_U, Us + (size_t)gbest * N * C, sizeof(double) * (size_t)N * C);
                memcpy(best_c, cs + (size_t)gbest * C, sizeof(double) * C);
            }
        }
        if (fitness_mode == 2) { /* LEADER: the shared state follows the gbest's step */
            memcpy(Us, Ut, sizeof(double) * (size_t)N * C);
            memcpy(cs, cg, sizeof(double) * C);
        }
        const double gf = pbf[gbest];
        if (gen > 0 && patience > 0) {
            const double rel = (prev_gf - gf) / (gf > 0.0 ? gf : 1.0);
            if (rel < tol) calm++; else calm = 0;
            if (calm >= patience) { prev_gf = gf; gen++; break; }
        }
        prev_gf = gf;
    }
    free(pos); free(vel); free(pbf); free(pbx); free(f); free(Us); free(Ut); free(cs);
    free(eval_pos);
    return gen; /* generations run */
}

/* IFCM (or FCM when lam = xi = 0) iterated until max|du| < eps or max_iter
 * (Alg. 1 step 11; R14).  U and c are updated in place.
 * Returns the number of iterations run. */
static int ifcm_run_planes(const double *x, int nx, int ny, int nz, int zt0, int zt1, int C, double m,
                           double lam, double xi, int q_mode, int v, double h, double eps, int max_iter,
                           double *U, double *c, double *J_out);
int orc_ifcm_run(const double *x, int nx, int ny, int nz, int C, double m, double lam,
                 double xi, int q_mode, int v, double h, double eps, int max_iter,
                 double *U, double *c, double *J_out) {
    return ifcm_run_planes(x, nx, ny, nz, 0, nz, C, m, lam, xi, q_mode, v, h, eps, max_iter, U, c, J_out);
}
static int ifcm_run_planes(const double *x, int nx, int ny, int nz, int zt0, int zt1, int C, double m,
                           double lam, double xi, int q_mode, int v, double h, double eps, int max_iter,
                           double *U, double *c, double *J_out) {
    const long N = (long)nx * ny * nz;
    double *Ut = (double *)malloc(sizeof(double) * (size_t)N * C);
    int it = 0;
    double J = 0.0;
    for (it = 1; it <= max_iter; ++it) {
        double cn[8], du;
        orc_ifcm_step_planes(x, nx, ny, nz, zt0, zt1, C, m, lam, xi, q_mode, v, h, U, c, Ut, cn, &J, &du);
        memcpy(U, Ut, sizeof(double) * (size_t)N * C);
        memcpy(c, cn, sizeof(double) * C);
        if (du < eps) break;
    }
    if (it > max_iter) it = max_iter;
    free(Ut);
    if (J_out) *J_out = J;
    return it;
}

/* FCM initialisation (Alg. 1 step 2; Alg. 2 step 5; R14):
 * t = 1: U_1 = Eq. 2 from c0, c_1 = Eq. 3; then repeat until
 * max |U_t - U_{t-1}| < eps (checked from t = 2) or max_iter.  Returns t. */
int orc_fcm_run(const double *x, long N, int C, double m, double eps, int max_iter,
                const double *c0, double *U, double *c) {
    double *Ut = (double *)malloc(sizeof(double) * (size_t)N * C);
    double cc[8], cn[8];
    memcpy(cc, c0, sizeof(double) * C);
    int t;
    for (t = 1; t <= max_iter; ++t) {
        double J, du;
        orc_fcm_step(x, N, C, m, cc, t > 1 ? U : NULL, Ut, cn, &J, &du);
        memcpy(U, Ut, sizeof(double) * (size_t)N * C);
        memcpy(cc, cn, sizeof(double) * C);
        if (t > 1 && du < eps) break;
    }
    if (t > max_iter) t = max_iter;
    memcpy(c, cc, sizeof(double) * C);
    free(Ut);
    return t;
}

/* The whole pipeline (Alg. 1 / Alg. 2) on a u8 volume:
 * normalise -> histogram + GMM -> FCM -> PSO (fitness_mode) -> final IFCM at the
 * gbest (lambda*, xi*) from the gbest's (U, c) -> argmax labels.
 * Parity unpinned end to end (only oracle-vs-GPU agreement); its parts are
 * pinned individually. */
static int segment_core(const double *xin, const int64_t *histin, int nx, int ny, int nz, int C, double m,
                        int q_mode, int v, double h, double eps, int max_iter, int P, int ring_k, int max_gen,
                        int patience, double tol, double v0, double vmax, uint64_t seed, uint8_t *labels,
                        double *U_out, double *c_out, double *lam_xi_out, double *J_out, int *gens_out,
                        int *final_iters_out, double *c_init_out, int fitness_mode);

/* dtype 0 u8, 1 u16, 2 f32 (pifcm_dtype): normalise + histogram by type, then
 * the pipeline of orc_segment_u8. */
int orc_segment_typed(const void *vol, int dtype, int nx, int ny, int nz, int C, double m, int q_mode,
                      int v, double h, double eps, int max_iter,
                      int P, int ring_k, int max_gen, int patience, double tol, double v0,
                      double vmax, uint64_t seed,
                      uint8_t *labels, double *U_out, double *c_out,
                      double *lam_xi_out, double *J_out, int *gens_out, int *final_iters_out,
                      double *c_init_out, int fitness_mode) {
    const long N = (long)nx * ny * nz;
    double *x = (double *)malloc(sizeof(double) * (size_t)N);
    int64_t hist[256];
    if (dtype == 1) {
        orc_normalize_u16((const uint16_t *)vol, N, x);
        orc_histogram_u16((const uint16_t *)vol, N, hist);
    } else if (dtype == 2) {
        orc_normalize_f32((const float *)vol, N, x);
        orc_histogram_f32((const float *)vol, N, hist);
    } else {
        orc_normalize_u8((const uint8_t *)vol, N, x);
        orc_histogram_u8((const uint8_t *)vol, N, hist);
    }
    const int r = segment_core(x, hist, nx, ny, nz, C, m, q_mode, v, h, eps, max_iter, P, ring_k, max_gen,
                               patience, tol, v0, vmax, seed, labels, U_out, c_out, lam_xi_out, J_out, gens_out,
                               final_iters_out, c_init_out, fitness_mode);
    free(x);
    return r;
}

int orc_segment_u8(const uint8_t *vol, int nx, int ny, int nz, int C, double m, int q_mode,
                   int v, double h, double eps, int max_iter,
                   int P, int ring_k, int max_gen, int patience, double tol, double v0,
                   double vmax, uint64_t seed,
                   uint8_t *labels, double *U_out /*[N][C] nullable*/, double *c_out /*[C]*/,
                   double *lam_xi_out /*[2]*/, double *J_out, int *gens_out, int *final_iters_out,
                   double *c_init_out /*[C] nullable: GMM centres*/, int fitness_mode) {
    return orc_segment_typed(vol, 0, nx, ny, nz, C, m, q_mode, v, h, eps, max_iter, P, ring_k, max_gen, patience,
                             tol, v0, vmax, seed, labels, U_out, c_out, lam_xi_out, J_out, gens_out,
                             final_iters_out, c_init_out, fitness_mode);
}

static int segment_core(const double *xin, const int64_t *histin, int nx, int ny, int nz, int C, double m,
                        int q_mode, int v, double h, double eps, int max_iter, int P, int ring_k, int max_gen,
                        int patience, double tol, double v0, double vmax, uint64_t seed, uint8_t *labels,
                        double *U_out, double *c_out, double *lam_xi_out, double *J_out, int *gens_out,
                        int *final_iters_out, double *c_init_out, int fitness_mode) {
    const long N = (long)nx * ny * nz;
    const double *x = xin;
    double *U = (double *)malloc(sizeof(double) * (size_t)N * C);
    double *Ub = (double *)malloc(sizeof(double) * (size_t)N * C);
    int64_t hist[256];
    memcpy(hist, histin, sizeof hist);
    double c0[8], c1[8], cb[8], lx[2], Jb = 0.0;
    orc_gmm_init(hist, C, 100, c0);
    if (c_init_out) memcpy(c_init_out, c0, sizeof(double) * C);
    orc_fcm_run(x, N, C, m, eps, max_iter, c0, U, c1);
    const int gens = orc_pso_run(x, nx, ny, nz, C, m, q_mode, v, h, U, c1, P, ring_k, max_gen,
                                 patience, tol, v0, vmax, seed, lx, &Jb, Ub, cb, NULL, NULL, NULL,
                                 fitness_mode);
    double Jf = 0.0;
    const int fi = orc_ifcm_run(x, nx, ny, nz, C, m, lx[0], lx[1], q_mode, v, h, eps, max_iter,
                                Ub, cb, &Jf);
    orc_argmax(Ub, N, C, labels);
    if (U_out) memcpy(U_out, Ub, sizeof(double) * (size_t)N * C);
    memcpy(c_out, cb, sizeof(double) * C);
    lam_xi_out[0] = lx[0];
    lam_xi_out[1] = lx[1];
    *J_out = Jb;
    *gens_out = gens;
    *final_iters_out = fi;
    free(U); free(Ub);
    return 0;
}

/* The literal slice mode (R25; Alg. 1 with its input z: "The z
 * slice is assigned to a new variable"; "running through each voxel
 * in the slice of a particular z axis image"): the whole volume is normalised
 * (Alg. 2 step 1); the R15 histogram of slice z on the volume's levels feeds the
 * GMM; FCM runs on the slice; the rows of the neighbouring planes z - 1, z + 1
 * (where they exist) are the Eq. 2 memberships at the FCM centres c1 and stay
 * fixed; the PSO (CHAINED) and the final IFCM update only slice z (3D
 * neighbourhood, Eq. 3 / Eq. 1 over the slice).  Outputs: labels [ny][nx] and
 * optionally U_out [ny*nx][C] of the slice.  Pins: nz = 1 equals
 * orc_segment_u8; the plane-restricted step equals the whole step on the
 * target rows (tests/test_oracle_pso.py); end to end parity unpinned. */
int orc_segment_slice_u8(const uint8_t *vol, int nx, int ny, int nz, int z, int C, double m, int q_mode,
                         int v, double h, double eps, int max_iter, int P, int ring_k, int max_gen, int patience,
                         double tol,
                         double v0, double vmax, uint64_t seed, uint8_t *labels, double *U_out, double *c_out,
                         double *lam_xi_out, double *J_out, int *gens_out, int *final_iters_out,
                         double *c_init_out, int *fcm_iters_out) {
    if (z < 0 || z >= nz) return -1;
    const long N = (long)nx * ny * nz, pl = (long)nx * ny;
    double *x = (double *)malloc(sizeof(double) * (size_t)N);
    orc_normalize_u8(vol, N, x);
    int mn = 255, mx = 0;
    for (long i = 0; i < N; ++i) {
        if (vol[i] < mn) mn = vol[i];
        if (vol[i] > mx) mx = vol[i];
    }
    int64_t hist[256];
    orc_histogram_u8_range(vol + (long)z * pl, pl, mn, mx, hist);
    double c0[8], c1[8], cb[8], lx[2], Jb = 0.0;
    orc_gmm_init(hist, C, 100, c0);
    if (c_init_out) memcpy(c_init_out, c0, sizeof(double) * C);
    /* the neighbourhood planes of slice z (Eq. 9 radius v in z): sub-volume
     * [zs0, zs1), target t */
    const int zs0 = z - v > 0 ? z - v : 0, zs1 = z + v + 1 < nz ? z + v + 1 : nz, nzs = zs1 - zs0,
              t = z - zs0;
    const double *xs = x + (long)zs0 * pl;
    double *Us = (double *)malloc(sizeof(double) * (size_t)nzs * pl * C);
    double *Ub = (double *)malloc(sizeof(double) * (size_t)nzs * pl * C);
    const int fi0 = orc_fcm_run(xs + (long)t * pl, pl, C, m, eps, max_iter, c0, Us + (long)t * pl * C, c1);
    if (fcm_iters_out) *fcm_iters_out = fi0;
    for (int k = 0; k < nzs; ++k) {
        if (k == t) continue;
        double cn[8], Jh, duh;
        orc_fcm_step(xs + (long)k * pl, pl, C, m, c1, NULL, Us + (long)k * pl * C, cn, &Jh, &duh);
    }
    const int gens = pso_core(xs, nx, ny, nzs, t, t + 1, C, m, q_mode, v, h, Us, c1, P, ring_k, max_gen,
                              patience, tol, v0, vmax, seed, lx, &Jb, Ub, cb, NULL, NULL, NULL, 0);
    double Jf = 0.0;
    const int fi = ifcm_run_planes(xs, nx, ny, nzs, t, t + 1, C, m, lx[0], lx[1], q_mode, v, h, eps,
                                   max_iter, Ub, cb, &Jf);
    orc_argmax(Ub + (long)t * pl * C, pl, C, labels);
    if (U_out) memcpy(U_out, Ub + (long)t * pl * C, sizeof(double) * (size_t)pl * C);
    memcpy(c_out, cb, sizeof(double) * C);
    lam_xi_out[0] = lx[0];
    lam_xi_out[1] = lx[1];
    *J_out = Jb;
    *gens_out = gens;
    *final_iters_out = fi;
    free(x); free(Us); free(Ub);
    return 0;
}

/* incS ("incorrect segmentation", defined in the paper's
 * ref. [1]) on a phantom with known truth (R26): cluster j is mapped to the
 * tissue class of its rank among the centres (ascending; ties to the lower
 * index), classes being numbered by ascending intensity level; incS = the
 * number of voxels whose mapped label differs from the truth label. */
long orc_incs(const uint8_t *labels, const uint8_t *truth, long N, int C, const double *centers) {
    int rank[8];
    for (int j = 0; j < C; ++j) {
        int r = 0;
        for (int k = 0; k < C; ++k)
            if (centers[k] < centers[j] || (centers[k] == centers[j] && k < j)) ++r;
        rank[j] = r;
    }
    long bad = 0;
    for (long i = 0; i < N; ++i)
        if (rank[labels[i]] != truth[i]) ++bad;
    return bad;
}

/* Eq. 11: the speed / quality trade-off of A algorithms over
 * k image sizes, J_a(alpha) = 1/k sum_i alpha (incS_ia - min_i incS) /
 * (max_i incS - min_i incS) + (1 - alpha) (S_ia - min_i S) / (max_i S - min_i S),
 * min / max over the algorithms at size i; a term whose max equals its min
 * is 0 (R26).  incs, secs: [k][A] row-major. */
void orc_eq11(const double *incs, const double *secs, int k, int A, double alpha, double *J) {
    for (int a = 0; a < A; ++a) J[a] = 0.0;
    for (int i = 0; i < k; ++i) {
        double lo_q = incs[i * A], hi_q = incs[i * A], lo_s = secs[i * A], hi_s = secs[i * A];
        for (int a = 1; a < A; ++a) {
            if (incs[i * A + a] < lo_q) lo_q = incs[i * A + a];
            if (incs[i * A + a] > hi_q) hi_q = incs[i * A + a];
            if (secs[i * A + a] < lo_s) lo_s = secs[i * A + a];
            if (secs[i * A + a] > hi_s) hi_s = secs[i * A + a];
        }
        for (int a = 0; a < A; ++a) {
            const double q = hi_q > lo_q ? (incs[i * A + a] - lo_q) / (hi_q - lo_q) : 0.0;
            const double t = hi_s > lo_s ? (secs[i * A + a] - lo_s) / (hi_s - lo_s) : 0.0;
            J[a] += alpha * q + (1.0 - alpha) * t;
        }
    }
    for (int a = 0; a < A; ++a) J[a] /= (double)k;
}
