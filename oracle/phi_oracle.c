/*
 * phi_oracle.c -- CPU restatement of the reference fine propagator Phi.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path and the "port" CPU baseline timed by `bench.py --impl reference`.  It
 * is never linked into, loaded by, or called from the product library
 * paper_2104_09404_b200/libmgrit_phi.so.
 *
 * It restates, operation by operation, what the reference computes with
 * NumPy for RungeKuttaStepper.advance (stepper.py:50-82) over
 * SemiDiscreteOperator.rhs (flux.py:129-161):
 *   - periodic windows (weno.py:191-199, 219-221): left window of interface
 *     i+1/2 = cells i-k..i+k, right window = cells i+1+k, ..., i+1-k, both
 *     through reconstruct_left (weno.py:234-235);
 *   - candidates  q_r = sum_t cw[r,t] w_t                      (weno.py:175)
 *       summed sequentially when advance() got >= 2 fields, and in "2-lane"
 *       order (even window slots) + (odd window slots) for a single field --
 *       the NumPy einsum contiguity quirk;
 *   - smoothness  beta_r = sum_a sum_b (w_a B[r,a,b]) w_b, a-major, from +0
 *                                                         (weno.py:154-158);
 *   - weights     raw_r = d_r/((eps+beta_r)(eps+beta_r)), S = sum_r raw_r,
 *                 omega_r = raw_r/S, value = sum_r omega_r q_r
 *                                                 (weno.py:161-168,176-177);
 *   - global LF:  alpha = NaN-propagating max over |uL|, |uR| of the field
 *                 (flux.py:70-79, models.py:115-117), advection: |a|;
 *                 F = (0.5 (f(uL)+f(uR))) - ((0.5 alpha)(uR-uL))
 *                 with f(u) = (0.5 u) u (models.py:107-109)  (flux.py:82-88);
 *   - rhs         A_i = (-(F_i - F_{i-1})) / dx               (flux.py:159-161);
 *   - SSP RK 1/2/3 in Shu-Osher form with Python's left-to-right evaluation
 *     (scalar products such as 0.25*dt first)                (stepper.py:50-62).
 * Zero table entries are skipped; for finite windows this is exact (0*w is a
 * signed zero), and a window holding any non-finite value reconstructs to
 * NaN, which is what the reference's 0*inf terms produce.
 *
 * Build: oracle/Makefile (gcc -O3 -ffp-contract=off, no fast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define ORA_MODEL_BURGERS 0
#define ORA_MODEL_ADVECTION 1
#define ORA_MODEL_SHALLOW_WATER 2   /* D = 2: (h, hu), characteristic WENO */
#define ORA_MODEL_EULER 3           /* D = 3: (rho, rho u, E)               */
/* bad_state bits (the reference's PhysicalStateError cases) */
#define ORA_BAD_DEPTH 1       /* models.py:147-153 */
#define ORA_BAD_DENSITY 2     /* models.py:228-232 */
#define ORA_BAD_PRESSURE 4    /* models.py:235-238 */
#define ORA_BAD_ROE 8         /* models.py:290-293 */
#define ORA_SUM_SEQ 0
#define ORA_SUM_LANE2 1

typedef struct {
    int32_t model;     /* 0 burgers, 1 linear advection                     */
    int32_t k;         /* WENO degree 0..3 (order 2k+1)                      */
    int32_t rk_order;  /* 1 FE, 2 SSP-RK2, 3 SSP-RK3; 0 = semi-discrete rhs  */
    int32_t regime;    /* ORA_SUM_SEQ / ORA_SUM_LANE2                        */
    double dt, dx, eps, speed;
    int32_t scheme;    /* 0 RK/WENO, 1 one-step LF, 2 matched LF (coarse)    */
    int32_t lf_order;  /* matched: 0 or 1                                     */
    int32_t m_eff;     /* matched: fine steps emulated                        */
    int32_t repeats;   /* composition count (ComposedStepper), >= 1           */
    double gravity;    /* shallow water g                                     */
    double gamma;      /* Euler ratio of specific heats                       */
    int32_t characteristic;  /* systems: 1 characteristic, 0 componentwise  */
    int32_t reserved;
} ora_params;

static int ncomp(const ora_params *p) {
    return p->model == ORA_MODEL_SHALLOW_WATER ? 2 : (p->model == ORA_MODEL_EULER ? 3 : 1);
}

/* ---- exact rational tables, weno.py:43-86.  IEEE division of the small
 * integers gives the correctly rounded double, i.e. float(Fraction(p, q)). */
static const int CW_NUM[4][4][4] = {
    {{1}},
    {{1, 1}, {-1, 3}},
    {{2, 5, -1}, {-1, 5, 2}, {2, -7, 11}},
    {{3, 13, -5, 1}, {-1, 7, 7, -1}, {1, -5, 13, 3}, {-3, 13, -23, 25}}};
static const int CW_DEN[4] = {1, 2, 6, 12};
static const int D_NUM[4][4] = {{1}, {2, 1}, {3, 6, 1}, {4, 18, 12, 1}};
static const int D_DEN[4] = {1, 3, 10, 35};
static const int SM_NUM[4][4][4][4] = {
    {{{0}}},
    {{{1, -1}, {-1, 1}}, {{1, -1}, {-1, 1}}},
    {{{20, -31, 11}, {-31, 50, -19}, {11, -19, 8}},
     {{8, -13, 5}, {-13, 26, -13}, {5, -13, 8}},
     {{8, -19, 11}, {-19, 50, -31}, {11, -31, 20}}},
    {{{2107, -4701, 3521, -927}, {-4701, 11003, -8623, 2321},
      {3521, -8623, 7043, -1941}, {-927, 2321, -1941, 547}},
     {{547, -1261, 961, -247}, {-1261, 3443, -2983, 801},
      {961, -2983, 2843, -821}, {-247, 801, -821, 267}},
     {{267, -821, 801, -247}, {-821, 2843, -2983, 961},
      {801, -2983, 3443, -1261}, {-247, 961, -1261, 547}},
     {{547, -1941, 2321, -927}, {-1941, 7043, -8623, 3521},
      {2321, -8623, 11003, -4701}, {-927, 3521, -4701, 2107}}}};
static const int SM_DEN[4] = {1, 1, 6, 240};

typedef struct {
    int k;
    double eps;
    double cw[4][4];      /* cw[r][j] multiplies window slot (k-r)+j        */
    double d[4];
    double sm[4][4][4];   /* sm[r][i][j] pairs window slots (k-r)+i, (k-r)+j */
} ora_tables;

static void build_tables(int k, double eps, ora_tables *t) {
    memset(t, 0, sizeof(*t));
    t->k = k;
    t->eps = eps;
    for (int r = 0; r <= k; ++r) {
        t->d[r] = (double)D_NUM[k][r] / (double)D_DEN[k];
        for (int j = 0; j <= k; ++j) {
            t->cw[r][j] = (double)CW_NUM[k][r][j] / (double)CW_DEN[k];
            for (int i = 0; i <= k; ++i)
                t->sm[r][i][j] = (double)SM_NUM[k][r][i][j] / (double)SM_DEN[k];
        }
    }
}

/* Exported for the table-equality test (tables vs float(Fraction)). */
int ora_get_tables(int k, double *cw16, double *d4, double *sm64) {
    if (k < 0 || k > 3) return 1;
    ora_tables t;
    build_tables(k, 1e-6, &t);
    memcpy(cw16, t.cw, sizeof(t.cw));
    memcpy(d4, t.d, sizeof(t.d));
    memcpy(sm64, t.sm, sizeof(t.sm));
    return 0;
}

/* reconstruct_left (weno.py:171-177) on the window w[0..2k] */
static double recon(const ora_tables *t, int regime, const double *w) {
    const int k = t->k;
    for (int s = 0; s <= 2 * k; ++s)
        if (!isfinite(w[s])) return NAN;
    double q[4] = {0, 0, 0, 0}, raw[4] = {0, 0, 0, 0};
    for (int r = 0; r <= k; ++r) {
        const int lo = k - r;
        if (regime == ORA_SUM_SEQ) {
            double acc = t->cw[r][0] * w[lo];
            for (int j = 1; j <= k; ++j) acc = acc + t->cw[r][j] * w[lo + j];
            q[r] = acc;
        } else {
            double ev = 0.0, od = 0.0;
            int he = 0, ho = 0;
            for (int j = 0; j <= k; ++j) {
                const int s = lo + j;
                const double p = t->cw[r][j] * w[s];
                if ((s & 1) == 0) { ev = he ? ev + p : p; he = 1; }
                else { od = ho ? od + p : p; ho = 1; }
            }
            q[r] = he ? (ho ? ev + od : ev) : od;
        }
        double b = 0.0;
        for (int i = 0; i <= k; ++i)
            for (int j = 0; j <= k; ++j)
                b = b + (w[lo + i] * t->sm[r][i][j]) * w[lo + j];
        const double e = t->eps + b;
        raw[r] = t->d[r] / (e * e);
    }
    double S = raw[0];
    for (int r = 1; r <= k; ++r) S = S + raw[r];
    double v = (raw[0] / S) * q[0];
    for (int r = 1; r <= k; ++r) v = v + (raw[r] / S) * q[r];
    return v;
}

typedef struct {
    int64_t nx;    /* cells */
    int64_t len;   /* doubles per state: ncomp * nx */
    double *pad;   /* field with k+1 periodic halo cells on both sides */
    double *ul, *ur, *F, *A, *u1, *u2, *tmp;
    int bad_state; /* PhysicalStateError: non-positive depth met */
} ora_work;

static int work_alloc(ora_work *w, int64_t nx, int k, int D) {
    w->nx = nx;
    w->len = D * nx;
    w->bad_state = 0;
    const int64_t H = k + 1;
    w->pad = (double *)malloc(sizeof(double) * (size_t)(D * (nx + 2 * H)));
    w->ul = (double *)malloc(sizeof(double) * (size_t)w->len * 7);
    if (!w->pad || !w->ul) { free(w->pad); free(w->ul); return 1; }
    w->ur = w->ul + w->len;
    w->F = w->ur + w->len;
    w->A = w->F + w->len;
    w->u1 = w->A + w->len;
    w->u2 = w->u1 + w->len;
    w->tmp = w->u2 + w->len;
    return 0;
}

static void work_free(ora_work *w) { free(w->pad); free(w->ul); }

/* SemiDiscreteOperator.rhs (flux.py:159-161) for one field v -> A */
static void rhs_field(const ora_params *p, const ora_tables *t, ora_work *wk,
                      const double *v, double *A) {
    const int64_t nx = wk->nx;
    const int k = t->k, H = k + 1;
    double *pad = wk->pad;
    for (int64_t i = 0; i < nx; ++i) pad[H + i] = v[i];
    for (int h = 0; h < H; ++h) {
        pad[h] = v[((nx - H + h) % nx + nx) % nx];
        pad[H + nx + h] = v[h % nx];
    }

    double w[7];
    for (int64_t i = 0; i < nx; ++i) {
        const double *c = pad + H + i;              /* cell i */
        for (int s = 0; s <= 2 * k; ++s) w[s] = c[s - k];
        wk->ul[i] = recon(t, p->regime, w);
        for (int s = 0; s <= 2 * k; ++s) w[s] = c[1 + k - s];
        wk->ur[i] = recon(t, p->regime, w);
    }
    if (p->scheme == 3) {
        /* Roe flux with Harten-Hyman entropy fix, Burgers (flux.py:91-126,
         * models.py:125-128): strength = 1*jump, speed from entropy_fix,
         * F = 0.5 (fL + fR) - 0.5 (speed * jump). */
        for (int64_t i = 0; i < nx; ++i) {
            const double l = wk->ul[i], r = wk->ur[i];
            const double fl = (0.5 * l) * l, fr = (0.5 * r) * r;
            const double lam = 0.5 * (l + r);
            const double a = lam - l, b = r - lam;
            const double inner = (a >= b || isnan(a)) ? a : b;      /* np.maximum */
            const double delta = (0.0 >= inner) ? 0.0 : inner;      /* NaN -> inner */
            const double alam = fabs(lam);
            const double speed = (alam < delta) ? 0.5 * ((lam * lam) / delta + delta) : alam;
            wk->F[i] = (0.5 * (fl + fr)) - (0.5 * (speed * (r - l)));
        }
        for (int64_t i = 0; i < nx; ++i) {
            const double fm = wk->F[i == 0 ? nx - 1 : i - 1];
            A[i] = (-(wk->F[i] - fm)) / p->dx;
        }
        return;
    }
    double alpha;
    if (p->model == ORA_MODEL_BURGERS) {
        /* np.max over interfaces (NaN-propagating), then np.maximum */
        double ml = 0.0, mr = 0.0;
        int nan = 0;
        for (int64_t i = 0; i < nx; ++i) {
            const double a = fabs(wk->ul[i]), b = fabs(wk->ur[i]);
            if (isnan(a) || isnan(b)) nan = 1;
            if (a > ml) ml = a;
            if (b > mr) mr = b;
        }
        alpha = nan ? NAN : (ml > mr ? ml : mr);
    } else {
        alpha = fabs(p->speed);
    }
    const double half_alpha = 0.5 * alpha;
    for (int64_t i = 0; i < nx; ++i) {
        const double l = wk->ul[i], r = wk->ur[i];
        double fl, fr;
        if (p->model == ORA_MODEL_BURGERS) { fl = (0.5 * l) * l; fr = (0.5 * r) * r; }
        else { fl = p->speed * l; fr = p->speed * r; }
        wk->F[i] = (0.5 * (fl + fr)) - (half_alpha * (r - l));
    }
    for (int64_t i = 0; i < nx; ++i) {
        const double fm = wk->F[i == 0 ? nx - 1 : i - 1];
        A[i] = (-(wk->F[i] - fm)) / p->dx;
    }
}

/* ---- systems: shallow water (models.py:136-211) and Euler (models.py:
 * 214-308); characteristic WENO (weno.py:203-233), LF or Roe flux
 * (flux.py:70-126).  States are component-major rows of D*nx.  Checked
 * against the reference bit for bit for shallow water; for Euler the left
 * eigenvectors are np.linalg.inv of the right ones (models.py:270), restated
 * by inv3() below (LU with partial pivoting), which agrees with LAPACK to
 * rounding -- everything else is pinned bit for bit by running the
 * reference with inv3 substituted (tests/golden/make_golden.py "euler").
 * The einsum contractions over the component axis accumulate in two lanes
 * from +0 -- (0 + x0 + x2) + (0 + x1) -- (lane2(), verified per call site
 * against the reference); the characteristic windows are fresh contiguous
 * arrays, so their candidate sums use the 2-lane order too. */
static double lane2(const double *x, int n) {
    double ev = 0.0, od = 0.0;
    for (int i = 0; i < n; ++i) {
        if (i & 1) od = od + x[i];
        else ev = ev + x[i];
    }
    return ev + od;
}

typedef struct {
    double lam[3];
    double R[3][3];   /* columns: right eigenvectors */
    double L[3][3];   /* rows: left eigenvectors     */
} ora_eig;

/* np.linalg.inv for 3x3: LU with partial pivoting (first maximal |pivot|),
 * multipliers scaled by the reciprocal pivot, rank-1 updates, then forward
 * (unit lower) and backward (dividing by the pivot) substitution of each
 * column of P I, skipping zero entries -- LAPACK dgetf2/dgetrs order */
static void inv3(const double A[3][3], double X[3][3]) {
    double a[3][3];
    int perm[3] = {0, 1, 2};
    memcpy(a, A, sizeof a);
    for (int j = 0; j < 3; ++j) {
        int pv = j;
        double best = fabs(a[j][j]);
        for (int i = j + 1; i < 3; ++i)
            if (fabs(a[i][j]) > best) { best = fabs(a[i][j]); pv = i; }
        if (pv != j) {
            for (int c = 0; c < 3; ++c) { double t = a[j][c]; a[j][c] = a[pv][c]; a[pv][c] = t; }
            int t = perm[j]; perm[j] = perm[pv]; perm[pv] = t;
        }
        const double rp = 1.0 / a[j][j];
        for (int i = j + 1; i < 3; ++i) a[i][j] = a[i][j] * rp;
        for (int i = j + 1; i < 3; ++i)
            for (int c = j + 1; c < 3; ++c) a[i][c] = a[i][c] - a[i][j] * a[j][c];
    }
    for (int col = 0; col < 3; ++col) {
        double b[3];
        for (int i = 0; i < 3; ++i) b[i] = perm[i] == col ? 1.0 : 0.0;
        for (int kk = 0; kk < 3; ++kk)
            if (b[kk] != 0.0)
                for (int i = kk + 1; i < 3; ++i) b[i] = b[i] - b[kk] * a[i][kk];
        for (int kk = 2; kk >= 0; --kk)
            if (b[kk] != 0.0) {
                b[kk] = b[kk] / a[kk][kk];
                for (int i = 0; i < kk; ++i) b[i] = b[i] - b[kk] * a[i][kk];
            }
        for (int i = 0; i < 3; ++i) X[i][col] = b[i];
    }
}

/* velocity (and Euler pressure) of a state, flagging inadmissible ones */
static double sys_vel(const ora_params *p, ora_work *wk, const double *s, double *pr) {
    if (p->model == ORA_MODEL_SHALLOW_WATER) {
        if (s[0] <= 0.0) wk->bad_state |= ORA_BAD_DEPTH;
        return s[1] / s[0];
    }
    if (s[0] <= 0.0) wk->bad_state |= ORA_BAD_DENSITY;
    const double vel = s[1] / s[0];
    *pr = (p->gamma - 1.0) * (s[2] - ((0.5 * s[0]) * vel) * vel);
    if (*pr <= 0.0) wk->bad_state |= ORA_BAD_PRESSURE;
    return vel;
}

/* wave speed c of a state with velocity vel (and pressure pr) */
static double sys_c(const ora_params *p, const double *s, double pr) {
    if (p->model == ORA_MODEL_SHALLOW_WATER) return sqrt(p->gravity * s[0]);
    return sqrt((p->gamma * pr) / s[0]);
}

static void sys_flux(const ora_params *p, ora_work *wk, const double *s, double *f) {
    double pr = 0.0;
    const double vel = sys_vel(p, wk, s, &pr);
    if (p->model == ORA_MODEL_SHALLOW_WATER) {
        f[0] = s[1];
        f[1] = ((s[0] * vel) * vel) + (((0.5 * p->gravity) * s[0]) * s[0]);
    } else {
        f[0] = s[1];
        f[1] = (s[1] * vel) + pr;
        f[2] = (s[2] + pr) * vel;
    }
}

static double sys_speed(const ora_params *p, ora_work *wk, const double *s) {
    double pr = 0.0;
    const double vel = sys_vel(p, wk, s, &pr);
    return fabs(vel) + sys_c(p, s, pr);
}

static void sys_eigenvalues(const ora_params *p, ora_work *wk, const double *s, double *lam) {
    double pr = 0.0;
    const double vel = sys_vel(p, wk, s, &pr);
    const double c = sys_c(p, s, pr);
    if (p->model == ORA_MODEL_SHALLOW_WATER) {
        lam[0] = vel - c; lam[1] = vel + c;
    } else {
        lam[0] = vel - c; lam[1] = vel; lam[2] = vel + c;
    }
}

/* eigen structure from (vel, c[, enthalpy]) -- models.py:159-176, 262-271 */
static void sys_eigen_from(const ora_params *p, double vel, double c, double H, ora_eig *e) {
    if (p->model == ORA_MODEL_SHALLOW_WATER) {
        const double inv2c = 0.5 / c;
        e->lam[0] = vel - c; e->lam[1] = vel + c;
        e->R[0][0] = 1.0; e->R[0][1] = 1.0; e->R[1][0] = vel - c; e->R[1][1] = vel + c;
        e->L[0][0] = (vel + c) * inv2c; e->L[0][1] = -1.0 * inv2c;
        e->L[1][0] = (-(vel - c)) * inv2c; e->L[1][1] = 1.0 * inv2c;
        return;
    }
    e->lam[0] = vel - c; e->lam[1] = vel; e->lam[2] = vel + c;
    e->R[0][0] = 1.0; e->R[0][1] = 1.0; e->R[0][2] = 1.0;
    e->R[1][0] = vel - c; e->R[1][1] = vel; e->R[1][2] = vel + c;
    e->R[2][0] = H - vel * c; e->R[2][1] = (0.5 * vel) * vel; e->R[2][2] = H + vel * c;
    inv3(e->R, e->L);
}

static void sys_eigen_cell(const ora_params *p, ora_work *wk, const double *s, ora_eig *e) {
    double pr = 0.0;
    const double vel = sys_vel(p, wk, s, &pr);
    const double c = sys_c(p, s, pr);
    const double H = p->model == ORA_MODEL_EULER ? (s[2] + pr) / s[0] : 0.0;
    sys_eigen_from(p, vel, c, H, e);
}

/* Roe linearisation (models.py:178-200, 280-300) */
static void sys_eigen_roe(const ora_params *p, ora_work *wk, const double *l, const double *r,
                          ora_eig *e) {
    double pl = 0.0, prr = 0.0;
    const double vl = sys_vel(p, wk, l, &pl), vr = sys_vel(p, wk, r, &prr);
    const double sl = sqrt(l[0]), sr = sqrt(r[0]);
    if (p->model == ORA_MODEL_SHALLOW_WATER) {
        const double hh = 0.5 * (l[0] + r[0]);
        const double uh = (sl * vl + sr * vr) / (sl + sr);
        sys_eigen_from(p, uh, sqrt(p->gravity * hh), 0.0, e);
        return;
    }
    const double hl = (l[2] + pl) / l[0], hr = (r[2] + prr) / r[0];
    const double uh = (sl * vl + sr * vr) / (sl + sr);
    const double Hh = (sl * hl + sr * hr) / (sl + sr);
    const double csq = (p->gamma - 1.0) * (Hh - (0.5 * uh) * uh);
    if (csq <= 0.0) wk->bad_state |= ORA_BAD_ROE;
    sys_eigen_from(p, uh, sqrt(csq), Hh, e);
}

static double entropy_fix1(double lh, double ll, double lr) {
    const double a = lh - ll, b = lr - lh;
    const double inner = (a >= b || isnan(a)) ? a : b;
    const double delta = (0.0 >= inner) ? 0.0 : inner;
    const double alam = fabs(lh);
    return (alam < delta) ? 0.5 * ((lh * lh) / delta + delta) : alam;
}

static void sys_rhs_field(const ora_params *p, const ora_tables *t, ora_work *wk,
                          const double *v, double *A) {
    const int64_t nx = wk->nx;
    const int k = t->k, W = 2 * k + 1, D = ncomp(p);
    double *sl = wk->ul, *sr = wk->ur, *F = wk->F;   /* component-major (D, nx) */
    for (int64_t i = 0; i < nx; ++i) {
        const int64_t ip = (i + 1) % nx;
        ora_eig e[2];
        if (p->characteristic) {
            double s0[3], s1[3];
            for (int d = 0; d < D; ++d) { s0[d] = v[d * nx + i]; s1[d] = v[d * nx + ip]; }
            sys_eigen_cell(p, wk, s0, &e[0]);
            sys_eigen_cell(p, wk, s1, &e[1]);
        }
        for (int side = 0; side < 2; ++side) {
            double win[3][7], rec[3];
            for (int s2 = 0; s2 < W; ++s2) {
                /* left window: cells i-k+s2; right window: cells i+1+k-s2 */
                const int64_t c = side == 0 ? (i - k + s2) : (i + 1 + k - s2);
                const int64_t cc = ((c % nx) + nx) % nx;
                for (int d = 0; d < D; ++d) win[d][s2] = v[d * nx + cc];
            }
            double *dst = side == 0 ? sl : sr;
            if (!p->characteristic) {
                /* (..., D, N, W) windows: >= 2 fields, sequential sums */
                for (int d = 0; d < D; ++d) dst[d * nx + i] = recon(t, ORA_SUM_SEQ, win[d]);
                continue;
            }
            const ora_eig *E = &e[side];
            double ch[3][7];
            double term[3];
            for (int s2 = 0; s2 < W; ++s2)
                for (int q = 0; q < D; ++q) {
                    for (int d = 0; d < D; ++d) term[d] = E->L[q][d] * win[d][s2];
                    ch[q][s2] = lane2(term, D);
                }
            for (int q = 0; q < D; ++q) rec[q] = recon(t, ORA_SUM_LANE2, ch[q]);
            for (int d = 0; d < D; ++d) {
                for (int q = 0; q < D; ++q) term[q] = E->R[d][q] * rec[q];
                dst[d * nx + i] = lane2(term, D);
            }
        }
    }
    if (p->scheme == 3) {                       /* Roe, flux.py:91-126 */
        for (int64_t i = 0; i < nx; ++i) {
            double l[3], r[3], jump[3], lamL[3], lamR[3], fl[3], fr[3], ss[3];
            for (int d = 0; d < D; ++d) {
                l[d] = sl[d * nx + i];
                r[d] = sr[d * nx + i];
                jump[d] = r[d] - l[d];
            }
            ora_eig e;
            sys_eigen_roe(p, wk, l, r, &e);
            sys_eigenvalues(p, wk, l, lamL);
            sys_eigenvalues(p, wk, r, lamR);
            double term[3];
            for (int kk = 0; kk < D; ++kk) {
                for (int d = 0; d < D; ++d) term[d] = e.L[kk][d] * jump[d];
                ss[kk] = entropy_fix1(e.lam[kk], lamL[kk], lamR[kk]) * lane2(term, D);
            }
            sys_flux(p, wk, l, fl);
            sys_flux(p, wk, r, fr);
            for (int d = 0; d < D; ++d) {
                for (int kk = 0; kk < D; ++kk) term[kk] = ss[kk] * e.R[d][kk];
                F[d * nx + i] = (0.5 * (fl[d] + fr[d])) - (0.5 * lane2(term, D));
            }
        }
    } else {                                    /* global LF, flux.py:70-88 */
        double ml = 0.0, mr = 0.0;
        int nan = 0;
        for (int64_t i = 0; i < nx; ++i) {
            double l[3], r[3];
            for (int d = 0; d < D; ++d) { l[d] = sl[d * nx + i]; r[d] = sr[d * nx + i]; }
            const double a = sys_speed(p, wk, l), b = sys_speed(p, wk, r);
            if (isnan(a) || isnan(b)) nan = 1;
            if (a > ml) ml = a;
            if (b > mr) mr = b;
        }
        const double alpha = nan ? NAN : (ml > mr ? ml : mr);
        const double ha = 0.5 * alpha;
        for (int64_t i = 0; i < nx; ++i) {
            double l[3], r[3], fl[3], fr[3];
            for (int d = 0; d < D; ++d) { l[d] = sl[d * nx + i]; r[d] = sr[d * nx + i]; }
            sys_flux(p, wk, l, fl);
            sys_flux(p, wk, r, fr);
            for (int d = 0; d < D; ++d)
                F[d * nx + i] = (0.5 * (fl[d] + fr[d])) - (ha * (r[d] - l[d]));
        }
    }
    for (int d = 0; d < D; ++d)
        for (int64_t i = 0; i < nx; ++i) {
            const double fm = F[d * nx + (i == 0 ? nx - 1 : i - 1)];
            A[d * nx + i] = (-(F[d * nx + i] - fm)) / p->dx;
        }
}

/* E(u)_i = 0.5 (u_{i+1} + u_{i-1})  (stepper.py:85-87) */
static void ora_E(const double *u, double *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        out[i] = 0.5 * (u[i + 1 == n ? 0 : i + 1] + u[i == 0 ? n - 1 : i - 1]);
}

/* D(f)_i = (f_{i+1} - f_{i-1}) / (2 dx)  (stepper.py:90-92) */
static void ora_D(const double *f, double dx, double *out, int64_t n) {
    const double twodx = 2.0 * dx;
    for (int64_t i = 0; i < n; ++i)
        out[i] = (f[i + 1 == n ? 0 : i + 1] - f[i == 0 ? n - 1 : i - 1]) / twodx;
}

/* MatchedLFFine / RediscretizedLF (stepper.py:102-114,155-167) and
 * MatchedLFCoarse (stepper.py:117-152); Burgers flux (0.5 u) u. */
static void lf_field(const ora_params *p, ora_work *wk, const double *u, double *out) {
    const int64_t n = wk->nx;
    double *f = wk->ul, *d = wk->ur, *v = wk->F, *v2 = wk->A, *acc = wk->u1, *e = wk->u2;
    for (int64_t i = 0; i < n; ++i) f[i] = (0.5 * u[i]) * u[i];
    if (p->scheme == 1) {
        ora_E(u, v, n);
        ora_D(f, p->dx, d, n);
        for (int64_t i = 0; i < n; ++i) out[i] = v[i] - (p->dt * d[i]);
        return;
    }
    if (p->lf_order == 0) {
        memcpy(v, u, sizeof(double) * (size_t)n);
        for (int j = 0; j < p->m_eff; ++j) {
            ora_E(v, v2, n);
            memcpy(v, v2, sizeof(double) * (size_t)n);
        }
        ora_D(f, p->dx, d, n);
        for (int64_t i = 0; i < n; ++i) out[i] = v[i] - (p->dt * d[i]);
        return;
    }
    ora_D(f, p->dx, acc, n);
    memcpy(v, u, sizeof(double) * (size_t)n);
    for (int j = 0; j < p->m_eff - 1; ++j) {
        ora_E(v, v2, n);
        memcpy(v, v2, sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < n; ++i) f[i] = (0.5 * v[i]) * v[i];
        ora_E(acc, e, n);
        ora_D(f, p->dx, d, n);
        for (int64_t i = 0; i < n; ++i) acc[i] = e[i] + d[i];
    }
    ora_E(v, v2, n);
    for (int64_t i = 0; i < n; ++i) out[i] = v2[i] - (p->dt * acc[i]);
}

/* RungeKuttaStepper.advance (stepper.py:50-82) + optional relaxation "+ g" */
static void phi_once(const ora_params *p, const ora_tables *t, ora_work *wk,
                     const double *u, double *out);

/* ComposedStepper (stepper.py:170-188): inner^repeats, then "+ g" */
static void phi_field(const ora_params *p, const ora_tables *t, ora_work *wk,
                      const double *u, const double *g, double *out) {
    const int64_t nx = wk->len;
    phi_once(p, t, wk, u, out);
    for (int r = 1; r < p->repeats; ++r) {
        memcpy(wk->tmp, out, sizeof(double) * (size_t)nx);
        phi_once(p, t, wk, wk->tmp, out);
    }
    if (g)
        for (int64_t i = 0; i < nx; ++i) out[i] = out[i] + g[i];
}

static void any_rhs(const ora_params *p, const ora_tables *t, ora_work *wk,
                    const double *v, double *A) {
    if (ncomp(p) > 1) sys_rhs_field(p, t, wk, v, A);
    else rhs_field(p, t, wk, v, A);
}

static void phi_once(const ora_params *p, const ora_tables *t, ora_work *wk,
                     const double *u, double *out) {
    const int64_t nx = wk->len;   /* elementwise RK over every component */
    double *A = wk->A, *u1 = wk->u1, *u2 = wk->u2;
    if (p->scheme == 1 || p->scheme == 2) {
        lf_field(p, wk, u, out);
        return;
    }
    if (p->rk_order == 0) {
        any_rhs(p, t, wk, u, out);
        return;
    }
    const double dt = p->dt;
    any_rhs(p, t, wk, u, A);
    for (int64_t i = 0; i < nx; ++i) u1[i] = u[i] + dt * A[i];
    if (p->rk_order == 1) {
        for (int64_t i = 0; i < nx; ++i) out[i] = u1[i];
    } else if (p->rk_order == 2) {
        const double hdt = 0.5 * dt;
        any_rhs(p, t, wk, u1, A);
        for (int64_t i = 0; i < nx; ++i)
            out[i] = ((0.5 * u[i]) + (0.5 * u1[i])) + (hdt * A[i]);
    } else {
        const double qdt = 0.25 * dt;
        const double two3 = 2.0 / 3.0;
        const double tdt = two3 * dt;
        any_rhs(p, t, wk, u1, A);
        for (int64_t i = 0; i < nx; ++i)
            u2[i] = ((0.75 * u[i]) + (0.25 * u1[i])) + (qdt * A[i]);
        any_rhs(p, t, wk, u2, A);
        for (int64_t i = 0; i < nx; ++i)
            out[i] = ((u[i] / 3.0) + (two3 * u2[i])) + (tdt * A[i]);
    }
}

static int check_params(const ora_params *p, int64_t nx) {
    if (!p || p->repeats < 1) return 1;
    if (p->scheme == 1 || p->scheme == 2)
        return (p->model != ORA_MODEL_BURGERS || nx < 1 ||
                (p->scheme == 2 && (p->m_eff < 1 || p->lf_order < 0 || p->lf_order > 1)));
    if (p->scheme != 0 && p->scheme != 3) return 1;
    if (p->scheme == 3 && p->model == ORA_MODEL_ADVECTION) return 1;
    if (p->model == ORA_MODEL_SHALLOW_WATER && !(p->gravity > 0.0)) return 1;
    if (p->model == ORA_MODEL_EULER && !(p->gamma > 1.0)) return 1;
    if (p->k < 0 || p->k > 3) return 1;
    if (p->rk_order < 0 || p->rk_order > 3) return 1;
    if (p->model < ORA_MODEL_BURGERS || p->model > ORA_MODEL_EULER) return 1;
    if (p->regime != ORA_SUM_SEQ && p->regime != ORA_SUM_LANE2) return 1;
    if (nx < 2 * p->k + 1) return 1;
    return 0;
}

/* worker pool: fields are independent, threads take them off a shared counter */
typedef struct {
    const ora_params *p;
    const ora_tables *t;
    const double *u, *g;
    double *out;
    int64_t u_stride, g_stride, out_stride, batch, nx;
    int64_t next;
    pthread_mutex_t lock;
    int err;
    int bad;
} ora_job;

static void *ora_worker(void *arg) {
    ora_job *job = (ora_job *)arg;
    ora_work wk;
    if (work_alloc(&wk, job->nx, job->p->k, ncomp(job->p))) {
        pthread_mutex_lock(&job->lock);
        job->err = 1;
        pthread_mutex_unlock(&job->lock);
        return NULL;
    }
    for (;;) {
        pthread_mutex_lock(&job->lock);
        const int64_t b = job->next++;
        pthread_mutex_unlock(&job->lock);
        if (b >= job->batch) break;
        phi_field(job->p, job->t, &wk, job->u + b * job->u_stride,
                  job->g ? job->g + b * job->g_stride : NULL,
                  job->out + b * job->out_stride);
    }
    if (wk.bad_state) {
        pthread_mutex_lock(&job->lock);
        job->bad |= wk.bad_state;
        pthread_mutex_unlock(&job->lock);
    }
    work_free(&wk);
    return NULL;
}

int ora_max_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

/*
 * out[b] = Phi(u[b]) (+ g[b] when g != NULL) for b < batch; rows of nx
 * doubles with the given strides (in elements).  u_stride 0 broadcasts one
 * state.  Fields are independent and are spread over nthreads POSIX threads
 * (nthreads <= 0: one per online core).  Rows hold ncomp(model) * nx doubles
 * (component-major).  Returns 0, 1 on bad arguments, 2 on allocation failure,
 * 2 + (ORA_BAD_* bits) when an inadmissible state was met (the reference's
 * PhysicalStateError).
 */
int ora_phi_apply(const ora_params *p, const double *u, int64_t u_stride,
                  const double *g, int64_t g_stride, double *out,
                  int64_t out_stride, int64_t batch, int64_t nx, int nthreads) {
    if (check_params(p, nx) || batch < 0) return 1;
    ora_tables t;
    build_tables(p->k, p->eps, &t);
    if (nthreads <= 0) nthreads = ora_max_threads();
    if (nthreads > batch) nthreads = batch > 0 ? (int)batch : 1;
    ora_job job = {p, &t, u, g, out, u_stride, g_stride, out_stride, batch, nx,
                   0, PTHREAD_MUTEX_INITIALIZER, 0, 0};
    if (nthreads == 1) {
        ora_worker(&job);
        return job.err ? 2 : (job.bad ? 2 + job.bad : 0);
    }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    if (!th) return 2;
    int started = 0;
    for (int i = 0; i < nthreads; ++i)
        if (pthread_create(&th[i], NULL, ora_worker, &job) == 0) ++started;
    if (started == 0) ora_worker(&job);
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
    free(th);
    return job.err ? 2 : (job.bad ? 2 + job.bad : 0);
}

/*
 * Sequential marching (MgritHierarchy.coarse_solve, mgrit.py:219-226, and
 * solve_serial, serial.py:40-61): u[i] = Phi(u[i-1]) (+ g[i]) for
 * i = 1..n_steps; u and g hold n_steps+1 rows of nx doubles.
 */
int ora_march(const ora_params *p, double *u, const double *g, int64_t n_steps,
              int64_t nx) {
    if (check_params(p, nx) || n_steps < 0) return 1;
    ora_tables t;
    build_tables(p->k, p->eps, &t);
    ora_work wk;
    if (work_alloc(&wk, nx, p->k, ncomp(p))) return 2;
    const int64_t len = wk.len;
    for (int64_t i = 1; i <= n_steps; ++i)
        phi_field(p, &t, &wk, u + (i - 1) * len, g ? g + i * len : NULL, u + i * len);
    const int bad = wk.bad_state;
    work_free(&wk);
    return bad ? 2 + bad : 0;
}
