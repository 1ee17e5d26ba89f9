/*
 * mgrit_phi.h -- C ABI of the B200 MGRIT fine-propagator library
 * (paper_2104_09404_b200/libmgrit_phi.so).
 *
 * The reference (arxiv 2104.09404, package `mgritlab`) is pure Python/NumPy;
 * its "FFI" for this path is Python calling the functions below through
 * ctypes.  Each entry point replaces one reference
 * interface, cited as pkg/src/mgritlab/<file>:<lines>:
 *
 *   mgp_sweep        -- the batched propagator and every level operation
 *                       built from it:
 *                         RungeKuttaStepper.advance   stepper.py:50-82
 *                         SemiDiscreteOperator.rhs    flux.py:129-161
 *                         MgritHierarchy.f_relax      mgrit.py:168-180
 *                         MgritHierarchy.c_relax      mgrit.py:182-191
 *                         MgritHierarchy.restrict     mgrit.py:199-217
 *                         MgritHierarchy.coarse_solve mgrit.py:219-226
 *                         MgritHierarchy.residual_norm mgrit.py:264-270
 *                         rel_l2_spacetime_error      grid.py:96-108
 *                         solve_serial                serial.py:40-61
 *   mgp_relax_fcf    -- MgritHierarchy.relax(0) (mgrit.py:193-197) of the
 *                       C-points-only finest level as one launch, optionally
 *                       with fine_values() (mgrit.py:272-273) of the relaxed
 *                       iterate fused in
 *   mgp_sum_partials -- deterministic reduction of the per-chunk partial sums
 *                       the sweep writes (residual^2, error^2, non-finite
 *                       count), replacing np.linalg.norm (mgrit.py:270,
 *                       grid.py:105-108) and np.isfinite (mgrit.py:323).
 *
 * Conventions: all pointers are device pointers owned by the caller; states
 * are rows of D*nx float64 values (D = 1 for the scalar models; D = 2 for
 * shallow water, component-major: nx depths h then nx momenta hu, the
 * reference's (..., D, N) layout); strides are in elements (float64), may be
 * 0 to broadcast one row.  Every call is asynchronous on `stream`
 * (a cudaStream_t, NULL = legacy default stream).  Return codes: MGP_OK,
 * MGP_EINVAL (bad argument: the Python layer raises ConfigError, mirroring
 * the reference's constructor checks), MGP_ECUDA (launch/CUDA failure:
 * RuntimeError).  Non-finite data never fails a call: NaN/inf propagate like
 * NumPy.  The library owns no device memory.
 */
#ifndef MGRIT_PHI_H
#define MGRIT_PHI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGP_OK 0
#define MGP_EINVAL 1
#define MGP_ECUDA 2

/* models.py:101-133 (Burgers) and the linear-advection model BASELINE.json
 * config 1 needs (flux a*u, |lambda| = |a|). */
#define MGP_MODEL_BURGERS 0
#define MGP_MODEL_ADVECTION 1
/* ShallowWater (models.py:136-211): state (h, hu), flux (hu, h u^2 + g h^2/2),
 * characteristic WENO (weno.py:222-233) with the LF or Roe flux; rows of
 * 2*nx, nx <= 2048, candidate sums always in the 2-lane order (the
 * characteristic windows are fresh contiguous arrays in the reference). */
#define MGP_MODEL_SHALLOW_WATER 2
/* Euler (models.py:214-308): state (rho, rho u, E), ideal gas gamma; rows of
 * 3*nx, nx <= 2048; left eigenvectors = inv(right) by LU with partial
 * pivoting (the reference's np.linalg.inv agrees to rounding). */
#define MGP_MODEL_EULER 3

/* bits OR-ed into *mgp_sweep_args.status where the reference raises
 * PhysicalStateError */
#define MGP_STATUS_NONPOSITIVE_DEPTH 1      /* models.py:147-153 */
#define MGP_STATUS_NONPOSITIVE_DENSITY 2    /* models.py:228-232 */
#define MGP_STATUS_NONPOSITIVE_PRESSURE 4   /* models.py:235-238 */
#define MGP_STATUS_ROE_NONHYPERBOLIC 8      /* models.py:290-293 */

/* NumPy candidate-sum order of weno.py:175:
 * SEQ when advance() received >= 2 fields, LANE2 for a single field. */
#define MGP_SUM_SEQ 0
#define MGP_SUM_LANE2 1

/* propagator family (mgp_phi.scheme) */
#define MGP_SCHEME_RK_WENO 0     /* RungeKuttaStepper over WENO + global LF (stepper.py:68-82) */
#define MGP_SCHEME_LF_ONESTEP 1  /* MatchedLFFine / RediscretizedLF (stepper.py:102-114,155-167) */
#define MGP_SCHEME_LF_MATCHED 2  /* MatchedLFCoarse order 0/1 (stepper.py:117-152) */
#define MGP_SCHEME_RK_WENO_ROE 3 /* as 0 with the Roe flux + entropy fix, Burgers
                                    (flux.py:91-126), nx <= 4096 */

/* how "+ g" is applied after a propagator application */
#define MGP_G_NONE 0   /* no addition (advance, serial march)              */
#define MGP_G_ZERO 1   /* + 0.0 (finest-level g, zero past node 0)         */
#define MGP_G_ARRAY 2  /* + g[row]                                         */

/* what the sweep does after its chained steps */
#define MGP_TAIL_NONE 0
#define MGP_TAIL_PHI 1       /* tail_out = Phi(x) (+ g_tail per tail_g_mode)  */
#define MGP_TAIL_RESTRICT 2  /* FAS restriction, mgrit.py:209-215 (below)    */
#define MGP_TAIL_RESID 3     /* residual (g + Phi(x)) - target, mgrit.py:268 */

#define MGP_GUESS_LAST_STEP 0
#define MGP_GUESS_INJECTION 1

/* One propagator Phi_l: SSP-RK(rk_order) over the WENO(2k+1)/global-LF
 * semi-discrete operator on a periodic mesh of nx cells
 * (harness.py:350-355 builds one per level with dt = dt0 * m**l), or a
 * member of the one-step Lax-Friedrichs family (scheme != 0; Burgers, nx <=
 * 2048; dt is the step the formula multiplies: dt for one-step and matched
 * order 0 (= dt_fine * m_eff), dt_fine for matched order 1). */
typedef struct mgp_phi {
    int32_t model;      /* MGP_MODEL_*                                        */
    int32_t weno_k;     /* reconstruction degree 0..3 (order 2k+1), flux.py:35 */
    int32_t rk_order;   /* 1 FE, 2 SSP-RK2, 3 SSP-RK3; 0 = semi-discrete rhs */
    int32_t regime;     /* MGP_SUM_* for chained steps                        */
    int64_t nx;         /* cells, >= 2k+1 (flux.py:138-141)                   */
    double dt;          /* step size of this level                             */
    double dx;          /* SpatialGrid.dx = length / nx (grid.py:35-37)        */
    double epsilon;     /* WENO epsilon > 0 (weno.py:30)                       */
    double speed;       /* advection speed a (ignored for Burgers)             */
    int32_t scheme;     /* MGP_SCHEME_* (0 for the WENO/RK propagators)        */
    int32_t lf_order;   /* MGP_SCHEME_LF_MATCHED: truncation order 0 or 1      */
    int32_t m_eff;      /* MGP_SCHEME_LF_MATCHED: fine steps emulated (m^l)    */
    int32_t repeats;    /* >= 1: Phi = inner^repeats (ComposedStepper,
                           stepper.py:170-188); 1 otherwise                    */
    double gravity;     /* shallow water: g > 0 (models.py:139-143)            */
    double gamma;       /* Euler: gamma > 1 (models.py:219-223)                */
    int32_t characteristic;  /* systems: 1 characteristic-field WENO, 0 per
                                component (WenoConfig.characteristic)      */
    int32_t reserved;
} mgp_phi;

/*
 * mgp_sweep: for every chunk b in [0, n_chunks), independently:
 *
 *   x = start[b*start_stride]                                   (row)
 *   [err/nonfinite accounting of x against ref[b*ref_cs]]
 *   for s = 1 .. n_steps:                                      (chained steps)
 *       x = Phi(x) (+ g[b*g_cs + (s-1)*g_ss] per g_mode)
 *       if store: store[b*st_cs + (s-1)*st_ss] = x
 *       [err/nonfinite accounting of x against ref[b*ref_cs + s*ref_ss]]
 *   tail (with the tail regime `tail_regime`):
 *     MGP_TAIL_PHI:      y = Phi(x) (+ tail_g[b*tg_s] per tail_g_mode);
 *                        tail_out[b*to_s] = y
 *     MGP_TAIL_RESTRICT: psi = Phi(x);  gf = tail_g row (tail_g_mode),
 *                        phi = aux[b*aux_s];
 *                        tail_out[b*to_s]  = (gf + phi) - psi      (coarse g)
 *                        tail_out2[b*to2_s] = guess == LAST_STEP
 *                                             ? phi + gf : aux2[b*aux2_s]
 *     MGP_TAIL_RESID:    r = (gf + Phi(x)) - aux[b*aux_s];
 *                        partials[3b+0] = sum over cells of r*r;
 *                        if tail_out: tail_out[b*to_s] = gf + Phi(x)  (the value
 *                        the next C-relaxation of the chunk computes)
 *                        (last chunk also accounts aux row in err/nonfinite
 *                         against ref[(b+1)*ref_cs] when ref_last_next != 0)
 *   partials (if non-NULL): [3b+0] residual^2, [3b+1] error^2 (ref non-NULL),
 *   [3b+2] number of non-finite cells seen (when count_nonfinite != 0).
 *
 * When n_steps > 0 and tail != MGP_TAIL_NONE, tail_regime must equal
 * phi.regime (each launch runs in one summation regime).
 *
 * n_chunks = 1 with store of every step is the sequential coarse solve /
 * serial march.  Chunks never read rows another chunk writes in the same
 * call (the caller guarantees it, e.g. by writing new C-points to a
 * separate buffer), so all chunks run concurrently.
 */
typedef struct mgp_sweep_args {
    mgp_phi phi;
    int64_t n_chunks;
    const double *start;  int64_t start_stride;
    int32_t n_steps;      int32_t g_mode;
    const double *g;      int64_t g_cs, g_ss;
    double *store;        int64_t st_cs, st_ss;
    int32_t tail;         int32_t tail_regime;
    int32_t tail_g_mode;  int32_t guess;
    const double *tail_g; int64_t tg_s;
    double *tail_out;     int64_t to_s;
    double *tail_out2;    int64_t to2_s;
    const double *aux;    int64_t aux_s;
    const double *aux2;   int64_t aux2_s;
    const double *ref;    int64_t ref_cs, ref_ss;
    int32_t ref_last_next;
    int32_t count_nonfinite;
    double *partials;
    int32_t *status;      /* optional device word: MGP_STATUS_* bits are OR-ed
                             in when a state the reference rejects is met
                             (the sweep still completes; the caller checks the
                             word after synchronising and raises) */
} mgp_sweep_args;

int mgp_sweep(const mgp_sweep_args *args, void *stream);

/*
 * mgp_relax_fcf: the finest level's relaxation over C-points only, as ONE
 * launch (MgritHierarchy.relax(0), mgrit.py:193-197, with the F-points
 * implicit -- c_relax after the F-relaxation they derive from):
 *
 *   for every CF-interval j in [0, n_chunks):
 *       x = cs[j*cs_s];  m-1 times x = Phi(x) (+ 0.0 per g_mode)   (F)
 *       x = Phi(x) (+ 0.0);  cd[(j+1)*cd_s] = x                     (C)
 *   and, when fstore != NULL, the final F-relaxation of the relaxed iterate:
 *       for every interval i: x = (i == 0 ? c0 : new C-point i);
 *       for s = 1..m-1: x = Phi(x) (+ 0.0); fstore[i*f_cs + (s-1)*f_ss] = x
 *   where c0 = f0_start if non-NULL (the new C-point 0 of a call that
 *   continues an earlier one, e.g. a later piece of a pipelined relaxation),
 *   else cs[0], which is then also copied to cd[0] (node 0 is kept).
 *   cstore (optional) receives every C-point of the relaxed iterate, rows
 *   0..n_chunks at cstore[i*cst_s] (e.g. the C-point rows of a trajectory
 *   buffer whose F-point rows are fstore).
 *
 * i.e. exactly mgp_sweep(n_steps = m-1, TAIL_PHI) followed by
 * mgp_sweep(n_steps = m-1, store) on the new C-points, bit for bit.  Each
 * interval's C-step runs straight into the next interval's final F-steps
 * (one chain of 2m-1 steps); persistent CTAs (one per resident slot) take
 * whole chains from a ticket counter.  With more intervals than slots the
 * first wave of chains runs only its F- and C-steps and queues the final
 * F-steps (split plan), which later CTAs take in completion order, starting
 * from the new C-point in cd; optionally the last chains are cut into
 * segments handed over through an L2-resident ring (segment > 0).  cd must
 * not alias cs.
 * workspace: at least mgp_relax_fcf_workspace() bytes, zero-filled once
 * before first use (every call leaves it clean again, so CUDA graph replays
 * work; calls sharing a workspace must be stream-ordered); epoch: non-zero
 * (reserved).  Scalar Burgers RK-WENO fields of nx <= 4096 (one CTA per
 * field) in the batched sum regime; anything else returns MGP_EINVAL and
 * the caller uses the two mgp_sweep launches.
 */
typedef struct mgp_fcf_args {
    mgp_phi phi;
    int64_t n_chunks;     /* CF-intervals (N_t / m)                  */
    int32_t m;            /* coarsening factor >= 1                   */
    int32_t g_mode;       /* MGP_G_NONE or MGP_G_ZERO                 */
    const double *cs;     int64_t cs_s;
    double *cd;           int64_t cd_s;
    double *fstore;       int64_t f_cs, f_ss;
    double *cstore;       int64_t cst_s;
    const double *f0_start;
    void *workspace;      int64_t workspace_bytes;
    uint32_t epoch;
    int32_t segment;      /* steps per hand-over segment of the chains taken
                             last (0 = whole chains, the measured default) */
    int32_t split;        /* split plan with F-point storage and segment 0:
                             0 = automatic (one CTA slot's worth of chains
                             run F+C only and queue their final F-steps when
                             intervals outnumber slots), -1 = off (whole
                             chains), > 0 = that many split chains */
    int32_t reserved;
} mgp_fcf_args;
int mgp_relax_fcf(const mgp_fcf_args *args, void *stream);
/* Workspace bytes mgp_relax_fcf needs for this propagator and interval
 * count on the current device (0 if the fused path does not apply). */
int64_t mgp_relax_fcf_workspace(const mgp_phi *phi, int64_t n_chunks, int32_t m);
/* out[j] = sum_b partials[width*b + j] for j < width (width <= 4), summed in a
 * fixed order independent of launch timing (deterministic). */
int mgp_sum_partials(const double *partials, int64_t n, int32_t width,
                     double *out, void *stream);

/* Largest nx supported for a propagator: 4096 cells per CTA (whole field in
 * shared memory); WENO5 Burgers fields up to 16 x 4096 cells are split over a
 * thread-block cluster (nx must then divide into power-of-two slabs);
 * shallow water 2048 cells. */
int64_t mgp_max_nx(int32_t weno_k, int32_t model);

/* Library/ABI version and the compile-time WENO tables of degree k, written
 * as cw[4][4], d[4], sm[4][4][4] (row-major, zero padded) so tests can check
 * them against float(Fraction(p, q)) of weno.py:43-86. */
int32_t mgp_abi_version(void);
int mgp_weno_tables(int32_t k, double *cw16, double *d4, double *sm64);

/* Number of kernel launches issued by this library since load (for the
 * bench's gpu_launches accounting). */
int64_t mgp_launch_count(void);

/* ABI self-description for binding checks: writes sizeof(mgp_phi),
 * sizeof(mgp_sweep_args) and then offsetof() of every mgp_sweep_args field
 * in declaration order to out[0..n); returns the number of entries written. */
int32_t mgp_sweep_args_layout(int64_t *out, int32_t n);

#ifdef __cplusplus
}
#endif

#endif /* MGRIT_PHI_H */
