// mgrit_phi.cu -- B200 (sm_100a) kernels for the MGRIT fine-propagator path.
//
// One CTA owns one whole field (a chunk's state, nx cells) in shared memory
// for every Runge-Kutta stage of every chained step of a relaxation sweep:
// the field is read from HBM once per sweep and written once per stored node;
// the WENO windows, the global Lax-Friedrichs speed (a CTA-wide NaN-propagating
// max per stage) and the periodic halo never leave the SM.  Compiled with
// -fmad=false: every a*b+c of the reference stays a separately rounded DMUL
// and DADD, and every "/" is an IEEE division, so results are bit-identical to
// the NumPy reference (SURVEY.md 8(c) "parity arithmetic contract").
//
// Reference semantics followed (pkg/src/mgritlab/...):
//   weno.py:154-236  reconstruction (windows, candidates, beta, weights)
//   flux.py:70-88    global LF speed and flux;  flux.py:159-161 rhs
//   models.py:107-117 Burgers flux / speed
//   stepper.py:50-62 SSP-RK1/2/3;  mgrit.py:168-270 level operations.
#include <cooperative_groups.h>
#include <vector>
#include <type_traits>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/mgrit_phi.h"
#include "div_shared.cuh"

// ---------------------------------------------------------------------------
// WENO tables (weno.py:43-86): numerators over a common denominator; the
// initialisers are IEEE-rounded quotients, i.e. float(Fraction(p, q)).
// Layout [k][r][j] (cw), [k][r] (d), [k][r][i][j] (smoothness), zero padded.
// ---------------------------------------------------------------------------
#define MGP_CW_TABLE                                                        \
    {{{1.0, 0, 0, 0}},                                                       \
     {{1.0 / 2, 1.0 / 2}, {-1.0 / 2, 3.0 / 2}},                              \
     {{2.0 / 6, 5.0 / 6, -1.0 / 6}, {-1.0 / 6, 5.0 / 6, 2.0 / 6},            \
      {2.0 / 6, -7.0 / 6, 11.0 / 6}},                                        \
     {{3.0 / 12, 13.0 / 12, -5.0 / 12, 1.0 / 12},                            \
      {-1.0 / 12, 7.0 / 12, 7.0 / 12, -1.0 / 12},                            \
      {1.0 / 12, -5.0 / 12, 13.0 / 12, 3.0 / 12},                            \
      {-3.0 / 12, 13.0 / 12, -23.0 / 12, 25.0 / 12}}}
#define MGP_D_TABLE                                                         \
    {{1.0}, {2.0 / 3, 1.0 / 3}, {3.0 / 10, 6.0 / 10, 1.0 / 10},              \
     {4.0 / 35, 18.0 / 35, 12.0 / 35, 1.0 / 35}}
#define S6(a) ((a) / 6.0)
#define S240(a) ((a) / 240.0)
#define MGP_SM_TABLE                                                        \
    {{{{0.0}}},                                                              \
     {{{1.0, -1.0}, {-1.0, 1.0}}, {{1.0, -1.0}, {-1.0, 1.0}}},               \
     {{{S6(20.0), S6(-31.0), S6(11.0)},                                      \
       {S6(-31.0), S6(50.0), S6(-19.0)},                                     \
       {S6(11.0), S6(-19.0), S6(8.0)}},                                      \
      {{S6(8.0), S6(-13.0), S6(5.0)},                                        \
       {S6(-13.0), S6(26.0), S6(-13.0)},                                     \
       {S6(5.0), S6(-13.0), S6(8.0)}},                                       \
      {{S6(8.0), S6(-19.0), S6(11.0)},                                       \
       {S6(-19.0), S6(50.0), S6(-31.0)},                                     \
       {S6(11.0), S6(-31.0), S6(20.0)}}},                                    \
     {{{S240(2107.0), S240(-4701.0), S240(3521.0), S240(-927.0)},            \
       {S240(-4701.0), S240(11003.0), S240(-8623.0), S240(2321.0)},          \
       {S240(3521.0), S240(-8623.0), S240(7043.0), S240(-1941.0)},           \
       {S240(-927.0), S240(2321.0), S240(-1941.0), S240(547.0)}},            \
      {{S240(547.0), S240(-1261.0), S240(961.0), S240(-247.0)},              \
       {S240(-1261.0), S240(3443.0), S240(-2983.0), S240(801.0)},            \
       {S240(961.0), S240(-2983.0), S240(2843.0), S240(-821.0)},             \
       {S240(-247.0), S240(801.0), S240(-821.0), S240(267.0)}},              \
      {{S240(267.0), S240(-821.0), S240(801.0), S240(-247.0)},               \
       {S240(-821.0), S240(2843.0), S240(-2983.0), S240(961.0)},             \
       {S240(801.0), S240(-2983.0), S240(3443.0), S240(-1261.0)},            \
       {S240(-247.0), S240(961.0), S240(-1261.0), S240(547.0)}},             \
      {{S240(547.0), S240(-1941.0), S240(2321.0), S240(-927.0)},             \
       {S240(-1941.0), S240(7043.0), S240(-8623.0), S240(3521.0)},           \
       {S240(2321.0), S240(-8623.0), S240(11003.0), S240(-4701.0)},          \
       {S240(-927.0), S240(3521.0), S240(-4701.0), S240(2107.0)}}}}

static const double h_cw[4][4][4] = MGP_CW_TABLE;
static const double h_d[4][4] = MGP_D_TABLE;
static const double h_sm[4][4][4][4] = MGP_SM_TABLE;
__constant__ double c_cw[4][4][4] = MGP_CW_TABLE;
__constant__ double c_d[4][4] = MGP_D_TABLE;
__constant__ double c_sm[4][4][4][4] = MGP_SM_TABLE;

// The same tables as compile-time literals for the kernels: after unrolling
// every index is a constant, so each coefficient becomes an immediate
// constant of the instruction stream and equal values are shared, instead of
// one constant-bank load per table entry (the __constant__ copies above stay
// the single source for host-side checks, mgp_weno_tables).
#ifndef MGP_CONST_BANK
__device__ __forceinline__ constexpr double tab_cw(int k, int r, int j) {
    constexpr double t[4][4][4] = MGP_CW_TABLE;
    return t[k][r][j];
}
__device__ __forceinline__ constexpr double tab_d(int k, int r) {
    constexpr double t[4][4] = MGP_D_TABLE;
    return t[k][r];
}
__device__ __forceinline__ constexpr double tab_sm(int k, int s, int a, int b) {
    constexpr double t[4][4][4][4] = MGP_SM_TABLE;
    return t[k][s][a][b];
}
#define CW(k, r, j) tab_cw(k, r, j)
#define DW(k, r) tab_d(k, r)
#define SM(k, s, a, b) tab_sm(k, s, a, b)
#else
#define CW(k, r, j) c_cw[k][r][j]
#define DW(k, r) c_d[k][r]
#define SM(k, s, a, b) c_sm[k][s][a][b]
#endif

namespace mgp_parts {
extern unsigned long long launches;
}

// Translation-unit split (see the end of the file): every compilation gets
// its own namespace for the internal code -- nvcc names an anonymous
// namespace after the source file, so identical units would collide.
#ifndef MGP_PART
#define MGP_PART 0
#endif
#define MGP_CAT2(a, b) a##b
#define MGP_CAT(a, b) MGP_CAT2(a, b)
#define MGP_UNIT MGP_CAT(mgp_unit_, MGP_PART)

namespace MGP_UNIT {

using mgp::SharedRcp;
using mgp::div_shared;
using mgp::shared_rcp;

constexpr int kMaxThreads = 512;
constexpr int kMaxRun = 8;
constexpr int64_t kMaxNx = (int64_t)kMaxThreads * kMaxRun;

// one launch counter for the whole library, whichever translation unit
// (MGP_PART, below) the launch sits in
unsigned long long &g_launches = mgp_parts::launches;
#ifdef MGP_FCF_TRACE
__device__ unsigned long long g_fcf_trace[4 * 8192];
#endif

#ifdef MGP_TRACE
__device__ long long g_trace[8192];
__device__ int g_trace_n;
__device__ __forceinline__ void trace(int tag) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int i = g_trace_n;
        if (i < 4096) {
            long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            g_trace[2 * i] = tag;
            g_trace[2 * i + 1] = t;
            g_trace_n = i + 1;
        }
    }
}
#else
__device__ __forceinline__ void trace(int) {}
#endif

__device__ __forceinline__ bool is_finite(double x) {
    return (__double2hiint(x) & 0x7FF00000) != 0x7FF00000;
}

__device__ __forceinline__ unsigned long long abs_bits(double x) {
    return (unsigned long long)__double_as_longlong(x) & 0x7FFFFFFFFFFFFFFFull;
}

__device__ __forceinline__ unsigned long long umax64(unsigned long long a,
                                                     unsigned long long b) {
    return a > b ? a : b;
}

constexpr unsigned long long kNaNBits = 0x7FF8000000000000ull;

// Warp-wide unsigned 64-bit max (alpha bits of non-negative doubles): the max
// high word, then the max low word among the lanes holding it -- two REDUX
// instead of five 64-bit shuffle rounds.
__device__ __forceinline__ unsigned long long warp_umax64(unsigned long long v) {
    const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return ((unsigned long long)mh << 32) | ml;
}

// kernel-internal model id: Burgers with the Roe flux (mgp_phi.scheme ==
// MGP_SCHEME_RK_WENO_ROE), no global alpha, NaN kept local like the reference
constexpr int kModelBurgersRoe = 8;

#ifndef MGP_SLIDE_UNROLL
#define MGP_SLIDE_UNROLL 1
#endif
// Unroll factor of the centred reconstruction: half a run per block (two
// blocks of 4 windows for runs of 8 cells, of 2 for runs of 4).  Measured on
// B200 (profiles/r02_fcf_unroll.txt; runs of 16: blocks of 4): C3 16.3 -> 17.8 G point-updates/s --
// the 8-window block spilled 824 bytes at 128 registers, the 4-window block
// none inside the loop, and its static schedule has 19 % fewer stall cycles
// per window; C2 (runs of 4) 14.2 -> 14.6 G.  WENO3 windows are small enough
// to unroll the whole run without spilling (+ 3-4 %, profiles/r02_order_probe.txt).
// MGP_CENTRED_UNROLL overrides.
#ifdef MGP_CENTRED_UNROLL
#define MGP_CU(pc) MGP_CENTRED_UNROLL
#else
#define MGP_CU(pc) (K <= 1 ? (pc) : ((pc) >= 8 ? 4 : ((pc) >= 4 ? (pc) / 2 : (pc))))
#endif
#define MGP_PRAGMA(x) _Pragma(#x)
#define MGP_UNROLL_(n) MGP_PRAGMA(unroll n)
#define MGP_UNROLL(n) MGP_UNROLL_(n)

// Shared-memory index of element t: one pad word per 2^LG elements, so that
// the lanes of a warp walking runs of P consecutive cells hit distinct banks.
// LG = log2(P) for runs of 4 or 8 cells (a thread's first cell i0 is then a
// multiple of 2^LG, so sk(i0 + x) = sk(i0) + x + (x >> LG) for any x: every
// address of the unrolled hot loops is the thread's base plus a literal),
// one pad per 16 elements otherwise.  A half-warp's 64-bit accesses at
// thread stride 2^LG + 1 words fall into 16 distinct bank pairs.
__host__ __device__ constexpr int pad_log(int p) { return p == 8 ? 3 : (p == 4 ? 2 : 4); }
template <int LG>
__host__ __device__ constexpr int skp(int t) { return t + (t >> LG); }
template <int LG>
__host__ __device__ constexpr int skp_size(int n) { return n + (n >> LG) + 1; }

// The dynamic shared memory of every kernel of the WENO/RK Field family, as
// one array: Field addresses it by element offsets, so every access is a
// shared-space LDS/STS with a 32-bit address (pointers kept in the Field
// struct decayed to generic 64-bit loads and stores).
extern __shared__ double mgp_sm[];

// ---------------------------------------------------------------------------
// WENO reconstruction, reference weno.py:154-177, for a run of consecutive
// interfaces.  Notation: c_j = cell j; the left state at interface i+1/2 uses
// the window c_{i-K..i+K}, the right state the reversed window
// c_{i+1+K..i+1-K} (weno.py:191-199).
//
//   left  q_r(i) = sum_j cw[r][j] c_{i-r+j}
//   right q_r(i) = sum_j cw[r][j] c_{i+1+r-j}
//   left  beta_s(i) = sum_{a,b} (c_{i-s+a} S_s[a][b]) c_{i-s+b}     (a-major)
//   right beta_r(i) = the same nine products as left beta_{K-r}(i+1),
//                     summed in exactly the reverse order
// (S_{K-r} is S_r flipped; checked for every table by test_abi.py), so the
// products of the left state at i+1 are formed once and summed twice.  The
// candidate sums follow NumPy: sequential for batches of >= 2 fields, (even
// window slots) + (odd window slots) for a single field.
// ---------------------------------------------------------------------------

// win[0..2K] = c_{m-K..m+K} for the window centre m.
template <int K, int REG>
__device__ __forceinline__ double cand_left(const double *win, int r) {
    // left q_r(m): cells m-r+j -> win[K-r+j], window slot K-r+j
    if (REG == MGP_SUM_SEQ || K < 2) {
        double acc = CW(K, r, 0) * win[K - r];
#pragma unroll
        for (int j = 1; j <= K; ++j) acc = acc + CW(K, r, j) * win[K - r + j];
        return acc;
    }
    double ev = 0.0, od = 0.0;
    bool he = false, ho = false;
#pragma unroll
    for (int j = 0; j <= K; ++j) {
        const int slot = K - r + j;
        const double p = CW(K, r, j) * win[K - r + j];
        if ((slot & 1) == 0) { ev = he ? ev + p : p; he = true; }
        else { od = ho ? od + p : p; ho = true; }
    }
    return he ? (ho ? ev + od : ev) : od;
}

template <int K, int REG>
__device__ __forceinline__ double cand_right(const double *win, int r) {
    // right q_r(m-1): cells (m-1)+1+r-j = m+r-j -> win[K+r-j], slot K-r+j
    if (REG == MGP_SUM_SEQ || K < 2) {
        double acc = CW(K, r, 0) * win[K + r];
#pragma unroll
        for (int j = 1; j <= K; ++j) acc = acc + CW(K, r, j) * win[K + r - j];
        return acc;
    }
    double ev = 0.0, od = 0.0;
    bool he = false, ho = false;
#pragma unroll
    for (int j = 0; j <= K; ++j) {
        const int slot = K - r + j;
        const double p = CW(K, r, j) * win[K + r - j];
        if ((slot & 1) == 0) { ev = he ? ev + p : p; he = true; }
        else { od = ho ? od + p : p; ho = true; }
    }
    return he ? (ho ? ev + od : ev) : od;
}

// Products of left beta_s(m): cells m-s+a -> win[K-s+a].  Returns the
// forward (a-major) sum; when RIGHT, also the reverse-order sum, which is
// right beta_{K-s}(m-1).
template <int K, bool RIGHT, bool LEFT = true>
__device__ __forceinline__ void beta_block(const double *win, int s, double &fwd,
                                           double &rev) {
    constexpr int N = (K + 1) * (K + 1);
    double p[N];
#pragma unroll
    for (int a = 0; a <= K; ++a)
#pragma unroll
        for (int b = 0; b <= K; ++b)
            p[a * (K + 1) + b] = (win[K - s + a] * SM(K, s, a, b)) * win[K - s + b];
    if (LEFT) {
        double f = p[0];
#pragma unroll
        for (int t = 1; t < N; ++t) f = f + p[t];
        fwd = f;
    }
    if (RIGHT) {
        double g = p[N - 1];
#pragma unroll
        for (int t = N - 2; t >= 0; --t) g = g + p[t];
        rev = g;
    }
}

// nonlinear weights and combination (weno.py:161-168, 176-177):
// raw_r = d_r / ((eps+beta_r)(eps+beta_r)), S = (raw_0 + raw_1) + ...,
// value = ((raw_0/S) q_0 + (raw_1/S) q_1) + ...  The divisions take the
// compiler's own fast path branch-free (div_shared.cuh); if any of them was
// outside its validity range the value is recomputed with IEEE `/`.
template <int K>
__device__ __forceinline__ double weno_value_ieee(const double *beta, const double *q, double eps) {
    double raw[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) {
        const double e = eps + beta[r];
        raw[r] = DW(K, r) / (e * e);
    }
    double S = raw[0];
#pragma unroll
    for (int r = 1; r <= K; ++r) S = S + raw[r];
    double v = (raw[0] / S) * q[0];
#pragma unroll
    for (int r = 1; r <= K; ++r) v = v + (raw[r] / S) * q[r];
    return v;
}

// The rare exact path out of line (keeps the hot loop compact in the
// instruction cache); operands by value so nothing is spilled to call it.
template <int K>
__device__ __noinline__ double weno_value_slow_(double b0, double b1, double b2, double b3,
                                                double q0, double q1, double q2, double q3,
                                                double eps) {
    const double beta[4] = {b0, b1, b2, b3};
    const double q[4] = {q0, q1, q2, q3};
    return weno_value_ieee<K>(beta, q, eps);
}

template <int K>
__device__ __forceinline__ double weno_value_slow(const double *beta, const double *q, double eps) {
    return weno_value_slow_<K>(beta[0], K >= 1 ? beta[1] : 0.0, K >= 2 ? beta[2] : 0.0,
                               K >= 3 ? beta[3] : 0.0, q[0], K >= 1 ? q[1] : 0.0,
                               K >= 2 ? q[2] : 0.0, K >= 3 ? q[3] : 0.0, eps);
}

template <int K>
__device__ __forceinline__ double weno_value(const double *beta, const double *q, double eps,
                                             const double *moot_win = nullptr,
                                             bool moot_extra = false) {
    bool bad = false;
    double raw[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) {
        const double e = eps + beta[r];
        raw[r] = mgp::div_fast_cnum(DW(K, r), shared_rcp(e * e), bad);
    }
    double S = raw[0];
#pragma unroll
    for (int r = 1; r <= K; ++r) S = S + raw[r];
    const SharedRcp R = shared_rcp(S);
    double v = mgp::div_fast(raw[0], R, bad) * q[0];
#pragma unroll
    for (int r = 1; r <= K; ++r) v = v + mgp::div_fast(raw[r], R, bad) * q[r];
    if (bad) {
        // `moot`: the value cannot reach the result (Burgers with a non-finite
        // cell in the field: alpha is NaN and every flux NaN), so skip the
        // slow exact recomputation on such data.  Checked only on this rare
        // path.
        bool moot = moot_extra;
        if (moot_win) {
#pragma unroll
            for (int t = 0; t <= 2 * K; ++t) moot |= !is_finite(moot_win[t]);
        }
        if (!moot) v = weno_value_slow<K>(beta, q, eps);
    }
    return v;
}

// As weno_value, with the validity of all 2K+2 fast-path divisions shown by
// one range test: if every e_r = eps + beta_r lies in [2^-60, 2^61) then
// e_r^2 is in [2^-120, 2^122), raw_r = d_r / e_r^2 (d_r >= 1/35) in
// [2^-128, 2^120), S = sum raw_r in [2^-128, 2^120] and omega_r = raw_r / S
// in [2^-248, 1] -- every divisor finite, every numerator above 2^-967 and
// every quotient normal, which is exactly the fast-path predicate of
// div_shared.cuh.  Otherwise (huge or non-finite fields) the value is
// recomputed with IEEE `/` unless `moot`.  Two integer operations per e_r
// replace the per-division checks.
template <int K>
__device__ __forceinline__ double weno_value_rc(const double *beta, const double *q, double eps,
                                                const double *moot_win) {
    constexpr unsigned kLo = 963u << 20;      // high word of 2^-60
    constexpr unsigned kSpan = 121u << 20;    // [2^-60, 2^61)
    double e[K + 1];
    bool ok = true;
#pragma unroll
    for (int r = 0; r <= K; ++r) {
        e[r] = eps + beta[r];
        ok &= ((unsigned)__double2hiint(e[r]) - kLo) < kSpan;
    }
    double raw[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) raw[r] = mgp::div_nocheck(DW(K, r), shared_rcp(e[r] * e[r]));
    double S = raw[0];
#pragma unroll
    for (int r = 1; r <= K; ++r) S = S + raw[r];
    const SharedRcp R = shared_rcp(S);
    double v = mgp::div_nocheck(raw[0], R) * q[0];
#pragma unroll
    for (int r = 1; r <= K; ++r) v = v + mgp::div_nocheck(raw[r], R) * q[r];
    if (!ok) {
        bool moot = false;
        if (moot_win) {
#pragma unroll
            for (int t = 0; t <= 2 * K; ++t) moot |= !is_finite(moot_win[t]);
        }
        if (!moot) v = weno_value_slow<K>(beta, q, eps);
    }
    return v;
}

// weno_value_rc without its branch: the range test is AND-ed into `ok` and
// the caller redoes the values exactly when it fails (reconstruct_centred).
template <int K>
__device__ __forceinline__ double weno_value_nc(const double *beta, const double *q, double eps,
                                                bool &ok) {
    constexpr unsigned kLo = 963u << 20;      // high word of 2^-60
    constexpr unsigned kSpan = 121u << 20;    // [2^-60, 2^61)
    double e[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) {
        e[r] = eps + beta[r];
        ok &= ((unsigned)__double2hiint(e[r]) - kLo) < kSpan;
    }
    double raw[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) raw[r] = mgp::div_nocheck(DW(K, r), shared_rcp(e[r] * e[r]));
    double S = raw[0];
#pragma unroll
    for (int r = 1; r <= K; ++r) S = S + raw[r];
    const SharedRcp R = shared_rcp(S);
    double v = mgp::div_nocheck(raw[0], R) * q[0];
#pragma unroll
    for (int r = 1; r <= K; ++r) v = v + mgp::div_nocheck(raw[r], R) * q[r];
    return v;
}

struct Consts {
    double dt, hdt, qdt, tdt, two3, inv_dx, dx, eps, speed, half_alpha_adv;
    double k0_omega;
    double twodx, inv_twodx;   // one-step LF family: central difference 2 dx
    int dx_pow2, twodx_pow2;
    int lf_order, m_eff;
    double gravity;            // shallow water
    double gamma, gm1;         // Euler: gamma, gamma - 1
};

namespace cg = cooperative_groups;

// Barrier over the CTAs that share one field: the CTA itself (CS = 1) or its
// thread-block cluster (CS > 1; release/acquire, so shared-memory writes into
// other CTAs of the cluster are visible after it).
template <int CS>
__device__ __forceinline__ void field_sync() {
    if (CS == 1) {
        __syncthreads();
    } else {
        cg::this_cluster().sync();
    }
}

// ---------------------------------------------------------------------------
// LL exchange: a "virtual cluster" of CS co-resident CTAs that share one field
// and talk through global memory instead of distributed shared memory, so the
// group is not tied to one GPC (16-CTA hardware clusters fit 7 times on a
// B200: 112 of 148 SMs; 9 groups of 16 co-resident CTAs use 144).  A double
// travels as two 8-byte words, each carrying half the payload and the
// exchange's 32-bit tag (the words validate themselves: no fence, no flag;
// measured 1.5k cycles for an all-to-all among 16 CTAs x 9 groups against
// 4.6k with fence + counter, profiles/r02_ll_exchange.txt).  Boxes are
// double-buffered by tag parity; the per-stage alpha all-to-all keeps every
// CTA within one exchange of its peers, which makes the reuse safe (see
// Field::sync).  The mailbox is zeroed by the launch, tags start at 1.
// ---------------------------------------------------------------------------
constexpr int kLLHalo = 4;                       // halo cells per side, K <= 3
// words per CTA and parity: alpha 2 | states from the left 6 | halo from the
// left 2*kLLHalo | halo from the right 2*kLLHalo | partial sums 6 | ack 2
constexpr int kLLAlpha = 0, kLLStates = 2, kLLFromLeft = 8, kLLFromRight = 8 + 2 * kLLHalo,
              kLLPsum = 8 + 4 * kLLHalo, kLLAck = 14 + 4 * kLLHalo, kLLWords = 16 + 4 * kLLHalo;
constexpr int kLLSpinLimit = 1 << 22;            // ~ seconds: a lost peer must not hang the GPU

__device__ __forceinline__ void ll_send(unsigned long long *w, double v, unsigned tag) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const unsigned long long t = (unsigned long long)tag << 32;
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(w),
                 "l"(t | (bits & 0xffffffffull)), "l"(t | (bits >> 32))
                 : "memory");
}
__device__ __forceinline__ double ll_recv(const unsigned long long *w, unsigned tag,
                                          unsigned long long *fail) {
    unsigned long long lo, hi;
    int spins = 0;
    do {
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(w)
                     : "memory");
    } while (((unsigned)(lo >> 32) != tag || (unsigned)(hi >> 32) != tag) &&
             ++spins < kLLSpinLimit);
    // a peer that never answered: the result is void; the launch that follows
    // on this stream reports it (launch_t)
    if (spins >= kLLSpinLimit) *fail = 1ull;
    return __longlong_as_double((long long)((hi << 32) | (lo & 0xffffffffull)));
}

// One field, held in shared memory by one CTA (CS = 1) or split into CS
// contiguous slabs over a thread-block cluster (CS > 1, for meshes larger
// than one SM's shared memory and for short sequential marches).  Local cell
// t of the slab is global cell c0 + t; thread `run` owns local interfaces
// and cells [run*P, run*P + P).  With CS > 1 the periodic halo comes from
// the neighbouring CTAs (their boundary cells are stored straight into this
// CTA's halo through distributed shared memory when committed), the states of
// the interface just left of the slab are pushed by the left neighbour, and
// alpha is reduced over the cluster.
// 256-bit global accesses (sm_100): a thread's slice of its CTA's RK-base row
__device__ __forceinline__ void ldg_cg4(const double *p, double *v) {
    asm volatile("ld.global.L1::no_allocate.L2::evict_last.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                 : "l"(p)
                 : "memory");
}
__device__ __forceinline__ void stg_cg4(double *p, const double *v) {
    asm volatile("st.global.L1::no_allocate.L2::evict_last.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]),
                 "d"(v[2]), "d"(v[3])
                 : "memory");
}

__device__ __forceinline__ void stg_stream4(double *p, const double *v) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(
                     p),
                 "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
}

// U0G: the Runge-Kutta base state lives in a global scratch row of the CTA
// (L2-resident, each thread reads and writes only its own run) instead of a
// fourth shared-memory array: a 4096-cell field then needs 105 KB and two
// CTAs fit one SM (256 threads x runs of 16 cells x 128 registers each).
// Measured: equal work on smaller meshes runs 0.84-0.88 of the FP64 peak with
// 2-4 CTAs per SM against 0.77 with one (profiles/r02_fcf_u0g.txt) -- one
// CTA's stage tails and barriers hide behind the other's reconstruction.
// Only full runs, only the fused-commit propagator (phi_commit).
template <int K, int REG, int MODEL, int P, int CS, bool LL = false, bool U0G = false>
struct Field {
    double *u0g;              // U0G: this CTA's RK-base row (global)
    // LL: the CS CTAs exchange through the global mailbox `mbox` (this
    // group's region) instead of distributed shared memory
    unsigned long long *mbox;
    unsigned long long *ll_fail;   // set when a poll gave up (word after the mailbox)
    unsigned eA, eB, eC;      // tags of the last alpha / halo / partial-sum exchange
    bool halo_pending;        // halo cells were sent since the last sync()
    __device__ __forceinline__ unsigned long long *box(int par, int cta, int off) const {
        return mbox + ((size_t)(par * CS + cta) * kLLWords + off);
    }
    __device__ __forceinline__ int left() const { return (q + CS - 1) % CS; }
    __device__ __forceinline__ int right() const { return (q + 1) % CS; }
    static constexpr int H = K + 1;  // halo cells on each side
    // P = 0: latency mode for sequential marches -- two threads per interface
    // (warps alternate between left and right states), one cell per thread
    // in the cell phases.  Otherwise P cells/interfaces per thread.
    static constexpr int PC = P == 0 ? 1 : P;
    static constexpr int LG = pad_log(P);
    static __host__ __device__ constexpr int sk(int t) { return skp<LG>(t); }
    static __host__ __device__ constexpr int sk_size(int n) { return skp_size<LG>(n); }
    int ns, run, i0, q;
    // element offsets into mgp_sm (shared-space addressing):
    int o_u;    // stage input, local cell t at o_u + sk(t + H), t in [-H, ns + H)
    int o_L;    // left states, then interface fluxes, at o_L + sk(i)
    int o_R;    // right states, then results, at o_R + sk(i)
    int o_u0;   // RK base state of the cells, at o_u0 + sk(t)
    int o_red;  // [32] per-warp alpha bits
    int o_edge;                    // [2] states of the interface left of the slab
    int o_cmax;                    // [CS] per-CTA alpha bits
    int b;                         // sk(i0): the thread's base (i0 a multiple of 2^LG)
    double *r_u_left, *r_u_right;  // neighbours' s_u (distributed shared memory)
    double *r_edge_right;          // right neighbour's s_edge
    double *r_L_right;             // right neighbour's s_L (centred reconstruction)
    // lay the arrays out from element offset `at`; returns the end offset
    __device__ __forceinline__ int layout(int at, int ns_, int tid) {
        ns = ns_;
        run = tid;
        i0 = tid * PC;
        b = sk(i0);
        o_u = at;
        o_L = o_u + sk_size(ns + 2 * H);
        o_R = o_L + sk_size(ns);
        o_u0 = o_R + sk_size(ns);
        return U0G ? o_u0 : o_u0 + sk_size(ns);
    }
    __device__ __forceinline__ double &s_u(int idx) const { return mgp_sm[o_u + idx]; }
    __device__ __forceinline__ double &s_L(int idx) const { return mgp_sm[o_L + idx]; }
    __device__ __forceinline__ double &s_R(int idx) const { return mgp_sm[o_R + idx]; }
    __device__ __forceinline__ double &s_u0(int idx) const { return mgp_sm[o_u0 + idx]; }
    __device__ __forceinline__ unsigned long long &s_red(int w) const {
        return reinterpret_cast<unsigned long long *>(mgp_sm)[o_red + w];
    }
    __device__ __forceinline__ double &s_edge(int j) const { return mgp_sm[o_edge + j]; }
    __device__ __forceinline__ unsigned long long &s_cmax(int j) const {
        return reinterpret_cast<unsigned long long *>(mgp_sm)[o_cmax + j];
    }
    // thread-relative accessors (runs of 4 or 8 cells): element i0 + x with
    // x a literal after unrolling -> base register + immediate
    static constexpr bool kRel = (P == 4 || P == 8 || P == 16);
    static constexpr bool kFusedCommit = true;   // phi_commit available (sweep_body)
    static constexpr bool kLL = LL && CS > 1;
    static __host__ __device__ constexpr int rel(int x) { return x + (x >> LG); }
    __device__ __forceinline__ double &u_rel(int x) const { return mgp_sm[o_u + b + rel(x + H)]; }
    __device__ __forceinline__ double &L_rel(int x) const { return mgp_sm[o_L + b + rel(x)]; }
    __device__ __forceinline__ double &R_rel(int x) const { return mgp_sm[o_R + b + rel(x)]; }
    __device__ __forceinline__ double &u0_rel(int x) const { return mgp_sm[o_u0 + b + rel(x)]; }
    // barrier over the CTAs sharing the field (hardware cluster barrier; an
    // mbarrier-based all-to-all with one arriving thread per CTA measured
    // 1.8-2.5x slower per stage on B200)
    __device__ __forceinline__ void sync() {
        if (!LL) {
            field_sync<CS>();
            return;
        }
        // LL: the barrier is local.  The neighbours' boundary cells sent at
        // their last commit are fetched afterwards by the two warps that read
        // them -- with runs of P >= H cells the left halo is read only by the
        // slab's first thread and the right halo only by its last -- so the
        // other warps start their reconstruction without waiting for the
        // neighbours.  Reuse of a box two exchanges later is safe: a sender
        // reaches that commit only after this CTA's next alpha, sent after
        // these reads.
        if (halo_pending && ns % PC != 0) {
            // a partial last run: the right halo has readers in two warps;
            // fetch both halos before the barrier instead
            const int tid = threadIdx.x;
            if (tid < 2 * H) {
                const int par = eB & 1;
                if (tid < H)
                    s_u(sk(ns + H + tid)) = ll_recv(box(par, q, kLLFromRight + 2 * tid), eB, ll_fail);
                else
                    s_u(sk(tid - H)) = ll_recv(box(par, q, kLLFromLeft + 2 * (tid - H)), eB, ll_fail);
            }
            halo_pending = false;
        }
        __syncthreads();
        if (halo_pending) {
            static_assert(!LL || (P >= 4 && K >= 1), "LL mode: merged runs of >= 4 cells");
            const int tid = threadIdx.x, lane = tid & 31;
            const int par = eB & 1;
            if (tid < 32) {            // cells [-H, 0) = the left neighbour's last H cells
                if (lane < H) s_u(sk(lane)) = ll_recv(box(par, q, kLLFromLeft + 2 * lane), eB, ll_fail);
                __syncwarp();
            }
            if (tid >> 5 == (ns / PC - 1) >> 5) {   // warp of the slab's last run
                // cells [ns, ns + H) = the right neighbour's first H cells
                if (lane < H)
                    s_u(sk(ns + H + lane)) = ll_recv(box(par, q, kLLFromRight + 2 * lane), eB, ll_fail);
                __syncwarp();
            }
            halo_pending = false;
        }
    }
    // LL: the commit / put phase that follows sends halo cells with this tag
    __device__ __forceinline__ void begin_halo_exchange() {
        if (LL && !halo_pending) {
            ++eB;
            halo_pending = true;
        }
    }
    __device__ __forceinline__ void send_halo(int t, double v) {
        // local cell t < H -> the left neighbour's right halo; t >= ns - H ->
        // the right neighbour's left halo
        if (t < H) ll_send(box(eB & 1, left(), kLLFromRight + 2 * t), v, eB);
        if (t >= ns - H) ll_send(box(eB & 1, right(), kLLFromLeft + 2 * (t - (ns - H))), v, eB);
    }

    static constexpr int HALO = H;
    __device__ __forceinline__ double cell(int t) const { return s_u(sk(t + H)); }
    __device__ __forceinline__ void load(int t, double v) { s_u(sk(t + H)) = v; }
    // centred reconstruction with the merged flux / rhs pass: each thread
    // forms the flux of the interface left of its run itself; the stage
    // values are committed into s_u after the alpha barrier, when every
    // reconstruction has read it.  On a
    // cluster (CS > 1) the slab's last window (centred on the right
    // neighbour's cell 0) is the neighbour's left state of its interface 0,
    // pushed into its s_L; the states of the interface left of the slab
    // arrive in s_edge as before.
    static constexpr bool kMerged =
#ifdef MGP_SLIDING_RECON
        false;
#else
        P > 0 && K > 0;
#endif
    __device__ __forceinline__ void put(int t, double v) {
        s_u(sk(t + H)) = v;
        if (CS == 1) {
            if (t < H) s_u(sk(ns + H + t)) = v;
            if (t >= ns - H) s_u(sk(t - (ns - H))) = v;
        } else if (LL) {
            send_halo(t, v);
        } else {
            if (t < H) r_u_left[sk(ns + H + t)] = v;
            if (t >= ns - H) r_u_right[sk(t - ns + H)] = v;
        }
    }

    // Left/right interface states of the owned run -> s_L, s_R; returns the
    // bits of this thread's NaN-propagating max |u| (Burgers).
    __device__ __forceinline__ unsigned long long reconstruct(const Consts &k) {
        unsigned long long m = 0;
        constexpr bool kCheck = (MODEL != MGP_MODEL_BURGERS);
        if (P == 0 && K > 0) {
            const int tid = threadIdx.x;
            const int side = (tid >> 5) & 1;              // warp-uniform
            const int i = ((tid >> 6) << 5) + (tid & 31);
            if (i >= ns) return 0;
            const int ctr = i + side;                      // window centre
            double win[2 * K + 1];
#pragma unroll
            for (int t = 0; t <= 2 * K; ++t) win[t] = cell(ctr - K + t);
            bool badw = false;
#pragma unroll
            for (int t = 0; t <= 2 * K; ++t) badw |= !is_finite(win[t]);
            double b[K + 1], q[K + 1];
            if (side == 0) {
#pragma unroll
                for (int s2 = 0; s2 <= K; ++s2) {
                    double dummy;
                    beta_block<K, false, true>(win, s2, b[s2], dummy);
                }
#pragma unroll
                for (int r = 0; r <= K; ++r) q[r] = cand_left<K, REG>(win, r);
            } else {
#pragma unroll
                for (int s2 = 0; s2 <= K; ++s2) {
                    double dummy;
                    beta_block<K, true, false>(win, s2, dummy, b[K - s2]);
                }
#pragma unroll
                for (int r = 0; r <= K; ++r) q[r] = cand_right<K, REG>(win, r);
            }
            double v = weno_value<K>(b, q, k.eps, nullptr, MODEL == MGP_MODEL_BURGERS && badw);
            if (kCheck && badw) v = __longlong_as_double(kNaNBits);
            if (side == 0) s_L(sk(i)) = v;
            else s_R(sk(i)) = v;
            if (CS > 1 && i == ns - 1) push_edge(side, v);
            if (MODEL == MGP_MODEL_BURGERS) {
                m = abs_bits(v);
                if (side == 0 && !is_finite(win[K])) m = kNaNBits;
            }
            return m;
        }
        if (kMerged) return reconstruct_centred(k);
        const int n = (ns - i0 < PC) ? ns - i0 : PC;
        if (n <= 0) return 0;
        if (K == 0) {
            // beta = 0, omega = raw/raw (1, or NaN when 1/eps^2 overflows)
            double c0 = cell(i0);
#pragma unroll 1
            for (int p = 0; p < n; ++p) {
                const int i = i0 + p;
                const double c1 = cell(i + 1);
                double ul = k.k0_omega * (CW(0, 0, 0) * c0);
                double ur = k.k0_omega * (CW(0, 0, 0) * c1);
                if (kCheck) {
                    if (!is_finite(c0)) ul = __longlong_as_double(kNaNBits);
                    if (!is_finite(c1)) ur = __longlong_as_double(kNaNBits);
                }
                s_L(sk(i)) = ul;
                s_R(sk(i)) = ur;
                if (CS > 1 && i == ns - 1) {
                    push_edge(0, ul);
                    push_edge(1, ur);
                }
                if (MODEL == MGP_MODEL_BURGERS) {
                    m = umax64(m, umax64(abs_bits(ul), abs_bits(ur)));
                    if (!is_finite(c0)) m = kNaNBits;
                }
                c0 = c1;
            }
            return m;
        }
        double win[2 * K + 1];
#pragma unroll
        for (int t = 0; t <= 2 * K; ++t) win[t] = cell(i0 - K + t);
        // warm-up: left state data of the first interface
        double bl[K + 1], ql[K + 1];
#pragma unroll
        for (int s = 0; s <= K; ++s) {
            double dummy;
            beta_block<K, false>(win, s, bl[s], dummy);
        }
#pragma unroll
        for (int r = 0; r <= K; ++r) ql[r] = cand_left<K, REG>(win, r);
        MGP_UNROLL(MGP_SLIDE_UNROLL)
        for (int p = 0; p < n; ++p) {
            const int i = i0 + p;
            // window of the left state at i+1; the nonfinite flag covers the
            // left window of interface i (Burgers: any non-finite cell makes
            // the reference's alpha NaN)
            const bool bad_here = !is_finite(win[K]);
            bool bad_left = false;
            if (kCheck) {
#pragma unroll
                for (int t = 0; t <= 2 * K; ++t) bad_left |= !is_finite(win[t]);
            }
#pragma unroll
            for (int t = 0; t < 2 * K; ++t) win[t] = win[t + 1];
            win[2 * K] = cell(i + 1 + K);
            bool bad_right = false;
            if (kCheck) {
#pragma unroll
                for (int t = 0; t <= 2 * K; ++t) bad_right |= !is_finite(win[t]);
            }
            double bl_next[K + 1], br[K + 1], ql_next[K + 1], qr[K + 1];
#pragma unroll
            for (int s = 0; s <= K; ++s) beta_block<K, true>(win, s, bl_next[s], br[K - s]);
#pragma unroll
            for (int r = 0; r <= K; ++r) {
                ql_next[r] = cand_left<K, REG>(win, r);
                qr[r] = cand_right<K, REG>(win, r);
            }
            const bool burg = MODEL == MGP_MODEL_BURGERS;
            double ul = weno_value<K>(bl, ql, k.eps, burg ? win : nullptr, burg && bad_here);
            double ur = weno_value<K>(br, qr, k.eps, burg ? win : nullptr, burg && bad_here);
            if (kCheck) {
                if (bad_left) ul = __longlong_as_double(kNaNBits);
                if (bad_right) ur = __longlong_as_double(kNaNBits);
            }
            s_L(sk(i)) = ul;
            s_R(sk(i)) = ur;
            if (CS > 1 && i == ns - 1) {
                push_edge(0, ul);
                push_edge(1, ur);
            }
            if (MODEL == MGP_MODEL_BURGERS) {
                m = umax64(m, umax64(abs_bits(ul), abs_bits(ur)));
                if (bad_here) m = kNaNBits;
            }
#pragma unroll
            for (int s = 0; s <= K; ++s) {
                bl[s] = bl_next[s];
                ql[s] = ql_next[s];
            }
        }
        return m;
    }

    // Whole-field CTA (CS = 1), P cells per thread: iteration p takes the
    // window centred on cell c = i0 + 1 + p and produces the two states that
    // window defines -- the left state of interface c (stored at c mod ns)
    // and the right state of interface c - 1 -- from one set of beta
    // products (forward and reverse sums, see beta_block).  The left state of
    // the thread's first interface i0 is the previous thread's last
    // iteration, so no window is evaluated twice and nothing is carried
    // between iterations; the fully unrolled loop keeps the sliding window
    // in registers without copies.
    // states owed to the right neighbour: the two states of this slab's last
    // interface (its s_edge) and the left state of its interface 0.  The
    // alpha exchange that follows the reconstruction carries tag eA + 1.
    __device__ __forceinline__ void push_edge(int side, double v) {
        if (LL) ll_send(box((eA + 1) & 1, right(), kLLStates + 2 * side), v, eA + 1);
        else r_edge_right[side] = v;
    }
    __device__ __forceinline__ void push_L0(double v) {
        if (LL) ll_send(box((eA + 1) & 1, right(), kLLStates + 4), v, eA + 1);
        else r_L_right[0] = v;
    }
    __device__ __forceinline__ void store_states(int c, double ul, double ur) {
        if (CS == 1) {
            s_L(sk(c == ns ? 0 : c)) = ul;
        } else if (c == ns) {
            push_L0(ul);                // L state of the neighbour's interface 0
            push_edge(1, ur);           // R state of the slab's last interface
        } else {
            s_L(sk(c)) = ul;
            if (c == ns - 1) push_edge(0, ul);
        }
        s_R(sk(c - 1)) = ur;
    }
    // the same for window p of a full run (c = i0 + 1 + p <= ns, equality
    // only for the last window of the field's last run): literal offsets
    __device__ __forceinline__ void store_states_rel(int p, double ul, double ur) {
        const int c = i0 + 1 + p;
        if (p == PC - 1 && c == ns) {
            if (CS == 1) {
                s_L(0) = ul;
            } else {
                push_L0(ul);
                push_edge(1, ur);
            }
        } else {
            L_rel(1 + p) = ul;
            if (CS > 1 && p >= PC - 2 && c == ns - 1) push_edge(0, ul);
        }
        R_rel(p) = ur;
    }

    // The whole run with the fast-path division sequences and NO branch: the
    // validity tests of every state of the run are AND-ed into one flag that
    // is examined after the loop, so the fully unrolled loop is one basic
    // block and the scheduler can overlap one window's beta products with
    // the previous window's division chains (and the left with the right
    // state's).  A run with any state outside the fast-path range is redone
    // by reconstruct_run_exact (out of line).
    __device__ __forceinline__ unsigned long long reconstruct_centred(const Consts &k) {
        unsigned long long m = 0;
        constexpr bool kCheck = (MODEL != MGP_MODEL_BURGERS);
        constexpr bool burg = (MODEL == MGP_MODEL_BURGERS);
        const int n = (ns - i0 < PC) ? ns - i0 : PC;
        if (n <= 0) return 0;
        if (n < PC) return reconstruct_run_exact(k, n, true);
        double win[2 * K + 1];
#pragma unroll
        for (int t = 0; t < 2 * K; ++t)
            win[t + 1] = kRel ? u_rel(1 - K + t) : cell(i0 + 1 - K + t);
        bool ok = true;
        constexpr int kCU = MGP_CU(PC);
#pragma unroll(kCU)
        for (int p = 0; p < PC; ++p) {
            const int c = i0 + 1 + p;
#pragma unroll
            for (int t = 0; t < 2 * K; ++t) win[t] = win[t + 1];
            win[2 * K] = kRel ? u_rel(1 + p + K) : cell(c + K);
            double bl[K + 1], br[K + 1], ql[K + 1], qr[K + 1];
#pragma unroll
            for (int s = 0; s <= K; ++s) beta_block<K, true>(win, s, bl[s], br[K - s]);
#pragma unroll
            for (int r = 0; r <= K; ++r) {
                ql[r] = cand_left<K, REG>(win, r);
                qr[r] = cand_right<K, REG>(win, r);
            }
            double ul = weno_value_nc<K>(bl, ql, k.eps, ok);
            double ur = weno_value_nc<K>(br, qr, k.eps, ok);
            if (kCheck) {
                bool bad = false;
#pragma unroll
                for (int t = 0; t <= 2 * K; ++t) bad |= !is_finite(win[t]);
                if (bad) {
                    ul = __longlong_as_double(kNaNBits);
                    ur = ul;
                }
            }
            if (kRel) store_states_rel(p, ul, ur);
            else store_states(c, ul, ur);
            if (burg) {
                m = umax64(m, umax64(abs_bits(ul), abs_bits(ur)));
                // a non-finite cell makes the reference's alpha NaN
                if (!is_finite(win[K])) m = kNaNBits;
            }
        }
        // A non-finite centre cell already made this run's alpha bits NaN:
        // the field's alpha is NaN and every flux NaN whatever the states
        // are, so the exact pass has nothing to repair (diverged iterates
        // are mostly such fields).
        if (!ok && !(burg && m == kNaNBits)) m = reconstruct_run_exact(k, n, false);
        return m;
    }

    // The run's states with IEEE division (weno.py:161-177 as written):
    // `all` = every state of the run (a partial run); otherwise only the
    // states the fast pass could not take exactly.  Burgers: a window with a
    // non-finite cell means a non-finite cell in the field, hence a NaN alpha
    // and NaN fluxes everywhere (flux.py:77-88) -- its states cannot reach the
    // result and keep the fast values (`moot`), and the run's alpha bits are
    // NaN.  Returns the run's alpha bits.
    __device__ __noinline__ unsigned long long reconstruct_run_exact(const Consts &k, int n,
                                                                     bool all) {
        unsigned long long m = 0;
        constexpr bool kCheck = (MODEL != MGP_MODEL_BURGERS);
        constexpr bool burg = (MODEL == MGP_MODEL_BURGERS);
        for (int p = 0; p < n; ++p) {
            const int c = i0 + 1 + p;
            double win[2 * K + 1];
#pragma unroll
            for (int t = 0; t <= 2 * K; ++t) win[t] = cell(c - K + t);
            bool bad = false;
#pragma unroll
            for (int t = 0; t <= 2 * K; ++t) bad |= !is_finite(win[t]);
            if (burg && bad && !all) {
                m = kNaNBits;
                continue;
            }
            double bl[K + 1], br[K + 1], ql[K + 1], qr[K + 1];
#pragma unroll
            for (int s = 0; s <= K; ++s) beta_block<K, true>(win, s, bl[s], br[K - s]);
#pragma unroll
            for (int r = 0; r <= K; ++r) {
                ql[r] = cand_left<K, REG>(win, r);
                qr[r] = cand_right<K, REG>(win, r);
            }
            double ul = weno_value_ieee<K>(bl, ql, k.eps);
            double ur = weno_value_ieee<K>(br, qr, k.eps);
            if (kCheck && bad) {
                ul = __longlong_as_double(kNaNBits);
                ur = ul;
            }
            store_states(c, ul, ur);
            if (burg) {
                m = umax64(m, umax64(abs_bits(ul), abs_bits(ur)));
                if (!is_finite(win[K]) || bad) m = kNaNBits;
            }
        }
        return m;
    }

    // A = SemiDiscreteOperator.rhs(s_u) for the owned cells (flux.py:70-88,
    // 159-161).  Precondition: s_u complete (caller synchronised).  On
    // return A[] holds the owned cells' rhs; s_u is unchanged.
    __device__ __forceinline__ double lf(const Consts &k, double ul, double ur,
                                         double half_alpha) const {
        double fl, fr;
        if (MODEL == kModelBurgersRoe) {
            // Roe flux with Harten-Hyman entropy fix for Burgers
            // (flux.py:91-126, models.py:125-128): lam = 0.5 (uL + uR),
            // delta = max(0, max(lam - uL, uR - lam)) (np.maximum, NaN-
            // propagating), speed = |lam| < delta ? 0.5 (lam lam / delta + delta)
            // : |lam|; F = 0.5 (f(uL) + f(uR)) - 0.5 (speed (uR - uL))
            fl = (0.5 * ul) * ul;
            fr = (0.5 * ur) * ur;
            const double lam = 0.5 * (ul + ur);
            const double a = lam - ul, b = ur - lam;
            const double inner = (a >= b || a != a) ? a : b;
            const double delta = (0.0 >= inner || 0.0 != 0.0) ? 0.0 : inner;
            const double alam = fabs(lam);
            const double speed = (alam < delta) ? 0.5 * ((lam * lam) / delta + delta) : alam;
            const double diss = speed * (ur - ul);
            return (0.5 * (fl + fr)) - (0.5 * diss);
        }
        if (MODEL == MGP_MODEL_BURGERS) {
            fl = (0.5 * ul) * ul;
            fr = (0.5 * ur) * ur;
        } else {
            fl = k.speed * ul;
            fr = k.speed * ur;
        }
        return (0.5 * (fl + fr)) - (half_alpha * (ur - ul));
    }

    // First order (K = 0) on full runs, one CTA per field: the "interface
    // states" are the cells themselves (left state of i+1/2 = omega c_i, right
    // state = omega c_{i+1}, omega = raw/raw), so a thread keeps the P + 2
    // states of its run and its two neighbours in registers and forms alpha's
    // contribution, the P + 1 fluxes and the rhs from them -- no interface
    // arrays, no flux pass, one barrier (alpha) instead of three.  Same
    // operations on the same values as the staged path (bit-identical).
    static constexpr bool kReg0 = (K == 0 && kRel && CS == 1);
    __device__ __forceinline__ void rhs_first_order(const Consts &k, double *A) {
        constexpr bool kCheck = (MODEL != MGP_MODEL_BURGERS);
        double sv[PC + 2];     // states of cells i0 - 1 .. i0 + PC
        unsigned long long m = 0;
        if (i0 < ns) {
#pragma unroll
            for (int x = 0; x < PC + 2; ++x) {
                const double c = u_rel(x - 1);
                double v = k.k0_omega * (CW(0, 0, 0) * c);
                if (kCheck && !is_finite(c)) v = __longlong_as_double(kNaNBits);
                sv[x] = v;
                if (MODEL == MGP_MODEL_BURGERS && x >= 1) {
                    // interfaces i0 .. i0 + PC - 1: left states sv[1..PC],
                    // right states sv[2..PC+1]; a non-finite cell of the
                    // run makes the reference's alpha NaN
                    m = umax64(m, abs_bits(v));
                    if (x <= PC && !is_finite(c)) m = kNaNBits;
                }
            }
        }
        double half_alpha;
        if (MODEL == MGP_MODEL_BURGERS) {
            m = warp_umax64(m);
            const int tid = threadIdx.x;
            if ((tid & 31) == 0) s_red(tid >> 5) = m;
            __syncthreads();
            const int nw = (blockDim.x + 31) >> 5;
            m = warp_umax64((tid & 31) < nw ? s_red(tid & 31) : 0ull);
            half_alpha = 0.5 * __longlong_as_double((long long)m);
        } else {
            half_alpha = k.half_alpha_adv;
            __syncthreads();   // every run has read its neighbours' cells before any commit
        }
        if (i0 < ns) {
            double fm = lf(k, sv[0], sv[1], half_alpha);
            double neg[PC];
#pragma unroll
            for (int p = 0; p < PC; ++p) {
                const double f = lf(k, sv[p + 1], sv[p + 2], half_alpha);
                neg[p] = -(f - fm);
                fm = f;
            }
            if (k.dx_pow2) {
#pragma unroll
                for (int p = 0; p < PC; ++p) A[p] = neg[p] * k.inv_dx;
            } else {
#pragma unroll
                for (int p = 0; p < PC; ++p) A[p] = neg[p] / k.dx;
            }
        }
    }

    __device__ __forceinline__ void rhs(const Consts &k, double *A, double *u0r = nullptr,
                                        int sg = 0) {
        if (kReg0 && ns % PC == 0) {   // uniform over the CTA
            rhs_first_order(k, A);
            return;
        }
        trace(1);
        unsigned long long m = reconstruct(k);
        trace(2);
        if (U0G && sg > 0) {
            // the RK base of the run, issued ahead of the alpha barrier that
            // hides its L2 latency (a thread beyond the field reads its own
            // padding slice of the row)
#pragma unroll
            for (int p = 0; p < (U0G ? PC : 0); p += 4) ldg_cg4(u0g + i0 + p, u0r + p);
        }
        double half_alpha;
        if (MODEL == MGP_MODEL_BURGERS) {
            m = warp_umax64(m);
            const int tid = threadIdx.x;
            if ((tid & 31) == 0) s_red(tid >> 5) = m;
            __syncthreads();
            // at most kMaxThreads / 32 = 16 warps: one slot per lane
            const int nw = (blockDim.x + 31) >> 5;
            m = warp_umax64((tid & 31) < nw ? s_red(tid & 31) : 0ull);
            if (CS > 1 && LL) {
                // all-to-all of the CTAs' alpha bits through the mailbox, and
                // the three states the left neighbour computed for this slab
                ++eA;
                const int par = eA & 1;
                if (tid < 32) {
                    if (tid == 0)
                        ll_send(box(par, q, kLLAlpha), __longlong_as_double((long long)m), eA);
                    unsigned long long v = 0;
                    if (tid < CS)
                        v = (unsigned long long)__double_as_longlong(
                            ll_recv(box(par, tid, kLLAlpha), eA, ll_fail));
                    v = warp_umax64(v);
                    if (tid == 0) s_cmax(0) = v;
                    if (tid < 3) {
                        const double sv = ll_recv(box(par, q, kLLStates + 2 * tid), eA, ll_fail);
                        if (tid < 2) s_edge(tid) = sv;
                        else s_L(0) = sv;
                    }
                }
                __syncthreads();
                m = s_cmax(0);
            } else if (CS > 1) {
                if (threadIdx.x == 0) {
                    cg::cluster_group cl = cg::this_cluster();
#pragma unroll
                    for (int j = 0; j < CS; ++j) cl.map_shared_rank(&s_cmax(0), j)[q] = m;
                }
                sync();   // also publishes the pushed edge states
                m = s_cmax(0);
#pragma unroll
                for (int j = 1; j < CS; ++j) m = umax64(m, s_cmax(j));
            }
            half_alpha = 0.5 * __longlong_as_double((long long)m);
        } else {
            half_alpha = k.half_alpha_adv;
            // CS = 1: the left state of each run's first interface was
            // written by the previous thread (reconstruct_centred)
            if (CS > 1) sync();
            else if (P > 0 && K > 0) __syncthreads();
        }
        trace(3);
        if (kMerged) {
            // each thread forms the flux of the interface left of its run
            // itself (one extra flux per run) instead of a flux pass, a
            // barrier and a re-read
            if (i0 < ns) {
                // interface left of the run: sk(i0 - 1) = b + rel(-1)
                const int il = (i0 == 0) ? sk(ns - 1) : (kRel ? b + rel(-1) : sk(i0 - 1));
                double fm = (CS > 1 && i0 == 0)
                                ? lf(k, s_edge(0), s_edge(1), half_alpha)
                                : lf(k, s_L(il), s_R(il), half_alpha);
                if (kRel && i0 + PC <= ns) {
                    // full run: straight-line code, literal offsets
                    double neg[PC];
#pragma unroll
                    for (int p = 0; p < PC; ++p) {
                        const double f = lf(k, L_rel(p), R_rel(p), half_alpha);
                        neg[p] = -(f - fm);
                        fm = f;
                    }
                    if (k.dx_pow2) {
#pragma unroll
                        for (int p = 0; p < PC; ++p) A[p] = neg[p] * k.inv_dx;
                    } else {
#pragma unroll
                        for (int p = 0; p < PC; ++p) A[p] = neg[p] / k.dx;
                    }
                } else {
#pragma unroll
                    for (int p = 0; p < PC; ++p) {
                        const int c = i0 + p;
                        if (c < ns) {
                            const double f = kRel ? lf(k, L_rel(p), R_rel(p), half_alpha)
                                                  : lf(k, s_L(sk(c)), s_R(sk(c)), half_alpha);
                            const double neg = -(f - fm);
                            A[p] = k.dx_pow2 ? neg * k.inv_dx : neg / k.dx;
                            fm = f;
                        }
                    }
                }
            }
            trace(4);
            return;
        }
#pragma unroll
        for (int p = 0; p < PC; ++p) {
            const int i = i0 + p;
            if (i < ns) s_L(sk(i)) = lf(k, s_L(sk(i)), s_R(sk(i)), half_alpha);
        }
        __syncthreads();
#pragma unroll
        for (int p = 0; p < PC; ++p) {
            const int c = i0 + p;
            if (c < ns) {
                double fm;
                if (c > 0) fm = s_L(sk(c - 1));
                else if (CS == 1) fm = s_L(sk(ns - 1));
                else fm = lf(k, s_edge(0), s_edge(1), half_alpha);
                const double neg = -(s_L(sk(c)) - fm);
                A[p] = k.dx_pow2 ? neg * k.inv_dx : neg / k.dx;
            }
        }
        trace(4);
    }

    // The RK base and the stage values live in shared memory (s_u0, s_u; the
    // base in a global row with U0G), so no per-cell state is held in
    // registers across the reconstruction.
    __device__ __forceinline__ double u0(int p) const {
        return (i0 + p < ns) ? (kRel ? u0_rel(p) : s_u0(sk(i0 + p))) : 0.0;
    }

    // Runge-Kutta stage value of the run's cells from the stage's rhs A
    // (stepper.py:50-62, Python's left-to-right scalars); the stage is
    // selected once, outside the cell loop.
    // FULL: a full run addressed by literal offsets (no per-cell range test)
    template <bool FULL>
    __device__ __forceinline__ double u0v(int p, const double *u0r) const {
        if (U0G) return u0r[p];
        if (FULL) return u0_rel(p);
        return u0(p);
    }
    template <bool FULL>
    __device__ __forceinline__ double stv(int p) const {
        if (FULL) return u_rel(p);
        return stage(p);
    }
    template <bool FULL = false>
    __device__ __forceinline__ void rk_update(const Consts &k, int rk, int sg, const double *A,
                                              double *st, const double *u0r) {
        const int code = rk == 0 ? 0 : (sg == 0 ? 1 : (rk == 2 ? 2 : (sg == 1 ? 3 : 4)));
        switch (code) {
            case 0:
#pragma unroll
                for (int p = 0; p < PC; ++p) st[p] = A[p];
                break;
            case 1:
#pragma unroll
                for (int p = 0; p < PC; ++p) st[p] = u0v<FULL>(p, u0r) + k.dt * A[p];
                break;
            case 2:
#pragma unroll
                for (int p = 0; p < PC; ++p)
                    st[p] = ((0.5 * u0v<FULL>(p, u0r)) + (0.5 * stv<FULL>(p))) + (k.hdt * A[p]);
                break;
            case 3:
#pragma unroll
                for (int p = 0; p < PC; ++p)
                    st[p] = ((0.75 * u0v<FULL>(p, u0r)) + (0.25 * stv<FULL>(p))) + (k.qdt * A[p]);
                break;
            default: {
                // u0 / 3.0: the reciprocal of 3 refined once for the run
                // (div_shared.cuh: the compiler's own fast-path sequence and
                // validity test, IEEE `/` otherwise -- bit-identical to `/`)
                const SharedRcp R3 = shared_rcp(3.0);
                bool bad = false;
                double third[PC];
#pragma unroll
                for (int p = 0; p < PC; ++p) third[p] = mgp::div_fast(u0v<FULL>(p, u0r), R3, bad);
                if (bad) {
#pragma unroll 1
                    for (int p = 0; p < PC; ++p) third[p] = mgp::div_slow(u0v<FULL>(p, u0r), 3.0);
                }
#pragma unroll
                for (int p = 0; p < PC; ++p)
                    st[p] = (third[p] + (k.two3 * stv<FULL>(p))) + (k.tdt * A[p]);
            }
        }
    }

    // Phi = RungeKuttaStepper.advance(s_u) (stepper.py:50-62) for the owned
    // cells; rk_order 0 gives the rhs.  The last stage's values (+ 0.0 for
    // g_mode ZERO, sweep_body's add_g for the modes without an array) are
    // committed straight into s_u with their halo copies: the next step's
    // input, and where every epilogue reads the result (cell(t)) after the
    // barrier that publishes it.
    __device__ __forceinline__ void phi_commit(const Consts &k, int rk, int g_mode) {
        static_assert(!U0G || ((P % 4 == 0) && (CS == 1 || LL)),
                      "U0G: full runs of a multiple of 4 cells, no hardware cluster");
        if (!U0G) {
#pragma unroll
            for (int p = 0; p < PC; ++p)
                if (i0 + p < ns) {
                    if (kRel) u0_rel(p) = u_rel(p);
                    else s_u0(sk(i0 + p)) = cell(i0 + p);
                }
        }
        const int stages = rk == 0 ? 1 : rk;
        // one call site of the reconstruction for every stage (code size)
#pragma unroll 1
        for (int sg = 0; sg < stages; ++sg) {
            if (sg > 0) {
                trace(5);
                sync();  // committed stage values (and halos) visible
            }
            double A[PC];
            double u0r[U0G ? PC : 1];
            rhs(k, A, u0r, sg);
            double st[PC];
            if (U0G) {
                if (sg == 0) {
                    // the stage input is the RK base: keep it for the later
                    // stages (this thread's slice of the CTA's global row)
#pragma unroll
                    for (int p = 0; p < (U0G ? PC : 0); ++p) u0r[p] = u_rel(p);
                    if (stages > 1) {
#pragma unroll
                        for (int p = 0; p < (U0G ? PC : 0); p += 4) stg_cg4(u0g + i0 + p, u0r + p);
                    }
                }
                rk_update<true>(k, rk, sg, A, st, u0r);
            } else if (kMerged && kRel && i0 + PC <= ns) {
                rk_update<true>(k, rk, sg, A, st, u0r);
            } else {
                rk_update<false>(k, rk, sg, A, st, u0r);
            }
            if (sg == stages - 1 && g_mode == MGP_G_ZERO) {
#pragma unroll
                for (int p = 0; p < PC; ++p) st[p] = st[p] + 0.0;
            }
            commit(st);
        }
    }

    __device__ __forceinline__ double stage(int p) const {
        return (i0 + p < ns) ? (kRel ? u_rel(p) : cell(i0 + p)) : 0.0;
    }

    __device__ __forceinline__ void commit(const double *v) {
        begin_halo_exchange();
        if (kRel && ns >= 2 * PC && (i0 + PC + H <= ns || i0 + PC == ns)) {
            // full run: literal offsets; the periodic halo copies (cells
            // [0, H) and [ns - H, ns), H <= PC) belong to the first and the
            // last run
#pragma unroll
            for (int p = 0; p < PC; ++p) u_rel(p) = v[p];
            if (i0 == 0) {
#pragma unroll
                for (int p = 0; p < H; ++p) {
                    if (CS == 1) s_u(sk(ns + H + p)) = v[p];
                    else if (LL) send_halo(p, v[p]);
                    else r_u_left[sk(ns + H + p)] = v[p];
                }
            }
            if (i0 + PC == ns) {
#pragma unroll
                for (int p = PC - H; p < PC; ++p) {
                    if (CS == 1) s_u(sk(p - (PC - H))) = v[p];
                    else if (LL) send_halo(ns - PC + p, v[p]);
                    else r_u_right[sk(p - (PC - H))] = v[p];
                }
            }
            return;
        }
#pragma unroll
        for (int p = 0; p < PC; ++p)
            if (i0 + p < ns) put(i0 + p, v[p]);
    }
};

__device__ __forceinline__ double add_g(double y, int mode, const double *g, int c) {
    if (mode == MGP_G_ZERO) return y + 0.0;
    if (mode == MGP_G_ARRAY) return y + g[c];
    return y;
}

__device__ __forceinline__ double g_value(int mode, const double *g, int c) {
    return mode == MGP_G_ARRAY ? g[c] : 0.0;
}

// The sweep over chunks (mgp_sweep semantics, include/mgrit_phi.h), generic
// over the propagator held in shared memory (WENO/RK Field or LFField).
template <class F, int CS>
__device__ __forceinline__ void sweep_body(const mgp_sweep_args &a, const Consts &k, F &f,
                                           const int ns, const int q, const int c0,
                                           double *s_sum, double *s_psum, const int nx) {
    // nx: row length in elements (periodic wrap of the halo loads)
    const int tid = threadIdx.x, nt = blockDim.x;
    const int rk = a.phi.rk_order;
    const int total = a.n_steps + (a.tail != MGP_TAIL_NONE ? 1 : 0);
    const int64_t first = blockIdx.x / CS, stride = gridDim.x / CS;

    for (int64_t b = first; b < a.n_chunks; b += stride) {
        double acc_r = 0.0, acc_e = 0.0, acc_n = 0.0;
        const double *x0 = a.start + b * a.start_stride;
        const double *ref = a.ref ? a.ref + b * a.ref_cs : nullptr;
        // slab and halo straight from global memory (periodic)
        for (int t = tid - F::HALO; t < ns + F::HALO; t += nt) {
            int c = c0 + t;
            c = c < 0 ? c + nx : (c >= nx ? c - nx : c);
            const double v = x0[c];
            f.load(t, v);
            if (t >= 0 && t < ns) {
                if (ref) {
                    const double d = v - ref[c];
                    acc_e = acc_e + d * d;
                }
                if (a.count_nonfinite && !is_finite(v)) acc_n += 1.0;
            }
        }
        // WENO/RK fields (Field): every propagator application commits its
        // last stage straight into s_u (Field::phi_commit) -- the next step's
        // input, and where every epilogue reads the result (cell(t)) after
        // the barrier that publishes it.  Plain chained steps without a g
        // array add their + 0.0 in the commit and leave the step's store /
        // error / non-finite count pending: they read s_u back in coalesced
        // order while the next step's reconstruction starts.
        const bool fused = F::kFusedCommit && a.g_mode != MGP_G_ARRAY;
        bool pending = false;
        double *p_st = nullptr;
        const double *p_rs = nullptr;
        auto flush = [&]() {
            if (p_st || p_rs || a.count_nonfinite) {
                for (int t = tid; t < ns; t += nt) {
                    const int c = c0 + t;
                    double v = 0.0;
                    if constexpr (F::kFusedCommit) v = f.cell(t);
                    if (p_st) p_st[c] = v;
                    if (p_rs) {
                        const double d = v - p_rs[c];
                        acc_e = acc_e + d * d;
                    }
                    if (a.count_nonfinite && !is_finite(v)) acc_n += 1.0;
                }
            }
            pending = false;
        };
        for (int s = 1; s <= total; ++s) {
            f.sync();  // s_u and halos complete
            if (pending) flush();
            if constexpr (F::kFusedCommit) {
                const bool step = s <= a.n_steps;
                // ComposedStepper (stepper.py:170-188): Phi = inner^repeats
#pragma unroll 1
                for (int rep = a.phi.repeats; rep > 0; --rep) {
                    f.phi_commit(k, rk, (rep == 1 && step && fused) ? a.g_mode : MGP_G_NONE);
                    if (rep > 1) f.sync();
                }
                if (step && fused) {
                    p_st = a.store ? a.store + b * a.st_cs + (int64_t)(s - 1) * a.st_ss : nullptr;
                    p_rs = ref ? ref + (int64_t)s * a.ref_ss : nullptr;
                    pending = true;
                    continue;
                }
                f.sync();   // the committed result (and its halos) visible
                if (step) {
                    // + g in place: each thread updates the cells it reads
                    f.begin_halo_exchange();
                    const double *g = a.g ? a.g + b * a.g_cs + (int64_t)(s - 1) * a.g_ss : nullptr;
                    double *st = a.store ? a.store + b * a.st_cs + (int64_t)(s - 1) * a.st_ss : nullptr;
                    const double *rs = ref ? ref + (int64_t)s * a.ref_ss : nullptr;
                    for (int t = tid; t < ns; t += nt) {
                        const int c = c0 + t;
                        const double v = add_g(f.cell(t), a.g_mode, g, c);
                        f.put(t, v);
                        if (st) st[c] = v;
                        if (rs) {
                            const double d = v - rs[c];
                            acc_e = acc_e + d * d;
                        }
                        if (a.count_nonfinite && !is_finite(v)) acc_n += 1.0;
                    }
                    continue;
                }
            } else {
            f.phi(k, rk);
            __syncthreads();   // results complete
            // ComposedStepper (stepper.py:170-188): Phi = inner^repeats
            for (int rep = 1; rep < a.phi.repeats; ++rep) {
                for (int t = tid; t < ns; t += nt) f.put(t, f.result(t));
                f.sync();
                f.phi(k, rk);
                __syncthreads();
            }
            if (s <= a.n_steps) {
                const double *g = a.g ? a.g + b * a.g_cs + (int64_t)(s - 1) * a.g_ss : nullptr;
                double *st = a.store ? a.store + b * a.st_cs + (int64_t)(s - 1) * a.st_ss : nullptr;
                const double *rs = ref ? ref + (int64_t)s * a.ref_ss : nullptr;
                for (int t = tid; t < ns; t += nt) {
                    const int c = c0 + t;
                    const double v = add_g(f.result(t), a.g_mode, g, c);
                    f.put(t, v);
                    if (st) st[c] = v;
                    if (rs) {
                        const double d = v - rs[c];
                        acc_e = acc_e + d * d;
                    }
                    if (a.count_nonfinite && !is_finite(v)) acc_n += 1.0;
                }
                continue;
            }
            }   // propagators with result slots (one-step LF family, systems)
            // the tail's Phi(x): Field committed it into s_u, the others hold
            // it in their result slots
            auto res = [&](int t) {
                if constexpr (F::kFusedCommit) return f.cell(t);
                else return f.result(t);
            };
            const double *tg = a.tail_g ? a.tail_g + b * a.tg_s : nullptr;
            if (a.tail == MGP_TAIL_PHI) {
                double *out = a.tail_out + b * a.to_s;
                for (int t = tid; t < ns; t += nt)
                    out[c0 + t] = add_g(res(t), a.tail_g_mode, tg, c0 + t);
            } else if (a.tail == MGP_TAIL_RESTRICT) {
                // mgrit.py:211-215: g_c = (g_f + phi) - psi;
                // u_c = phi + g_f (last-step) or u_f (injection)
                const double *phi = a.aux + b * a.aux_s;
                const double *uf = a.aux2 ? a.aux2 + b * a.aux2_s : nullptr;
                double *gc = a.tail_out + b * a.to_s;
                double *uc = a.tail_out2 + b * a.to2_s;
                for (int t = tid; t < ns; t += nt) {
                    const int c = c0 + t;
                    const double p = phi[c];
                    const double left =
                        (a.tail_g_mode == MGP_G_NONE) ? p : g_value(a.tail_g_mode, tg, c) + p;
                    gc[c] = left - res(t);
                    uc[c] = (a.guess == MGP_GUESS_LAST_STEP) ? add_g(p, a.tail_g_mode, tg, c)
                                                             : uf[c];
                }
            } else {  // MGP_TAIL_RESID, mgrit.py:268: (g + Phi(u_prev)) - u
                const double *tgt = a.aux + b * a.aux_s;
                const bool last = (b == a.n_chunks - 1) && a.ref_last_next;
                const double *rn = (last && a.ref) ? a.ref + (b + 1) * a.ref_cs : nullptr;
                // optional: keep g + Phi(x), which is the value the next
                // C-relaxation of this chunk computes (mgrit.py:182-191)
                double *keep = a.tail_out ? a.tail_out + b * a.to_s : nullptr;
                for (int t = tid; t < ns; t += nt) {
                    const int c = c0 + t;
                    const double y = res(t);
                    const double pred =
                        (a.tail_g_mode == MGP_G_NONE) ? y : g_value(a.tail_g_mode, tg, c) + y;
                    if (keep) keep[c] = pred;
                    const double u = tgt[c];
                    const double r = pred - u;
                    acc_r = acc_r + r * r;
                    if (last) {
                        if (rn) {
                            const double d = u - rn[c];
                            acc_e = acc_e + d * d;
                        }
                        if (a.count_nonfinite && !is_finite(u)) acc_n += 1.0;
                    }
                }
            }
        }
        if (pending) {
            f.sync();
            flush();
        }
        if (a.partials) {
            // fixed-order reduction: warps, CTA, then cluster ranks in order
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                acc_r += __shfl_xor_sync(0xffffffffu, acc_r, o);
                acc_e += __shfl_xor_sync(0xffffffffu, acc_e, o);
                acc_n += __shfl_xor_sync(0xffffffffu, acc_n, o);
            }
            __syncthreads();
            if ((tid & 31) == 0) {
                s_sum[3 * (tid >> 5) + 0] = acc_r;
                s_sum[3 * (tid >> 5) + 1] = acc_e;
                s_sum[3 * (tid >> 5) + 2] = acc_n;
            }
            __syncthreads();
            if (tid < 3) {
                double t = 0.0;
                const int nw = (nt + 31) >> 5;
                for (int w = 0; w < nw; ++w) t = t + s_sum[3 * w + tid];
                if (CS == 1) {
                    a.partials[3 * b + tid] = t;
                } else if constexpr (F::kLL) {
                    // ranks' partials through the mailbox, summed by rank 0
                    // in rank order (as the cluster path).  A chunk may hold
                    // no alpha exchange (no steps), so this exchange carries
                    // its own back-pressure: nobody passes the chunk's last
                    // barrier before rank 0 has read every word.
                    const unsigned e = f.eC + 1;
                    ll_send(f.box(0, q, kLLPsum + 2 * tid), t, e);
                    if (q == 0) {
                        double tt = 0.0;
                        for (int j = 0; j < CS; ++j)
                            tt = tt + ll_recv(f.box(0, j, kLLPsum + 2 * tid), e, f.ll_fail);
                        a.partials[3 * b + tid] = tt;
                    }
                } else {
                    cg::cluster_group cl = cg::this_cluster();
                    cl.map_shared_rank(s_psum, 0)[3 * q + tid] = t;
                }
            }
            if constexpr (F::kLL) {
                ++f.eC;
                if (tid < 32) {
                    __syncwarp();   // rank 0's three readers are done
                    if (tid == 0) {
                        if (q == 0) ll_send(f.box(0, 0, kLLAck), 0.0, f.eC);
                        else (void)ll_recv(f.box(0, 0, kLLAck), f.eC, f.ll_fail);
                    }
                }
            } else if (CS > 1) {
                f.sync();
                if (q == 0 && tid < 3) {
                    double t = 0.0;
                    for (int j = 0; j < CS; ++j) t = t + s_psum[3 * j + tid];
                    a.partials[3 * b + tid] = t;
                }
            }
        }
        f.sync();  // shared buffers are reused by the next chunk
    }
}

template <int K, int REG, int MODEL, int P, int REGS, int CS, bool LL = false>
__global__ void __maxnreg__(REGS) sweep_kernel(const mgp_sweep_args a, const Consts k,
                                               unsigned long long *mbox) {
    using F = Field<K, REG, MODEL, P, CS, LL>;
    F f;
    f.u0g = nullptr;
    f.eA = f.eB = f.eC = 0;
    f.halo_pending = false;
    // LL: this group's region of the mailbox (zeroed by the launch)
    f.mbox = LL ? mbox + (size_t)(blockIdx.x / CS) * 2 * CS * kLLWords : nullptr;
    f.ll_fail = LL ? mbox + (size_t)(gridDim.x / CS) * 2 * CS * kLLWords : nullptr;
    const int nx = (int)a.phi.nx;
    const int ns = nx / CS;            // cells of this CTA's slab
    const int q = (CS == 1) ? 0 : (int)(blockIdx.x % CS);
    const int c0 = q * ns;             // global index of local cell 0
    const int tid = threadIdx.x;
    f.q = q;
    const int o_sum = f.layout(0, ns, tid);    // the four field arrays (smem_bytes)
    double *s_sum = mgp_sm + o_sum;            // [3 * 32]
    double *s_psum = s_sum + 3 * 32;           // [3 * CS] cluster partials
    f.o_edge = o_sum + 3 * 32 + 3 * CS;        // [2]
    f.o_cmax = f.o_edge + 2;                   // [CS]
    f.o_red = f.o_cmax + CS;                   // [32]
    if (CS > 1 && !LL) {
        cg::cluster_group cl = cg::this_cluster();
        f.r_u_left = cl.map_shared_rank(&f.s_u(0), (q + CS - 1) % CS);
        f.r_u_right = cl.map_shared_rank(&f.s_u(0), (q + 1) % CS);
        f.r_edge_right = cl.map_shared_rank(&f.s_edge(0), (q + 1) % CS);
        f.r_L_right = cl.map_shared_rank(&f.s_L(0), (q + 1) % CS);
    }
    sweep_body<F, CS>(a, k, f, ns, q, c0, s_sum, s_psum, nx);
}

// ---------------------------------------------------------------------------
// Sequential march of ONE field over a thread-block cluster (coarse solve
// mgrit.py:219-226, serial solve serial.py:40-61) with ONE cluster barrier
// per Runge-Kutta stage.  CTA q owns the slab of cells [c0, c0 + ns) and
// also keeps G = K+1 ghost cells on each side, which it updates itself: the
// interface states its neighbours computed next to its slab (G+1 on the
// left, G on the right) arrive through distributed shared memory together
// with alpha, before the one barrier, so the ghost cells' fluxes, rhs and
// Runge-Kutta updates are formed locally with the neighbours' exact
// operations (bit-identical values) and the next stage needs no halo
// exchange.  Per stage: reconstruction of the owned interfaces (two
// threads per interface, one per side, as the latency mode of Field), warp
// max -> the alpha slots of every CTA, the barrier, alpha from the slots,
// then one thread per held cell forms both of its interface fluxes and the
// stage value.  Interface states and alpha slots are double-buffered by
// stage parity (a CTA is at most one barrier ahead of its neighbours).
// Same arithmetic as Field::phi + sweep_body (bit-identical); used for
// plain marches (no tail, no partial sums, no repeats).
// ---------------------------------------------------------------------------
// Exchange primitive of the march (round 2): the pushed interface states and
// alpha slots travel as st.async stores that complete on the RECEIVER's
// mbarrier (complete_tx), and every thread of the receiver arrives on the same
// mbarrier after its own shared-memory stores -- so one mbarrier phase per
// stage and CTA replaces the cluster barrier.  A cluster-scope release
// compiles to MEMBAR.ALL.GPU on sm_100a (it waited for the acknowledgement of
// every pushed word: 1.57 `membar` stalls per issue in round 1's ncu); the
// mbarrier needs none.  MGP_MARCH_CLSYNC builds the cluster-barrier variant.
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned mapa_u32(unsigned addr, int rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_b64(unsigned raddr, unsigned long long v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                     raddr),
                 "l"(v), "r"(rbar)
                 : "memory");
}

template <int K, int REG, int CS>
__global__ void __launch_bounds__(512, 1) march_kernel(const mgp_sweep_args a, const Consts k) {
#ifdef MGP_MARCH_CLSYNC
    constexpr bool kAsync = false;
#else
    constexpr bool kAsync = true;
#endif
    __shared__ alignas(8) unsigned long long s_mbar[2];   // one per stage parity
    constexpr int G = K + 1;   // ghost cells per side
    constexpr int IL = G + 1;  // interfaces held left of the slab: local [-IL, -1]
    constexpr int IR = G;      // and right of it: [ns, ns + IR)
    extern __shared__ double smem[];
    const int nx = (int)a.phi.nx;
    const int ns = nx / CS;
    const int q = (int)(blockIdx.x % CS);
    const int c0 = q * ns;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const int ncell = ns + 2 * G;         // cells held: local [-G, ns + G)
    const int ni = ns + IL + IR;          // interfaces held: local [-IL, ns + IR)
    double *s_u0 = smem;                  // RK base, local cell t at [t + G]
    double *s_v = s_u0 + ncell;           // stage input
    double *s_L = s_v + ncell;            // [2][ni] left states, interface i at [i + IL]
    double *s_R = s_L + 2 * ni;           // [2][ni] right states
    // [2][CS][warps] alpha bits by stage parity: every warp of the cluster
    // stores its max into its slot of every CTA
    unsigned long long *s_am = reinterpret_cast<unsigned long long *>(s_R + 2 * ni);
    cg::cluster_group cl = cg::this_cluster();
    double *rl_L = cl.map_shared_rank(s_L, (q + CS - 1) % CS);
    double *rl_R = cl.map_shared_rank(s_R, (q + CS - 1) % CS);
    double *rr_L = cl.map_shared_rank(s_L, (q + 1) % CS);
    double *rr_R = cl.map_shared_rank(s_R, (q + 1) % CS);
    unsigned long long *r_am = cl.map_shared_rank(s_am, lane < CS ? lane : 0);

    for (int t = tid - G; t < ns + G; t += nt) {
        int c = c0 + t;
        c = c < 0 ? c + nx : (c >= nx ? c - nx : c);
        const double v = a.start[c];
        s_u0[t + G] = v;
        s_v[t + G] = v;
    }
    // st.async targets: the neighbours' state arrays and mbarriers, every
    // CTA's alpha slots and mbarriers (lane j < CS addresses CTA j)
    const unsigned a_L = smem_u32(s_L), a_R = smem_u32(s_R), a_am = smem_u32(s_am);
    const unsigned a_bar = smem_u32(s_mbar);
    const int ql = (q + CS - 1) % CS, qr = (q + 1) % CS;
    const unsigned al_L = mapa_u32(a_L, ql), al_R = mapa_u32(a_R, ql), al_bar = mapa_u32(a_bar, ql);
    const unsigned ar_L = mapa_u32(a_L, qr), ar_R = mapa_u32(a_R, qr), ar_bar = mapa_u32(a_bar, qr);
    const unsigned aj_am = mapa_u32(a_am, lane < CS ? lane : 0);
    const unsigned aj_bar = mapa_u32(a_bar, lane < CS ? lane : 0);
    if (kAsync && tid == 0) {
        for (int p2 = 0; p2 < 2; ++p2)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a_bar + 8 * p2), "r"(nt));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl.sync();   // every CTA of the cluster running, loaded, mbarriers initialised
    // bytes a CTA receives per stage: 2 IL states from the left neighbour,
    // 2 IR from the right one, CS * nw alpha slots
    const unsigned tx_bytes = 8u * (unsigned)(2 * IL + 2 * IR + CS * nw);

    const int side = warp & 1;                     // warp-uniform
    const int i = ((warp >> 1) << 5) + lane;       // interface i + 1/2 (local)
    const int t = tid - G;                         // held cell of the update phase
    int cg_ = c0 + t;                              // its global index (periodic)
    cg_ = cg_ < 0 ? cg_ + nx : (cg_ >= nx ? cg_ - nx : cg_);
    const bool upd = t < ns + G;
    const bool own = t >= 0 && t < ns;
    const int rk = a.phi.rk_order;
    const int stages = rk == 0 ? 1 : rk;
    int par = 0;
    int stage_no = 0;        // stages completed: parity par, mbarrier phase (stage_no >> 1) & 1
#ifdef MGP_TRACE
    long long prof[6] = {0, 0, 0, 0, 0, 0}, pt0 = clock64(), pt1;
#define MARCH_PROF(ph) do { pt1 = clock64(); prof[ph] += pt1 - pt0; pt0 = pt1; } while (0)
#else
#define MARCH_PROF(ph) do { } while (0)
#endif
    for (int s = 1; s <= a.n_steps; ++s) {
        // this step's g, loaded ahead of the stages that hide its latency
        double gv = 0.0;
        if (upd && a.g_mode == MGP_G_ARRAY) gv = a.g[(int64_t)(s - 1) * a.g_ss + cg_];
        for (int sg = 0; sg < stages; ++sg, par ^= 1) {
            double *L = s_L + par * ni, *R = s_R + par * ni;
            unsigned long long m = 0;
            if (i < ns) {
                const int ctr = i + side;          // window centre
                double win[2 * K + 1];
#pragma unroll
                for (int w = 0; w <= 2 * K; ++w) win[w] = s_v[ctr - K + w + G];
                double v;
                if constexpr (K == 0) {
                    // first order: beta = 0, omega = raw/raw (Field::reconstruct)
                    v = k.k0_omega * (CW(0, 0, 0) * win[0]);
                } else {
                double b[K + 1], qv[K + 1];
                if (side == 0) {
#pragma unroll
                    for (int s2 = 0; s2 <= K; ++s2) {
                        double dummy;
                        beta_block<K, false, true>(win, s2, b[s2], dummy);
                    }
#pragma unroll
                    for (int r = 0; r <= K; ++r) qv[r] = cand_left<K, REG>(win, r);
                } else {
#pragma unroll
                    for (int s2 = 0; s2 <= K; ++s2) {
                        double dummy;
                        beta_block<K, true, false>(win, s2, dummy, b[K - s2]);
                    }
#pragma unroll
                    for (int r = 0; r <= K; ++r) qv[r] = cand_right<K, REG>(win, r);
                }
                // one range test validates every fast-path division; a
                // window with a non-finite cell is moot (alpha NaN)
                v = weno_value_rc<K>(b, qv, k.eps, win);
                }
                const int o = par * ni;
                (side == 0 ? L : R)[i + IL] = v;
                if (kAsync) {
                    const unsigned long long vb = (unsigned long long)__double_as_longlong(v);
                    if (i < IR)
                        st_async_b64((side == 0 ? al_L : al_R) + 8u * (unsigned)(o + ns + i + IL),
                                     vb, al_bar + 8 * par);
                    if (i >= ns - IL)
                        st_async_b64((side == 0 ? ar_L : ar_R) + 8u * (unsigned)(o + i - ns + IL),
                                     vb, ar_bar + 8 * par);
                } else {
                    if (i < IR) (side == 0 ? rl_L : rl_R)[o + ns + i + IL] = v;
                    if (i >= ns - IL) (side == 0 ? rr_L : rr_R)[o + i - ns + IL] = v;
                }
                m = abs_bits(v);
                // a non-finite cell makes the reference's alpha NaN
                if (side == 0 && !is_finite(win[K])) m = kNaNBits;
            }
            MARCH_PROF(0);
            m = warp_umax64(m);
            if (kAsync) {
                if (lane < CS)
                    st_async_b64(aj_am + 8u * (unsigned)(par * CS * nw + q * nw + warp), m,
                                 aj_bar + 8 * par);
                MARCH_PROF(1);
                // every thread arrives (release: its own shared-memory stores)
                // and waits for the phase: all local arrivals + all pushed bytes
                if (tid == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                                     a_bar + 8 * par),
                                 "r"(tx_bytes)
                                 : "memory");
                else
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a_bar + 8 * par)
                                 : "memory");
                const unsigned phase = (unsigned)(stage_no >> 1) & 1u;
                unsigned done = 0;
                while (!done)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\t"
                        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                        "selp.u32 %0, 1, 0, p;\n\t}"
                        : "=r"(done)
                        : "r"(a_bar + 8 * par), "r"(phase)
                        : "memory");
                ++stage_no;
            } else {
                if (lane < CS) r_am[par * CS * nw + q * nw + warp] = m;
                MARCH_PROF(1);
                cl.sync();   // release / acquire: states, ghosts' interfaces, alpha slots
            }
            MARCH_PROF(2);
            unsigned long long mm = 0;
            for (int l = lane; l < CS * nw; l += 32) mm = umax64(mm, s_am[par * CS * nw + l]);
            mm = warp_umax64(mm);
            const double half_alpha = 0.5 * __longlong_as_double((long long)mm);
            MARCH_PROF(3);
            if (upd) {
                // flux.py:82-88 (Burgers f = (0.5 u) u), flux.py:159-161
                const double ulp = L[t + IL], urp = R[t + IL];
                const double ulm = L[t - 1 + IL], urm = R[t - 1 + IL];
                const double fp = (0.5 * ((0.5 * ulp) * ulp + (0.5 * urp) * urp)) -
                                  (half_alpha * (urp - ulp));
                const double fm = (0.5 * ((0.5 * ulm) * ulm + (0.5 * urm) * urm)) -
                                  (half_alpha * (urm - ulm));
                const double neg = -(fp - fm);
                const double A = k.dx_pow2 ? neg * k.inv_dx : neg / k.dx;
                double st;
                const double u0 = s_u0[tid], stg = s_v[tid];
                if (rk == 0) st = A;
                else if (sg == 0) st = u0 + k.dt * A;
                else if (rk == 2) st = ((0.5 * u0) + (0.5 * stg)) + (k.hdt * A);
                else if (sg == 1) st = ((0.75 * u0) + (0.25 * stg)) + (k.qdt * A);
                else st = ((u0 / 3.0) + (k.two3 * stg)) + (k.tdt * A);
                if (sg == stages - 1) {
                    // sweep_body: + g, store, next step's base
                    if (a.g_mode == MGP_G_ZERO) st = st + 0.0;
                    else if (a.g_mode == MGP_G_ARRAY) st = st + gv;
                    if (own && a.store) a.store[(int64_t)(s - 1) * a.st_ss + c0 + t] = st;
                    s_u0[tid] = st;
                }
                s_v[tid] = st;
            }
            MARCH_PROF(4);
            __syncthreads();
            MARCH_PROF(5);
        }
    }
    if (kAsync) cl.sync();   // no CTA leaves while a peer's pushes may be in flight
#ifdef MGP_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int ph = 0; ph < 6; ++ph) {
            g_trace[2 * ph] = ph;
            g_trace[2 * ph + 1] = prof[ph];
        }
        g_trace_n = 6;
    }
#endif
#undef MARCH_PROF
}

Consts make_consts(const mgp_phi &p);

// Kernel attributes (dynamic shared memory above 48 KB, 16-CTA clusters) are
// per device context: one flag bit per device index, set on first use there.
template <class Kern>
bool ensure_attrs(Kern kern, unsigned long long &devs, bool nonportable_cluster) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    const unsigned long long bit = 1ull << (dev & 63);
    if (devs & bit) return true;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
        cudaSuccess)
        return false;
    if (nonportable_cluster &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
            cudaSuccess)
        return false;
    devs |= bit;
    return true;
}

template <int K, int REG, int CS>
int launch_march(const mgp_sweep_args &a, cudaStream_t st) {
    const int ns = (int)(a.phi.nx / CS);
    const int nt = 2 * ((ns + 31) / 32 * 32);
    const int G = K + 1;
    const size_t sm = sizeof(double) * (size_t)(2 * (ns + 2 * G) + 4 * (ns + 2 * G + 1)) +
                      sizeof(unsigned long long) * (size_t)(2 * CS * (nt / 32));
    auto kern = march_kernel<K, REG, CS>;
    static unsigned long long attr_devs = 0;
    if (!ensure_attrs(kern, attr_devs, CS > 8)) return MGP_ECUDA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)CS);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const Consts kk = make_consts(a.phi);
    if (cudaLaunchKernelEx(&cfg, kern, a, kk) != cudaSuccess) return MGP_ECUDA;
    ++g_launches;
    return cudaPeekAtLastError() == cudaSuccess ? MGP_OK : MGP_ECUDA;
}

// ---------------------------------------------------------------------------
// Fused FCF relaxation of the finest level (mgp_relax_fcf, include/
// mgrit_phi.h).  Chain j (j < nc) = interval j's m-1 F-steps, its C-step
// (new C-point j+1) and, with F-point storage, interval j+1's m-1 final
// F-steps; chain nc = interval 0's final F-steps.  Persistent CTAs (one per
// resident slot) take work from a ticket counter: first whole chains, then
// the last R <= G chains cut into segments of S steps, segment-major, so
// the work still handed out at the end is short and a segment's
// predecessor (the same chain's previous segment) was taken about R
// tickets earlier; the field travels between segments through an
// L2-resident row per split chain.  Dynamic assignment keeps every slot busy
// to the end: co-resident CTAs do not progress at equal rates (the warp
// scheduler favours older warps; measured up to 1.4x on B200), which a
// static split of the steps turns into an idle tail, and hand-overs cost
// about a tenth of a step each (exposed L2 latency), hence whole chains
// wherever the tail allows.
// ---------------------------------------------------------------------------
struct FcfPlan {
    int64_t nc, nchains, W;   // intervals, chains (+1 with F-point storage), tickets
    int64_t K, R;             // chains taken whole; the last R = nchains - K are split
    int64_t Gmax;             // resident CTA slots (workspace layout)
    int64_t A;                // split plan: chains 0..A-1 run their first m steps only
                              // (F-steps + C-step) and queue their final F-steps
    int m, L, S;              // coarsening factor, regular chain length, segment steps
    bool fstore;
    int ordered;              // > 0: chain starts read C-points from host memory (zero-copy);
                              // keep at most `ordered` rows in flight, in ticket order
    int64_t u0_off;           // U0G kernels: byte offset of the CTAs' RK-base rows in the workspace
    __host__ __device__ int len(int64_t j) const {
        if (!fstore) return m;
        if (j < nc - 1) return L;
        return j == nc - 1 ? m : m - 1;
    }
    __host__ __device__ int nseg(int n) const { return (n + S - 1) / S; }
    // split chains with more than t segments (lengths never increase with j)
    __host__ __device__ int64_t count(int t) const {
        int64_t c = R;
        if (fstore) {
            if (nc - 1 >= K && nseg(m) <= t) --c;
            if (nc >= K && nseg(m - 1) <= t) --c;
        }
        return c;
    }
    __host__ __device__ int64_t n_units() const {
        int64_t w = K;
        for (int t = 0; t < nseg(L); ++t) w += count(t);
        return w;
    }
    // ticket i -> chain j and segment t (steps [t S, min((t+1) S, len(j)))),
    // t = -1 for a chain taken whole
    __host__ __device__ void unit(int64_t i, int64_t &j, int &t) const {
        if (i < K) {
            j = i;
            t = -1;
            return;
        }
        i -= K;
        for (int u = 0; u < nseg(L); ++u) {
            const int64_t c = count(u);
            if (i < c) {
                j = K + i;
                t = u;
                return;
            }
            i -= c;
        }
        j = -1;
        t = 0;
    }
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// ring-row tag: chain j has completed s steps (0 = row never used)
__device__ __forceinline__ unsigned long long fcf_tag(int64_t j, int s) {
    return ((unsigned long long)(j + 1) << 20) | (unsigned)s;
}

template <class F>
__device__ __forceinline__ void fcf_load(F &f, const double *x0, int ns, bool coherent) {
    for (int t = (int)threadIdx.x - F::HALO; t < ns + F::HALO; t += blockDim.x) {
        int c = t < 0 ? t + ns : (t >= ns ? t - ns : t);
        f.load(t, coherent ? __ldcg(x0 + c) : x0[c]);
    }
}

template <int K, int REG, int MODEL, int P, int REGS>
__global__ void __maxnreg__(REGS) fcf_kernel(const mgp_fcf_args a, const Consts k,
                                             const FcfPlan pl) {
    __shared__ long long s_ticket, s_chain;
    constexpr bool kU0G = (P == 16);   // runs of 16: two CTAs per SM for 4096-cell fields
    using F = Field<K, REG, MODEL, P, 1, false, kU0G>;
    F f;
    // one row of blockDim.x runs per CTA (threads beyond the field, where the
    // block size is rounded up to a warp, own padding slices)
    f.u0g = kU0G ? reinterpret_cast<double *>(static_cast<char *>(a.workspace) + pl.u0_off) +
                       (size_t)blockIdx.x * (size_t)blockDim.x * P
                 : nullptr;
    const int ns = (int)a.phi.nx;
    const int tid = threadIdx.x, nt = blockDim.x;
    f.q = 0;
    f.o_red = f.layout(0, ns, tid);
    f.o_edge = f.o_cmax = f.o_red;   // unused without a cluster
    // workspace (layout fixed per device and mesh, whatever the call's
    // interval count): ticket, exit and queue counters, one spare | Gmax
    // tags (segment mode) or queue slots (split plan) | Gmax rows
    unsigned long long *ctr = static_cast<unsigned long long *>(a.workspace);
    unsigned long long *tags = ctr + 4;
    unsigned long long *queue = tags;   // split plan (tags are segment-mode only)
    double *ring = reinterpret_cast<double *>(tags + pl.Gmax);
    const double *c0 = a.f0_start ? a.f0_start : a.cs;   // new C-point 0
    const int m = pl.m;
    if (blockIdx.x == 0) {
        for (int c = tid; c < ns; c += nt) {
            const double v = c0[c];
            if (!a.f0_start) a.cd[c] = v;
            if (a.cstore) a.cstore[c] = v;
        }
    }
    for (;;) {
        if (tid == 0) s_ticket = (long long)atomicAdd(ctr, 1ull);
        __syncthreads();   // also: the previous unit's stores to s_u are done
        const int64_t i = s_ticket;
        if (i >= pl.W) break;
#ifdef MGP_FCF_TRACE
        unsigned long long t_unit0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_unit0));
#endif
        int64_t j;
        int seg;
        int s0, s1, len;
        const bool a_only = i < pl.A;              // split plan, first half
        const bool b_unit = pl.A > 0 && i > pl.nc; // split plan, second half
        if (b_unit) {
            // the final F-steps of a chain whose first half has completed, in
            // completion order (queue slot i - nc - 1; 0 = not yet published)
            if (tid == 0) {
                unsigned long long v;
                while ((v = ld_acquire_u64(queue + (i - pl.nc - 1))) == 0ull) __nanosleep(64);
                s_chain = (long long)v - 1;
            }
            __syncthreads();
            j = s_chain;
            seg = -1;
            len = pl.L;
            s0 = m;
            s1 = pl.L;
        } else {
            if (a_only) {
                j = i;
                seg = -1;
            } else {
                pl.unit(i, j, seg);
            }
            len = pl.len(j);
            s0 = seg < 0 ? 0 : seg * pl.S;
            s1 = a_only ? m : (seg < 0 || s0 + pl.S >= len) ? len : s0 + pl.S;
        }
        const bool seg_mode = seg >= 0;
        const int64_t row = j - pl.K;               // split chains only
        double *rrow = ring + (row < 0 ? 0 : row) * ns;
        if (seg_mode && s0 > 0) {
            // a later segment needs the chain's previous one (taken about R
            // tickets earlier, normally long done)
            if (tid == 0)
                while (ld_acquire_u64(tags + row) != fcf_tag(j, s0)) __nanosleep(32);
            __syncthreads();
        }
        if (s0 == 0 && pl.ordered) {
            // zero-copy input: the first wave's rows would otherwise arrive
            // interleaved, every CTA waiting for the whole wave; in ticket
            // order with a bounded window, ticket i's row arrives ~i rows in
            if (i >= pl.ordered) {
                if (tid == 0)
                    while (ld_acquire_u64(ctr + 3) + (unsigned long long)pl.ordered <=
                           (unsigned long long)i)
                        __nanosleep(32);
                __syncthreads();
            }
            fcf_load(f, j == pl.nc ? c0 : a.cs + j * a.cs_s, ns, false);
            __syncthreads();
            if (tid == 0) atomicAdd(ctr + 3, 1ull);
        } else if (s0 == 0) {
            fcf_load(f, j == pl.nc ? c0 : a.cs + j * a.cs_s, ns, false);
        } else if (b_unit) {
            fcf_load(f, a.cd + (j + 1) * a.cd_s, ns, true);
        } else {
            fcf_load(f, rrow, ns, true);
        }
        // Every step's last stage commits its state straight into s_u (the
        // next step's input).  After the barrier that publishes it, the
        // state is flushed from s_u to wherever the step's result goes, in
        // coalesced order, while the next step's reconstruction starts (s_u
        // is next written after that step's alpha barrier).
        double *dst = nullptr, *dst2 = nullptr, *dst3 = nullptr;
        for (int st = s0; st <= s1; ++st) {
            f.sync();
            if (dst || dst2 || dst3) {
                const bool wide = !dst3 && ns % 4 == 0 &&
                                  ((reinterpret_cast<uintptr_t>(dst) |
                                    reinterpret_cast<uintptr_t>(dst2)) & 31) == 0;
                if (wide) {
                    // streaming output: 256-bit stores with L2 evict-first
                    // priority (written once, never read by this launch)
                    for (int c = 4 * tid; c < ns; c += 4 * nt) {
                        double v[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) v[i] = f.cell(c + i);
                        if (dst) stg_stream4(dst + c, v);
                        if (dst2) stg_stream4(dst2 + c, v);
                    }
                } else {
                    for (int c = tid; c < ns; c += nt) {
                        const double v = f.cell(c);
                        if (dst) dst[c] = v;
                        if (dst2) dst2[c] = v;
                        if (dst3) __stcg(dst3 + c, v);
                    }
                }
            }
            if (st == s1) break;
            // ComposedStepper: Phi = inner^repeats, + g after the last (one
            // call site: the propagator's code exists once in the kernel)
#pragma unroll 1
            for (int rep = a.phi.repeats; rep > 0; --rep) {
                f.phi_commit(k, a.phi.rk_order, rep == 1 ? a.g_mode : MGP_G_NONE);
                if (rep > 1) f.sync();
            }
            // where this step's state goes
            dst = dst2 = dst3 = nullptr;
            if (j == pl.nc) {                       // interval 0's final F-steps
                dst = a.fstore + (int64_t)st * a.f_ss;
            } else if (st == m - 1) {               // C-step: new C-point j+1
                dst = a.cd + (j + 1) * a.cd_s;
                if (a.cstore) dst2 = a.cstore + (j + 1) * a.cst_s;
            } else if (st >= m) {                   // interval j+1's final F-steps
                dst = a.fstore + (j + 1) * a.f_cs + (int64_t)(st - m) * a.f_ss;
            }
            if (seg_mode && (st == s1 - 1) && (s1 < len)) dst3 = rrow;   // hand the field on
        }
        if (seg_mode && s1 < len) {
            __threadfence();   // every thread's row stores before the release
            __syncthreads();
            if (tid == 0) st_release_u64(tags + row, fcf_tag(j, s1));
        }
        if (a_only) {
            // new C-point j+1 is in cd: queue the chain's final F-steps
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                const unsigned long long pos = atomicAdd(ctr + 2, 1ull);
                st_release_u64(queue + pos, (unsigned long long)j + 1);
            }
        }
#ifdef MGP_FCF_TRACE
        if (tid == 0 && i < 8192) {
            unsigned long long t1;
            unsigned smid;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            g_fcf_trace[4 * i] = t_unit0;
            g_fcf_trace[4 * i + 1] = t1;
            g_fcf_trace[4 * i + 2] = blockIdx.x;
            g_fcf_trace[4 * i + 3] = smid | ((unsigned long long)(s1 - s0) << 32);
        }
#endif
    }
    // the last CTA out leaves the workspace clean for the next call
    if (tid == 0) {
        __threadfence();
        const unsigned long long done = atomicAdd(ctr + 1, 1ull);
        if (done == (unsigned long long)gridDim.x - 1) {
            for (int64_t r = 0; r < pl.R; ++r) tags[r] = 0ull;
            for (int64_t r = 0; r < pl.A; ++r) queue[r] = 0ull;
            ctr[0] = 0ull;
            ctr[1] = 0ull;
            ctr[2] = 0ull;
            ctr[3] = 0ull;
            __threadfence();
        }
    }
}

// ---------------------------------------------------------------------------
// One-step Lax-Friedrichs family (stepper.py:85-167), Burgers only:
//   E(u)_i = 0.5 (u_{i+1} + u_{i-1}),  D(f)_i = (f_{i+1} - f_{i-1}) / (2 dx)
//   one-step (matched-lf-fine, rediscretized-lf):  Phi(u) = E u - dt D f(u)
//   matched order 0:  E^m u - (m dt) D f(u)
//   matched order 1:  acc = D f(u); v = u; m-1 times { v = E v;
//                     acc = E acc + D f(v) };  Phi(u) = E v - dt_fine acc
// Elementwise NumPy arithmetic: no summation-order subtleties.  The whole
// field lives in shared memory (nx <= kMaxLfNx); one CTA per chunk.
// ---------------------------------------------------------------------------
constexpr int kMaxLfNx = 2048;

template <int MODE>   // 1 = one-step, 2 = matched coarse
struct LFField {
    static constexpr int HALO = 0;
    static constexpr bool kFusedCommit = false;
    static constexpr bool kLL = false;
    int ns;
    double *s_u, *s_R, *s_va, *s_vb, *s_aa, *s_ab, *s_f;

    __device__ __forceinline__ void load(int t, double v) {
        if (t >= 0 && t < ns) s_u[t] = v;
    }
    __device__ __forceinline__ void put(int t, double v) { s_u[t] = v; }
    __device__ __forceinline__ double result(int t) const { return s_R[t]; }
    __device__ __forceinline__ void sync() { __syncthreads(); }
    __device__ __forceinline__ int up(int c) const { return c + 1 == ns ? 0 : c + 1; }
    __device__ __forceinline__ int dn(int c) const { return c == 0 ? ns - 1 : c - 1; }
    __device__ __forceinline__ double E(const double *v, int c) const {
        return 0.5 * (v[up(c)] + v[dn(c)]);
    }
    __device__ __forceinline__ double D(const Consts &k, const double *f, int c) const {
        const double d = f[up(c)] - f[dn(c)];
        return k.twodx_pow2 ? d * k.inv_twodx : d / k.twodx;
    }

    __device__ void phi(const Consts &k, int) {
        const int tid = threadIdx.x, nt = blockDim.x;
        for (int c = tid; c < ns; c += nt) s_f[c] = (0.5 * s_u[c]) * s_u[c];
        __syncthreads();
        if (MODE == 1) {
            for (int c = tid; c < ns; c += nt) s_R[c] = E(s_u, c) - (k.dt * D(k, s_f, c));
            return;
        }
        if (k.lf_order == 0) {
            const double *src = s_u;
            double *dst = s_va;
            for (int j = 0; j < k.m_eff; ++j) {
                for (int c = tid; c < ns; c += nt) dst[c] = E(src, c);
                __syncthreads();
                src = dst;
                dst = (dst == s_va) ? s_vb : s_va;
            }
            for (int c = tid; c < ns; c += nt) s_R[c] = src[c] - (k.dt * D(k, s_f, c));
            return;
        }
        double *acc = s_aa, *accn = s_ab;
        for (int c = tid; c < ns; c += nt) acc[c] = D(k, s_f, c);
        __syncthreads();
        const double *v = s_u;
        double *vn = s_va;
        for (int j = 0; j < k.m_eff - 1; ++j) {
            for (int c = tid; c < ns; c += nt) vn[c] = E(v, c);
            __syncthreads();
            for (int c = tid; c < ns; c += nt) s_f[c] = (0.5 * vn[c]) * vn[c];
            __syncthreads();
            for (int c = tid; c < ns; c += nt) accn[c] = E(acc, c) + D(k, s_f, c);
            __syncthreads();
            v = vn;
            vn = (vn == s_va) ? s_vb : s_va;
            double *t = acc;
            acc = accn;
            accn = t;
        }
        for (int c = tid; c < ns; c += nt) s_R[c] = E(v, c) - (k.dt * acc[c]);
    }
};

template <int MODE>
__global__ void __launch_bounds__(256) lf_kernel(const mgp_sweep_args a, const Consts k) {
    extern __shared__ double smem[];
    LFField<MODE> f;
    const int nx = (int)a.phi.nx;
    f.ns = nx;
    f.s_u = smem;
    f.s_R = f.s_u + nx;
    f.s_va = f.s_R + nx;
    f.s_vb = f.s_va + nx;
    f.s_aa = f.s_vb + nx;
    f.s_ab = f.s_aa + nx;
    f.s_f = f.s_ab + nx;
    double *s_sum = f.s_f + nx;
    double *s_psum = s_sum + 3 * 32;
    sweep_body<LFField<MODE>, 1>(a, k, f, nx, 0, 0, s_sum, s_psum, nx);
}

// ---------------------------------------------------------------------------
// Hyperbolic systems: shallow water (D = 2, models.py:136-211) and Euler
// (D = 3, models.py:214-308); component-major rows of D nx.
// Characteristic WENO (weno.py:203-233, flux.py:127-161): the window of cell
// c is projected onto the left eigenvectors L(c) of cell c, every
// characteristic field is reconstructed (left state of interface c and right
// state of interface c-1 from the same window, sharing the beta products)
// and mapped back with the right eigenvectors R(c).  Shallow water has L in
// closed form (models.py:159-170); Euler takes L = inv(R) (models.py:270),
// computed by inv3() -- LU with partial pivoting in LAPACK's operation order
// (the reference's np.linalg.inv agrees with it to rounding).
// Every contraction over the component axis is summed like the reference's
// einsum: two lanes from +0, (0 + t0 + t2) + (0 + t1); candidate sums use
// the 2-lane order (componentwise reconstruction, characteristic = false:
// the sequential order).  Flux: global LF (alpha = NaN-propagating max of
// |u| + c over both interface states) or Roe with the Harten-Hyman entropy
// fix per wave (flux.py:91-126).  States the reference rejects with
// PhysicalStateError set MGP_STATUS_* bits in *status; the sweep completes.
// One CTA per field, whole field in shared memory (nx <= kMaxSysNx).
// ---------------------------------------------------------------------------
constexpr int kMaxSysNx = 2048;

__device__ __forceinline__ double entropy_fix(double lh, double ll, double lr) {
    const double a = lh - ll, b = lr - lh;
    const double inner = (a >= b || a != a) ? a : b;      // np.maximum
    const double delta = (0.0 >= inner) ? 0.0 : inner;
    const double alam = fabs(lh);
    return (alam < delta) ? 0.5 * ((lh * lh) / delta + delta) : alam;
}

// the reference einsum's component-axis sum
template <int D>
__device__ __forceinline__ double lane_sum(const double *t) {
    double ev = 0.0, od = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        if (i & 1) od = od + t[i];
        else ev = ev + t[i];
    }
    return ev + od;
}

// np.linalg.inv of a 3x3 (models.py:270): LU with partial pivoting (first
// maximal |pivot|), multipliers scaled by the reciprocal pivot, rank-1
// updates, then unit-lower forward and pivot-dividing backward substitution
// of each column of P I, skipping zero entries (LAPACK dgetf2 / dgetrs)
__device__ __forceinline__ void inv3(const double (&A)[3][3], double (&X)[3][3]) {
    double a[3][3];
    int perm[3] = {0, 1, 2};
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c) a[i][c] = A[i][c];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        int pv = j;
        double best = fabs(a[j][j]);
#pragma unroll
        for (int i = j + 1; i < 3; ++i)
            if (fabs(a[i][j]) > best) { best = fabs(a[i][j]); pv = i; }
        // row swap without dynamic register indexing
#pragma unroll
        for (int i = j + 1; i < 3; ++i)
            if (pv == i) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double t = a[j][c];
                    a[j][c] = a[i][c];
                    a[i][c] = t;
                }
                const int t = perm[j];
                perm[j] = perm[i];
                perm[i] = t;
            }
        const double rp = 1.0 / a[j][j];
#pragma unroll
        for (int i = j + 1; i < 3; ++i) a[i][j] = a[i][j] * rp;
#pragma unroll
        for (int i = j + 1; i < 3; ++i)
#pragma unroll
            for (int c = j + 1; c < 3; ++c) a[i][c] = a[i][c] - a[i][j] * a[j][c];
    }
#pragma unroll
    for (int col = 0; col < 3; ++col) {
        double b[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) b[i] = perm[i] == col ? 1.0 : 0.0;
#pragma unroll
        for (int kk = 0; kk < 3; ++kk)
            if (b[kk] != 0.0)
#pragma unroll
                for (int i = kk + 1; i < 3; ++i) b[i] = b[i] - b[kk] * a[i][kk];
#pragma unroll
        for (int kk = 2; kk >= 0; --kk)
            if (b[kk] != 0.0) {
                b[kk] = b[kk] / a[kk][kk];
#pragma unroll
                for (int i = 0; i < kk; ++i) b[i] = b[i] - b[kk] * a[i][kk];
            }
#pragma unroll
        for (int i = 0; i < 3; ++i) X[i][col] = b[i];
    }
}

template <int D>
struct Eig {
    double lam[D];
    double R[D][D];
    double L[D][D];
};

template <int K, bool ROE, int D>
struct SysField {
    static constexpr int HALO = 0;   // halos are maintained by load/put
    static constexpr bool kFusedCommit = false;
    static constexpr bool kLL = false;
    static constexpr int H = K;      // window reach
    int nx, pitch;                   // cells; per-component stride of s_u
    bool charwise;                   // characteristic reconstruction
    double *s_u;    // stage input: component d, cell c at s_u[d*pitch + H + c]
    double *s_u0;   // RK base, element e = d*nx + c
    double *s_L;    // left states at interface i (e = d*nx + i), then fluxes
    double *s_R;    // right states at interface i, then results
    unsigned long long *s_red;   // [32] per-warp alpha bits
    int32_t *status;
    int bad;

    __device__ __forceinline__ double cellv(int d, int c) const {
        return s_u[d * pitch + H + c];
    }
    __device__ __forceinline__ void load(int e, double v) {
        const int d = e / nx;
        const int c = e - d * nx;
        double *row = s_u + d * pitch + H;
        row[c] = v;
        if (c < H) row[nx + c] = v;
        if (c >= nx - H) row[c - nx] = v;
    }
    __device__ __forceinline__ void put(int e, double v) { load(e, v); }
    __device__ __forceinline__ double result(int e) const { return s_R[e]; }
    __device__ __forceinline__ void sync() { __syncthreads(); }

    // velocity (and Euler pressure) of a state; flags inadmissible states
    __device__ __forceinline__ double vel_of(const Consts &k, const double *s, double &p) {
        if (D == 2) {
            if (s[0] <= 0.0) bad |= MGP_STATUS_NONPOSITIVE_DEPTH;
            p = 0.0;
            return s[1] / s[0];
        }
        if (s[0] <= 0.0) bad |= MGP_STATUS_NONPOSITIVE_DENSITY;
        const double vel = s[1] / s[0];
        p = k.gm1 * (s[D - 1] - ((0.5 * s[0]) * vel) * vel);
        if (p <= 0.0) bad |= MGP_STATUS_NONPOSITIVE_PRESSURE;
        return vel;
    }
    __device__ __forceinline__ double c_of(const Consts &k, const double *s, double p) const {
        return D == 2 ? sqrt(k.gravity * s[0]) : sqrt((k.gamma * p) / s[0]);
    }
    __device__ __forceinline__ void flux(const Consts &k, const double *s, double *f) {
        double p;
        const double vel = vel_of(k, s, p);
        f[0] = s[1];
        if (D == 2) {
            f[1] = ((s[0] * vel) * vel) + (((0.5 * k.gravity) * s[0]) * s[0]);
        } else {
            f[1] = (s[1] * vel) + p;
            f[D - 1] = (s[D - 1] + p) * vel;
        }
    }
    __device__ __forceinline__ void eigen_from(double vel, double c, double Hh, Eig<D> &e) const {
        if (D == 2) {
            const double inv2c = 0.5 / c;
            e.lam[0] = vel - c;
            e.lam[D - 1] = vel + c;
            e.R[0][0] = 1.0; e.R[0][D - 1] = 1.0;
            e.R[D - 1][0] = vel - c; e.R[D - 1][D - 1] = vel + c;
            e.L[0][0] = (vel + c) * inv2c; e.L[0][D - 1] = -1.0 * inv2c;
            e.L[D - 1][0] = (-(vel - c)) * inv2c; e.L[D - 1][D - 1] = 1.0 * inv2c;
        } else {
            double R3[3][3], L3[3][3];
            e.lam[0] = vel - c; e.lam[1] = vel; e.lam[D - 1] = vel + c;
            R3[0][0] = 1.0; R3[0][1] = 1.0; R3[0][2] = 1.0;
            R3[1][0] = vel - c; R3[1][1] = vel; R3[1][2] = vel + c;
            R3[2][0] = Hh - vel * c; R3[2][1] = (0.5 * vel) * vel; R3[2][2] = Hh + vel * c;
            inv3(R3, L3);
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    e.R[i][j] = R3[i % 3][j % 3];
                    e.L[i][j] = L3[i % 3][j % 3];
                }
        }
    }

    // WENO of one window: left state (interface m) and right state (m-1)
    template <int REG>
    __device__ __forceinline__ void recon2(const Consts &k, const double *w, double &l,
                                           double &r) const {
        double bl[K + 1], br[K + 1], ql[K + 1], qr[K + 1];
#pragma unroll
        for (int s2 = 0; s2 <= K; ++s2) beta_block<K, true>(w, s2, bl[s2], br[K - s2]);
#pragma unroll
        for (int q = 0; q <= K; ++q) {
            ql[q] = cand_left<K, REG>(w, q);
            qr[q] = cand_right<K, REG>(w, q);
        }
        l = weno_value<K>(bl, ql, k.eps);
        r = weno_value<K>(br, qr, k.eps);
    }

    // interface states of every interface; returns this thread's alpha bits
    __device__ __forceinline__ unsigned long long reconstruct(const Consts &k) {
        unsigned long long m = 0;
        for (int c = threadIdx.x; c < nx; c += blockDim.x) {
            double sl[D], sr[D];
            if (charwise) {
                double s0[D], p;
#pragma unroll
                for (int d = 0; d < D; ++d) s0[d] = cellv(d, c);
                const double vel = vel_of(k, s0, p);
                const double cs = c_of(k, s0, p);
                const double Hh = D == 3 ? (s0[D - 1] + p) / s0[0] : 0.0;
                Eig<D> e;
                eigen_from(vel, cs, Hh, e);
                double lrec[D], rrec[D];
#pragma unroll
                for (int q = 0; q < D; ++q) {
                    double w[2 * K + 1];
#pragma unroll
                    for (int s2 = 0; s2 <= 2 * K; ++s2) {
                        double t[D];
#pragma unroll
                        for (int d = 0; d < D; ++d) t[d] = e.L[q][d] * cellv(d, c - K + s2);
                        w[s2] = lane_sum<D>(t);
                    }
                    recon2<MGP_SUM_LANE2>(k, w, lrec[q], rrec[q]);
                }
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    double t[D], u[D];
#pragma unroll
                    for (int q = 0; q < D; ++q) {
                        t[q] = e.R[d][q] * lrec[q];
                        u[q] = e.R[d][q] * rrec[q];
                    }
                    sl[d] = lane_sum<D>(t);
                    sr[d] = lane_sum<D>(u);
                }
            } else {
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    double w[2 * K + 1];
#pragma unroll
                    for (int s2 = 0; s2 <= 2 * K; ++s2) w[s2] = cellv(d, c - K + s2);
                    recon2<MGP_SUM_SEQ>(k, w, sl[d], sr[d]);
                }
            }
            const int im = c == 0 ? nx - 1 : c - 1;
#pragma unroll
            for (int d = 0; d < D; ++d) {
                s_L[d * nx + c] = sl[d];
                s_R[d * nx + im] = sr[d];
            }
            if (!ROE) {
                double p;
                const double vl = vel_of(k, sl, p);
                const double al = fabs(vl) + c_of(k, sl, p);
                const double vr = vel_of(k, sr, p);
                const double ar = fabs(vr) + c_of(k, sr, p);
                m = umax64(m, umax64(abs_bits(al), abs_bits(ar)));
            }
        }
        return m;
    }

    __device__ __forceinline__ void roe(const Consts &k, const double *l, const double *r,
                                        double *F) {
        double pl, pr;
        const double vl = vel_of(k, l, pl), vr = vel_of(k, r, pr);
        const double sql = sqrt(l[0]), sqr = sqrt(r[0]);
        Eig<D> e;
        if (D == 2) {
            const double hh = 0.5 * (l[0] + r[0]);
            const double uh = (sql * vl + sqr * vr) / (sql + sqr);
            eigen_from(uh, sqrt(k.gravity * hh), 0.0, e);
        } else {
            const double hl = (l[D - 1] + pl) / l[0], hr = (r[D - 1] + pr) / r[0];
            const double uh = (sql * vl + sqr * vr) / (sql + sqr);
            const double Hh = (sql * hl + sqr * hr) / (sql + sqr);
            const double csq = k.gm1 * (Hh - (0.5 * uh) * uh);
            if (csq <= 0.0) bad |= MGP_STATUS_ROE_NONHYPERBOLIC;
            eigen_from(uh, sqrt(csq), Hh, e);
        }
        const double cl = c_of(k, l, pl), cr = c_of(k, r, pr);
        double laml[D], lamr[D];
        laml[0] = vl - cl; laml[D - 1] = vl + cl;
        lamr[0] = vr - cr; lamr[D - 1] = vr + cr;
        if (D == 3) { laml[1 % D] = vl; lamr[1 % D] = vr; }
        double ss[D], t[D];
#pragma unroll
        for (int q = 0; q < D; ++q) {
#pragma unroll
            for (int d = 0; d < D; ++d) t[d] = e.L[q][d] * (r[d] - l[d]);
            ss[q] = entropy_fix(e.lam[q], laml[q], lamr[q]) * lane_sum<D>(t);
        }
        double fl[D], fr[D];
        flux(k, l, fl);
        flux(k, r, fr);
#pragma unroll
        for (int d = 0; d < D; ++d) {
#pragma unroll
            for (int q = 0; q < D; ++q) t[q] = ss[q] * e.R[d][q];
            F[d] = (0.5 * (fl[d] + fr[d])) - (0.5 * lane_sum<D>(t));
        }
    }

    __device__ __forceinline__ void rhs(const Consts &k) {
        unsigned long long m = reconstruct(k);
        double half_alpha = 0.0;
        if (!ROE) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = umax64(m, __shfl_xor_sync(0xffffffffu, m, o));
            if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
        }
        __syncthreads();
        if (!ROE) {
            m = s_red[0];
            const int nw = (blockDim.x + 31) >> 5;
            for (int w = 1; w < nw; ++w) m = umax64(m, s_red[w]);
            half_alpha = 0.5 * __longlong_as_double((long long)m);
        }
        for (int i = threadIdx.x; i < nx; i += blockDim.x) {
            double l[D], r[D], F[D];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                l[d] = s_L[d * nx + i];
                r[d] = s_R[d * nx + i];
            }
            if (ROE) {
                roe(k, l, r, F);
            } else {
                double fl[D], fr[D];
                flux(k, l, fl);
                flux(k, r, fr);
#pragma unroll
                for (int d = 0; d < D; ++d)
                    F[d] = (0.5 * (fl[d] + fr[d])) - (half_alpha * (r[d] - l[d]));
            }
#pragma unroll
            for (int d = 0; d < D; ++d) s_L[d * nx + i] = F[d];
        }
        __syncthreads();
    }

    __device__ __forceinline__ double A(const Consts &k, int e) const {
        const int d = e / nx;
        const int c = e - d * nx;
        const double fm = s_L[d * nx + (c == 0 ? nx - 1 : c - 1)];
        const double neg = -(s_L[e] - fm);
        return k.dx_pow2 ? neg * k.inv_dx : neg / k.dx;
    }

    __device__ void phi(const Consts &k, int rk) {
        const int tid = threadIdx.x, nt = blockDim.x, n = D * nx;
        bad = 0;
        for (int e = tid; e < n; e += nt) {
            const int d = e / nx;
            s_u0[e] = cellv(d, e - d * nx);
        }
        const int stages = rk == 0 ? 1 : rk;
#pragma unroll 1
        for (int sg = 0; sg < stages; ++sg) {
            if (sg > 0) __syncthreads();   // committed stage values visible
            rhs(k);
            const bool last = (sg == stages - 1);
            for (int e = tid; e < n; e += nt) {
                const double a = A(k, e);
                const double u0 = s_u0[e];
                double st;
                if (rk == 0) {
                    st = a;
                } else if (sg == 0) {
                    st = u0 + k.dt * a;
                } else {
                    const int d = e / nx;
                    const double cur = cellv(d, e - d * nx);
                    if (rk == 2) st = ((0.5 * u0) + (0.5 * cur)) + (k.hdt * a);
                    else if (sg == 1) st = ((0.75 * u0) + (0.25 * cur)) + (k.qdt * a);
                    else st = ((u0 / 3.0) + (k.two3 * cur)) + (k.tdt * a);
                }
                if (last) s_R[e] = st;
                else put(e, st);
            }
        }
        if (bad && status) atomicOr(status, bad);
    }
};

template <int K, bool ROE, int D>
__global__ void __launch_bounds__(256) sys_kernel(const mgp_sweep_args a, const Consts k) {
    extern __shared__ double smem[];
    SysField<K, ROE, D> f;
    const int nx = (int)a.phi.nx;
    f.nx = nx;
    f.pitch = nx + 2 * K;
    f.charwise = a.phi.characteristic != 0;
    f.s_u = smem;
    f.s_u0 = f.s_u + D * f.pitch;
    f.s_L = f.s_u0 + D * nx;
    f.s_R = f.s_L + D * nx;
    double *s_sum = f.s_R + D * nx;            // [3 * 32]
    double *s_psum = s_sum + 3 * 32;           // [3]
    f.s_red = reinterpret_cast<unsigned long long *>(s_psum + 3);
    f.status = a.status;
    f.bad = 0;
    sweep_body<SysField<K, ROE, D>, 1>(a, k, f, D * nx, 0, 0, s_sum, s_psum, D * nx);
}

__global__ void __launch_bounds__(1024, 1)
    sum_partials_kernel(const double *p, int64_t n, int width, double *out) {
    __shared__ double s[1024];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int j = 0; j < width; ++j) {
        // each thread sums a contiguous block, then a fixed binary tree
        const int64_t per = (n + nt - 1) / nt;
        const int64_t lo = tid * per, hi = lo + per < n ? lo + per : n;
        double t = 0.0;
        for (int64_t i = lo; i < hi; ++i) t = t + p[width * i + j];
        s[tid] = t;
        __syncthreads();
        for (int h = nt / 2; h > 0; h >>= 1) {
            if (tid < h) s[tid] = s[tid] + s[tid + h];
            __syncthreads();
        }
        if (tid == 0) out[j] = s[0];
        __syncthreads();
    }
}

bool pow2_normal(double x) {
    uint64_t bits;
    memcpy(&bits, &x, 8);
    const uint64_t mant = bits & 0x000FFFFFFFFFFFFFull;
    const uint64_t ex = (bits >> 52) & 0x7FF;
    return mant == 0 && ex != 0 && ex != 0x7FF && !(bits >> 63);
}

Consts make_consts(const mgp_phi &p) {
    Consts k;
    k.dt = p.dt;
    k.hdt = 0.5 * p.dt;
    k.qdt = 0.25 * p.dt;
    k.two3 = 2.0 / 3.0;
    k.tdt = k.two3 * p.dt;
    k.dx = p.dx;
    k.dx_pow2 = pow2_normal(p.dx);
    k.inv_dx = 1.0 / p.dx;
    k.eps = p.epsilon;
    k.speed = p.speed;
    k.half_alpha_adv = 0.5 * (p.speed < 0 ? -p.speed : p.speed);
    const double raw = 1.0 / (p.epsilon * p.epsilon);
    k.k0_omega = raw / raw;
    k.twodx = 2.0 * p.dx;
    k.inv_twodx = 1.0 / k.twodx;
    k.twodx_pow2 = pow2_normal(k.twodx);
    k.lf_order = p.lf_order;
    k.m_eff = p.m_eff;
    k.gravity = p.gravity;
    k.gamma = p.gamma;
    k.gm1 = p.gamma - 1.0;
    return k;
}

// Cells per thread run.  Single-field launches (the sequential coarse solve)
// use the most threads (shortest per-step latency); batched launches use
// longer runs, which share more reconstruction products per interface.
int run_length(int64_t nx, int64_t n_chunks) {
    static int env = -1;
    if (env < 0) {
        const char *e = getenv("MGP_RUN");
        env = e ? atoi(e) : 0;
    }
    int p = 1;
    while ((nx + p - 1) / p > kMaxThreads) p *= 2;
    if (n_chunks > 1) {
        const int want = env > 0 ? env : (nx >= 1024 ? 8 : 4);
        while (p < want && p < kMaxRun) p *= 2;
    } else if (env > 0 && n_chunks == 1) {
        // keep the latency-oriented choice for single fields
    }
    return p;
}

int threads_for(int64_t ns, int p) {
    int64_t nt = p == 0 ? 2 * ((ns + 31) / 32 * 32) : (ns + p - 1) / p;
    nt = (nt + 31) / 32 * 32;
    return (int)nt;
}

size_t smem_bytes(int64_t ns, int k, int cs, int p) {
    const int H = k + 1;
    const auto size = [p](int n) {   // Field::sk_size for run length p
        return p == 8 ? skp_size<3>(n) : (p == 4 ? skp_size<2>(n) : skp_size<4>(n));
    };
    // runs of 16 (fcf_kernel, Field U0G): no RK-base array
    const int arrays = p == 16 ? 2 : 3;
    return sizeof(double) * (size_t)(size((int)ns + 2 * H) + arrays * size((int)ns) + 3 * 32 +
                                     3 * cs + 2) +
           sizeof(unsigned long long) * (size_t)(cs + 32);
}

// Library-owned device scratch, one allocation per (kind, device, stream),
// grown on demand: kind 0 = the LL mailbox (Field, LL mode; zeroed by every
// launch that uses it, tags restart at 1).
void *device_scratch(int kind, size_t bytes, cudaStream_t st, bool zero) {
    struct Box {
        int kind, dev;
        cudaStream_t st;
        void *p;
        size_t bytes;
    };
    static std::vector<Box> boxes;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    Box *bx = nullptr;
    for (auto &b : boxes)
        if (b.kind == kind && b.dev == dev && b.st == st) bx = &b;
    if (!bx) {
        boxes.push_back(Box{kind, dev, st, nullptr, 0});
        bx = &boxes.back();
    }
    if (bx->bytes < bytes) {
        if (bx->p) {
            // work of earlier launches on this stream may still use the old block
            if (cudaStreamSynchronize(st) != cudaSuccess) return nullptr;
            cudaFree(bx->p);
        }
        bx->p = nullptr;
        bx->bytes = 0;
        if (cudaMalloc(&bx->p, bytes) != cudaSuccess) return nullptr;
        bx->bytes = bytes;
    }
    if (zero && cudaMemsetAsync(bx->p, 0, bytes, st) != cudaSuccess) return nullptr;
    return bx->p;
}

// Pinned host word per (device, stream) that receives the LL give-up flag of
// the last LL launch on that stream.
unsigned long long *ll_fail_flag(cudaStream_t st) {
    struct Flag {
        int dev;
        cudaStream_t st;
        unsigned long long *p;
    };
    static std::vector<Flag> flags;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    for (auto &f : flags)
        if (f.dev == dev && f.st == st) return f.p;
    unsigned long long *p = nullptr;
    if (cudaHostAlloc(&p, sizeof(unsigned long long), cudaHostAllocDefault) != cudaSuccess)
        return nullptr;
    *p = 0;
    flags.push_back(Flag{dev, st, p});
    return p;
}

template <int K, int REG, int MODEL, int P, int REGS, int CS, bool LL = false>
int launch_t(const mgp_sweep_args &a, cudaStream_t st) {
    const int64_t ns = a.phi.nx / CS;
    const int nt = threads_for(ns, P);
    const size_t sm = smem_bytes(ns, K, CS, P);
    auto kern = sweep_kernel<K, REG, MODEL, P, REGS, CS, LL>;
    static unsigned long long attr_devs = 0;
    if (!ensure_attrs(kern, attr_devs, CS > 8 && !LL)) return MGP_ECUDA;
    int64_t grid = a.n_chunks;
    if (grid > ((int64_t)1 << 30) / CS) grid = ((int64_t)1 << 30) / CS;
    const Consts k = make_consts(a.phi);
    unsigned long long *mbox = nullptr;
    int dev = 0, nsm = 0, per = 0;
    if (LL) {
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, nt, sm) != cudaSuccess)
            return MGP_ECUDA;
        // one field (group) per resident slot; the kernel strides over the chunks
        const int64_t groups = (int64_t)per * nsm / CS;
        if (groups < 1) return MGP_ECUDA;
        if (grid > groups) grid = groups;
    }
    if (CS == 1) {
        kern<<<(unsigned)grid, nt, sm, st>>>(a, k, mbox);
    } else if (LL) {
        // groups of CS co-resident CTAs (cooperative launch: all resident or
        // the launch fails), as many groups as fit the device
        // the previous LL launch on this stream gave up on a peer (its result is
        // void): surface it now -- the flag travels back without a host wait
        unsigned long long *fail_host = ll_fail_flag(st);
        if (!fail_host) return MGP_ECUDA;
        if (*fail_host) {
            *fail_host = 0;
            return MGP_ECUDA;
        }
        const size_t words = (size_t)grid * 2 * CS * kLLWords;
        mbox = static_cast<unsigned long long *>(
            device_scratch(0, (words + 1) * sizeof(unsigned long long), st, true));
        if (!mbox) return MGP_ECUDA;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(grid * CS));
        cfg.blockDim = dim3(nt);
        cfg.dynamicSmemBytes = sm;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, kern, a, k, mbox) != cudaSuccess) return MGP_ECUDA;
        cudaMemcpyAsync(fail_host, mbox + words, sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost, st);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(grid * CS));
        cfg.blockDim = dim3(nt);
        cfg.dynamicSmemBytes = sm;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, kern, a, k, mbox) != cudaSuccess) return MGP_ECUDA;
    }
    ++g_launches;
    return cudaPeekAtLastError() == cudaSuccess ? MGP_OK : MGP_ECUDA;
}

#ifndef MGP_REGS
#define MGP_REGS 128
#endif

int env_int(const char *name) {
    const char *e = getenv(name);
    return e ? atoi(e) : 0;
}

// Cluster size for a field: meshes above one SM's capacity must be split
// (WENO5 Burgers only, up to 16 x 4096 cells); single-field marches of the
// sequential coarse solve are split for latency (MGP_MARCH_CS overrides).
// Smallest cluster size cs in {2, 4, 8, 16} that splits a mesh of nx > kMaxNx
// cells into equal slabs of at most kMaxNx cells, or 0 if none does.
int split_cs(int64_t nx) {
    for (int cs = 2; cs <= 16; cs *= 2)
        if (nx % cs == 0 && nx / cs <= kMaxNx) return cs;
    return 0;
}

int cluster_size(const mgp_sweep_args &a) {
    const int64_t nx = a.phi.nx;
    const bool cl_ok = a.phi.weno_k == 2 && a.phi.model == MGP_MODEL_BURGERS &&
                       a.phi.scheme == MGP_SCHEME_RK_WENO;
    if (nx > kMaxNx) return split_cs(nx);   // validate() guarantees a size exists
    if (cl_ok && a.n_chunks == 1) {
        const int env = env_int("MGP_MARCH_CS");   // per call (tests switch it)
        // default: slabs of >= 64 cells, at most 16 CTAs (measured, latency
        // mode: C2 nx=512 -> 8 CTAs, 5.5 us/step; C3 nx=4096 -> 16 CTAs,
        // 9.0 us/step)
        int cs = env > 0 ? env : 16;
        if (env <= 0)
            while (cs > 1 && nx / cs < 64) cs /= 2;
        while (cs > 1 && (nx % cs || nx / cs < 64)) cs /= 2;
        return cs;
    }
    return 1;
}

// Cluster size of the one-exchange-per-stage march (march_kernel), or 0 when
// the call is not a plain single-field march it covers (Burgers RK-WENO,
// WENO1/3/5).  At most 16 CTAs and 256 cells per CTA.  Measured on B200 with
// the st.async / mbarrier exchange, us per SSP-RK3 step
// (profiles/r02_march_async.txt; round 1's cluster-barrier exchange in
// brackets), Field path -> best march_kernel cluster:
//   WENO5 nx 128  4.04 -> 2.20 (2 CTAs)   nx 512 4.67 -> 2.43 (16) [3.32]   nx 4096 7.97 -> 5.01 (16) [6.29]
//   WENO3 nx 128  2.10 -> 1.87 (2)        nx 512 3.54 -> 2.19 (16) [3.05]   nx 4096 15.4 -> 4.09 (16) [5.24]
//   WENO1 nx 128  1.61 -> 1.39 (2)        nx 512 2.10 -> 1.68 (16) [2.31]   nx 4096 9.79 -> 3.23 (16) [4.63]
// Small meshes run on 2 CTAs (the cheapest exchange), meshes from 512 cells
// (WENO5: 256) on as many CTAs as divide them, up to 16.  MGP_MARCH_CS forces
// the size, MGP_MARCH_MIN_SLAB the smallest slab, MGP_MARCH2=0 selects the
// Field path.
int march_cluster_size(const mgp_sweep_args &a) {
    // read per call (a getenv per launch), so tests can switch paths in-process
    const char *e = getenv("MGP_MARCH2");
    const int on = (e && atoi(e) == 0) ? 0 : 1;
    const int min_slab_env = env_int("MGP_MARCH_MIN_SLAB");
    const int force = env_int("MGP_MARCH_CS");
    const int64_t nx = a.phi.nx;
    if (!on || a.n_chunks != 1 || a.tail != MGP_TAIL_NONE || a.phi.repeats != 1 || a.ref ||
        a.count_nonfinite || a.partials || a.n_steps < 1 ||
        a.phi.weno_k < 0 || a.phi.weno_k > 2 ||
        a.phi.model != MGP_MODEL_BURGERS || a.phi.scheme != MGP_SCHEME_RK_WENO ||
        a.phi.rk_order < 0 || a.phi.rk_order > 3 ||
        (a.g_mode != MGP_G_NONE && a.g_mode != MGP_G_ZERO && a.g_mode != MGP_G_ARRAY) ||
        (a.g_mode == MGP_G_ARRAY && !a.g))
        return 0;
    int cs = force > 0 ? force : 16;
    if (force <= 0) {
        if (min_slab_env > 0) {
            while (cs > 2 && (nx % cs || nx / cs < min_slab_env)) cs /= 2;
        } else if (nx >= (a.phi.weno_k == 2 ? 256 : 512)) {
            while (cs > 2 && (nx % cs || nx / cs < 16)) cs /= 2;
        } else {
            cs = 2;
        }
    }
    if (cs != 2 && cs != 4 && cs != 8 && cs != 16) return 0;
    if (nx % cs || nx / cs < 8 || nx / cs > 256) return 0;
    return cs;
}

template <int K, int REG, int MODEL, int P>
int launch_r(const mgp_sweep_args &a, cudaStream_t st) {
#ifdef MGP_EXPERIMENT
    // register-budget experiments (tools/): MGP_MAXREG selects the variant
    static int env = -1;
    if (env < 0) env = env_int("MGP_MAXREG");
    if (K == 2 && MODEL == MGP_MODEL_BURGERS && P >= 4) {
        switch (env) {
            case 96: return launch_t<K, REG, MODEL, P, 96, 1>(a, st);
            case 112: return launch_t<K, REG, MODEL, P, 112, 1>(a, st);
            default: break;
        }
    }
#endif
    return launch_t<K, REG, MODEL, P, MGP_REGS, 1>(a, st);
}

// The runs-of-16 / RK-base-in-global variant (Field U0G, two CTAs per SM for
// 4096-cell fields) pays for the fused FCF launch only: the batched sweeps
// measured slower with it (C3 F+C sweep 20.2 -> 19.7 G point-updates/s, C5 LL
// sweep 15.8 -> 15.3; profiles/r02_fcf_u0g.txt), so they keep runs of 8.
template <int K, int REG, int MODEL>
int launch_p(const mgp_sweep_args &a, cudaStream_t st) {
    const int cs = cluster_size(a);
#ifdef MGP_QUICK
    if (cs > 1) return MGP_EINVAL;
    if constexpr (K != 2) {
        return MGP_EINVAL;
    } else {
        switch (run_length(a.phi.nx, a.n_chunks)) {
            case 4: return launch_r<K, REG, MODEL, 4>(a, st);
            case 8: return launch_r<K, REG, MODEL, 8>(a, st);
        }
        return MGP_EINVAL;
    }
#else
    if constexpr (K <= 2 && MODEL == MGP_MODEL_BURGERS) {
        switch (march_cluster_size(a)) {
            case 2: return launch_march<K, REG, 2>(a, st);
            case 4: return launch_march<K, REG, 4>(a, st);
            case 8: return launch_march<K, REG, 8>(a, st);
            case 16: return launch_march<K, REG, 16>(a, st);
            default: break;
        }
    }
    if (cs > 1) {
      if constexpr (K != 2 || MODEL != MGP_MODEL_BURGERS) {
        return MGP_EINVAL;
      } else {
        // slabs: P = 8 above 512 cells per CTA; below, the latency mode
        // (two threads per interface) for slabs <= 256 cells, else P = 1
        const int64_t nsl = a.phi.nx / cs;
        const int mode = nsl > 512 ? 8 : (nsl <= 256 ? 0 : 1);
        // batched sweeps of a split mesh: groups of co-resident CTAs that
        // exchange through global memory (every SM usable; hardware clusters
        // of 16 fit 7 times on a B200).  MGP_LL=0 keeps the cluster path.
        if (mode == 8 && a.n_chunks > 1 && a.phi.nx > kMaxNx) {
            const char *e = getenv("MGP_LL");
            if (!(e && atoi(e) == 0)) {
                switch (cs) {
                    case 2: return launch_t<K, REG, MODEL, 8, MGP_REGS, 2, true>(a, st);
                    case 4: return launch_t<K, REG, MODEL, 8, MGP_REGS, 4, true>(a, st);
                    case 8: return launch_t<K, REG, MODEL, 8, MGP_REGS, 8, true>(a, st);
                    case 16: return launch_t<K, REG, MODEL, 8, MGP_REGS, 16, true>(a, st);
                }
            }
        }
        switch (cs) {
            case 2: return mode == 8 ? launch_t<K, REG, MODEL, 8, MGP_REGS, 2>(a, st)
                         : mode == 0 ? launch_t<K, REG, MODEL, 0, MGP_REGS, 2>(a, st)
                                     : launch_t<K, REG, MODEL, 1, MGP_REGS, 2>(a, st);
            case 4: return mode == 8 ? launch_t<K, REG, MODEL, 8, MGP_REGS, 4>(a, st)
                         : mode == 0 ? launch_t<K, REG, MODEL, 0, MGP_REGS, 4>(a, st)
                                     : launch_t<K, REG, MODEL, 1, MGP_REGS, 4>(a, st);
            case 8: return mode == 8 ? launch_t<K, REG, MODEL, 8, MGP_REGS, 8>(a, st)
                         : mode == 0 ? launch_t<K, REG, MODEL, 0, MGP_REGS, 8>(a, st)
                                     : launch_t<K, REG, MODEL, 1, MGP_REGS, 8>(a, st);
            case 16: return mode == 8 ? launch_t<K, REG, MODEL, 8, MGP_REGS, 16>(a, st)
                          : mode == 0 ? launch_t<K, REG, MODEL, 0, MGP_REGS, 16>(a, st)
                                      : launch_t<K, REG, MODEL, 1, MGP_REGS, 16>(a, st);
        }
        return MGP_EINVAL;
      }
    }
    switch (run_length(a.phi.nx, a.n_chunks)) {
        case 1: return launch_r<K, REG, MODEL, 1>(a, st);
        case 2: return launch_r<K, REG, MODEL, 2>(a, st);
        case 4: return launch_r<K, REG, MODEL, 4>(a, st);
        case 8: return launch_r<K, REG, MODEL, 8>(a, st);
    }
    return MGP_EINVAL;
#endif
}

// KSET selects the instantiated kernels (translation-unit split, below):
// bit 0 K = 0, bit 1 K = 1, bit 2 K = 2 sequential sums, bit 3 K = 2
// two-lane sums, bit 4 K = 3
constexpr int kKAll = 31;
template <int MODEL, int KSET = kKAll>
int launch_m(const mgp_sweep_args &a, cudaStream_t st) {
    const int reg = a.n_steps > 0 ? a.phi.regime : a.tail_regime;
    switch (a.phi.weno_k) {
        case 0:
            if constexpr ((KSET & 1) != 0) return launch_p<0, MGP_SUM_SEQ, MODEL>(a, st);
            break;
        case 1:
            if constexpr ((KSET & 2) != 0) return launch_p<1, MGP_SUM_SEQ, MODEL>(a, st);
            break;
        case 2:
            if (reg == MGP_SUM_SEQ) {
                if constexpr ((KSET & 4) != 0) return launch_p<2, MGP_SUM_SEQ, MODEL>(a, st);
            } else {
                if constexpr ((KSET & 8) != 0) return launch_p<2, MGP_SUM_LANE2, MODEL>(a, st);
            }
            break;
        case 3:
            if constexpr ((KSET & 16) != 0)
                return reg == MGP_SUM_SEQ ? launch_p<3, MGP_SUM_SEQ, MODEL>(a, st)
                                          : launch_p<3, MGP_SUM_LANE2, MODEL>(a, st);
            break;
    }
    return MGP_EINVAL;
}

template <int MODE>
int launch_lf(const mgp_sweep_args &a, cudaStream_t st) {
    const int64_t nx = a.phi.nx;
    int nt = (int)((nx + 31) / 32 * 32);
    if (nt > 256) nt = 256;
    const size_t sm = sizeof(double) * (size_t)(7 * nx + 3 * 32 + 3);
    auto kern = lf_kernel<MODE>;
    static unsigned long long attr_devs = 0;
    if (!ensure_attrs(kern, attr_devs, false)) return MGP_ECUDA;
    int64_t grid = a.n_chunks;
    if (grid > (int64_t)1 << 30) grid = (int64_t)1 << 30;
    kern<<<(unsigned)grid, nt, sm, st>>>(a, make_consts(a.phi));
    ++g_launches;
    return cudaPeekAtLastError() == cudaSuccess ? MGP_OK : MGP_ECUDA;
}

template <int K, bool ROE, int D>
int launch_sys_t(const mgp_sweep_args &a, cudaStream_t st) {
    const int64_t nx = a.phi.nx;
    int nt = (int)((nx + 31) / 32 * 32);
    if (nt > 256) nt = 256;
    const size_t sm = sizeof(double) * (size_t)(D * (nx + 2 * K) + 3 * D * nx + 3 * 32 + 3) +
                      sizeof(unsigned long long) * 32;
    auto kern = sys_kernel<K, ROE, D>;
    static unsigned long long attr_devs = 0;
    if (!ensure_attrs(kern, attr_devs, false)) return MGP_ECUDA;
    int64_t grid = a.n_chunks;
    if (grid > (int64_t)1 << 30) grid = (int64_t)1 << 30;
    kern<<<(unsigned)grid, nt, sm, st>>>(a, make_consts(a.phi));
    ++g_launches;
    return cudaPeekAtLastError() == cudaSuccess ? MGP_OK : MGP_ECUDA;
}

template <bool ROE, int D>
int launch_sys_k(const mgp_sweep_args &a, cudaStream_t st) {
    switch (a.phi.weno_k) {
        case 0: return launch_sys_t<0, ROE, D>(a, st);
        case 1: return launch_sys_t<1, ROE, D>(a, st);
        case 2: return launch_sys_t<2, ROE, D>(a, st);
        case 3: return launch_sys_t<3, ROE, D>(a, st);
    }
    return MGP_EINVAL;
}

// a template so that only the translation unit that calls it instantiates
// the system kernels
template <int UNUSED = 0>
int launch_sys(const mgp_sweep_args &a, cudaStream_t st) {
    const bool roe = a.phi.scheme == MGP_SCHEME_RK_WENO_ROE;
    if (a.phi.model == MGP_MODEL_EULER)
        return roe ? launch_sys_k<true, 3>(a, st) : launch_sys_k<false, 3>(a, st);
    return roe ? launch_sys_k<true, 2>(a, st) : launch_sys_k<false, 2>(a, st);
}

// --- fused FCF relaxation (mgp_relax_fcf) ----------------------------------
struct FcfLaunch {
    int G = 0, nt = 0;
    size_t smem = 0;
    int64_t R = 0, Gmax = 0, bytes = 0, u0_off = 0;
};

template <int K, int P>
int fcf_setup(const mgp_phi &phi, int64_t nc, bool fstore, FcfLaunch &L) {
    auto kern = fcf_kernel<K, MGP_SUM_SEQ, MGP_MODEL_BURGERS, P, MGP_REGS>;
    const int ns = (int)phi.nx;
    L.nt = threads_for(ns, P);
    L.smem = smem_bytes(ns, K, 1, P);
    static unsigned long long attr_devs = 0;
    if (!ensure_attrs(kern, attr_devs, false)) return MGP_ECUDA;
    int dev = 0, nsm = 0, per = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, L.nt, L.smem) != cudaSuccess)
        return MGP_ECUDA;
    // one CTA per resident slot, at most one per chain; with more chains
    // than CTAs the last G chains are split
    const int64_t nchains = nc + (fstore ? 1 : 0);
    L.Gmax = (int64_t)per * nsm;
    int64_t G = L.Gmax;
    if (G > nchains) G = nchains;
    if (G < 1) return MGP_EINVAL;
    L.G = (int)G;
    L.R = nchains > G ? G : 0;
    L.bytes = (4 + L.Gmax) * 8 + L.Gmax * ns * (int64_t)sizeof(double);
    L.u0_off = 0;
    if (P == 16) {   // U0G: one RK-base row per resident CTA, 256-byte aligned
        L.u0_off = (L.bytes + 255) / 256 * 256;
        L.bytes = L.u0_off + L.Gmax * (int64_t)L.nt * P * (int64_t)sizeof(double);
    }
    return MGP_OK;
}

template <int K, int P>
int fcf_launch(const mgp_fcf_args &a, cudaStream_t st) {
    FcfLaunch L;
    const bool fstore = a.fstore != nullptr;
    const int rc = fcf_setup<K, P>(a.phi, a.n_chunks, fstore, L);
    if (rc != MGP_OK) return rc;
    if (a.workspace_bytes < L.bytes) return MGP_EINVAL;
    FcfPlan pl;
    pl.nc = a.n_chunks;
    pl.m = a.m;
    pl.fstore = fstore;
    pl.nchains = a.n_chunks + (fstore ? 1 : 0);
    pl.L = fstore ? 2 * a.m - 1 : a.m;
    pl.R = L.R;
    pl.Gmax = L.Gmax;
    pl.u0_off = L.u0_off;
    pl.K = pl.nchains - L.R;
    // segment length of the chains taken last; measured on B200 for C2
    // shapes: whole chains (S = L) and S = 1, 2 within 1-2 %
    pl.S = (a.segment > 0 && a.segment < pl.L) ? a.segment : pl.L;
    pl.W = pl.n_units();
    // zero-copy input (relax_to_host): ordered chain-start loads.  In every
    // plan the chain-start units hold a prefix of the tickets, so a load
    // only ever waits for loads of smaller tickets, already taken by
    // running CTAs.
    pl.ordered = 0;
    {
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, a.cs) == cudaSuccess && pa.type == cudaMemoryTypeHost) {
            const char *e = getenv("MGP_FCF_ORDERED");
            pl.ordered = e ? atoi(e) : 192;   // measured plateau 96-256 (profiles/)
        }
        cudaGetLastError();
    }
    // split plan (F-point storage, whole chains): with more intervals than
    // CTA slots, the first A chains run only their F- and C-steps and queue
    // their final F-steps, so the second wave draws from whole chains and
    // 3-step units instead of idling on a partial wave of 7-step chains
    pl.A = 0;
    if (fstore && pl.S == pl.L && a.split >= 0 && pl.nc >= 2) {
        int64_t A = a.split > 0 ? a.split : (pl.nc > L.G ? (int64_t)L.G : 0);
        if (A > pl.nc - 1) A = pl.nc - 1;
        if (A > L.Gmax) A = L.Gmax;          // queue slots
        pl.A = A;
        pl.K = pl.nchains;
        pl.R = 0;
        pl.W = pl.nchains + A;
    }
    fcf_kernel<K, MGP_SUM_SEQ, MGP_MODEL_BURGERS, P, MGP_REGS>
        <<<L.G, L.nt, L.smem, st>>>(a, make_consts(a.phi), pl);
    ++g_launches;
    return cudaPeekAtLastError() == cudaSuccess ? MGP_OK : MGP_ECUDA;
}

// the fused path covers scalar Burgers RK-WENO fields of one CTA in the
// batched (sequential-sum) regime; MGP_EINVAL otherwise
bool fcf_supported(const mgp_phi &p, int64_t nc) {
    return p.model == MGP_MODEL_BURGERS && p.scheme == MGP_SCHEME_RK_WENO &&
           p.regime == MGP_SUM_SEQ && p.weno_k >= 0 && p.weno_k <= 3 &&
           p.rk_order >= 0 && p.rk_order <= 3 && p.repeats >= 1 &&
           p.nx >= 2 * p.weno_k + 1 && p.nx <= kMaxNx && p.dx > 0.0 && p.epsilon > 0.0 &&
           nc >= 1;
}

template <class Fn>
int fcf_dispatch(const mgp_phi &p, int64_t nc, Fn &&fn) {
    int run = run_length(p.nx, nc > 1 ? nc : 2);
    // WENO5 fields above 2048 cells (one CTA per SM with four shared arrays):
    // runs of 16 cells with the RK base in global memory, two CTAs per SM
    // (Field U0G).  MGP_FCF_U0G=0 keeps the runs of 8; MGP_FCF_U0G=n > 1
    // applies the variant from n cells on (it also gains on smaller meshes
    // when every CTA slot is busy -- 2048 cells 0.856 -> 0.874, 512 cells
    // 0.839 -> 0.878 of the FP64 peak -- but loses on config 2 itself, whose
    // 1025 chains then occupy under half of the slots).
    if (p.weno_k == 2 && p.nx % 16 == 0) {
        const char *e = getenv("MGP_FCF_U0G");
        const int v = e ? atoi(e) : 1;             // 0: off, 1: default, > 1: smallest mesh
        const int64_t least = v > 1 ? v : 2049;
        if (v != 0 && p.nx >= least) run = 16;
    }
    switch (p.weno_k) {
#define MGP_FCF_K(KK)                                                   \
    case KK:                                                            \
        if (run == 4) return fn(std::integral_constant<int, KK>{},      \
                                std::integral_constant<int, 4>{});      \
        if (run == 8) return fn(std::integral_constant<int, KK>{},      \
                                std::integral_constant<int, 8>{});      \
        if (run == 16) {                                                \
            if constexpr (KK == 2)                                      \
                return fn(std::integral_constant<int, KK>{},            \
                          std::integral_constant<int, 16>{});           \
        }                                                               \
        return MGP_EINVAL;
#ifndef MGP_QUICK
        MGP_FCF_K(0)
        MGP_FCF_K(1)
        MGP_FCF_K(3)
#endif
        MGP_FCF_K(2)
#undef MGP_FCF_K
    }
    return MGP_EINVAL;
}

int64_t max_nx_for(int k, int model) {
    if (model == MGP_MODEL_SHALLOW_WATER || model == MGP_MODEL_EULER) return kMaxSysNx;
    return (k == 2 && model == MGP_MODEL_BURGERS) ? 16 * kMaxNx : kMaxNx;
}

int validate(const mgp_sweep_args *a) {
    if (!a) return MGP_EINVAL;
    const mgp_phi &p = a->phi;
    if (p.repeats < 1) return MGP_EINVAL;
    const bool system = p.model == MGP_MODEL_SHALLOW_WATER || p.model == MGP_MODEL_EULER;
    if (system) {
        if (p.scheme != MGP_SCHEME_RK_WENO && p.scheme != MGP_SCHEME_RK_WENO_ROE)
            return MGP_EINVAL;
        if (p.model == MGP_MODEL_SHALLOW_WATER && !(p.gravity > 0.0))
            return MGP_EINVAL;                        // models.py:139-143
        if (p.model == MGP_MODEL_EULER && !(p.gamma > 1.0))
            return MGP_EINVAL;                        // models.py:219-223
    } else if (p.scheme == MGP_SCHEME_RK_WENO_ROE &&
               (p.model != MGP_MODEL_BURGERS || p.nx > kMaxNx)) {
        return MGP_EINVAL;
    }
    if (p.scheme != MGP_SCHEME_RK_WENO && p.scheme != MGP_SCHEME_RK_WENO_ROE) {
        if (p.scheme != MGP_SCHEME_LF_ONESTEP && p.scheme != MGP_SCHEME_LF_MATCHED)
            return MGP_EINVAL;
        if (p.model != MGP_MODEL_BURGERS) return MGP_EINVAL;   // stepper.py:95-99
        if (p.nx < 1 || p.nx > kMaxLfNx || !(p.dx > 0.0)) return MGP_EINVAL;
        if (p.scheme == MGP_SCHEME_LF_MATCHED &&
            ((p.lf_order != 0 && p.lf_order != 1) || p.m_eff < 1))
            return MGP_EINVAL;
        if (a->n_chunks < 0 || a->n_steps < 0 || !a->start) return MGP_EINVAL;
        if (a->g_mode == MGP_G_ARRAY && !a->g && a->n_steps > 0) return MGP_EINVAL;
        if (a->tail == MGP_TAIL_PHI && !a->tail_out) return MGP_EINVAL;
        if (a->tail == MGP_TAIL_RESTRICT && (!a->tail_out || !a->tail_out2 || !a->aux))
            return MGP_EINVAL;
        if (a->tail == MGP_TAIL_RESTRICT && a->guess == MGP_GUESS_INJECTION && !a->aux2)
            return MGP_EINVAL;
        if (a->tail == MGP_TAIL_RESID && (!a->aux || !a->partials)) return MGP_EINVAL;
        return MGP_OK;
    }
    if (p.model != MGP_MODEL_BURGERS && p.model != MGP_MODEL_ADVECTION && !system)
        return MGP_EINVAL;
    if (p.weno_k < 0 || p.weno_k > 3) return MGP_EINVAL;
    if (p.rk_order < 0 || p.rk_order > 3) return MGP_EINVAL;
    if (p.regime != MGP_SUM_SEQ && p.regime != MGP_SUM_LANE2) return MGP_EINVAL;
    if (p.nx < 2 * p.weno_k + 1 || p.nx > max_nx_for(p.weno_k, p.model)) return MGP_EINVAL;
    // meshes above one CTA's capacity: equal power-of-two slabs of <= kMaxNx
    if (!system && p.nx > kMaxNx && split_cs(p.nx) == 0) return MGP_EINVAL;
    if (!(p.dx > 0.0) || !(p.epsilon > 0.0)) return MGP_EINVAL;
    if (a->n_chunks < 0 || a->n_steps < 0 || !a->start) return MGP_EINVAL;
    if (a->g_mode < MGP_G_NONE || a->g_mode > MGP_G_ARRAY) return MGP_EINVAL;
    if (a->g_mode == MGP_G_ARRAY && !a->g && a->n_steps > 0) return MGP_EINVAL;
    if (a->tail < MGP_TAIL_NONE || a->tail > MGP_TAIL_RESID) return MGP_EINVAL;
    if (a->tail != MGP_TAIL_NONE) {
        if (a->tail_regime != MGP_SUM_SEQ && a->tail_regime != MGP_SUM_LANE2) return MGP_EINVAL;
        if (a->tail_g_mode < MGP_G_NONE || a->tail_g_mode > MGP_G_ARRAY) return MGP_EINVAL;
        if (a->tail_g_mode == MGP_G_ARRAY && !a->tail_g) return MGP_EINVAL;
    }
    if (a->tail == MGP_TAIL_PHI && !a->tail_out) return MGP_EINVAL;
    if (a->tail == MGP_TAIL_RESTRICT) {
        if (!a->tail_out || !a->tail_out2 || !a->aux) return MGP_EINVAL;
        if (a->guess == MGP_GUESS_INJECTION && !a->aux2) return MGP_EINVAL;
        if (a->guess != MGP_GUESS_INJECTION && a->guess != MGP_GUESS_LAST_STEP) return MGP_EINVAL;
    }
    if (a->tail == MGP_TAIL_RESID && (!a->aux || !a->partials)) return MGP_EINVAL;
    // one summation regime per launch (the kernel is specialised on it)
    if (a->n_steps > 0 && a->tail != MGP_TAIL_NONE && a->tail_regime != p.regime)
        return MGP_EINVAL;
    return MGP_OK;
}

}  // namespace MGP_UNIT

using namespace MGP_UNIT;

// ---- translation-unit split ------------------------------------------------
// The library is built from MGP_NPARTS compilations of this file, run in
// parallel (MGP_PART = 1..7; undefined = everything in one unit).  Each part
// instantiates one group of kernels behind an externally visible entry;
// part 1 also holds the C ABI, the fused FCF relaxation and the one-step LF
// family.  Same code, flags and per-kernel compilation either way.
#define MGP_IN_PART(n) (MGP_PART == 0 || MGP_PART == (n))

namespace mgp_parts {
int sweep_burgers_k2seq(const mgp_sweep_args &a, cudaStream_t st);
int sweep_burgers_k2lane2(const mgp_sweep_args &a, cudaStream_t st);
int sweep_burgers_k013(const mgp_sweep_args &a, cudaStream_t st);
int sweep_roe(const mgp_sweep_args &a, cudaStream_t st);
int sweep_advection(const mgp_sweep_args &a, cudaStream_t st);
int sweep_systems(const mgp_sweep_args &a, cudaStream_t st);
#if MGP_IN_PART(1)
unsigned long long launches = 0;
#endif
#ifndef MGP_QUICK   // experiment builds: Burgers K = 2 through launch_m directly
#if MGP_IN_PART(2)
int sweep_burgers_k2seq(const mgp_sweep_args &a, cudaStream_t st) {
    return launch_m<MGP_MODEL_BURGERS, 4>(a, st);
}
#endif
#if MGP_IN_PART(3)
int sweep_burgers_k2lane2(const mgp_sweep_args &a, cudaStream_t st) {
    return launch_m<MGP_MODEL_BURGERS, 8>(a, st);
}
#endif
#if MGP_IN_PART(4)
int sweep_burgers_k013(const mgp_sweep_args &a, cudaStream_t st) {
    return launch_m<MGP_MODEL_BURGERS, 1 | 2 | 16>(a, st);
}
#endif
#if MGP_IN_PART(5)
int sweep_roe(const mgp_sweep_args &a, cudaStream_t st) {
    return launch_m<kModelBurgersRoe>(a, st);
}
#endif
#if MGP_IN_PART(6)
int sweep_advection(const mgp_sweep_args &a, cudaStream_t st) {
    return launch_m<MGP_MODEL_ADVECTION>(a, st);
}
#endif
#if MGP_IN_PART(7)
int sweep_systems(const mgp_sweep_args &a, cudaStream_t st) { return launch_sys<>(a, st); }
#endif
#endif  // MGP_QUICK
}  // namespace mgp_parts

#if MGP_IN_PART(1)
extern "C" {

int mgp_sweep(const mgp_sweep_args *args, void *stream) {
    const int rc = validate(args);
    if (rc != MGP_OK) return rc;
    if (args->n_chunks == 0) return MGP_OK;
    cudaStream_t st = (cudaStream_t)stream;
#ifdef MGP_QUICK
    // experiment builds (tools/): Burgers RK-WENO with the global LF flux only
    if (args->phi.model != MGP_MODEL_BURGERS || args->phi.scheme != MGP_SCHEME_RK_WENO)
        return MGP_EINVAL;
    return launch_m<MGP_MODEL_BURGERS>(*args, st);
#else
    const mgp_sweep_args &a = *args;
    if (a.phi.model == MGP_MODEL_SHALLOW_WATER || a.phi.model == MGP_MODEL_EULER)
        return mgp_parts::sweep_systems(a, st);
    if (a.phi.scheme == MGP_SCHEME_RK_WENO_ROE) return mgp_parts::sweep_roe(a, st);
    if (a.phi.scheme == MGP_SCHEME_LF_ONESTEP) return launch_lf<1>(a, st);
    if (a.phi.scheme == MGP_SCHEME_LF_MATCHED) return launch_lf<2>(a, st);
    if (a.phi.model == MGP_MODEL_BURGERS) {
        if (a.phi.weno_k != 2) return mgp_parts::sweep_burgers_k013(a, st);
        const int reg = a.n_steps > 0 ? a.phi.regime : a.tail_regime;
        return reg == MGP_SUM_SEQ ? mgp_parts::sweep_burgers_k2seq(a, st)
                                  : mgp_parts::sweep_burgers_k2lane2(a, st);
    }
    return mgp_parts::sweep_advection(a, st);
#endif
}

int mgp_relax_fcf(const mgp_fcf_args *args, void *stream) {
    if (!args) return MGP_EINVAL;
    const mgp_fcf_args &a = *args;
    if (!fcf_supported(a.phi, a.n_chunks) || a.m < 1 || !a.cs || !a.cd || !a.workspace ||
        a.segment < 0 ||
        a.epoch == 0 || (a.g_mode != MGP_G_NONE && a.g_mode != MGP_G_ZERO))
        return MGP_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    return fcf_dispatch(a.phi, a.n_chunks, [&](auto kk, auto pp) {
        return fcf_launch<decltype(kk)::value, decltype(pp)::value>(a, st);
    });
}

#ifdef MGP_FCF_TRACE
int mgp_debug_fcf_trace(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_fcf_trace, sizeof(unsigned long long) * 4 * 8192) ==
                   cudaSuccess ? 0 : 2;
}
#endif

int64_t mgp_relax_fcf_workspace(const mgp_phi *phi, int64_t n_chunks, int32_t m) {
    if (!phi || m < 1 || !fcf_supported(*phi, n_chunks)) return 0;
    int64_t bytes = 0;
    const int rc = fcf_dispatch(*phi, n_chunks, [&](auto kk, auto pp) {
        FcfLaunch L;   // with F-point storage (the larger of the two plans)
        const int r = fcf_setup<decltype(kk)::value, decltype(pp)::value>(*phi, n_chunks, true, L);
        bytes = L.bytes;
        return r;
    });
    return rc == MGP_OK ? bytes : 0;
}

int mgp_sum_partials(const double *partials, int64_t n, int32_t width, double *out,
                     void *stream) {
    if (!partials || !out || n < 0 || width < 1 || width > 4) return MGP_EINVAL;
    sum_partials_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(partials, n, width, out);
    ++g_launches;
    return cudaPeekAtLastError() == cudaSuccess ? MGP_OK : MGP_ECUDA;
}

int64_t mgp_max_nx(int32_t weno_k, int32_t model) { return max_nx_for(weno_k, model); }

int32_t mgp_abi_version(void) { return 6; }   // 6: MGP_TAIL_RESID honours tail_out

int mgp_weno_tables(int32_t k, double *cw16, double *d4, double *sm64) {
    if (k < 0 || k > 3 || !cw16 || !d4 || !sm64) return MGP_EINVAL;
    memcpy(cw16, h_cw[k], sizeof(h_cw[k]));
    memcpy(d4, h_d[k], sizeof(h_d[k]));
    memcpy(sm64, h_sm[k], sizeof(h_sm[k]));
    return MGP_OK;
}

int64_t mgp_launch_count(void) { return (int64_t)g_launches; }

#ifdef MGP_TRACE
int mgp_trace_read(long long *out, int n) {
    int cnt = 0;
    cudaMemcpyFromSymbol(&cnt, g_trace_n, sizeof(int));
    if (cnt > n / 2) cnt = n / 2;
    cudaMemcpyFromSymbol(out, g_trace, sizeof(long long) * 2 * cnt);
    int zero = 0;
    cudaMemcpyToSymbol(g_trace_n, &zero, sizeof(int));
    return cnt;
}
#endif

int32_t mgp_sweep_args_layout(int64_t *out, int32_t n) {
#define MGP_OFF(f) (int64_t) offsetof(mgp_sweep_args, f)
    const int64_t v[] = {
        (int64_t)sizeof(mgp_phi), (int64_t)sizeof(mgp_sweep_args),
        MGP_OFF(phi), MGP_OFF(n_chunks), MGP_OFF(start), MGP_OFF(start_stride),
        MGP_OFF(n_steps), MGP_OFF(g_mode), MGP_OFF(g), MGP_OFF(g_cs), MGP_OFF(g_ss),
        MGP_OFF(store), MGP_OFF(st_cs), MGP_OFF(st_ss), MGP_OFF(tail),
        MGP_OFF(tail_regime), MGP_OFF(tail_g_mode), MGP_OFF(guess), MGP_OFF(tail_g),
        MGP_OFF(tg_s), MGP_OFF(tail_out), MGP_OFF(to_s), MGP_OFF(tail_out2),
        MGP_OFF(to2_s), MGP_OFF(aux), MGP_OFF(aux_s), MGP_OFF(aux2), MGP_OFF(aux2_s),
        MGP_OFF(ref), MGP_OFF(ref_cs), MGP_OFF(ref_ss), MGP_OFF(ref_last_next),
        MGP_OFF(count_nonfinite), MGP_OFF(partials), MGP_OFF(status)};
#undef MGP_OFF
    const int32_t total = (int32_t)(sizeof(v) / sizeof(v[0]));
    int32_t i = 0;
    for (; i < n && i < total; ++i) out[i] = v[i];
    return i;
}

}  // extern "C"
#endif  // MGP_IN_PART(1)
