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
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#include "../../include/mgrit_phi.h"

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

namespace {

constexpr int kMaxThreads = 512;
constexpr int kMaxPerThread = 8;
constexpr int64_t kMaxNx = (int64_t)kMaxThreads * kMaxPerThread;

unsigned long long g_launches = 0;

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

// reconstruct_left (weno.py:171-177) on the window w[0..2K] (cells in
// increasing order for the left state, reversed for the right state).
// Zero table entries are skipped (exact for finite windows); CHECK = true
// turns a window with any non-finite cell into NaN as the reference's 0*inf
// terms do -- needed only where no NaN-propagating alpha covers it.
template <int K, bool CHECK>
__device__ __forceinline__ double reconstruct(const double *w, int regime,
                                              double eps, double k0_omega) {
    if (CHECK) {
        int bad = 0;
#pragma unroll
        for (int s = 0; s <= 2 * K; ++s) bad |= !is_finite(w[s]);
        if (bad) return __longlong_as_double(kNaNBits);
    }
    if (K == 0) {
        // beta = 0, omega = raw/raw (1, or NaN when 1/eps^2 overflows)
        return k0_omega * (c_cw[0][0][0] * w[0]);
    }
    double q[K + 1], raw[K + 1];
#pragma unroll
    for (int r = 0; r <= K; ++r) {
        const int lo = K - r;
        double acc;
        if (K < 2 || regime == MGP_SUM_SEQ) {
            acc = c_cw[K][r][0] * w[lo];
#pragma unroll
            for (int j = 1; j <= K; ++j) acc = acc + c_cw[K][r][j] * w[lo + j];
        } else {
            // NumPy's contiguous einsum: (even slots) + (odd slots)
            double ev = 0.0, od = 0.0;
            bool he = false, ho = false;
#pragma unroll
            for (int j = 0; j <= K; ++j) {
                const int s = lo + j;
                const double p = c_cw[K][r][j] * w[s];
                if ((s & 1) == 0) {
                    ev = he ? ev + p : p;
                    he = true;
                } else {
                    od = ho ? od + p : p;
                    ho = true;
                }
            }
            acc = he ? (ho ? ev + od : ev) : od;
        }
        q[r] = acc;
        double b = 0.0;
#pragma unroll
        for (int i = 0; i <= K; ++i)
#pragma unroll
            for (int j = 0; j <= K; ++j) {
                const double t = (w[lo + i] * c_sm[K][r][i][j]) * w[lo + j];
                b = (i == 0 && j == 0) ? t : b + t;
            }
        const double e = eps + b;
        raw[r] = c_d[K][r] / (e * e);
    }
    double S = raw[0];
#pragma unroll
    for (int r = 1; r <= K; ++r) S = S + raw[r];
    double v = (raw[0] / S) * q[0];
#pragma unroll
    for (int r = 1; r <= K; ++r) v = v + (raw[r] / S) * q[r];
    return v;
}

struct Consts {
    double dt, hdt, qdt, tdt, two3, inv_dx, dx, eps, speed, half_alpha_adv;
    double k0_omega;
    bool dx_pow2;
};

// Field: the shared-memory image of one field plus the per-stage machinery.
template <int K, int MODEL>
struct Field {
    static constexpr int H = K + 1;   // periodic halo on each side
    int nx;
    double *s_u;    // [nx + 2H]  stage input, cell c at s_u[c + H]
    double *s_u0;   // [nx]       RK base state
    double *s_L;    // [nx]       left states, then the interface flux
    double *s_R;    // [nx]       right states
    unsigned long long *s_red;  // [32]
    double *s_sum;  // [3 * 32]

    __device__ __forceinline__ void put(int c, double v) {
        s_u[c + H] = v;
        if (c < H) s_u[nx + H + c] = v;
        if (c >= nx - H) s_u[c - (nx - H)] = v;
    }
    __device__ __forceinline__ double get(int c) const { return s_u[c + H]; }

    // A = SemiDiscreteOperator.rhs(s_u), written to s_R[c] for the cells this
    // thread owns (c = tid + j*blockDim.x; the thread that reconstructs
    // interface c+1/2 is the one that owns cell c, so s_R[c] is free to
    // reuse once the flux is formed).  Starts with a barrier (s_u must be
    // complete) and ends after the flux barrier; s_u is not modified.
    __device__ void rhs(const Consts &k, int regime) {
        const int tid = threadIdx.x, nt = blockDim.x;
        __syncthreads();
        unsigned long long m = 0;
#pragma unroll 1
        for (int i = tid; i < nx; i += nt) {
            const double *c = s_u + H + i;
            double w[2 * K + 2];
#pragma unroll
            for (int s = 0; s < 2 * K + 2; ++s) w[s] = c[s - K];
            double wr[2 * K + 1];
#pragma unroll
            for (int s = 0; s <= 2 * K; ++s) wr[s] = w[2 * K + 1 - s];
            constexpr bool kCheck = (MODEL == MGP_MODEL_ADVECTION);
            const double ul = reconstruct<K, kCheck>(w, regime, k.eps, k.k0_omega);
            const double ur = reconstruct<K, kCheck>(wr, regime, k.eps, k.k0_omega);
            s_L[i] = ul;
            s_R[i] = ur;
            if (MODEL == MGP_MODEL_BURGERS) {
                m = umax64(m, umax64(abs_bits(ul), abs_bits(ur)));
                // a non-finite cell makes every window holding it NaN in the
                // reference, hence alpha NaN (np.max propagates it)
                if (!is_finite(w[K])) m = kNaNBits;
            }
        }
        double half_alpha;
        if (MODEL == MGP_MODEL_BURGERS) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                m = umax64(m, __shfl_xor_sync(0xffffffffu, m, o));
            if ((tid & 31) == 0) s_red[tid >> 5] = m;
            __syncthreads();
            m = s_red[0];
            const int nw = (nt + 31) >> 5;
            for (int w = 1; w < nw; ++w) m = umax64(m, s_red[w]);
            half_alpha = 0.5 * __longlong_as_double((long long)m);
        } else {
            half_alpha = k.half_alpha_adv;
        }
#pragma unroll 1
        for (int i = tid; i < nx; i += nt) {
            const double ul = s_L[i], ur = s_R[i];
            double fl, fr;
            if (MODEL == MGP_MODEL_BURGERS) {
                fl = (0.5 * ul) * ul;
                fr = (0.5 * ur) * ur;
            } else {
                fl = k.speed * ul;
                fr = k.speed * ur;
            }
            s_L[i] = (0.5 * (fl + fr)) - (half_alpha * (ur - ul));
        }
        __syncthreads();
#pragma unroll 1
        for (int c = tid; c < nx; c += nt) {
            const double fm = s_L[c == 0 ? nx - 1 : c - 1];
            const double neg = -(s_L[c] - fm);
            s_R[c] = k.dx_pow2 ? neg * k.inv_dx : neg / k.dx;
        }
    }

    // RungeKuttaStepper.advance(s_u) (stepper.py:50-62) for the owned cells,
    // result in s_R[c]; rk_order 0 gives the rhs.  s_u keeps the last stage
    // input (the caller commits the result with put()).
    __device__ void phi(const Consts &k, int rk, int regime) {
        const int tid = threadIdx.x, nt = blockDim.x;
        for (int c = tid; c < nx; c += nt) s_u0[c] = get(c);
        rhs(k, regime);
        if (rk == 0) return;
        for (int c = tid; c < nx; c += nt) {
            const double u1 = s_u0[c] + k.dt * s_R[c];
            s_R[c] = u1;
            if (rk > 1) put(c, u1);
        }
        if (rk == 1) return;
        rhs(k, regime);
        if (rk == 2) {
            for (int c = tid; c < nx; c += nt)
                s_R[c] = ((0.5 * s_u0[c]) + (0.5 * get(c))) + (k.hdt * s_R[c]);
            return;
        }
        for (int c = tid; c < nx; c += nt) {
            const double u2 = ((0.75 * s_u0[c]) + (0.25 * get(c))) + (k.qdt * s_R[c]);
            put(c, u2);
        }
        rhs(k, regime);
        for (int c = tid; c < nx; c += nt)
            s_R[c] = ((s_u0[c] / 3.0) + (k.two3 * get(c))) + (k.tdt * s_R[c]);
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

template <int K, int MODEL>
__global__ void __launch_bounds__(kMaxThreads, 1)
    sweep_kernel(const mgp_sweep_args a, const Consts k) {
    extern __shared__ double smem[];
    using F = Field<K, MODEL>;
    F f;
    const int nx = (int)a.phi.nx;
    f.nx = nx;
    f.s_u = smem;
    f.s_u0 = f.s_u + nx + 2 * F::H;
    f.s_L = f.s_u0 + nx;
    f.s_R = f.s_L + nx;
    f.s_sum = f.s_R + nx;
    f.s_red = reinterpret_cast<unsigned long long *>(f.s_sum + 3 * 32);

    const int tid = threadIdx.x, nt = blockDim.x;
    const int rk = a.phi.rk_order;

    for (int64_t b = blockIdx.x; b < a.n_chunks; b += gridDim.x) {
        double acc_r = 0.0, acc_e = 0.0, acc_n = 0.0;
        const double *x0 = a.start + b * a.start_stride;
        const double *ref = a.ref ? a.ref + b * a.ref_cs : nullptr;
        for (int c = tid; c < nx; c += nt) {
            const double v = x0[c];
            f.put(c, v);
            if (ref) {
                const double d = v - ref[c];
                acc_e = acc_e + d * d;
            }
            if (a.count_nonfinite && !is_finite(v)) acc_n += 1.0;
        }
        for (int s = 1; s <= a.n_steps; ++s) {
            f.phi(k, rk, a.phi.regime);
            const double *g = a.g ? a.g + b * a.g_cs + (int64_t)(s - 1) * a.g_ss : nullptr;
            double *st = a.store ? a.store + b * a.st_cs + (int64_t)(s - 1) * a.st_ss : nullptr;
            const double *rs = ref ? ref + (int64_t)s * a.ref_ss : nullptr;
            for (int c = tid; c < nx; c += nt) {
                const double v = add_g(f.s_R[c], a.g_mode, g, c);
                f.put(c, v);
                if (st) st[c] = v;
                if (rs) {
                    const double d = v - rs[c];
                    acc_e = acc_e + d * d;
                }
                if (a.count_nonfinite && !is_finite(v)) acc_n += 1.0;
            }
        }
        if (a.tail != MGP_TAIL_NONE) {
            f.phi(k, rk, a.tail_regime);
            const double *tg = a.tail_g ? a.tail_g + b * a.tg_s : nullptr;
            if (a.tail == MGP_TAIL_PHI) {
                double *out = a.tail_out + b * a.to_s;
                for (int c = tid; c < nx; c += nt)
                    out[c] = add_g(f.s_R[c], a.tail_g_mode, tg, c);
            } else if (a.tail == MGP_TAIL_RESTRICT) {
                // mgrit.py:211-215: g_c = (g_f + phi) - psi;
                // u_c = phi + g_f (last-step) or u_f (injection)
                const double *phi = a.aux + b * a.aux_s;
                const double *uf = a.aux2 ? a.aux2 + b * a.aux2_s : nullptr;
                double *gc = a.tail_out + b * a.to_s;
                double *uc = a.tail_out2 + b * a.to2_s;
                for (int c = tid; c < nx; c += nt) {
                    const double gf = g_value(a.tail_g_mode, tg, c);
                    const double p = phi[c];
                    const double left = (a.tail_g_mode == MGP_G_NONE) ? p : gf + p;
                    gc[c] = left - f.s_R[c];
                    uc[c] = (a.guess == MGP_GUESS_LAST_STEP)
                                ? add_g(p, a.tail_g_mode, tg, c)
                                : uf[c];
                }
            } else {  // MGP_TAIL_RESID, mgrit.py:268: (g + Phi(u_prev)) - u
                const double *tgt = a.aux + b * a.aux_s;
                const bool last = (b == a.n_chunks - 1) && a.ref_last_next;
                const double *rn = (last && a.ref) ? a.ref + (b + 1) * a.ref_cs : nullptr;
                for (int c = tid; c < nx; c += nt) {
                    const double pred = (a.tail_g_mode == MGP_G_NONE)
                                            ? f.s_R[c]
                                            : g_value(a.tail_g_mode, tg, c) + f.s_R[c];
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
        if (a.partials) {
            // fixed-order block reduction (deterministic for a given nt)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                acc_r += __shfl_xor_sync(0xffffffffu, acc_r, o);
                acc_e += __shfl_xor_sync(0xffffffffu, acc_e, o);
                acc_n += __shfl_xor_sync(0xffffffffu, acc_n, o);
            }
            __syncthreads();
            if ((tid & 31) == 0) {
                f.s_sum[3 * (tid >> 5) + 0] = acc_r;
                f.s_sum[3 * (tid >> 5) + 1] = acc_e;
                f.s_sum[3 * (tid >> 5) + 2] = acc_n;
            }
            __syncthreads();
            if (tid < 3) {
                double t = 0.0;
                const int nw = (nt + 31) >> 5;
                for (int w = 0; w < nw; ++w) t = t + f.s_sum[3 * w + tid];
                a.partials[3 * b + tid] = t;
            }
        }
        __syncthreads();  // s_u / s_sum reuse by the next chunk
    }
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
    return k;
}

int threads_for(int64_t nx) {
    int64_t nt = (nx + kMaxPerThread - 1) / kMaxPerThread;
    if (nt < 128) nt = nx < 128 ? nx : 128;  // keep >= 4 warps when possible
    nt = (nt + 31) / 32 * 32;
    if (nt > kMaxThreads) nt = kMaxThreads;
    return (int)nt;
}

size_t smem_bytes(int64_t nx, int k) {
    return sizeof(double) * (size_t)(nx + 2 * (k + 1) + 3 * nx + 3 * 32) +
           sizeof(unsigned long long) * 32;
}

template <int K, int MODEL>
int launch_t(const mgp_sweep_args &a, cudaStream_t st) {
    const int nt = threads_for(a.phi.nx);
    const size_t sm = smem_bytes(a.phi.nx, K);
    auto kern = sweep_kernel<K, MODEL>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024) != cudaSuccess)
            return MGP_ECUDA;
        attr_set = true;
    }
    int64_t grid = a.n_chunks;
    if (grid > (int64_t)1 << 30) grid = (int64_t)1 << 30;
    const Consts k = make_consts(a.phi);
    kern<<<(unsigned)grid, nt, sm, st>>>(a, k);
    ++g_launches;
    return cudaPeekAtLastError() == cudaSuccess ? MGP_OK : MGP_ECUDA;
}

template <int MODEL>
int launch_m(const mgp_sweep_args &a, cudaStream_t st) {
    switch (a.phi.weno_k) {
        case 0: return launch_t<0, MODEL>(a, st);
        case 1: return launch_t<1, MODEL>(a, st);
        case 2: return launch_t<2, MODEL>(a, st);
        case 3: return launch_t<3, MODEL>(a, st);
    }
    return MGP_EINVAL;
}

int validate(const mgp_sweep_args *a) {
    if (!a) return MGP_EINVAL;
    const mgp_phi &p = a->phi;
    if (p.model != MGP_MODEL_BURGERS && p.model != MGP_MODEL_ADVECTION) return MGP_EINVAL;
    if (p.weno_k < 0 || p.weno_k > 3) return MGP_EINVAL;
    if (p.rk_order < 0 || p.rk_order > 3) return MGP_EINVAL;
    if (p.regime != MGP_SUM_SEQ && p.regime != MGP_SUM_LANE2) return MGP_EINVAL;
    if (p.nx < 2 * p.weno_k + 1 || p.nx > kMaxNx) return MGP_EINVAL;
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
    return MGP_OK;
}

}  // namespace

extern "C" {

int mgp_sweep(const mgp_sweep_args *args, void *stream) {
    const int rc = validate(args);
    if (rc != MGP_OK) return rc;
    if (args->n_chunks == 0) return MGP_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (args->phi.model == MGP_MODEL_BURGERS) return launch_m<MGP_MODEL_BURGERS>(*args, st);
    return launch_m<MGP_MODEL_ADVECTION>(*args, st);
}

int mgp_sum_partials(const double *partials, int64_t n, int32_t width, double *out,
                     void *stream) {
    if (!partials || !out || n < 0 || width < 1 || width > 4) return MGP_EINVAL;
    sum_partials_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(partials, n, width, out);
    ++g_launches;
    return cudaPeekAtLastError() == cudaSuccess ? MGP_OK : MGP_ECUDA;
}

int64_t mgp_max_nx(void) { return kMaxNx; }

int32_t mgp_abi_version(void) { return 1; }

int mgp_weno_tables(int32_t k, double *cw16, double *d4, double *sm64) {
    if (k < 0 || k > 3 || !cw16 || !d4 || !sm64) return MGP_EINVAL;
    memcpy(cw16, h_cw[k], sizeof(h_cw[k]));
    memcpy(d4, h_d[k], sizeof(h_d[k]));
    memcpy(sm64, h_sm[k], sizeof(h_sm[k]));
    return MGP_OK;
}

int64_t mgp_launch_count(void) { return (int64_t)g_launches; }

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
        MGP_OFF(count_nonfinite), MGP_OFF(partials)};
#undef MGP_OFF
    const int32_t total = (int32_t)(sizeof(v) / sizeof(v[0]));
    int32_t i = 0;
    for (; i < n && i < total; ++i) out[i] = v[i];
    return i;
}

}  // extern "C"
