/*
 * ctmo.c — fp64 CPU ORACLE for collapsed Taylor mode AD (arXiv 2505.13644).
 *
 * TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py. The product path never
 * links, loads or calls it, and it shares no code with the CUDA path.
 *
 * Plain, slow, obviously correct: per-point loops in fp64, OpenMP over points,
 * no blocking or fusion. Each routine cites the passage it follows
 * ("P:<line>" = PAPER.md line).
 *
 * Parity pins (tests/test_oracle_*.py, all -m "not gpu"):
 *  - act_derivs: central finite differences of each activation; closed forms.
 *  - partitions / nu: the cheat-sheet integers and the partition
 *    counts p(k) = 1,2,3,5,7,11,15,22.
 *  - O1 (vanilla): per-direction finite differences of f along v; closed forms
 *    (quadratic nets, ||x||^4, sums of sines, 1-hidden-layer tanh nets);
 *    torch fp64 autograd Hessians / 4th derivatives on tiny nets.
 *  - O2 (tensors): O1 == O2 (independent derivations: integer vs set partitions).
 *  - O3 (collapsed): O3 == O1 (Eq. 7, the paper's claim).
 *  - gamma: the values printed in Fig. 3.
 *  - biharmonic set: equals the 4th-tensor contraction (O2) and closed forms.
 *  - splitmix64: the reference generator's published outputs for seed 0.
 *  - randomized: exact designs (Hadamard, all sign vectors) reproduce the exact
 *    Laplacian; mean over seeds is unbiased.
 */
#include "ctmo.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define KMAX 4      /* highest Taylor degree the operators need (biharmonic) */
#define PMAXK 8     /* partitions are enumerated up to k = 8 for the nu table */
#define PMAXN 32    /* p(8) = 22 partitions */

/* ------------------------------------------------------------------------ */
/* Activation derivatives sigma^(k)(z), k = 0..4.                            */
/* tanh: sigma' = 1 - t^2 (textbook); higher ones by the product rule:       */
/*   sigma'' = -2 t s, sigma''' = s (6 t^2 - 2), sigma'''' = 8 t s (2 - 3 t^2) */
/* with t = tanh z, s = 1 - t^2.  Pinned by finite differences in tests.     */
/* ------------------------------------------------------------------------ */
void ctmo_act_derivs(int32_t act, double z, double *d)
{
    switch (act) {
    case CTMO_TANH: {
        double t = tanh(z), s = 1.0 - t * t;
        d[0] = t;
        d[1] = s;
        d[2] = -2.0 * t * s;
        d[3] = s * (6.0 * t * t - 2.0);
        d[4] = 8.0 * t * s * (2.0 - 3.0 * t * t);
        break;
    }
    case CTMO_IDENTITY:
        d[0] = z; d[1] = 1.0; d[2] = 0.0; d[3] = 0.0; d[4] = 0.0;
        break;
    case CTMO_SQUARE:
        d[0] = z * z; d[1] = 2.0 * z; d[2] = 2.0; d[3] = 0.0; d[4] = 0.0;
        break;
    case CTMO_SIN:
        d[0] = sin(z); d[1] = cos(z); d[2] = -sin(z); d[3] = -cos(z); d[4] = sin(z);
        break;
    case CTMO_EXP:  /* every derivative of exp is exp */
        d[0] = d[1] = d[2] = d[3] = d[4] = exp(z);
        break;
    default:
        d[0] = d[1] = d[2] = d[3] = d[4] = NAN;
    }
}

/* ------------------------------------------------------------------------ */
/* Integer partitions P(k) and the multiplicity nu(sigma) of Eq. 3           */
/* (`eq:faa-di-bruno`):                                            */
/*   nu(sigma) = k! / ( prod_s n_s!  *  prod_{s in sigma} s! )                */
/* ------------------------------------------------------------------------ */
typedef struct {
    int nparts;
    int part[PMAXK];
    double nu;
    int64_t nu_int;
} partition_t;

static partition_t g_part[PMAXK + 1][PMAXN];
static int g_npart[PMAXK + 1];
static int g_part_ready = 0;

static int64_t factorial(int n)
{
    int64_t r = 1;
    for (int i = 2; i <= n; ++i) r *= i;
    return r;
}

/* Enumerate partitions of k as non-increasing part lists, largest first part
 * first ({k}, {k-1,1}, ...). */
static void gen_partitions(int k, int remaining, int maxpart, int *cur, int depth)
{
    if (remaining == 0) {
        partition_t *p = &g_part[k][g_npart[k]++];
        p->nparts = depth;
        for (int i = 0; i < depth; ++i) p->part[i] = cur[i];
        /* nu = k! / (prod_s n_s! * prod_{s in sigma} s!) */
        int64_t denom = 1;
        int count[PMAXK + 1];
        memset(count, 0, sizeof(count));
        for (int i = 0; i < depth; ++i) {
            count[cur[i]]++;
            denom *= factorial(cur[i]);
        }
        for (int s = 1; s <= k; ++s) denom *= factorial(count[s]);
        p->nu_int = factorial(k) / denom;
        p->nu = (double)p->nu_int;
        return;
    }
    for (int s = (remaining < maxpart ? remaining : maxpart); s >= 1; --s) {
        cur[depth] = s;
        gen_partitions(k, remaining - s, s, cur, depth + 1);
    }
}

static void init_partitions(void)
{
    if (g_part_ready) return;
    int cur[PMAXK];
    for (int k = 1; k <= PMAXK; ++k) {
        g_npart[k] = 0;
        gen_partitions(k, k, k, cur, 0);
    }
    g_part_ready = 1;
}

int32_t ctmo_partition(int32_t k, int32_t p, int32_t *parts, int64_t *nu)
{
    init_partitions();
    if (k < 1 || k > PMAXK || p < 0 || p >= g_npart[k]) return 0;
    const partition_t *q = &g_part[k][p];
    for (int i = 0; i < q->nparts; ++i) parts[i] = q->part[i];
    *nu = q->nu_int;
    return q->nparts;
}

/* Scalar (elementwise) Faa di Bruno, Eq. 3 with a diagonal derivative tensor:
 *   h_k = sum_{sigma in P(k)} nu(sigma) sigma^{(|sigma|)}(z0) prod_{s in sigma} z_s
 * zc[s] = z_s (s = 1..k).  skip_trivial drops sigma = {k} (Eq. 7). */
static double faa_di_bruno(int k, const double *d, const double *zc, int skip_trivial)
{
    double h = 0.0;
    for (int p = 0; p < g_npart[k]; ++p) {
        const partition_t *q = &g_part[k][p];
        if (skip_trivial && q->nparts == 1) continue; /* sigma = {k} */
        double term = q->nu * d[q->nparts];
        for (int i = 0; i < q->nparts; ++i) term *= zc[q->part[i]];
        h += term;
    }
    return h;
}

/* ------------------------------------------------------------------------ */
/* Network helpers                                                           */
/* ------------------------------------------------------------------------ */
static const double *layer_W(const ctmo_net *net, int l)
{
    const double *p = net->params;
    for (int i = 0; i < l; ++i) p += (size_t)net->widths[i + 1] * net->widths[i] + net->widths[i + 1];
    return p;
}
static const double *layer_b(const ctmo_net *net, int l)
{
    return layer_W(net, l) + (size_t)net->widths[l + 1] * net->widths[l];
}
static int max_width(const ctmo_net *net)
{
    int m = 0;
    for (int i = 0; i <= net->L; ++i)
        if (net->widths[i] > m) m = net->widths[i];
    return m;
}
static int check_net(const ctmo_net *net)
{
    if (!net || net->L < 1 || !net->widths || !net->params) return 1;
    for (int i = 0; i <= net->L; ++i)
        if (net->widths[i] < 1) return 1;
    if (net->widths[net->L] != 1) return 1;
    return 0;
}

/* y = W x (+ b if b != NULL), W [out, in] row-major */
static void affine(const double *W, const double *b, int out, int in, const double *x, double *y)
{
    for (int i = 0; i < out; ++i) {
        double acc = b ? b[i] : 0.0;
        const double *w = W + (size_t)i * in;
        for (int j = 0; j < in; ++j) acc += w[j] * x[j];
        y[i] = acc;
    }
}

int ctmo_forward(const ctmo_net *net, const double *X, int64_t N, double *f)
{
    if (check_net(net) || (N > 0 && (!X || !f))) return 1;
    const int D = net->widths[0], wm = max_width(net);
#pragma omp parallel
    {
        double *a = malloc(sizeof(double) * wm), *z = malloc(sizeof(double) * wm);
        double d[5];
#pragma omp for schedule(static)
        for (int64_t n = 0; n < N; ++n) {
            memcpy(a, X + n * D, sizeof(double) * D);
            for (int l = 0; l < net->L; ++l) {
                int in = net->widths[l], out = net->widths[l + 1];
                affine(layer_W(net, l), layer_b(net, l), out, in, a, z);
                if (l < net->L - 1) {
                    for (int i = 0; i < out; ++i) {
                        ctmo_act_derivs(net->act, z[i], d);
                        a[i] = d[0];
                    }
                } else {
                    memcpy(a, z, sizeof(double) * out);
                }
            }
            f[n] = a[0];
        }
        free(a);
        free(z);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Direction families: R directions u_r in R^D, each in one of G groups with  */
/* coefficient c_g; the operator is sum_g c_g sum_{r in g} <d^K f, u_r^{(x)K}>. */
/* (Eq. 5 `eq:sum-k-directional`; Eq. 14 for several groups.)     */
/* ------------------------------------------------------------------------ */
typedef struct {
    int K, R, G;
    const double *dirs;    /* [R, D] shared, or [N, R, D] when per_point */
    int per_point;
    const int *group;      /* [R] group index */
    const double *gcoef;   /* [G] */
} dirset_t;

/* O1 — standard (vanilla) Taylor mode, P:560-564 and Eq. D1:
 * the primal is shared (the "0th component is shared across all jets");
 * each direction r propagates its own coefficients x_{1,r}=u_r, x_{2..K,r}=0;
 * the output's top coefficients f_{K,r} are sliced then summed. */
static void route_o1(const ctmo_net *net, const dirset_t *ds, const double *X, int64_t N,
                     double *op, double *f, double *norm)
{
    const int D = net->widths[0], L = net->L, K = ds->K, wm = max_width(net);
    int nunits = 0;
    for (int l = 1; l < L; ++l) nunits += net->widths[l];
#pragma omp parallel
    {
        /* primal derivatives per hidden unit: deriv[unit][0..4] */
        double *deriv = malloc(sizeof(double) * 5 * (nunits > 0 ? nunits : 1));
        double *a0 = malloc(sizeof(double) * wm), *z0 = malloc(sizeof(double) * wm);
        double *xk = malloc(sizeof(double) * (KMAX + 1) * wm);
        double *zk = malloc(sizeof(double) * (KMAX + 1) * wm);
#pragma omp for schedule(dynamic, 1)
        for (int64_t n = 0; n < N; ++n) {
            const double *x = X + n * D;
            /* primal pass */
            memcpy(a0, x, sizeof(double) * D);
            int off = 0;
            for (int l = 0; l < L; ++l) {
                int in = net->widths[l], out = net->widths[l + 1];
                affine(layer_W(net, l), layer_b(net, l), out, in, a0, z0);
                if (l < L - 1) {
                    for (int i = 0; i < out; ++i) {
                        ctmo_act_derivs(net->act, z0[i], deriv + 5 * (off + i));
                        a0[i] = deriv[5 * (off + i)];
                    }
                    off += out;
                } else {
                    a0[0] = z0[0];
                }
            }
            double fval = a0[0];
            /* one K-jet per direction */
            double total = 0.0, absum = 0.0;
            const double *dirs = ds->per_point ? ds->dirs + (size_t)n * ds->R * D : ds->dirs;
            for (int r = 0; r < ds->R; ++r) {
                /* input jet coefficients x_1 = u_r, x_2 = ... = x_K = 0 */
                for (int k = 1; k <= K; ++k)
                    for (int i = 0; i < D; ++i)
                        xk[k * wm + i] = (k == 1) ? dirs[(size_t)r * D + i] : 0.0;
                off = 0;
                for (int l = 0; l < L; ++l) {
                    int in = net->widths[l], out = net->widths[l + 1];
                    /* affine rule: f_k = W x_k for k >= 1 (no bias) */
                    for (int k = 1; k <= K; ++k) affine(layer_W(net, l), NULL, out, in, xk + k * wm, zk + k * wm);
                    if (l < L - 1) {
                        for (int i = 0; i < out; ++i) {
                            double zc[KMAX + 1];
                            for (int k = 1; k <= K; ++k) zc[k] = zk[k * wm + i];
                            for (int k = 1; k <= K; ++k)
                                xk[k * wm + i] = faa_di_bruno(k, deriv + 5 * (off + i), zc, 0);
                        }
                        off += out;
                    } else {
                        for (int k = 1; k <= K; ++k) xk[k * wm] = zk[k * wm];
                    }
                }
                double c = ds->gcoef[ds->group ? ds->group[r] : 0];
                double term = c * xk[K * wm]; /* slice f_{K,r} */
                total += term;
                absum += fabs(term);
            }
            op[n] = total;
            if (f) f[n] = fval;
            if (norm) norm[n] = absum;
        }
        free(deriv); free(a0); free(z0); free(xk); free(zk);
    }
}

/* O3 — collapsed Taylor mode, Eq. 7 (`eq:faa-di-bruno-expanded`) and
 * Eq. D2/D4: propagate x_0, {x_{k,r}}_{k<K}, and one
 * summed top coefficient per group, X_K^g = sum_{r in g} x_{K,r}:
 *   sum_r h_{K,r} = sum_r sum_{sigma != {K}} nu(sigma) <d^|sigma| h, (x)_s h_{s,r}>
 *                 + <dh, sum_r z_{K,r}>.
 * The groups follow the paper's per-member collapse (one collapsed
 * coefficient per interpolation member), combined with c_g at the end. */
static void route_o3(const ctmo_net *net, const dirset_t *ds, const double *X, int64_t N,
                     double *op, double *f)
{
    const int D = net->widths[0], L = net->L, K = ds->K, R = ds->R, G = ds->G, wm = max_width(net);
#pragma omp parallel
    {
        double *a0 = malloc(sizeof(double) * wm), *z0 = malloc(sizeof(double) * wm);
        /* lower coefficients x_{k,r}, k = 1..K-1: [K][R][wm] */
        double *xl = malloc(sizeof(double) * (size_t)K * R * wm);
        double *zl = malloc(sizeof(double) * (size_t)K * R * wm);
        double *xt = malloc(sizeof(double) * (size_t)G * wm); /* collapsed tops */
        double *zt = malloc(sizeof(double) * (size_t)G * wm);
        double d[5];
#pragma omp for schedule(dynamic, 1)
        for (int64_t n = 0; n < N; ++n) {
            const double *dirs = ds->per_point ? ds->dirs + (size_t)n * R * D : ds->dirs;
            memcpy(a0, X + n * D, sizeof(double) * D);
            for (int r = 0; r < R; ++r)
                for (int k = 1; k < K; ++k)
                    for (int i = 0; i < D; ++i)
                        xl[((size_t)k * R + r) * wm + i] = (k == 1) ? dirs[(size_t)r * D + i] : 0.0;
            for (int g = 0; g < G; ++g)
                for (int i = 0; i < D; ++i) xt[(size_t)g * wm + i] = 0.0; /* sum_r x_{K,r} = 0 */
            for (int l = 0; l < L; ++l) {
                int in = net->widths[l], out = net->widths[l + 1];
                const double *W = layer_W(net, l);
                affine(W, layer_b(net, l), out, in, a0, z0);
                for (int r = 0; r < R; ++r)
                    for (int k = 1; k < K; ++k)
                        affine(W, NULL, out, in, xl + ((size_t)k * R + r) * wm, zl + ((size_t)k * R + r) * wm);
                for (int g = 0; g < G; ++g) affine(W, NULL, out, in, xt + (size_t)g * wm, zt + (size_t)g * wm);
                if (l == L - 1) {
                    a0[0] = z0[0];
                    for (int g = 0; g < G; ++g) xt[(size_t)g * wm] = zt[(size_t)g * wm];
                    break;
                }
                for (int i = 0; i < out; ++i) {
                    ctmo_act_derivs(net->act, z0[i], d);
                    a0[i] = d[0];
                    /* <dh, sum_r z_{K,r}> : the trivial partition, linear in the top */
                    for (int g = 0; g < G; ++g) xt[(size_t)g * wm + i] = d[1] * zt[(size_t)g * wm + i];
                    for (int r = 0; r < R; ++r) {
                        double zc[KMAX + 1];
                        for (int k = 1; k < K; ++k) zc[k] = zl[((size_t)k * R + r) * wm + i];
                        zc[K] = 0.0; /* not used: the trivial partition is skipped */
                        for (int k = 1; k < K; ++k)
                            xl[((size_t)k * R + r) * wm + i] = faa_di_bruno(k, d, zc, 0);
                        int g = ds->group ? ds->group[r] : 0;
                        xt[(size_t)g * wm + i] += faa_di_bruno(K, d, zc, 1);
                    }
                }
            }
            double total = 0.0;
            for (int g = 0; g < G; ++g) total += ds->gcoef[g] * xt[(size_t)g * wm];
            op[n] = total;
            if (f) f[n] = a0[0];
        }
        free(a0); free(z0); free(xl); free(zl); free(xt); free(zt);
    }
}

/* O2 — explicit derivative tensors. Forward propagation of the value, the
 * Jacobian and the higher derivative tensors of every unit w.r.t. x (the plain
 * definition of d^k f(x0) by the multivariate chain rule, with the set-partition
 * form of Faa di Bruno for an elementwise activation), then the contraction
 * <d^K f(x0), C> of Eq. 8/10/12 with the operator's coefficient tensor C.
 * K=2 needs orders 1-2; K=4 orders 1-4 (D^4 entries per unit). */
static int64_t ipow(int64_t b, int e) { int64_t r = 1; while (e-- > 0) r *= b; return r; }

/* C2 [D*D] coefficient matrix (K=2). For K=4: if dirs4 is NULL, C is the biharmonic
 * tensor sum_{a,b} e_a (x) e_a (x) e_b (x) e_b; otherwise C = sum_s c_s v_s^{(x)4} with
 * c_s = w4[s] (or c4 when w4 is NULL) and the directions dirs4 [N, S4, D] per point
 * (d4_per_point) or [S4, D] shared. Returns <d^K f, C> per point. */
static void route_o2(const ctmo_net *net, int K, const double *C2, int C2_per_point,
                     const double *dirs4, int S4, double c4, const double *w4, int d4_per_point,
                     const double *X, int64_t N, double *op, double *f)
{
    const int D = net->widths[0], L = net->L, wm = max_width(net);
    /* per unit: orders 1..K, sizes D, D^2, ..., D^K */
    int64_t tsz[KMAX + 1], toff[KMAX + 2];
    toff[1] = 0;
    for (int k = 1; k <= K; ++k) {
        tsz[k] = ipow(D, k);
        toff[k + 1] = toff[k] + tsz[k];
    }
    const int64_t per_unit = toff[K + 1];
#pragma omp parallel
    {
        double *a0 = malloc(sizeof(double) * wm), *z0 = malloc(sizeof(double) * wm);
        double *A = malloc(sizeof(double) * (size_t)wm * per_unit); /* input tensors of layer */
        double *Z = malloc(sizeof(double) * (size_t)wm * per_unit); /* pre-activation tensors */
        double d[5];
#pragma omp for schedule(dynamic, 1)
        for (int64_t n = 0; n < N; ++n) {
            memcpy(a0, X + n * D, sizeof(double) * D);
            /* input: d x_i / d x_a = delta_ia, higher derivatives zero */
            memset(A, 0, sizeof(double) * (size_t)D * per_unit);
            for (int i = 0; i < D; ++i) A[(size_t)i * per_unit + toff[1] + i] = 1.0;
            for (int l = 0; l < L; ++l) {
                int in = net->widths[l], out = net->widths[l + 1];
                const double *W = layer_W(net, l);
                affine(W, layer_b(net, l), out, in, a0, z0);
                /* tensors are linear in the inputs: Z_u = sum_i W_ui A_i */
                for (int u = 0; u < out; ++u) {
                    double *zu = Z + (size_t)u * per_unit;
                    memset(zu, 0, sizeof(double) * per_unit);
                    for (int i = 0; i < in; ++i) {
                        double w = W[(size_t)u * in + i];
                        const double *ai = A + (size_t)i * per_unit;
                        for (int64_t e = 0; e < per_unit; ++e) zu[e] += w * ai[e];
                    }
                }
                if (l == L - 1) {
                    a0[0] = z0[0];
                    memcpy(A, Z, sizeof(double) * per_unit);
                    break;
                }
                for (int u = 0; u < out; ++u) {
                    ctmo_act_derivs(net->act, z0[u], d);
                    a0[u] = d[0];
                    const double *z1 = Z + (size_t)u * per_unit + toff[1];
                    const double *z2 = Z + (size_t)u * per_unit + toff[2];
                    double *h = A + (size_t)u * per_unit;
                    /* h_a = s' z_a */
                    for (int a = 0; a < D; ++a) h[toff[1] + a] = d[1] * z1[a];
                    /* h_ab = s'' z_a z_b + s' z_ab */
                    for (int a = 0; a < D; ++a)
                        for (int b = 0; b < D; ++b)
                            h[toff[2] + a * D + b] = d[2] * z1[a] * z1[b] + d[1] * z2[a * D + b];
                    if (K >= 4) {
                        const double *z3 = Z + (size_t)u * per_unit + toff[3];
                        const double *z4 = Z + (size_t)u * per_unit + toff[4];
#define I2(a, b) ((a) * D + (b))
#define I3(a, b, c) (((a) * D + (b)) * D + (c))
#define I4(a, b, c, e) ((((a) * D + (b)) * D + (c)) * D + (e))
                        /* h_abc: set partitions of {a,b,c}: {a}{b}{c}; {ab}{c},{ac}{b},{bc}{a}; {abc} */
                        for (int a = 0; a < D; ++a)
                            for (int b = 0; b < D; ++b)
                                for (int c = 0; c < D; ++c)
                                    h[toff[3] + I3(a, b, c)] =
                                        d[3] * z1[a] * z1[b] * z1[c] +
                                        d[2] * (z2[I2(a, b)] * z1[c] + z2[I2(a, c)] * z1[b] + z2[I2(b, c)] * z1[a]) +
                                        d[1] * z3[I3(a, b, c)];
                        /* h_abce: the 15 set partitions of {a,b,c,e} */
                        for (int a = 0; a < D; ++a)
                            for (int b = 0; b < D; ++b)
                                for (int c = 0; c < D; ++c)
                                    for (int e = 0; e < D; ++e) {
                                        double t4 = z1[a] * z1[b] * z1[c] * z1[e];
                                        double t3 = z2[I2(a, b)] * z1[c] * z1[e] + z2[I2(a, c)] * z1[b] * z1[e] +
                                                    z2[I2(a, e)] * z1[b] * z1[c] + z2[I2(b, c)] * z1[a] * z1[e] +
                                                    z2[I2(b, e)] * z1[a] * z1[c] + z2[I2(c, e)] * z1[a] * z1[b];
                                        double t2 = z2[I2(a, b)] * z2[I2(c, e)] + z2[I2(a, c)] * z2[I2(b, e)] +
                                                    z2[I2(a, e)] * z2[I2(b, c)] + z3[I3(a, b, c)] * z1[e] +
                                                    z3[I3(a, b, e)] * z1[c] + z3[I3(a, c, e)] * z1[b] +
                                                    z3[I3(b, c, e)] * z1[a];
                                        h[toff[4] + I4(a, b, c, e)] =
                                            d[4] * t4 + d[3] * t3 + d[2] * t2 + d[1] * z4[I4(a, b, c, e)];
                                    }
                    }
                }
            }
            /* A now holds the output unit's derivative tensors */
            double val = 0.0;
            if (K == 2) {
                const double *H = A + toff[2];
                const double *C = C2_per_point ? C2 + (size_t)n * D * D : C2;
                for (int a = 0; a < D; ++a)
                    for (int b = 0; b < D; ++b) val += H[a * D + b] * C[a * D + b];
            } else if (!dirs4) {
                const double *T4 = A + toff[4];
                for (int a = 0; a < D; ++a)
                    for (int b = 0; b < D; ++b) val += T4[I4(a, a, b, b)];
            } else {
                const double *T4 = A + toff[4];
                for (int s = 0; s < S4; ++s) {
                    const double *v = dirs4 + ((size_t)(d4_per_point ? n * S4 : 0) + s) * D;
                    const double cs = w4 ? w4[s] : c4;
                    for (int a = 0; a < D; ++a)
                        for (int b = 0; b < D; ++b)
                            for (int c = 0; c < D; ++c)
                                for (int e = 0; e < D; ++e) val += cs * T4[I4(a, b, c, e)] * v[a] * v[b] * v[c] * v[e];
                }
            }
            op[n] = val;
            if (f) f[n] = a0[0];
        }
        free(a0); free(z0); free(A); free(Z);
    }
}
#undef I2
#undef I3
#undef I4

static void fill_nan(double *p, int64_t N)
{
    if (p)
        for (int64_t n = 0; n < N; ++n) p[n] = NAN;
}

/* ------------------------------------------------------------------------ */
/* Operators                                                                 */
/* ------------------------------------------------------------------------ */

/* Eq. 8 exact: directions e_d, d = 1..D, one group, c = 1. */
int ctmo_laplacian(const ctmo_net *net, const double *X, int64_t N, int32_t route,
                   double *op, double *f, double *norm)
{
    if (check_net(net) || N < 0 || (N > 0 && (!X || !op))) return 1;
    init_partitions();
    const int D = net->widths[0];
    if (route == CTMO_O2) {
        double *C = calloc((size_t)D * D, sizeof(double));
        for (int a = 0; a < D; ++a) C[a * D + a] = 1.0; /* <d^2 f, I_D> */
        route_o2(net, 2, C, 0, NULL, 0, 0.0, NULL, 0, X, N, op, f);
        free(C);
        fill_nan(norm, N);
        return 0;
    }
    double *E = calloc((size_t)D * D, sizeof(double));
    for (int d = 0; d < D; ++d) E[d * D + d] = 1.0;
    double one = 1.0;
    dirset_t ds = {2, D, 1, E, 0, NULL, &one};
    if (route == CTMO_O1) route_o1(net, &ds, X, N, op, f, norm);
    else if (route == CTMO_O3) { route_o3(net, &ds, X, N, op, f); fill_nan(norm, N); }
    else { free(E); return 1; }
    free(E);
    return 0;
}

/* Eq. 10 exact: directions s_r = columns of sigma. */
int ctmo_weighted_laplacian(const ctmo_net *net, const double *X, int64_t N,
                            const double *sigma, int32_t R, int32_t route,
                            double *op, double *f, double *norm)
{
    if (check_net(net) || N < 0 || R < 1 || !sigma || (N > 0 && (!X || !op))) return 1;
    init_partitions();
    const int D = net->widths[0];
    if (route == CTMO_O2) {
        /* D = sigma sigma^T */
        double *C = calloc((size_t)D * D, sizeof(double));
        for (int a = 0; a < D; ++a)
            for (int b = 0; b < D; ++b)
                for (int r = 0; r < R; ++r) C[a * D + b] += sigma[a * R + r] * sigma[b * R + r];
        route_o2(net, 2, C, 0, NULL, 0, 0.0, NULL, 0, X, N, op, f);
        free(C);
        fill_nan(norm, N);
        return 0;
    }
    double *S = malloc(sizeof(double) * (size_t)R * D);
    for (int r = 0; r < R; ++r)
        for (int d = 0; d < D; ++d) S[r * D + d] = sigma[d * R + r];
    double one = 1.0;
    dirset_t ds = {2, R, 1, S, 0, NULL, &one};
    if (route == CTMO_O1) route_o1(net, &ds, X, N, op, f, norm);
    else if (route == CTMO_O3) { route_o3(net, &ds, X, N, op, f); fill_nan(norm, N); }
    else { free(S); return 1; }
    free(S);
    return 0;
}

/* Eq. 8/10 stochastic: (1/S) sum_s <d^2 f, u_s (x) u_s>, u_s = sigma v_s
 * (P:654-663). */
int ctmo_randomized_laplacian(const ctmo_net *net, const double *X, int64_t N,
                              const double *V, int32_t S, const double *sigma, int32_t Rv,
                              int32_t route, double *op, double *f, double *norm)
{
    if (check_net(net) || N < 0 || S < 1 || Rv < 1 || (N > 0 && (!X || !op || !V))) return 1;
    init_partitions();
    const int D = net->widths[0];
    if (!sigma && Rv != D) return 1;
    /* u_{n,s} = sigma v_{n,s} */
    double *U = malloc(sizeof(double) * (size_t)(N > 0 ? N : 1) * S * D);
    for (int64_t n = 0; n < N; ++n)
        for (int s = 0; s < S; ++s) {
            const double *v = V + ((size_t)n * S + s) * Rv;
            double *u = U + ((size_t)n * S + s) * D;
            for (int d = 0; d < D; ++d) {
                if (!sigma) { u[d] = v[d]; continue; }
                double acc = 0.0;
                for (int r = 0; r < Rv; ++r) acc += sigma[d * Rv + r] * v[r];
                u[d] = acc;
            }
        }
    int rc = 0;
    if (route == CTMO_O2) {
        /* C_n = (1/S) sum_s u_s u_s^T */
        double *C = calloc((size_t)(N > 0 ? N : 1) * D * D, sizeof(double));
        for (int64_t n = 0; n < N; ++n)
            for (int s = 0; s < S; ++s) {
                const double *u = U + ((size_t)n * S + s) * D;
                for (int a = 0; a < D; ++a)
                    for (int b = 0; b < D; ++b) C[(size_t)n * D * D + a * D + b] += u[a] * u[b] / S;
            }
        route_o2(net, 2, C, 1, NULL, 0, 0.0, NULL, 0, X, N, op, f);
        free(C);
        fill_nan(norm, N);
    } else {
        double c = 1.0 / S;
        dirset_t ds = {2, S, 1, U, 1, NULL, &c};
        if (route == CTMO_O1) route_o1(net, &ds, X, N, op, f, norm);
        else if (route == CTMO_O3) { route_o3(net, &ds, X, N, op, f); fill_nan(norm, N); }
        else rc = 1;
    }
    free(U);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Exact rationals for gamma (Eq. F1)                                        */
/* ------------------------------------------------------------------------ */
typedef struct { __int128 n, d; } rat_t;

static __int128 gcd128(__int128 a, __int128 b)
{
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) { __int128 t = a % b; a = b; b = t; }
    return a;
}
static rat_t rat(__int128 n, __int128 d)
{
    if (d < 0) { n = -n; d = -d; }
    __int128 g = gcd128(n, d);
    if (g > 1) { n /= g; d /= g; }
    rat_t r = {n, d};
    return r;
}
static rat_t rat_mul(rat_t a, rat_t b) { return rat(a.n * b.n, a.d * b.d); }
static rat_t rat_add(rat_t a, rat_t b) { return rat(a.n * b.d + b.n * a.d, a.d * b.d); }
static rat_t rat_sub(rat_t a, rat_t b) { return rat(a.n * b.d - b.n * a.d, a.d * b.d); }

/* generalised binomial (a over b) = prod_{l=0}^{b-1} (a - l) / (b - l), 1 if b = 0 */
static rat_t gbinom(rat_t a, int b)
{
    rat_t r = rat(1, 1);
    for (int l = 0; l < b; ++l) r = rat_mul(r, rat_mul(rat_sub(a, rat(l, 1)), rat(1, b - l)));
    return r;
}

/* gamma_{i,j} = sum_{0 < m <= i} (-1)^{|i-m|} (i over m) (|i| m/|m| over j) (|m|/|i|)^{|i|}
 * (Eq. `eq:ttc_coeff`), for I = 2. */
int ctmo_gamma(int32_t i1, int32_t i2, int32_t j1, int32_t j2, int64_t *num, int64_t *den)
{
    if (i1 < 0 || i2 < 0 || j1 < 0 || j2 < 0 || !num || !den) return 1;
    const int ni = i1 + i2;
    if (ni == 0 || j1 + j2 != ni) return 1;
    rat_t g = rat(0, 1);
    for (int m1 = 0; m1 <= i1; ++m1)
        for (int m2 = 0; m2 <= i2; ++m2) {
            const int nm = m1 + m2;
            if (nm == 0) continue; /* |m|_1 > 0 */
            rat_t sign = rat(((ni - nm) % 2) ? -1 : 1, 1);
            rat_t b_im = rat_mul(gbinom(rat(i1, 1), m1), gbinom(rat(i2, 1), m2));
            rat_t b_mj = rat_mul(gbinom(rat((__int128)ni * m1, nm), j1), gbinom(rat((__int128)ni * m2, nm), j2));
            rat_t pw = rat(1, 1);
            for (int e = 0; e < ni; ++e) pw = rat_mul(pw, rat(nm, ni));
            g = rat_add(g, rat_mul(rat_mul(sign, b_im), rat_mul(b_mj, pw)));
        }
    *num = (int64_t)g.n;
    *den = (int64_t)g.d;
    return 0;
}

static double gamma_d(int i1, int i2, int j1, int j2)
{
    int64_t n, d;
    ctmo_gamma(i1, i2, j1, j2, &n, &d);
    return (double)n / (double)d;
}

/* Eq. `ttc_for_biharm_final`:
 *  Laplacian^2 f = 1/24 [ (2D g40 + 2 g31 + g22) sum_d <d^4 f, (4 e_d)^4>
 *                        + 2 g31 sum_{d1 != d2} <d^4 f, (3 e_d1 + e_d2)^4>
 *                        + 2 g22 sum_{d1 < d2} <d^4 f, (2 e_d1 + 2 e_d2)^4> ]
 * with g = gamma_{(2,2), j}. Directions are kept exactly as printed. */
int64_t ctmo_biharmonic_set(int32_t D, double *dirs, double *coef)
{
    if (D < 1) return -1;
    const int64_t J = (int64_t)D * (3 * D - 1) / 2;
    if (!dirs || !coef) return J;
    const double g40 = gamma_d(2, 2, 4, 0), g31 = gamma_d(2, 2, 3, 1), g22 = gamma_d(2, 2, 2, 2);
    const double cA = (2.0 * D * g40 + 2.0 * g31 + g22) / 24.0;
    const double cB = 2.0 * g31 / 24.0;
    const double cC = 2.0 * g22 / 24.0;
    memset(dirs, 0, sizeof(double) * (size_t)J * D);
    int64_t j = 0;
    for (int d = 0; d < D; ++d, ++j) { dirs[j * D + d] = 4.0; coef[j] = cA; }
    for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) {
            if (a == b) continue;
            dirs[j * D + a] = 3.0; dirs[j * D + b] = 1.0; coef[j] = cB; ++j;
        }
    for (int a = 0; a < D; ++a)
        for (int b = a + 1; b < D; ++b) {
            dirs[j * D + a] = 2.0; dirs[j * D + b] = 2.0; coef[j] = cC; ++j;
        }
    return J;
}

int ctmo_biharmonic(const ctmo_net *net, const double *X, int64_t N, int32_t route,
                    double *op, double *f, double *norm)
{
    if (check_net(net) || N < 0 || (N > 0 && (!X || !op))) return 1;
    init_partitions();
    const int D = net->widths[0];
    if (route == CTMO_O2) {
        route_o2(net, 4, NULL, 0, NULL, 0, 0.0, NULL, 0, X, N, op, f);
        fill_nan(norm, N);
        return 0;
    }
    const int64_t J = ctmo_biharmonic_set(D, NULL, NULL);
    double *dirs = malloc(sizeof(double) * (size_t)J * D), *coef = malloc(sizeof(double) * J);
    ctmo_biharmonic_set(D, dirs, coef);
    /* the three interpolation groups A, B, C (one collapsed slot each) */
    int *group = malloc(sizeof(int) * J);
    double gcoef[3];
    for (int64_t j = 0; j < J; ++j) group[j] = (j < D) ? 0 : (j < (int64_t)D * D) ? 1 : 2;
    gcoef[0] = coef[0];
    gcoef[1] = (J > D) ? coef[D] : 0.0;
    gcoef[2] = (J > (int64_t)D * D) ? coef[D * D] : 0.0;
    dirset_t ds = {4, (int)J, 3, dirs, 0, group, gcoef};
    int rc = 0;
    if (route == CTMO_O1) route_o1(net, &ds, X, N, op, f, norm);
    else if (route == CTMO_O3) { route_o3(net, &ds, X, N, op, f); fill_nan(norm, N); }
    else rc = 1;
    free(dirs); free(coef); free(group);
    return rc;
}

/* Stochastic biharmonic, Eq. 12 stochastic case: the paper prints the
 * scale D/S; with standard normal v, Isserlis' theorem gives
 * E <d^4 f, v^{(x)4}> = 3 Laplacian^2 f, so the unbiased scale is 1/(3S)
 * (reading Q1). One 4-jet per sample (x1 = v_s, x2 = x3 = x4 = 0),
 * collapsed over the S samples (1 + 3S + 1 vectors). */
int ctmo_stochastic_biharmonic(const ctmo_net *net, const double *X, int64_t N, const double *V, int32_t S,
                               int32_t route, double *op, double *f, double *norm)
{
    if (check_net(net) || N < 0 || S < 1 || (N > 0 && (!X || !op || !V))) return 1;
    init_partitions();
    const double c = 1.0 / (3.0 * S);
    if (route == CTMO_O2) {
        route_o2(net, 4, NULL, 0, V, S, c, NULL, 1, X, N, op, f);
        fill_nan(norm, N);
        return 0;
    }
    dirset_t ds = {4, S, 1, V, 1, NULL, &c};
    if (route == CTMO_O1) route_o1(net, &ds, X, N, op, f, norm);
    else if (route == CTMO_O3) { route_o3(net, &ds, X, N, op, f); fill_nan(norm, N); }
    else return 1;
    return 0;
}

/* General linear operator of degree K as a weighted sum of K-th directional
 * derivatives (Eq. 5 `eq:sum-k-directional` P:548-558 with coefficients; the form Eq. 15
 * `eq:ttc-general` P:824-839 reduces any <d^K f, C> to, with the gamma_{i,j}/K! of
 * Eq. F1 as weights):  op = sum_j w_j <d^K f(x0), u_j^{(x)K}>,  K in {2, 4}.
 * dirs [J, D] shared, or [N, J, D] per point (per_point != 0); w [J].
 * O1: one K-jet per direction; O3: collapsed, one summed top coefficient per group of
 * equal weights (Eq. 7); O2: the explicit tensor contracted with sum_j w_j u_j^{(x)K}. */
int ctmo_directional_sum(const ctmo_net *net, const double *X, int64_t N, int32_t K, int32_t J,
                         const double *dirs, int32_t per_point, const double *w, int32_t route,
                         double *op, double *f, double *norm)
{
    if (check_net(net) || N < 0 || J < 1 || !dirs || !w || (K != 2 && K != 4) ||
        (N > 0 && (!X || !op)))
        return 1;
    init_partitions();
    const int D = net->widths[0];
    if (route == CTMO_O2) {
        if (K == 2) {
            const int64_t nC = per_point ? (N > 0 ? N : 1) : 1;
            double *C = calloc((size_t)nC * D * D, sizeof(double));
            for (int64_t n = 0; n < nC; ++n)
                for (int j = 0; j < J; ++j) {
                    const double *u = dirs + ((size_t)n * J + j) * D;
                    for (int a = 0; a < D; ++a)
                        for (int b = 0; b < D; ++b) C[(size_t)n * D * D + a * D + b] += w[j] * u[a] * u[b];
                }
            route_o2(net, 2, C, per_point != 0, NULL, 0, 0.0, NULL, 0, X, N, op, f);
            free(C);
        } else {
            route_o2(net, 4, NULL, 0, dirs, J, 0.0, w, per_point != 0, X, N, op, f);
        }
        fill_nan(norm, N);
        return 0;
    }
    /* groups of equal weight (first-occurrence order) */
    int *group = malloc(sizeof(int) * J);
    double *gcoef = malloc(sizeof(double) * J);
    int G = 0;
    for (int j = 0; j < J; ++j) {
        int g = 0;
        while (g < G && gcoef[g] != w[j]) ++g;
        if (g == G) gcoef[G++] = w[j];
        group[j] = g;
    }
    dirset_t ds = {K, J, G, dirs, per_point != 0, group, gcoef};
    int rc = 0;
    if (route == CTMO_O1) route_o1(net, &ds, X, N, op, f, norm);
    else if (route == CTMO_O3) { route_o3(net, &ds, X, N, op, f); fill_nan(norm, N); }
    else rc = 1;
    free(group); free(gcoef);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Nested collapsed Laplacians: Laplacian^2 f = Laplacian (Laplacian f)      */
/* ("we simply nest the Laplacian implementations":   */
/* "nesting Taylor mode Laplacians ... while also allowing to apply our      */
/* collapsing technique").                                                   */
/*                                                                           */
/* The INNER computation is the collapsed Laplacian of Eq. 8/Eq. 7 (K = 2,   */
/* directions e_d): per unit (h0, h1_1..h1_D, sum h2) with                   */
/*   h0 = s(z0), h1_d = s'(z0) z1_d, sum h2 = s'(z0) sum z2 + s''(z0) sum_d z1_d^2 */
/* (Eq. 1, Eq. 7). The OUTER computation applies collapsed   */
/* Taylor mode again (K = 2, directions e_1..e_D) to every quantity of the   */
/* inner one: each becomes an outer 2-jet (value, first coefficients along   */
/* e_1..e_D, one collapsed second coefficient), and the inner rule is        */
/* evaluated in 2-jet arithmetic. Linear layers act on every component, the  */
/* bias on the (inner value, outer value) component only.            */
/* ------------------------------------------------------------------------ */

/* An outer jet is D + 2 doubles: [value, c_1 .. c_D, collapsed second]. */
/* g = phi(a) for phi with derivatives (p0, p1, p2) at a[0]:
 *   value p0, c_e = p1 a_e, second = p1 a_2 + p2 sum_e a_e^2  (Eq. 1/7, K = 2) */
static void jet_apply(int D, double p0, double p1, double p2, const double *a, double *g)
{
    double sq = 0.0;
    for (int e = 1; e <= D; ++e) { g[e] = p1 * a[e]; sq += a[e] * a[e]; }
    g[D + 1] = p1 * a[D + 1] + p2 * sq;
    g[0] = p0;
}

/* g = a * b (Leibniz; the collapsed second coefficient of a product of two
 * 2-jets along e is a b_2 + a_2 b + 2 sum_e a_e b_e) */
static void jet_mul(int D, const double *a, const double *b, double *g)
{
    double cross = 0.0;
    for (int e = 1; e <= D; ++e) cross += a[e] * b[e];
    const double v = a[0] * b[0];
    const double s2 = a[0] * b[D + 1] + a[D + 1] * b[0] + 2.0 * cross;
    for (int e = 1; e <= D; ++e) g[e] = a[0] * b[e] + a[e] * b[0];
    g[0] = v;
    g[D + 1] = s2;
}

int ctmo_biharmonic_nested(const ctmo_net *net, const double *X, int64_t N, double *op, double *f,
                           double *lap)
{
    if (check_net(net) || N < 0 || (N > 0 && (!X || !op))) return 1;
    const int D = net->widths[0];
    const int J = D + 2;           /* components of one outer jet */
    const int C = D + 2;           /* inner components: h0, h1_1..h1_D, sum h2 */
    const int U = C * J;           /* doubles per unit */
    const int wmax = max_width(net);
#pragma omp parallel
    {
        double *H = malloc(sizeof(double) * (size_t)wmax * U);
        double *Z = malloc(sizeof(double) * (size_t)wmax * U);
        double *t0 = malloc(sizeof(double) * J), *t1 = malloc(sizeof(double) * J);
        double *s0 = malloc(sizeof(double) * J), *s1 = malloc(sizeof(double) * J), *s2 = malloc(sizeof(double) * J);
        double *acc = malloc(sizeof(double) * J);
#pragma omp for schedule(dynamic, 1)
        for (int64_t n = 0; n < N; ++n) {
            /* input: x as an inner jet (x, e_d, 0); each inner quantity as an outer jet:
             * x_i -> (x_i, e_i, 0); the constants (e_d)_i and 0 -> (const, 0, 0) */
            memset(H, 0, sizeof(double) * (size_t)D * U);
            for (int i = 0; i < D; ++i) {
                double *u = H + (size_t)i * U;
                u[0 * J + 0] = X[n * D + i];
                u[0 * J + 1 + i] = 1.0;
                u[(1 + i) * J + 0] = 1.0;
            }
            for (int l = 0; l < net->L; ++l) {
                const int in = net->widths[l], out = net->widths[l + 1];
                const double *W = layer_W(net, l), *b = layer_b(net, l);
                for (int i = 0; i < out; ++i) {
                    double *z = Z + (size_t)i * U;
                    for (int k = 0; k < U; ++k) {
                        double a = 0.0;
                        for (int j = 0; j < in; ++j) a += W[(size_t)i * in + j] * H[(size_t)j * U + k];
                        z[k] = a;
                    }
                    z[0] += b[i];
                }
                if (l == net->L - 1) break;
                for (int i = 0; i < out; ++i) {
                    const double *z = Z + (size_t)i * U;
                    double *h = H + (size_t)i * U;
                    double d[5];
                    ctmo_act_derivs(net->act, z[0], d);
                    /* s(z0), s'(z0), s''(z0) as outer jets */
                    jet_apply(D, d[0], d[1], d[2], z, s0);
                    jet_apply(D, d[1], d[2], d[3], z, s1);
                    jet_apply(D, d[2], d[3], d[4], z, s2);
                    /* sum h2 = s'(z0) * sum z2 + s''(z0) * sum_d z1_d * z1_d */
                    memset(acc, 0, sizeof(double) * J);
                    for (int dd = 0; dd < D; ++dd) {
                        jet_mul(D, z + (1 + dd) * J, z + (1 + dd) * J, t0);
                        for (int k = 0; k < J; ++k) acc[k] += t0[k];
                    }
                    jet_mul(D, s2, acc, t0);
                    jet_mul(D, s1, z + (D + 1) * J, t1);
                    for (int k = 0; k < J; ++k) h[(D + 1) * J + k] = t0[k] + t1[k];
                    /* h1_d = s'(z0) * z1_d */
                    for (int dd = 0; dd < D; ++dd) jet_mul(D, s1, z + (1 + dd) * J, h + (1 + dd) * J);
                    /* h0 = s(z0) */
                    memcpy(h, s0, sizeof(double) * J);
                }
            }
            /* scalar output: outer second coefficient of the inner collapsed top */
            op[n] = Z[(D + 1) * J + (D + 1)];
            if (f) f[n] = Z[0];
            if (lap) lap[n] = Z[(D + 1) * J + 0];
        }
        free(H); free(Z); free(t0); free(t1); free(s0); free(s1); free(s2); free(acc);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Counter-based Rademacher directions: splitmix64         */
/* finaliser of seed + (idx + 1) * 0x9E3779B97F4A7C15; sign = top bit.        */
/* ------------------------------------------------------------------------ */
uint64_t ctmo_splitmix64(uint64_t seed, uint64_t idx)
{
    uint64_t z = seed + (idx + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void ctmo_rademacher(uint64_t seed, int64_t point_offset, int64_t N, int32_t S, int32_t Rv, double *V)
{
    for (int64_t n = 0; n < N; ++n)
        for (int s = 0; s < S; ++s)
            for (int d = 0; d < Rv; ++d) {
                uint64_t idx = ((uint64_t)(point_offset + n) * (uint64_t)S + (uint64_t)s) * (uint64_t)Rv + (uint64_t)d;
                V[((size_t)n * S + s) * Rv + d] = (ctmo_splitmix64(seed, idx) >> 63) ? -1.0 : 1.0;
            }
}

/* Host threads for the OpenMP loops over points (bench.py's reference arm runs on rank 0
 * alone under torchrun, which sets OMP_NUM_THREADS=1 for every rank). No arithmetic. */
void ctmo_set_num_threads(int32_t n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int32_t ctmo_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
