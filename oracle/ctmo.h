/*
 * ctmo.h — fp64 CPU ORACLE for collapsed Taylor mode (arXiv 2505.13644).
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product path (paper_2505_13644_b200/,
 * libctm.so) may include, link or call this. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may use it.
 *
 * It shares no code with the CUDA path (no headers, helpers, tables or constants).
 *
 * Citations "P:<line>" refer to the paper text, with the equation named.
 *
 * Parity pins: every exported function is pinned by -m "not gpu" tests
 * (tests/test_oracle_*.py); see DESIGN.md §Oracle for the pin of each function.
 */
#ifndef CTMO_H
#define CTMO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Elementwise activation of the hidden layers. The product path is tanh-only
 * (P:1032); the others exist so closed forms can be expressed as MLPs. */
enum { CTMO_TANH = 0, CTMO_IDENTITY = 1, CTMO_SQUARE = 2, CTMO_SIN = 3, CTMO_EXP = 4 };

/* Evaluation routes:
 *  O1 vanilla (standard) Taylor mode: one K-jet per direction, top coefficients
 *     sliced then summed (Eq. D1/D3 P:3066-3446);
 *  O2 explicit derivative tensors contracted with the operator's coefficient
 *     tensor (Eq. 8, 10, 12 read as definitions);
 *  O3 collapsed Taylor mode: the summed top coefficient is propagated
 *     (Eq. 7 `eq:faa-di-bruno-expanded`). */
enum { CTMO_O1 = 1, CTMO_O2 = 2, CTMO_O3 = 3 };

/* An MLP f: R^D -> R with L affine layers; activation after layers 1..L-1,
 * the last layer affine. widths[0]=D, widths[L]=1.
 * params = [W_1 (w1 x w0, row-major), b_1 (w1), W_2, b_2, ...]. */
typedef struct {
    int32_t L;
    const int32_t *widths;
    const double *params;
    int32_t act;
} ctmo_net;

/* All operator calls: X [N, D] row-major. Outputs op[N], f[N] (f may be NULL),
 * norm[N] (may be NULL) = the parity normaliser: the sum over directions of
 * |c_r f_{K,r}| (O1 only; other routes write NaN).  Return 0 on success,
 * nonzero on bad arguments. */

/* Exact Laplacian, Eq. 8 (exact case): sum_d <d^2 f, e_d (x) e_d>. */
int ctmo_laplacian(const ctmo_net *net, const double *X, int64_t N, int32_t route,
                   double *op, double *f, double *norm);

/* Weighted Laplacian, Eq. 10 (exact case), P:690-711:
 * sum_r <d^2 f, s_r (x) s_r>, sigma = (s_1..s_R) in R^{D x R} row-major [D, R]. */
int ctmo_weighted_laplacian(const ctmo_net *net, const double *X, int64_t N,
                            const double *sigma, int32_t R, int32_t route,
                            double *op, double *f, double *norm);

/* Randomized (Hutchinson) Laplacian, Eq. 8/10 (stochastic cases), P:654-722:
 * (1/S) sum_s <d^2 f, u_s (x) u_s>, u_s = sigma v_s (sigma [D, Rv]) or u_s = v_s
 * (sigma NULL, Rv = D).  V [N, S, Rv]: the drawn directions, per point. */
int ctmo_randomized_laplacian(const ctmo_net *net, const double *X, int64_t N,
                              const double *V, int32_t S, const double *sigma, int32_t Rv,
                              int32_t route, double *op, double *f, double *norm);

/* Exact biharmonic, Eq. 12 (exact case) P:739-753, evaluated by O1/O3 through
 * the interpolation family of Eq. `ttc_for_biharm_final`;
 * O2 contracts the 4th derivative tensor: sum_{a,b} T4[a,a,b,b]. */
int ctmo_biharmonic(const ctmo_net *net, const double *X, int64_t N, int32_t route,
                    double *op, double *f, double *norm);

/* Stochastic biharmonic, Eq. 12 stochastic case, with the unbiased scale
 * 1/(3S) for standard normal directions (the printed D/S is read as garbled, DESIGN.md
 * Q1): op = 1/(3S) sum_s <d^4 f, v_s^{(x)4}>, V [N, S, D] the drawn directions. */
int ctmo_stochastic_biharmonic(const ctmo_net *net, const double *X, int64_t N, const double *V, int32_t S,
                               int32_t route, double *op, double *f, double *norm);

/* Weighted sum of K-th directional derivatives, K in {2, 4} (Eq. 5 with weights; the
 * reduction target of the general approach Eq. 13-15):
 * op = sum_j w[j] <d^K f(x0), u_j^{(x)K}>, dirs [J, D] shared or [N, J, D] per point. */
int ctmo_directional_sum(const ctmo_net *net, const double *X, int64_t N, int32_t K, int32_t J,
                         const double *dirs, int32_t per_point, const double *w, int32_t route,
                         double *op, double *f, double *norm);

/* Biharmonic by NESTED collapsed Laplacians:
 * Laplacian^2 f = Laplacian(Laplacian f), the inner Laplacian in collapsed Taylor mode
 * (Eq. 7/8) evaluated in the 2-jet arithmetic of an outer collapsed Laplacian.
 * op[N] = Laplacian^2 f, f[N] (may be NULL), lap[N] = Laplacian f (may be NULL).
 * No normaliser: parity uses the O1 biharmonic's (same operator). */
int ctmo_biharmonic_nested(const ctmo_net *net, const double *X, int64_t N, double *op, double *f,
                           double *lap);

/* sigma^(k)(z), k = 0..4, of the activation (d must hold 5 doubles). */
void ctmo_act_derivs(int32_t act, double z, double *d);

/* Plain forward pass f(x). */
int ctmo_forward(const ctmo_net *net, const double *X, int64_t N, double *f);

/* gamma_{i,j} of Eq. F1 (`eq:ttc_coeff`) for I = 2, as an exact
 * reduced fraction num/den (den > 0). */
int ctmo_gamma(int32_t i1, int32_t i2, int32_t j1, int32_t j2, int64_t *num, int64_t *den);

/* Direction family of Eq. `ttc_for_biharm_final`, in the order
 * group A (4 e_d, d=0..D-1), group B (3 e_a + e_b, a != b, a-major),
 * group C (2 e_a + 2 e_b, a < b, a-major), with coefficients c_j such that
 * Laplacian^2 f = sum_j c_j <d^4 f, v_j^{(x)4}>.  J = D(3D-1)/2.
 * dirs [J, D], coef [J].  Returns J (or -1). Pass NULL to query J. */
int64_t ctmo_biharmonic_set(int32_t D, double *dirs, double *coef);

/* Faa di Bruno multiplicity nu(sigma) of Eq. 3 for the p-th integer
 * partition of k in the oracle's enumeration order; parts[] receives the parts
 * (non-increasing), returns the number of parts, or 0 when p is out of range. */
int32_t ctmo_partition(int32_t k, int32_t p, int32_t *parts, int64_t *nu);

/* Counter-based Rademacher draw (splitmix64 finaliser):
 * V[n, s, d] for global point index point_offset + n. */
void ctmo_rademacher(uint64_t seed, int64_t point_offset, int64_t N, int32_t S, int32_t Rv,
                     double *V);
uint64_t ctmo_splitmix64(uint64_t seed, uint64_t idx);

/* Number of OpenMP threads the oracle uses (for the cpu_baseline report). */
void ctmo_set_num_threads(int32_t n);
int32_t ctmo_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
