/*
 * ctm.h — C ABI of libctm: collapsed Taylor mode PDE operators of tanh MLPs on
 * NVIDIA B200 (sm_100a).  arXiv 2505.13644 ("collapsed Taylor mode AD").
 *
 * The library computes, for a batch of N points x_n in R^D and an MLP
 * f: R^D -> R (tanh on the hidden layers, affine output), the linear
 * PDE operators of the paper by COLLAPSED Taylor mode (Eq. 7,
 * `eq:faa-di-bruno-expanded`): every layer propagates the primal
 * x_0, the first-order coefficients {x_{1,r}} (K=2) or {x_{1,j},x_{2,j},x_{3,j}}
 * (K=4) and ONE summed top coefficient, so sum_r d^K f[v_r] is never
 * materialised per direction.
 *
 * Conventions (all calls):
 *  - Tensor pointers are DEVICE pointers on the handle's device, fp32,
 *    row-major, contiguous, 16-byte aligned (else CTM_ESHAPE).
 *  - Operator calls are ASYNCHRONOUS on `stream` (a cudaStream_t, NULL = the
 *    legacy default stream); the caller synchronises. Inputs must stay valid
 *    until the work on `stream` completes.
 *  - A handle is not re-entrant: concurrent calls on one handle are undefined
 *    (one handle per stream/thread). The handle owns a grow-only workspace.
 *  - Errors are status codes; nothing is thrown or aborted. Arguments are
 *    validated before any launch. N == 0 is a no-op returning CTM_OK (per-point
 *    arrays such as sigma_x or per-point dirs may then be NULL).
 *    ctm_last_error() gives a thread-local detail message.
 *  - Results are bitwise deterministic run to run, and independent of how a
 *    batch is split into calls (no reduction depends on N or on a point's
 *    position; random directions are keyed on the global point index).
 *  - Arithmetic (ctm_set_precision): fp32 values; the layer contractions run on
 *    tcgen05 tensor cores on bf16 planes of every operand. Default CTM_PRECISION_FP32:
 *    three planes (all 24 bits), six plane products, the five small ones over the
 *    whole K before the leading one (fp32 accumulation). CTM_PRECISION_BF16X3: two
 *    planes (~17 bits), three products per K step, half the tensor work. The Taylor
 *    rules run in fp32.  Accuracy target: |op - op_fp64| <= 1e-4 * sum_r
 *    |c_r f_{K,r}|.
 *  - Direction blocks: a point's R directions (K=4: J jets) may be split into nb
 *    blocks of rb, each propagated as its own slot group [x0; its directions; its
 *    partial collapsed top] of P = rb + 2 (K=2), 3 rb + 2 (K=4) or 1 + 2 rb
 *    (standard mode) slots; the partial tops are summed at the readout. This is exact
 *    because the top coefficient enters the Taylor rule of Eq. 7 linearly.
 *    A block must fit one MMA tile (P <= 256); the number of directions is otherwise
 *    bounded only by memory (N * nb * P < 2^31 slot rows) and, for weighted sums and
 *    K=4, by 2048 weights per point. The block size depends only on the operator and
 *    R (never on N), so results stay independent of how a batch is split; it is chosen
 *    by a cost model unless fixed with ctm_set_direction_block. Grad mode
 *    (ctm_grad_enable) uses one block per point (P <= 256).
 */
#ifndef CTM_H
#define CTM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ctm_mlp *ctm_mlp_t; /* opaque; owns device copies of the weights */

typedef enum {
    CTM_OK = 0,
    CTM_EINVAL = 1,       /* NULL required pointer, negative size, bad enum      */
    CTM_ESHAPE = 2,       /* width/D mismatch, misaligned pointer               */
    CTM_ENOMEM = 3,       /* device allocation failed                           */
    CTM_ECUDA = 4,        /* a CUDA runtime/driver call or a launch failed       */
    CTM_EUNSUPPORTED = 5  /* slot count over the cap, non-scalar output, ...     */
} ctm_status;

typedef enum { CTM_RADEMACHER = 0, CTM_GAUSSIAN = 1 } ctm_dist;

/* Load an MLP with n_layers affine layers (n_layers >= 2): tanh after layers
 * 1..n_layers-1, affine output.
 *   widths [n_layers+1] (HOST): widths[0] = D >= 1, widths[n_layers] = 1.
 *   W [n_layers] (HOST array of DEVICE pointers): W_l is [w_l, w_{l-1}] (nn.Linear).
 *   b [n_layers] (HOST array of DEVICE pointers): b_l is [w_l].
 * The weights are copied (pre-split into bf16 hi/lo pairs, padded); the call
 * synchronises the device before returning, so W and b may be freed after.
 * Errors: CTM_EINVAL (NULL, n_layers < 2, width < 1), CTM_EUNSUPPORTED
 * (widths[n_layers] != 1, D > 4096, hidden width > 8192), CTM_ECUDA, CTM_ENOMEM. */
ctm_status ctm_load_mlp(int32_t n_layers, const int32_t *widths, const float *const *W,
                        const float *const *b, int32_t device, ctm_mlp_t *out);

/* Free a handle (NULL-safe). Synchronises the handle's device. */
ctm_status ctm_free_mlp(ctm_mlp_t mlp);

/* Exact Laplacian, Eq. 8 exact case: op[n] = sum_d <d^2 f(x_n), e_d^{(x)2}>.
 *   X [N, D]; op_out [N]; f_out [N] or NULL (f(x_n)).
 * Slots per point P = D + 2 (split into direction blocks when that is faster). */
ctm_status ctm_laplacian(ctm_mlp_t mlp, const float *X, int64_t N, float *op_out, float *f_out,
                         void *stream);

/* Exact Laplacian by STANDARD (vanilla) Taylor mode, P:560-564 and Eq. D3:
 * the same value as ctm_laplacian, but every layer propagates 1 + 2D vectors
 * (x0, and per direction x_{1,d}, x_{2,d}); the top coefficients are sliced and
 * summed only at the output. The paper's baseline, exposed to measure the
 * collapsed/standard ratio of Table `tab:benchmark-ratios` on B200.
 * P = 1 + 2D per point, split into direction blocks of 1 + 2 rb slots. */
ctm_status ctm_laplacian_standard(ctm_mlp_t mlp, const float *X, int64_t N, float *op_out, float *f_out,
                                  void *stream);

/* Weighted Laplacian, Eq. 10 exact case:
 * op[n] = <d^2 f(x_n), sigma sigma^T> = sum_r <d^2 f, s_r^{(x)2}>,
 *   sigma [D, R] (columns s_r; constant across points), R >= 1 (R > 254 runs
 *   in direction blocks). */
ctm_status ctm_weighted_laplacian(ctm_mlp_t mlp, const float *X, int64_t N, const float *sigma,
                                  int32_t R, float *op_out, float *f_out, void *stream);

/* Randomized (Hutchinson) Laplacian, Eq. 8/10 stochastic cases:
 * op[n] = (1/S) sum_s <d^2 f(x_n), (sigma v_{n,s})^{(x)2}>, directions i.i.d. per
 * point.
 *   V [N, S, Rv] explicit directions, or NULL to generate them in-kernel from the
 *     counter i = ((point_offset+n)*S+s)*Rv+d: CTM_RADEMACHER = sign of splitmix64(seed, i)
 *     (top bit set -> -1); CTM_GAUSSIAN = Box-Muller on splitmix64
 *     counters 2i, 2i+1 (parity tests pass Gaussian V explicitly).
 *   point_offset: global index of X[0] (shard-invariant generation), >= 0.
 *   sigma [D, Rv] or NULL (then Rv must equal D), Rv <= 4096. S >= 1 (direction blocks
 *   of the S samples; the 1/S scale is applied once at the readout). */
ctm_status ctm_randomized_laplacian(ctm_mlp_t mlp, const float *X, int64_t N, int32_t S,
                                    const float *V, ctm_dist dist, uint64_t seed,
                                    int64_t point_offset, const float *sigma, int32_t Rv,
                                    float *op_out, float *f_out, void *stream);

/* Exact biharmonic, Eq. 12 exact case, by collapsed 4th-order Taylor
 * mode through the interpolation family of Eq. `ttc_for_biharm_final`
 * (gamma of Fig. 3): J = D(3D-1)/2 jets collapsed into
 * ONE weighted top slot per direction block (P = 3J + 2 for one block; D <= 7 fits one
 * tile, larger D runs in blocks of jets). CTM_EUNSUPPORTED for J > 2048 (D > 36). */
ctm_status ctm_biharmonic(ctm_mlp_t mlp, const float *X, int64_t N, float *op_out, float *f_out,
                          void *stream);

/* Direction blocks (see Conventions): rb > 0 fixes the directions (K=4: jets) per block
 * for later operator calls on this handle (clipped to the operator's R); 0 restores the
 * planner. The value changes the summation order of the collapsed top, not the operator:
 * results for different rb agree to rounding. Host-side. CTM_EINVAL for NULL or rb < 0. */
ctm_status ctm_set_direction_block(ctm_mlp_t mlp, int32_t rb);

/* Exact biharmonic by STANDARD (uncollapsed) 4th-order Taylor mode through the same
 * interpolation family as ctm_biharmonic: every layer propagates 1 + 4J vectors (x0 and,
 * per jet, x1..x4); the weighted top coefficients are summed only at the output. The
 * paper's baseline for the biharmonic rows of Table `tab:benchmark-ratios` (P:3850-3923:
 * 141 vs 109 vectors at D = 5); same value, arguments and errors as ctm_biharmonic.
 * Slots per direction block 1 + 4 rb. */
ctm_status ctm_biharmonic_standard(ctm_mlp_t mlp, const float *X, int64_t N, float *op_out, float *f_out,
                                   void *stream);

/* The randomized Laplacian and the stochastic biharmonic by STANDARD (uncollapsed) Taylor
 * mode: the same estimators, arguments, generated directions and errors as
 * ctm_randomized_laplacian / ctm_stochastic_biharmonic, with 1 + 2S (resp. 1 + 4S)
 * propagated vectors and the per-sample top coefficients summed only at the output. The
 * paper's baselines for the stochastic rows of Table `tab:benchmark-ratios`. */
ctm_status ctm_randomized_laplacian_standard(ctm_mlp_t mlp, const float *X, int64_t N, int32_t S,
                                             const float *V, ctm_dist dist, uint64_t seed,
                                             int64_t point_offset, const float *sigma, int32_t Rv,
                                             float *op_out, float *f_out, void *stream);
ctm_status ctm_stochastic_biharmonic_standard(ctm_mlp_t mlp, const float *X, int64_t N, int32_t S, const float *V,
                                              ctm_dist dist, uint64_t seed, int64_t point_offset, float *op_out,
                                              float *f_out, void *stream);

/* Replace the weights of a loaded MLP (same widths), e.g. after an optimizer step: the
 * library re-derives every weight-dependent array (bf16 pairs, W1^T, the fixed
 * directions' W1 V, W^T in grad mode) with kernels on `stream`, asynchronously; W, b as
 * in ctm_load_mlp (device, caller-owned; must stay valid until `stream` passes this
 * call). Clears the recorded tape. Errors: CTM_EINVAL, CTM_ESHAPE, CTM_ECUDA. */
ctm_status ctm_set_weights(ctm_mlp_t mlp, const float *const *W, const float *const *b, void *stream);

/* Hidden-layer activation of a loaded MLP (default CTM_ACT_TANH, the paper's).
 * Every operator applies the Taylor rules of the selected s with its derivatives
 * s', s'', s''', s'''' (sin: cos, -sin, -cos, sin; exp: all exp z, SPEC S:123 names sin/exp;
 * square z^2: 2z, 2, 0, 0; identity: 1, 0, 0, 0). Host-side setting, takes effect for the next call. CTM_EINVAL for an
 * unknown code or a NULL handle. */
typedef enum { CTM_ACT_TANH = 0, CTM_ACT_IDENTITY = 1, CTM_ACT_SQUARE = 2, CTM_ACT_SIN = 3, CTM_ACT_EXP = 4 } ctm_activation;
ctm_status ctm_set_activation(ctm_mlp_t mlp, ctm_activation act);

/* Arithmetic of the layer contractions for later calls on this handle.
 * The paper computes in fp32 (PyTorch); collapsing is exact,
 * so the arithmetic is the whole error budget of an operator value.
 *   CTM_PRECISION_FP32 (default): every operand as three bf16 planes p0 + p1 + p2 (the
 *     fp32 value to 2^-27), D = sum of the five correction products over the whole K, then
 *     p0*p0 over the whole K, fp32 accumulation in TMEM: fp32-class error.
 *   CTM_PRECISION_BF16X3: two planes, p1*p0 + p0*p1 + p0*p0 per K step ("3xBF16",
 *     ~17 operand bits): about half the tensor time, ~2^-16 per product.
 *   CTM_PRECISION_FP16X3: two fp16 planes (11 + 11 significant bits, the operand split of
 *     3xTF32) of power-of-two scaled values: weights per layer, slot blocks per slot type
 *     (primal / first order / collapsed top) from a rigorous bound on the block's values
 *     (the previous block's recorded max |value| and ||W||_inf), so no plane overflows;
 *     p1*p0 + p0*p1 over the whole K, then p0*p0: three products, ~2^-21 per product, the
 *     tensor time and energy of BF16X3. Covers the collapsed forward
 *     operators of tanh and sin nets with at least two points per MMA tile: K=2
 *     (laplacian, weighted, randomized without sigma, sigma(x), K=2 directional sums) and
 *     K=4 (biharmonic, stochastic biharmonic, K=4 directional sums), and in grad
 *     mode the whole differentiable path (forward, ctm_backward's adjoint layers and weight
 *     gradients) of the same K=2 operators (one scale per slot block, DESIGN.md §5 "fp16x3
 *     training"), the nested biharmonic (one scale per block) and the standard-mode
 *     baselines; other calls on an FP16X3 handle (the exp / identity / square activations,
 *     nets with one hidden layer) run in CTM_PRECISION_FP32.
 * Changing the precision invalidates a recorded tape (ctm_backward then fails).
 * Errors: CTM_EINVAL (NULL handle, unknown value). */
typedef enum { CTM_PRECISION_FP32 = 0, CTM_PRECISION_BF16X3 = 1, CTM_PRECISION_FP16X3 = 2 } ctm_precision;
ctm_status ctm_set_precision(ctm_mlp_t mlp, ctm_precision prec);

/* Weighted Laplacian with a point-dependent sigma (Eq. 10; "sigma can depend on x0",
 * P:686): op[n] = <d^2 f(x_n), sigma(x_n) sigma(x_n)^T> = sum_r <d^2 f(x_n), s_r(x_n)^2>.
 *   sigma_x [N, D, R] device, fp32: sigma(x_n) row-major [D, R] for each point (the
 *   caller evaluates sigma at its points). P = R + 2 (direction blocks for large R). Layer
 *   1 runs on the tensor cores as for ctm_randomized_laplacian with explicit V. Errors:
 *   CTM_EINVAL (NULL sigma_x, R < 1), CTM_ESHAPE (misaligned), CTM_EUNSUPPORTED (D > 4096). */
ctm_status ctm_weighted_laplacian_pointwise(ctm_mlp_t mlp, const float *X, int64_t N, const float *sigma_x,
                                            int32_t R, float *op_out, float *f_out, void *stream);

/* General linear operator of degree K as a weighted sum of K-th directional derivatives
 * (Eq. 5 `eq:sum-k-directional` P:548-558 with coefficients; the general approach of
 * Eq. 13-15, reduces <d^K f, C> to this form with the weights gamma_{i,j}/K!
 * of Eq. F1 and directions sum_i v_{d_i} [j]_i):
 *   op[n] = sum_j weights[j] <d^K f(x_n), u_j^{(x)K}>,   K in {2, 4},
 * collapsed: one summed, weighted top coefficient (Eq. 7).
 *   dirs [J, D] (per_point = 0: the same directions for every point; U = W1 u_j is
 *   computed once per call) or [N, J, D] (per_point = 1); weights [J]; device, fp32.
 *   P = J + 2 (K = 2) or 3J + 2 (K = 4) per point, in direction blocks; J <= 2048;
 *   per-point K = 4 also needs J*D <= 12288.
 * Errors: CTM_EINVAL (NULL dirs/weights, J < 1), CTM_ESHAPE (misaligned),
 * CTM_EUNSUPPORTED (K not 2 or 4, J > 2048, D > 4096). */
ctm_status ctm_directional_sum(ctm_mlp_t mlp, const float *X, int64_t N, int32_t K, int32_t J,
                               const float *dirs, int32_t per_point, const float *weights, float *op_out,
                               float *f_out, void *stream);

/* Exact biharmonic by NESTED collapsed Laplacians, Laplacian(Laplacian f) (P:1192,
 * "the most efficient way to compute biharmonics is by nesting
 * Laplacians ... while also allowing to apply our collapsing technique"). The slots of
 * the nest that are equal by symmetry of mixed partials are propagated once: per point
 * z, the gradient (D), the Hessian upper triangle (D(D+1)/2), the gradient of the
 * Laplacian (D) and the biharmonic (1): P = 2 + 2D + D(D+1)/2 <= 256, i.e. D <= 20
 * (27 vectors at D = 5 vs 107 for ctm_biharmonic). Same arguments, layout, ownership and
 * errors as ctm_biharmonic; CTM_EUNSUPPORTED for D > 20. */
ctm_status ctm_biharmonic_nested(ctm_mlp_t mlp, const float *X, int64_t N, float *op_out, float *f_out,
                                 void *stream);

/* Stochastic biharmonic, Eq. 12 stochastic case, collapsed over S samples
 * (1 + 3S + 1 vectors): op[n] = 1/(3S) sum_s <d^4 f(x_n), v_{n,s}^{(x)4}> with
 * standard normal v (the printed scale D/S is read as garbled: Isserlis gives
 * E<d^4 f, v^4> = 3 Laplacian^2 f, Q1).
 *   V [N, S, D] explicit directions, or NULL: generated in-kernel (Box-Muller on the
 *   splitmix64 counters 2i, 2i+1 of i = ((point_offset+n)*S+s)*D+d).
 *   dist must be CTM_GAUSSIAN. P = 3S + 2 per point, in blocks of samples; S <= 2048 and
 *   S*D <= 12288. */
ctm_status ctm_stochastic_biharmonic(ctm_mlp_t mlp, const float *X, int64_t N, int32_t S, const float *V,
                                     ctm_dist dist, uint64_t seed, int64_t point_offset, float *op_out,
                                     float *f_out, void *stream);

/* ---- Differentiable path (PINN training) ----------------
 * ctm_grad_enable(mlp, 1) makes every later K=2 operator call on this handle
 * (ctm_laplacian, ctm_weighted_laplacian, ctm_randomized_laplacian,
 * ctm_weighted_laplacian_pointwise, ctm_directional_sum with K = 2) record a tape of
 * what its adjoint needs, in library-owned device memory: the layer-1 input block and
 * every hidden layer's output block (bf16 pairs) and pre-activations (fp32), about
 * 8 * N * P * sum_l w_l bytes (C1, N = 16384: ~20 GB). Other operators clear the tape.
 * ctm_grad_enable(mlp, 0) stops recording (memory is kept until ctm_free_mlp).
 * Errors: CTM_EINVAL (NULL), CTM_ECUDA / CTM_ENOMEM (setup). */
ctm_status ctm_grad_enable(ctm_mlp_t mlp, int32_t enable);

/* Gradients of  L = sum_n gop[n] * op[n] + gf[n] * f[n]  with respect to every weight and
 * bias, for the LAST recorded call (its X, directions and N):
 *   gop [N] device (required), gf [N] device or NULL (= 0);
 *   dW, db: HOST arrays of L device pointers, dW[l] [w_{l+1}, w_l] row-major (nn.Linear
 *   layout, as passed to ctm_load_mlp), db[l] [w_{l+1}]; fp32, caller-owned;
 *   accumulate != 0 adds into dW/db, else overwrites.
 * The adjoint runs the transposed Taylor rules layer by layer (jet_layer_kernel<kBwd2>:
 * tcgen05 GEMM with A = W^T fused with the transposed rule) and dW_l = Z_bar_l^T B_{l-1}
 * as 3xBF16 GEMMs; deterministic. Asynchronous on `stream` (order it after the forward).
 * Errors: CTM_EUNSUPPORTED (no recorded differentiable call), CTM_EINVAL (NULL
 * pointers), CTM_ESHAPE (misaligned gop/gf), CTM_ECUDA. */
ctm_status ctm_backward(ctm_mlp_t mlp, const float *gop, const float *gf, float *const *dW, float *const *db,
                        int32_t accumulate, void *stream);

/* Static message for a status. */
const char *ctm_status_str(ctm_status s);

/* Thread-local detail of the last error on this thread ("" if none). */
const char *ctm_last_error(void);

/* Introspection for tests/bench (HOST-side, no device work):
 * number of kernel launches the last operator call on this handle issued,
 * and the slot plan of the last call: P (slots per point), points per tile,
 * MMA N of the hidden-layer GEMMs. */
ctm_status ctm_last_plan(ctm_mlp_t mlp, int32_t *launches, int32_t *slots_per_point,
                         int32_t *points_per_tile, int32_t *mma_n);

/* The direction blocks of the last operator call: blocks per point and directions (K=4:
 * jets) per block; slots_per_point of ctm_last_plan is the slot count of ONE block.
 * HOST-side. */
ctm_status ctm_last_blocks(ctm_mlp_t mlp, int32_t *blocks, int32_t *per_block);

/* The arithmetic the last operator call ran in (a ctm_precision value; an FP16X3 handle
 * runs the calls its mode does not cover in CTM_PRECISION_FP32, see ctm_set_precision).
 * HOST-side. CTM_EINVAL for a NULL handle or output. */
ctm_status ctm_last_precision(ctm_mlp_t mlp, int32_t *precision);

/* The planner itself (HOST-only, no device, no handle): for an operator of kind
 * order = 2 (collapsed K=2), 4 (collapsed K=4), 3 (standard K=2) or 5 (standard K=4) with R
 * directions (jets) and forced_rb as in ctm_set_direction_block, the block split and
 * tile plan an operator call would use. CTM_EINVAL for a bad order or R < 1;
 * CTM_EUNSUPPORTED if no block fits a tile. Any output pointer may be NULL. */
ctm_status ctm_plan_blocks(int32_t order, int32_t R, int32_t forced_rb, int32_t *blocks, int32_t *per_block,
                           int32_t *slots_per_block, int32_t *points_per_tile, int32_t *mma_n);

/* The layer contraction alone (a diagnostic for the GEMM-only accuracy test; SURVEY §8(c)
 * "Parity unpinned": the plane split and the tensor-core accumulation are covered by the
 * end-to-end parity plus this). Z = B W_l^T for hidden layer `layer` (2 <= layer <= L-1,
 * 1-based as W_l in ctm_load_mlp: W_l [w_l, w_{l-1}]), no bias, through the operator
 * path's own kernel (jet_layer_kernel, the handle's precision mode) with the Taylor rule
 * bypassed: the epilogue stores the raw fp32 accumulator of every slot row.
 *   B [rows, w_{l-1}] device fp32 (split into bf16 planes on the device), Z [rows, w_l]
 *   device fp32. Asynchronous on `stream`. Errors: CTM_EINVAL (NULL pointers, rows < 0,
 *   layer out of range), CTM_ESHAPE (misaligned). */
ctm_status ctm_gemm_probe(ctm_mlp_t mlp, int32_t layer, const float *B, int64_t rows, float *Z, void *stream);

/* Per-kernel timing (measurement support for bench.py; off by default).
 * When enabled, every launch of an operator call is bracketed by CUDA events
 * recorded on the call's stream. ctm_profile_read synchronises those events
 * and returns, per kernel kind, the summed device time (ms), the number of
 * launches, and the algorithmic work those launches did (FLOP for
 * CTM_KIND_LAYER = 2 * N * P * w_in * w_out useful products, P the point's slots with all
 * its directions in one block; bytes written for CTM_KIND_SEED = the layer-1 block's slot
 * rows x padded width x 2 bytes x planes; FLOP for CTM_KIND_WGRAD = 2 * N * P * w_l * w_{l-1}),
 * then clears the accumulators.
 * arrays: ms[CTM_KIND_COUNT], launches[CTM_KIND_COUNT], work[CTM_KIND_COUNT]. */
typedef enum {
    CTM_KIND_PREP = 0,    /* per-call direction matrices (W1 sigma)            */
    CTM_KIND_SEED = 1,    /* layer 1: seed + affine + tanh rule                 */
    CTM_KIND_LAYER = 2,   /* hidden layers: tcgen05 GEMM + Taylor epilogue      */
    CTM_KIND_FINAL = 3,   /* readout / finalize                                 */
    CTM_KIND_BWD = 4,     /* ctm_backward: adjoint layers (tcgen05, W^T GEMM + transposed rule) */
    CTM_KIND_WGRAD = 5,   /* ctm_backward: weight-gradient GEMMs Z_bar^T B (work = 2 rows K M)  */
    CTM_KIND_BAUX = 6,    /* ctm_backward: readout adjoint, bias sums, crops                    */
    CTM_KIND_COUNT = 7
} ctm_kernel_kind;

ctm_status ctm_profile_enable(ctm_mlp_t mlp, int32_t enable);
ctm_status ctm_profile_read(ctm_mlp_t mlp, double *ms, int64_t *launches, double *work);

#ifdef __cplusplus
}
#endif
#endif /* CTM_H */
