// jet_layer.cuh — one hidden layer of collapsed Taylor mode, fused:
//
//   Z^T[feature, slot] = W_l[feature, :] . B_{l-1}[slot, :]      (bf16 planes, tcgen05, TMEM accumulator)
//   B_l[slot, feature] = Taylor rule of tanh applied per point    (epilogue, registers)
//
// Swap-AB mapping: the MMA's M = 128 output features (one TMEM lane
// each), N = the slots of `pts_per_tile` points (one TMEM column each). Each epilogue
// thread owns one feature across all slots of a point, so the collapse
// sum_r (...) over directions is a sequential in-register sum inside one thread:
// X1 never round-trips HBM between the GEMM and the nonlinearity.
//
// K=2 epilogue (Eq. 1 P:327 + Eq. 7, Eq. D4):
//   h0 = tanh z0, h1_r = s' z1_r, sum h2 = s' sum z2 + s'' sum_r z1_r^2
// K=4 epilogue (cheat-sheet rows for k<=4, collapsed by Eq. 7):
//   h1 = s'z1, h2 = s''z1^2 + s'z2, h3 = s'''z1^3 + 3s''z1z2 + s'z3,
//   sum_w h4 = sum_j w_j (s''''z1^4 + 6s'''z1^2z2 + 4s''z1z3 + 3s''z2^2) + s' sum_w z4
//
// Layout in HBM: block B_l is [N*P rows, ld], row = n*P + slot, stored as
// bf16 planes (p0 = rn_bf16(v), p1 = rn_bf16(v - p0), p2 = rn_bf16(v - p0 - p1)), plane k at
// k * pstride elements. Arithmetic, chosen per handle:
//   fp32 mode (default), 3 planes: the five correction products p2*p0 + p1*p1 + p0*p2 +
//     p1*p0 + p0*p1 over the whole K first, then p0*p0 over the whole K into the same fp32
//     accumulator ("bf16x6, two phases": the main products see only K/16 accumulations);
//   fast mode, 2 planes: p1*p0 + p0*p1 + p0*p0 per K step ("3xBF16", ~17 operand bits).
#pragma once
#include <type_traits>

#include "ptx.cuh"

namespace ctm {

#ifdef CTM_EXP_STATS  // per-role cycle counters (experiment builds only)
__device__ unsigned long long g_stats[256][8];
#define STAT_T0() const long long t0_ = clock64()
#define STAT_ADD(i) atomicAdd(&g_stats[blockIdx.x][i], (unsigned long long)(clock64() - t0_))
#else
#define STAT_T0()
#define STAT_ADD(i)
#endif

constexpr int kBM = 128;                         // features per CTA = TMEM lanes (a CTA pair spans 256)
// bf16 K per stage: 128-byte rows, SWIZZLE_128B (descriptor layout code 2, 8-row core-matrix
// stride 1024 B). Measured against 64-byte rows / SWIZZLE_64B with twice the stages: the
// tensor pipe is fed better by 128-byte rows (C1 layers -8.5%, C4 -4.5%, S=8 -4.5%).
constexpr int kBK = 64;
constexpr uint32_t kSwLayout = 2, kSwSBO = 1024;
// The operand ring holds SLOTS of one bf16 plane of A and the same plane of B for one
// K block (kBK). A K step of the fp32 mode's first phase needs three slots (all planes), of
// its second phase one slot (p0 again), of the fast mode two slots.
constexpr int kMaxN = 256;                       // MMA N cap (TMEM columns per accumulator)
constexpr int kATileBytes = kBM * kBK * 2;       // 16 KB
constexpr int kSlots = 6;                        // 6 x 32 KB ring
constexpr int kBTileBytes = (kMaxN / 2) * kBK * 2;  // 16 KB: a CTA of the pair stages half of B
constexpr int kSlotBytes = kATileBytes + kBTileBytes;
constexpr int kStageBytes = kSlotBytes;          // (ring bytes = kSlots * kSlotBytes)
// kFlagRing7 instances (MMA N <= 208, e.g. C1's 4 points of 52 slots): 7 slots of 29 KB
constexpr int kSlots7 = 7;
constexpr int kSlotBytes7 = kATileBytes + 104 * kBK * 2;
constexpr int kRingBytes = (kSlots * kSlotBytes > kSlots7 * kSlotBytes7) ? kSlots * kSlotBytes : kSlots7 * kSlotBytes7;
constexpr int kMaxPtsPerTile = 128;              // P >= 2  ->  pts_per_tile <= 128
constexpr int kMaxJets = 84;                     // K=4: 3J+2 <= 256
constexpr int kMaxW = 2048;                      // per-direction weights in smem (all blocks of a point)
constexpr int kLayerThreads = 320;               // warp0 TMA, warp1 MMA, warps2-9 epilogue (2 groups)
constexpr int kLayerSmem = kRingBytes + 1024 /*align*/ + 256 /*barriers*/ +
                           4 * kMaxPtsPerTile * 2 * 4 /*readout*/ + kMaxW * 4 + 2 * kBM * 4 /*xacc*/;
constexpr uint32_t kTmemCols = 512;              // 1 CTA/SM; reads past N stay in range
// Epilogue modes (template parameter KORD): 2 = K=2 collapsed, 4 = K=4 collapsed (weighted
// top), kStd2 = K=2 STANDARD Taylor mode (1 + 2R slots, the per-direction top
// coefficients are propagated and only summed at the output) -- the paper's baseline.
constexpr int kStd2 = 3;
// kStd4: K=4 STANDARD Taylor mode for a weighted jet family (the biharmonic of Eq. 12 by
// the interpolation directions, uncollapsed): 1 + 4J slots, per jet (z1, z2, z3, z4); the
// per-jet top coefficients h4_j are weighted and summed only at the readout -- the
// paper's baseline for the biharmonic rows of Table `tab:benchmark-ratios`.
constexpr int kStd4 = 7;
// kNest: the biharmonic by NESTED collapsed Laplacians, with the slots
// of the nest that are equal by symmetry of partial derivatives stored once: per point
// [z | g_a = d_a z (D) | H_ab = d_a d_b z, a <= b packed row-major (D(D+1)/2) |
//  L_a = d_a Lap z (D) | Q = Lap^2 z], P = 2 + 2D + D(D+1)/2 (27 at D = 5, 252 at D = 20).
constexpr int kNest = 5;
constexpr int kNestMaxD = 20;
// kBwd2: the backward of the K=2 collapsed rule (differentiable path): the
// mainloop computes B_bar^T = W^T Z_bar^T (A = W^T), the epilogue applies the transposed
// Taylor rule with the saved pre-activations (epilogue_bwd2).
constexpr int kBwd2 = 6;

// Hidden-layer activation s and its derivatives s', s'', s''', s'''' at z (the Taylor
// rules only ever need these five numbers). tanh is the paper's; sin, exp, identity
// and square extend the path and turn closed forms into GPU tests.
enum : int { kActTanh = 0, kActIdentity = 1, kActSquare = 2, kActSin = 3, kActExp = 4 };
struct ActD {
  float d0, d1, d2, d3, d4;
};
__device__ __forceinline__ ActD act_derivs(int act, float z) {
  ActD r;
  if (act == kActTanh) {
    const float t = tanhf(z);
    const float s = 1.f - t * t;          // tanh'
    r.d0 = t;
    r.d1 = s;
    r.d2 = -2.f * t * s;                  // tanh''
    r.d3 = s * (6.f * t * t - 2.f);       // tanh'''
    r.d4 = 8.f * t * s * (2.f - 3.f * t * t);  // tanh''''
  } else if (act == kActSin) {
    float sn, cs;
    sincosf(z, &sn, &cs);
    r.d0 = sn; r.d1 = cs; r.d2 = -sn; r.d3 = -cs; r.d4 = sn;
  } else if (act == kActExp) {
    const float e = expf(z);
    r.d0 = e; r.d1 = e; r.d2 = e; r.d3 = e; r.d4 = e;
  } else if (act == kActSquare) {
    r.d0 = z * z; r.d1 = 2.f * z; r.d2 = 2.f; r.d3 = 0.f; r.d4 = 0.f;
  } else {
    r.d0 = z; r.d1 = 1.f; r.d2 = 0.f; r.d3 = 0.f; r.d4 = 0.f;
  }
  return r;
}

// Kept at 128 bytes: one more 8-byte word changed ptxas's unrolling of the epilogue and cost
// 3-5% of layer time (measured A/B, K=4 and K=2 instances).
struct LayerParams {
  const float* bias;      // [Mpad]
  uint16_t* out;          // [nplanes][rows, ldo] bf16 planes
  int64_t pstride;        // elements between planes
  int ldo;
  int m_tiles;
  int64_t n_points;
  int P;                  // slots per point
  int pts_per_tile;
  int n_mma;              // MMA N, multiple of 16, <= 256
  int k_iters;            // Kpad / kBK
  const float* jet_w;     // K=4: weights of the J jets in the collapsed slot; K=2 if weighted
  int J;                  // K=4: jets; kNest: D; K=2 weighted: directions
  // Direction blocks: a point's directions are split into `blocks` groups of
  // `rb` directions, each propagated as its own slot group [x0; its directions; partial top]
  // ("sub-point"). n_points counts sub-points; sub-point i holds directions
  // (i % blocks) * rb .. +rb-1 of point i / blocks, so its weights start at jw[(i % blocks) * rb].
  int blocks;
  int rb;
  int16_t weighted;       // K=2: collapse sum_r w_r z_{1,r}^2 (directional sums, Eq. 5 with weights)
  int16_t act;            // kAct*
  float* z_out;           // forward, grad mode: the pre-activations z of every slot (fp32) or nullptr
  int ldz;
  int16_t nplanes;        // 3: fp32 mode, 2: fast mode (operand planes read and written)
  int16_t readout;        // last hidden layer: reduce against w_out instead of storing
  const float* z_in;      // kBwd2: this layer's saved pre-activations (fp32)
  int ldzi;
  const float* w_out;     // [Mpad] output-layer weights (zero padded)
  float* partial;         // [n_points, m_tiles, 2]
};
static_assert(sizeof(LayerParams) == 128, "LayerParams grew past 128 bytes (see above)");

template <int NPL>
__device__ __forceinline__ void store_out(const LayerParams& p, size_t idx, float v) {
  ptx::store_planes<NPL>(p.out + idx, p.pstride, v);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One point (sub-point) of one tile, for the feature owned by this thread; jw points at
// the weights of its direction block. TMEM columns
// [tcol, tcol + P) hold z for slots 0..P-1. Writes the output slots (bf16 pairs) or, on
// the readout layer, returns w_out*h0 and w_out*(top) for the reduction.
// part 0: the whole point. A tile holding a single point (P > 128) is split between the
// two epilogue warp groups at a jet boundary `split`: part 1 = the primal and middle slots
// [1, split), part 2 = middle slots [split, ..) and the top; the partial collapsed sum of
// part 1 reaches part 2 through xacc (this thread's slot) and the named barrier bar_id.
// FLAGS (compile time, K=2 only): kFlagWeighted = collapse sum_r w_r z1_r^2 with the smem
// weights; kFlagSaveZ = also store the pre-activations (grad mode). The plain operators
// compile to the loop without either.
constexpr int kFlagWeighted = 1, kFlagSaveZ = 2;
// kFlagWide (plain K=2 only): 4 epilogue warp groups instead of 2, chosen by the host when a
// tile holds >= 8 points (small P: the epilogue, not the MMA, bounds the tile).
constexpr int kFlagWide = 4;
// kFlagNP2: the fast mode's two operand planes (ctm_set_precision); without it three (the
// fp32 mode). The plane count is a compile-time constant of every layer-kernel instance.
constexpr int kFlagNP2 = 8;
// kFlagF16 (K=2 only): the fp16x3 mode: two fp16 planes per operand with power-of-two scales
// (weights per layer, slot blocks per slot type), products p1*p0 + p0*p1 over the whole K,
// then p0*p0. Implies two planes.
constexpr int kFlagF16 = 16;
// kFlagRing7 (plain K=2, MMA N <= 208): a 7-slot operand ring of 29 KB slots instead of 6 x 32 KB
// (one more K block of TMA lookahead)
constexpr int kFlagRing7 = 32;
template <int FLAGS>
__host__ __device__ constexpr int planes_of() {
  return (FLAGS & (kFlagNP2 | kFlagF16)) ? 2 : 3;
}

// fp16x3 scale state of one slot block in device memory: the planes hold fp16 splits of
// v * scale[t], t the slot type (0 primal, 1 first order / K=4 h1, 2 collapsed top, 3 K=4 h2,
// 4 K=4 h3); the block's producer records max |v| per type (float bits, atomicMax) for the
// next layer's bound.
constexpr int kF16Types = 5;
struct F16Rec {
  float scale[kF16Types];
  unsigned maxabs[kF16Types];
};
// per-launch fp16x3 arguments of a layer kernel (zero for the other modes)
struct F16Args {
  const F16Rec* in;   // the B operand's block
  F16Rec* out;        // the output block, or nullptr (readout layer)
  const float* wsc;   // [0] 2^-(sa+11): the weights' factor in the accumulator (seed.cuh split_weights_f16_kernel),
                      // [1] ||W||_inf = max_m sum_k |W[m,k]|
  float s0, s1, s2;   // sup |s|, |s'|, |s''| of the activation
  float s3, s4;       // sup of the third and fourth derivatives (K=4)
  float rw;           // sum_r |w_r| over one sub-point's directions (< 0: from the smem weights)
  int uniform;        // grad mode: one scale for every slot type of the output block (the weight
                      // gradients contract over all slot rows, wgrad.cuh)
  // kBwd2 (the adjoint, fp16x3 training): bounds of the layer's saved pre-activations
  // zb = {max |z1|, max |z_top|} and of the backward seeds bb = {|c| max|gop| max|w_L|,
  // max|gf| max|w_L|, sum_r |w_r|, max_r |w_r|} (f16_bwd_prep_kernel)
  const float* zb;
  const float* bb;
};
// the registers an fp16x3 epilogue thread carries: unscale factors of the accumulator per
// slot type (2^-(sa+11) / scale_in[t]), scales of its output block, running max |output|
struct F16Ctx {
  float us[kF16Types];
  float os[kF16Types];
  float mx[kF16Types];
};
// output scale of a slot type from a bound B on |v|: 2^(14 - e), B = m 2^e, m in [0.5, 1), so
// |v * scale| <= 2^14 < 65504 (fp16 max)
__device__ __forceinline__ float f16_scale_for(float B) {
  if (!(B > 0.f) || !(B < 3.0e38f)) return 1.f;
  int e;
  frexpf(B, &e);
  e = e < -100 ? -100 : (e > 100 ? 100 : e);
  return ldexpf(1.f, 14 - e);
}
// Rigorous bounds of the next block's values from the input block's recorded maxima and the
// layer's ||W||_inf (Eq. 7 / the K=2 rule): |h0| <= s0; |h1_r| <= s1 G M1;
// |top| <= s1 G Mt + s2 Rw (G M1)^2.
__device__ __forceinline__ void f16_out_scales(const F16Args& a, float rw, float* os) {
  const float G = a.wsc[1];
  const float M1 = __uint_as_float(a.in->maxabs[1]), Mt = __uint_as_float(a.in->maxabs[2]);
  const float g1 = G * M1;
  os[0] = f16_scale_for(a.s0);
  os[1] = f16_scale_for(a.s1 * g1);
  os[2] = f16_scale_for(a.s1 * G * Mt + a.s2 * rw * g1 * g1);
  os[3] = os[4] = 1.f;
  if (a.uniform) os[0] = os[1] = os[2] = os[3] = os[4] = fminf(os[0], fminf(os[1], os[2]));
}
// The standard modes (the paper's baselines): per direction / jet, no collapse.
// K=2 pairs: |h1| <= s1 g1, |h2_r| <= s2 g1^2 + s1 g2 (g_k = G M_k, M2 = the input's type-2
// maximum); K=4 jets: |h1| <= s1 g1, |h2| <= s2 g1^2 + s1 g2, |h3| <= s3 g1^3 + 3 s2 g1 g2 +
// s1 g3, |h4| <= s4 g1^4 + 6 s3 g1^2 g2 + 4 s2 g1 g3 + 3 s2 g2^2 + s1 g4 (types 1, 3, 4, 2).
__device__ __forceinline__ void f16_std_scales(const F16Args& a, bool k4, float* os) {
  const float G = a.wsc[1];
  os[0] = f16_scale_for(a.s0);
  if (!k4) {
    const float g1 = G * __uint_as_float(a.in->maxabs[1]), g2 = G * __uint_as_float(a.in->maxabs[2]);
    os[1] = f16_scale_for(a.s1 * g1);
    os[2] = f16_scale_for(a.s2 * g1 * g1 + a.s1 * g2);
    os[3] = os[4] = 1.f;
    return;
  }
  const float g1 = G * __uint_as_float(a.in->maxabs[1]), g2 = G * __uint_as_float(a.in->maxabs[3]),
              g3 = G * __uint_as_float(a.in->maxabs[4]), g4 = G * __uint_as_float(a.in->maxabs[2]);
  os[1] = f16_scale_for(a.s1 * g1);
  os[3] = f16_scale_for(a.s2 * g1 * g1 + a.s1 * g2);
  os[4] = f16_scale_for(a.s3 * g1 * g1 * g1 + 3.f * a.s2 * g1 * g2 + a.s1 * g3);
  os[2] = f16_scale_for(a.s4 * g1 * g1 * g1 * g1 + 6.f * a.s3 * g1 * g1 * g2 + 4.f * a.s2 * g1 * g3 +
                        3.f * a.s2 * g2 * g2 + a.s1 * g4);
}
// The nested rule (epilogue_nested) with ONE scale per block: m = G M bounds every input slot
// value of the layer (M = the input block's max |value| over all slots, maxabs[0]), so
// |g'| <= s1 m, |H'| <= s2 m^2 + s1 m, |L'| <= s3 D m^3 + 3 s2 D m^2 + s1 m,
// |Q'| <= s4 D^2 m^4 + 6 s3 D^2 m^3 + 3 s2 D^2 m^2 + 4 s2 D m^2 + s1 m   (|g|^2 <= D m^2,
// tr H <= D m, g^T H g <= D^2 m^3, |H|_F^2 <= D^2 m^2, g^T L <= D m^2), |h0| <= s0.
__device__ __forceinline__ void f16_nest_scales(const F16Args& a, int D, float* os) {
  const float m = a.wsc[1] * __uint_as_float(a.in->maxabs[0]);
  const float Dm = (float)D * m, m2 = m * m;
  const float b = fmaxf(fmaxf(a.s0, a.s1 * m), fmaxf(a.s2 * m2 + a.s1 * m,
      fmaxf(a.s3 * Dm * m2 + 3.f * a.s2 * Dm * m + a.s1 * m,
            a.s4 * Dm * Dm * m2 + 6.f * a.s3 * Dm * Dm * m + 3.f * a.s2 * Dm * Dm + 4.f * a.s2 * Dm * m + a.s1 * m)));
  const float sc = f16_scale_for(b);
  for (int t = 0; t < kF16Types; ++t) os[t] = sc;
}
// The adjoint of the K=2 rule (epilogue_bwd2) with G = ||W^T||_inf and the input adjoint
// block's maxima Mb[t]: |hb_t| <= G Mb[t] =: H_t (hb = W^T zb per slot), and with Z1, Zt the
// bounds of the saved z1, z_top, R = P - 2 directions, Rw = sum |w_r|, w = max |w_r|:
//   |ztb| <= s1 Ht;  |z1b_r| <= s1 H1 + 2 s2 w Z1 Ht;
//   |z0b| <= s1 H0 + s2 R Z1 H1 + (s2 Zt + s3 Rw Z1^2) Ht.
// One scale for the whole output block (grad mode: uniform, see F16Args).
__device__ __forceinline__ void f16_bwd_scales(const F16Args& a, int R, float* os) {
  const float G = a.wsc[1];
  const float H0 = G * __uint_as_float(a.in->maxabs[0]), H1 = G * __uint_as_float(a.in->maxabs[1]),
              Ht = G * __uint_as_float(a.in->maxabs[2]);
  const float Z1 = a.zb[0], Zt = a.zb[1], Rw = a.bb[2], wm = a.bb[3];
  const float bt = a.s1 * Ht;
  const float b1 = a.s1 * H1 + 2.f * a.s2 * wm * Z1 * Ht;
  const float b0 = a.s1 * H0 + a.s2 * (float)R * Z1 * H1 + (a.s2 * Zt + a.s3 * Rw * Z1 * Z1) * Ht;
  const float sc = f16_scale_for(fmaxf(bt, fmaxf(b1, b0)));
  for (int t = 0; t < kF16Types; ++t) os[t] = sc;
}
// The K=4 rule (cheat-sheet rows k <= 4) with g_k = G M_k the bounds of the
// input jets' coefficients: |h1| <= s1 g1; |h2| <= s2 g1^2 + s1 g2;
// |h3| <= s3 g1^3 + 3 s2 g1 g2 + s1 g3;
// |top| <= Rw (s4 g1^4 + 6 s3 g1^2 g2 + 4 s2 g1 g3 + 3 s2 g2^2) + s1 G Mt.
__device__ __forceinline__ void f16_out_scales4(const F16Args& a, float rw, float* os) {
  const float G = a.wsc[1];
  const float g1 = G * __uint_as_float(a.in->maxabs[1]), g2 = G * __uint_as_float(a.in->maxabs[3]),
              g3 = G * __uint_as_float(a.in->maxabs[4]), gt = G * __uint_as_float(a.in->maxabs[2]);
  os[0] = f16_scale_for(a.s0);
  os[1] = f16_scale_for(a.s1 * g1);
  os[3] = f16_scale_for(a.s2 * g1 * g1 + a.s1 * g2);
  os[4] = f16_scale_for(a.s3 * g1 * g1 * g1 + 3.f * a.s2 * g1 * g2 + a.s1 * g3);
  os[2] = f16_scale_for(rw * (a.s4 * g1 * g1 * g1 * g1 + 6.f * a.s3 * g1 * g1 * g2 + 4.f * a.s2 * g1 * g3 +
                              3.f * a.s2 * g2 * g2) + a.s1 * gt);
}

template <int KORD, int FLAGS = 0>
__device__ __forceinline__ void epilogue_point(const LayerParams& p, uint32_t tcol, int64_t row, int m, float bias,
                                               float wo, const float* jw, int part, int split, float* xacc,
                                               int bar_id, float& fpart, float& opart, F16Ctx* fc = nullptr) {
  constexpr int NPL = planes_of<FLAGS>();
  constexpr bool F16 = (FLAGS & kFlagF16) != 0;  // fp16x3: unscale what is read, scale what is stored
  static_assert(!F16 || KORD == 2 || KORD == 4 || KORD == kBwd2 || KORD == kNest || KORD == kStd2 || KORD == kStd4,
                "fp16x3: an instance without fp16x3 support");
  const int P = p.P;
  const int ld = p.ldo;
  constexpr bool kStd = (KORD == kStd2) || (KORD == kStd4);  // no collapsed top slot
  const int nmid = kStd ? P - 1 : P - 2;  // middle slots are 1 .. nmid
  const int mb = (part == 2) ? split : 1;
  const int me = (part == 1) ? split : nmid + 1;
  // ---- slot 0: the primal; the bias enters here only (affine rule)
  const float z0 = (F16 ? ptx::tmem_ld1(tcol) * fc->us[0] : ptx::tmem_ld1(tcol)) + bias;
  ptx::tmem_ld_wait();
  const ActD A = act_derivs(p.act, z0);
  const float t = A.d0, d1 = A.d1, d2 = A.d2, d3 = A.d3, d4 = A.d4;
  fpart = (part == 2) ? 0.f : wo * t;
  opart = 0.f;
  if (!p.readout && part != 2) {
    if constexpr (F16) {
      uint16_t* const r0 = p.out + (size_t)row * ld + m;
      ptx::store_f16_off(r0, r0 + p.pstride, 0u, t * fc->os[0]);
      fc->mx[0] = fmaxf(fc->mx[0], fabsf(t));
    } else {
      store_out<NPL>(p, (size_t)row * ld + m, t);
    }
  }
  constexpr bool kSaveZ = (FLAGS & kFlagSaveZ) != 0;
  float* zp = kSaveZ ? p.z_out + (size_t)(row + mb) * p.ldz + m : nullptr;
  if (kSaveZ && part != 2) p.z_out[(size_t)row * p.ldz + m] = z0;
  // plane bases of slot mb; the slot after it is a running 32-bit element offset
  uint16_t* const q0 = p.out + (size_t)(row + mb) * ld + m;
  uint16_t* const q1 = q0 + p.pstride;
  uint16_t* const q2 = q1 + p.pstride;
  uint32_t off = 0;
  // ---- middle slots: first-order coefficients (K=2), jets (z1, z2, z3) (K=4), or the
  //      standard-mode pairs (z1_r, z2_r) with no collapse
  float acc = 0.f;  // the collapsed sum over directions (standard: sum_r h2_r at readout)
  int jj = (KORD == 4) ? (mb - 1) / 3 : (KORD == kStd4) ? (mb - 1) / 4 : mb - 1;  // first direction / jet
  // type: the fp16x3 slot type of the stored value (1 first order / h1, 3 h2, 4 h3)
  auto put = [&](float h, int type = 1) {
    if (!p.readout) {
      if constexpr (F16) {
        ptx::store_f16_off(q0, q1, off, h * fc->os[type]);
        fc->mx[type] = fmaxf(fc->mx[type], fabsf(h));
      } else {
        ptx::store_planes_off<NPL>(q0, q1, q2, off, h);
      }
    }
    off += (uint32_t)ld;
  };
  if constexpr (KORD == 4) {
    // jets (z1, z2, z3), read 5 at a time (15 of 16 columns) so each slot's role is a
    // compile-time index in the unrolled loop
    auto jet = [&](float z1, float z2, float z3) {
      if constexpr (F16) {  // fp16x3: the jet's coefficients carry the scales of types 1, 3, 4
        z1 *= fc->us[1];
        z2 *= fc->us[3];
        z3 *= fc->us[4];
      }
      put(d1 * z1, 1);
      put(d2 * z1 * z1 + d1 * z2, 3);
      put(d3 * z1 * z1 * z1 + 3.f * d2 * z1 * z2 + d1 * z3, 4);
      const float nl = d4 * z1 * z1 * z1 * z1 + 6.f * d3 * z1 * z1 * z2 + 4.f * d2 * z1 * z3 + 3.f * d2 * z2 * z2;
      acc = fmaf(jw[jj], nl, acc);
      ++jj;
    };
    const int nj = (me - mb) / 3;
    int j = 0;
    for (; j + 5 <= nj; j += 5) {
      float v[16];
      ptx::tmem_ld16(tcol + (uint32_t)(mb + 3 * j), v);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 5; ++u) jet(v[3 * u], v[3 * u + 1], v[3 * u + 2]);
    }
    for (; j < nj; ++j) {
      float v[4];
      ptx::tmem_ld4(tcol + (uint32_t)(mb + 3 * j), v);
      ptx::tmem_ld_wait();
      jet(v[0], v[1], v[2]);
    }
  } else if constexpr (KORD == kStd4) {
    // standard K=4 mode: per jet (h1, h2, h3, h4), the weighted h4 summed for the readout
    // (cheat-sheet rows k <= 4, per jet); 4 jets per 16 columns
    auto jet4 = [&](float z1, float z2, float z3, float z4) {
      if constexpr (F16) {  // fp16x3: the jet's coefficients carry the scales of types 1, 3, 4, 2
        z1 *= fc->us[1];
        z2 *= fc->us[3];
        z3 *= fc->us[4];
        z4 *= fc->us[2];
      }
      put(d1 * z1, 1);
      put(d2 * z1 * z1 + d1 * z2, 3);
      put(d3 * z1 * z1 * z1 + 3.f * d2 * z1 * z2 + d1 * z3, 4);
      const float h4 = d4 * z1 * z1 * z1 * z1 + 6.f * d3 * z1 * z1 * z2 + 4.f * d2 * z1 * z3 + 3.f * d2 * z2 * z2 +
                       d1 * z4;
      put(h4, 2);
      acc = fmaf(jw[jj], h4, acc);
      ++jj;
    };
    const int nj = (me - mb) / 4;
    int j = 0;
    for (; j + 4 <= nj; j += 4) {
      float v[16];
      ptx::tmem_ld16(tcol + (uint32_t)(mb + 4 * j), v);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 4; ++u) jet4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
    }
    for (; j < nj; ++j) {
      float v[4];
      ptx::tmem_ld4(tcol + (uint32_t)(mb + 4 * j), v);
      ptx::tmem_ld_wait();
      jet4(v[0], v[1], v[2], v[3]);
    }
  } else if constexpr (KORD == kStd2) {
    // standard mode: per direction (h1_r, h2_r) with no collapse, 8 pairs per 16 columns
    auto pair = [&](float z1, float z2) {
      if constexpr (F16) {  // fp16x3: first- and second-order coefficients, types 1 and 2
        z1 *= fc->us[1];
        z2 *= fc->us[2];
      }
      put(d1 * z1, 1);                          // h_{1,r}
      const float h2 = fmaf(d2 * z1, z1, d1 * z2);  // h_{2,r} = tanh'' z1^2 + tanh' z2 (Eq. 1)
      acc += h2;
      put(h2, 2);
    };
    const int np = (me - mb) / 2;
    int j = 0;
    for (; j + 8 <= np; j += 8) {
      float v[16];
      ptx::tmem_ld16(tcol + (uint32_t)(mb + 2 * j), v);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 8; ++u) pair(v[2 * u], v[2 * u + 1]);
    }
    for (; j < np; ++j) {
      float v[2];
      ptx::tmem_ld2(tcol + (uint32_t)(mb + 2 * j), v);
      ptx::tmem_ld_wait();
      pair(v[0], v[1]);
    }
  } else {
    constexpr bool wsum = (FLAGS & kFlagWeighted) != 0;
    auto middle = [&](float z) {
      put(d1 * z);  // h_{1,r} = tanh' z_{1,r}
      if constexpr (wsum)
        acc = fmaf(jw[jj++] * z, z, acc);  // sum_r w_r z_{1,r}^2
      else
        acc = fmaf(z, z, acc);  // sum_r z_{1,r}^2
      if constexpr (kSaveZ) {
        *zp = z;
        zp += p.ldz;
      }
    };
    const int cnt = me - mb;
    const float us1 = F16 ? fc->us[1] : 1.f;
    int s = 0;
    for (; s + 16 <= cnt; s += 16) {
      float v[16];
      ptx::tmem_ld16(tcol + (uint32_t)(mb + s), v);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) middle(F16 ? v[i] * us1 : v[i]);
    }
    const int rem = cnt - s;  // 0..15, warp-uniform
    if (rem > 0) {
      float v[15];
#pragma unroll
      for (int i = 0; i < 15; ++i)
        if (i < rem) v[i] = ptx::tmem_ld1(tcol + (uint32_t)(mb + s + i));
      ptx::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 15; ++i)
        if (i < rem) middle(F16 ? v[i] * us1 : v[i]);
    }
  }
  if (part != 0) {  // part 1 hands its partial collapsed sum to part 2 (one barrier site for both)
    if (part == 1) *xacc = acc;
    asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
    if (part == 1) return;
    acc += *xacc;
  }
  if (kStd) {  // standard mode: the top coefficients are sliced and summed only here
    opart = wo * acc;
    return;
  }
  // ---- slot P-1: the collapsed top, <dh, sum z_K> + the collapsed non-linear terms (Eq. 7)
  const float zt = F16 ? ptx::tmem_ld1(tcol + (uint32_t)(P - 1)) * fc->us[2] : ptx::tmem_ld1(tcol + (uint32_t)(P - 1));
  ptx::tmem_ld_wait();
  const float top = d1 * zt + (KORD == 2 ? d2 * acc : acc);
  if constexpr (kSaveZ) *zp = zt;
  opart = wo * top;
  if (!p.readout) {
    if constexpr (F16) {
      ptx::store_f16_off(q0, q1, off, top * fc->os[2]);
      fc->mx[2] = fmaxf(fc->mx[2], fabsf(top));
    } else {
      ptx::store_planes_off<NPL>(q0, q1, q2, off, top);
    }
  }
}

// The K=2 rule for a point of P <= 16 slots whose 16 columns lie in the accumulator buffer:
// one TMEM load and one wait for the whole point (the general loop waits for the primal,
// the middle slots and the top separately). Same operations in the same order as
// epilogue_point, so the two give identical bits.
template <int FLAGS, int PC = 0>
__device__ __forceinline__ void epilogue_point_small(const LayerParams& p, uint32_t tcol, int64_t row, int m,
                                                     float bias, float wo, const float* jw, float& fpart,
                                                     float& opart, F16Ctx* fc = nullptr) {
  constexpr bool F16 = (FLAGS & kFlagF16) != 0;
  constexpr bool kSaveZ = (FLAGS & kFlagSaveZ) != 0;
  constexpr int NPL = planes_of<FLAGS>();
  constexpr bool wsum = (FLAGS & kFlagWeighted) != 0;
  const int P = PC > 0 ? PC : p.P;  // PC: the slot count as a compile-time constant
  const uint32_t ld = (uint32_t)p.ldo;
  float v[16];
  ptx::tmem_ld16(tcol, v);
  ptx::tmem_ld_wait();
  if constexpr (F16) {
    v[0] *= fc->us[0];
#pragma unroll
    for (int i = 1; i < 16; ++i) v[i] *= (i == P - 1) ? fc->us[2] : fc->us[1];
  }
  const float z0 = v[0] + bias;
  const ActD A = act_derivs(p.act, z0);
  fpart = wo * A.d0;
  // plane bases of the point's slot 0; slot i of plane k is q_k[i * ld]
  uint16_t* const q0 = p.out + (size_t)row * ld + m;
  uint16_t* const q1 = q0 + p.pstride;
  uint16_t* const q2 = q1 + p.pstride;
  float* zp = kSaveZ ? p.z_out + (size_t)row * p.ldz + m : nullptr;
  if constexpr (kSaveZ) zp[0] = z0;
  // one loop per value of p.readout (uniform): no per-store test of the flag
  auto body = [&](auto ro) {
    constexpr bool kRO = decltype(ro)::value;
    // one store: fp16x3 scales by the slot type and records the output's max per type
    auto st = [&](uint32_t off, float h, int type) {
      if constexpr (F16) {
        ptx::store_f16_off(q0, q1, off, h * fc->os[type]);
        fc->mx[type] = fmaxf(fc->mx[type], fabsf(h));
      } else {
        ptx::store_planes_off<NPL>(q0, q1, q2, off, h);
      }
    };
    if (!kRO) st(0u, A.d0, 0);
    float acc = 0.f, zt = 0.f;
#pragma unroll
    for (int i = 1; i < 16; ++i) {
      if (i < P - 1) {
        const float z = v[i];
        if (!kRO) st((uint32_t)i * ld, A.d1 * z, 1);
        if constexpr (wsum)
          acc = fmaf(jw[i - 1] * z, z, acc);
        else
          acc = fmaf(z, z, acc);
        if constexpr (kSaveZ) zp[(size_t)i * p.ldz] = z;
      } else if (i == P - 1) {
        zt = v[i];
      }
    }
    const float top = A.d1 * zt + A.d2 * acc;
    if constexpr (kSaveZ) zp[(size_t)(P - 1) * p.ldz] = zt;
    opart = wo * top;
    if (!kRO) st((uint32_t)(P - 1) * ld, top, 2);
  };
  if (p.readout)
    body(std::true_type{});
  else
    body(std::false_type{});
}

// Nested-Laplacian biharmonic epilogue (kNest) for one point, the whole point in this
// thread (no split). With s = tanh and the slots of the layout above (multivariate chain
// rule for h = s(z)):
//   h_a   = s' g_a
//   H'_ab = s'' g_a g_b + s' H_ab
//   L'_a  = s''' g_a |g|^2 + 2 s'' (H g)_a + s'' g_a tr H + s' L_a
//   Q'    = s'''' |g|^4 + 2 s''' |g|^2 tr H + 4 s''' g^T H g + 2 s'' |H|_F^2 + s'' (tr H)^2
//           + 4 s'' g^T L + s' Q
// (D = 1 gives the K=4 Faa di Bruno row of the cheat sheet.) Register
// arrays are sized kNestMaxD and indexed with compile-time indices under runtime guards.
// fp16x3 (F16): every accumulator column is unscaled by us (uniform over the block's slots),
// every stored value scaled by os and its max |value| recorded in mx[0]
template <int NPL, bool F16 = false>
__device__ __forceinline__ void epilogue_nested(const LayerParams& p, uint32_t tcol, int64_t row, int m, float bias,
                                                float wo, float& fpart, float& opart, F16Ctx* fc = nullptr) {
  const int D = p.J;
  const int ld = p.ldo;
  const float us = F16 ? fc->us[0] : 1.f;
  const float z0 = ptx::tmem_ld1(tcol) * us + bias;
  float g[kNestMaxD];
#pragma unroll
  for (int a = 0; a < kNestMaxD; ++a) g[a] = (a < D) ? ptx::tmem_ld1(tcol + 1u + (uint32_t)a) : 0.f;
  ptx::tmem_ld_wait();
#pragma unroll
  for (int a = 0; a < kNestMaxD; ++a) g[a] *= us;
  auto sto = [&](const LayerParams& pp, size_t idx, float v) {
    if constexpr (F16) {
      ptx::store_f16_off(pp.out + idx, pp.out + idx + pp.pstride, 0u, v * fc->os[0]);
      fc->mx[0] = fmaxf(fc->mx[0], fabsf(v));
    } else {
      ctm::store_out<NPL>(pp, idx, v);
    }
  };
  const ActD A = act_derivs(p.act, z0);
  const float t = A.d0, d1 = A.d1, d2 = A.d2, d3 = A.d3, d4 = A.d4;
  const bool store = !p.readout;
  fpart = wo * t;
  if (store) sto(p, (size_t)row * ld + m, t);
  float gg = 0.f;
#pragma unroll
  for (int a = 0; a < kNestMaxD; ++a)
    if (a < D) {
      gg = fmaf(g[a], g[a], gg);
      if (store) sto(p, (size_t)(row + 1 + a) * ld + m, d1 * g[a]);
    }
  // Hessian slots, one packed row at a time
  float hg[kNestMaxD];
#pragma unroll
  for (int a = 0; a < kNestMaxD; ++a) hg[a] = 0.f;
  float trH = 0.f, HF = 0.f;
  int slot = 1 + D;
#pragma unroll
  for (int a = 0; a < kNestMaxD; ++a) {
    if (a < D) {
      float hr[kNestMaxD];
#pragma unroll
      for (int b = a; b < kNestMaxD; ++b) hr[b] = (b < D) ? ptx::tmem_ld1(tcol + (uint32_t)(slot + b - a)) : 0.f;
      ptx::tmem_ld_wait();
#pragma unroll
      for (int b = a; b < kNestMaxD; ++b) hr[b] *= us;
#pragma unroll
      for (int b = a; b < kNestMaxD; ++b)
        if (b < D) {
          const float h = hr[b];
          if (store)
            sto(p, (size_t)(row + slot + b - a) * ld + m, fmaf(d2 * g[a], g[b], d1 * h));
          if (b == a) {
            trH += h;
            HF = fmaf(h, h, HF);
            hg[a] = fmaf(h, g[a], hg[a]);
          } else {
            HF = fmaf(2.f * h, h, HF);
            hg[a] = fmaf(h, g[b], hg[a]);
            hg[b] = fmaf(h, g[a], hg[b]);
          }
        }
      slot += D - a;
    }
  }
  // gradient-of-Laplacian slots and the top
  float Lv[kNestMaxD];
#pragma unroll
  for (int a = 0; a < kNestMaxD; ++a) Lv[a] = (a < D) ? ptx::tmem_ld1(tcol + (uint32_t)(slot + a)) : 0.f;
  float zq = ptx::tmem_ld1(tcol + (uint32_t)(slot + D));
  ptx::tmem_ld_wait();
  zq *= us;
#pragma unroll
  for (int a = 0; a < kNestMaxD; ++a) Lv[a] *= us;
  float gL = 0.f, gHg = 0.f;
#pragma unroll
  for (int a = 0; a < kNestMaxD; ++a)
    if (a < D) {
      gL = fmaf(g[a], Lv[a], gL);
      gHg = fmaf(g[a], hg[a], gHg);
      if (store) {
        const float v = d3 * g[a] * gg + 2.f * d2 * hg[a] + d2 * g[a] * trH + d1 * Lv[a];
        sto(p, (size_t)(row + slot + a) * ld + m, v);
      }
    }
  const float q = d4 * gg * gg + 2.f * d3 * gg * trH + 4.f * d3 * gHg + 2.f * d2 * HF + d2 * trH * trH +
                  4.f * d2 * gL + d1 * zq;
  opart = wo * q;
  if (store) sto(p, (size_t)(row + slot + D) * ld + m, q);
}

// The same rule with D known at compile time (D <= 8, P <= 54): the point's P columns
// are read with one burst of x16/x8/x4/x2/x1 loads and a single wait, and every slot
// index is a constant, so the whole point lives in registers.
template <int D, int NPL, bool F16 = false>
__device__ __forceinline__ void epilogue_nested_d(const LayerParams& p, uint32_t tcol, int64_t row, int m,
                                                  float bias, float wo, float& fpart, float& opart,
                                                  F16Ctx* fc = nullptr) {
  constexpr int T = D * (D + 1) / 2;
  constexpr int P = 2 + 2 * D + T;
  constexpr int oH = 1 + D, oL = 1 + D + T;
  float v[P];
  ptx::tmem_ld_cols<P>(tcol, v);
  ptx::tmem_ld_wait();
  if constexpr (F16) {
#pragma unroll
    for (int i = 0; i < P; ++i) v[i] *= fc->us[0];
  }
  const int ld = p.ldo;
  const ActD A = act_derivs(p.act, v[0] + bias);
  const float t = A.d0, d1 = A.d1, d2 = A.d2, d3 = A.d3, d4 = A.d4;
  const float* g = v + 1;
  float gg = 0.f, trH = 0.f, HF = 0.f, gL = 0.f, gHg = 0.f;
  float hg[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    gg = fmaf(g[a], g[a], gg);
    gL = fmaf(g[a], v[oL + a], gL);
    hg[a] = 0.f;
  }
  {
    int k = oH;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = a; b < D; ++b, ++k) {
        const float h = v[k];
        if (b == a) {
          trH += h;
          HF = fmaf(h, h, HF);
          hg[a] = fmaf(h, g[a], hg[a]);
        } else {
          HF = fmaf(2.f * h, h, HF);
          hg[a] = fmaf(h, g[b], hg[a]);
          hg[b] = fmaf(h, g[a], hg[b]);
        }
      }
  }
#pragma unroll
  for (int a = 0; a < D; ++a) gHg = fmaf(g[a], hg[a], gHg);
  const float q = d4 * gg * gg + 2.f * d3 * gg * trH + 4.f * d3 * gHg + 2.f * d2 * HF + d2 * trH * trH +
                  4.f * d2 * gL + d1 * v[P - 1];
  fpart = wo * t;
  opart = wo * q;
  if (p.readout) return;
  uint16_t* po = p.out + (size_t)row * ld + m;
  auto put = [&](size_t off, float v) {
    if constexpr (F16) {
      ptx::store_f16_off(po + off, po + off + p.pstride, 0u, v * fc->os[0]);
      fc->mx[0] = fmaxf(fc->mx[0], fabsf(v));
    } else {
      ptx::store_planes<NPL>(po + off, p.pstride, v);
    }
  };
  put(0, t);
#pragma unroll
  for (int a = 0; a < D; ++a) put((size_t)(1 + a) * ld, d1 * g[a]);
  {
    int k = oH;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = a; b < D; ++b, ++k) put((size_t)k * ld, fmaf(d2 * g[a], g[b], d1 * v[k]));
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
    put((size_t)(oL + a) * ld, d3 * g[a] * gg + 2.f * d2 * hg[a] + d2 * g[a] * trH + d1 * v[oL + a]);
  put((size_t)(P - 1) * ld, q);
}

template <int NPL, bool F16 = false>
__device__ __forceinline__ void epilogue_nested_any(const LayerParams& p, uint32_t tcol, int64_t row, int m,
                                                    float bias, float wo, float& fpart, float& opart,
                                                    F16Ctx* fc = nullptr) {
  switch (p.J) {
    case 1: epilogue_nested_d<1, NPL, F16>(p, tcol, row, m, bias, wo, fpart, opart, fc); break;
    case 2: epilogue_nested_d<2, NPL, F16>(p, tcol, row, m, bias, wo, fpart, opart, fc); break;
    case 3: epilogue_nested_d<3, NPL, F16>(p, tcol, row, m, bias, wo, fpart, opart, fc); break;
    case 4: epilogue_nested_d<4, NPL, F16>(p, tcol, row, m, bias, wo, fpart, opart, fc); break;
    case 5: epilogue_nested_d<5, NPL, F16>(p, tcol, row, m, bias, wo, fpart, opart, fc); break;
    case 6: epilogue_nested_d<6, NPL, F16>(p, tcol, row, m, bias, wo, fpart, opart, fc); break;
    case 7: epilogue_nested_d<7, NPL, F16>(p, tcol, row, m, bias, wo, fpart, opart, fc); break;
    case 8: epilogue_nested_d<8, NPL, F16>(p, tcol, row, m, bias, wo, fpart, opart, fc); break;
    default: epilogue_nested<NPL, F16>(p, tcol, row, m, bias, wo, fpart, opart, fc);
  }
}

// Backward of the K=2 collapsed tanh rule (kBwd2), for one point and the feature owned
// by this thread. The accumulator holds the adjoints of the layer's OUTPUT slots,
// (h0b, h1b_r, tb) = B_bar[slot] = (Z_bar_next W)[slot], computed by the mainloop with
// A = W^T; the saved pre-activations z (p.z_in, fp32) give the forward rule
//   h0 = s(z0), h1_r = s'(z0) z1_r, top = s'(z0) zt + s''(z0) sum_r w_r z1_r^2
// whose transpose is
//   zt_bar  = s' tb
//   z1_bar_r = s' h1b_r + 2 s'' w_r z1_r tb
//   z0_bar  = s' h0b + s'' sum_r z1_r h1b_r + (s'' zt + s''' sum_r w_r z1_r^2) tb
// (w_r = 1 unless p.weighted). Writes Z_bar of this layer as bf16 pairs.
// kB: slots per TMEM load / z-load batch (16; 8 keeps the register count of the 4-group
// adjoint instance low)
template <int kB, int NPL, bool F16 = false>
__device__ __forceinline__ void epilogue_bwd2(const LayerParams& p, uint32_t tcol, int64_t row, int m,
                                              const float* jw, F16Ctx* fc = nullptr) {
  // fp16x3 (F16): the accumulator carries the weights' and the input adjoint block's scales
  // (us, uniform over the slot types in grad mode); outputs are stored scaled by os and their
  // maxima recorded per slot type (0 z0b, 1 z1b, 2 ztb) for the next layer's bound
  const int P = p.P;
  const int ld = p.ldo;
  const uint32_t ldz = (uint32_t)p.ldzi;  // slot offsets are 32-bit (one wide multiply-add per address)
  const float* zr = p.z_in + (size_t)row * ldz + m;
  float hb0 = ptx::tmem_ld1(tcol);
  float tb = ptx::tmem_ld1(tcol + (uint32_t)(P - 1));
  const float z0 = zr[0];
  const float zt = zr[(uint32_t)(P - 1) * ldz];
  ptx::tmem_ld_wait();
  float us1 = 1.f;
  if constexpr (F16) {
    hb0 *= fc->us[0];
    tb *= fc->us[2];
    us1 = fc->us[1];
  }
  const ActD A = act_derivs(p.act, z0);
  const float two_s2_tb = 2.f * A.d2 * tb;
  const bool wsum = p.weighted;
  float szh = 0.f, szz = 0.f;
  uint16_t* const q0 = p.out + (size_t)(row + 1) * ld + m;  // plane bases of slot 1
  uint16_t* const q1 = q0 + p.pstride;
  uint16_t* const q2 = q1 + p.pstride;
  uint32_t off = 0;
  const int nmid = P - 2;
  int s = 0;
  auto put = [&](float v, int type) {
    if constexpr (F16) {
      ptx::store_f16_off(q0, q1, off, v * fc->os[type]);
      fc->mx[type] = fmaxf(fc->mx[type], fabsf(v));
    } else {
      ptx::store_planes_off<NPL>(q0, q1, q2, off, v);
    }
  };
  auto one = [&](float hb, float z1, int r) {
    if constexpr (F16) hb *= us1;
    const float w = wsum ? jw[r] : 1.f;
    szh = fmaf(z1, hb, szh);
    szz = fmaf(w * z1, z1, szz);
    put(fmaf(A.d1, hb, w * two_s2_tb * z1), 1);
    off += (uint32_t)ld;
  };
  for (; s + kB <= nmid; s += kB) {
    float v[kB], z[kB];
    ptx::tmem_ld_cols<kB>(tcol + (uint32_t)(1 + s), v);
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      z[i] = zr[(uint32_t)(1 + s + i) * ldz];
    }
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < kB; ++i) one(v[i], z[i], s + i);
  }
  const int rem = nmid - s;
  if (rem > 0) {
    float v[kB - 1], z[kB - 1];
#pragma unroll
    for (int i = 0; i < kB - 1; ++i)
      if (i < rem) {
        v[i] = ptx::tmem_ld1(tcol + (uint32_t)(1 + s + i));
        z[i] = zr[(uint32_t)(1 + s + i) * ldz];
      }
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < kB - 1; ++i)
      if (i < rem) one(v[i], z[i], s + i);
  }
  put(A.d1 * tb, 2);  // slot P-1
  const float z0b = A.d1 * hb0 + A.d2 * szh + (A.d2 * zt + A.d3 * szz) * tb;
  if constexpr (F16) {
    uint16_t* const r0 = p.out + (size_t)row * ld + m;
    ptx::store_f16_off(r0, r0 + p.pstride, 0u, z0b * fc->os[0]);
    fc->mx[0] = fmaxf(fc->mx[0], fabsf(z0b));
  } else {
    store_out<NPL>(p, (size_t)row * ld + m, z0b);
  }
}

// The k-th tile of CTA pair `pair`: tile t = pair + k * npairs, feature pair t % m_pairs of
// point group t / m_pairs. Consecutive tiles run on consecutive pairs at the same time, so
// the m_pairs feature tiles of a point group read its B operand together: one HBM read,
// the other reads hit L2 (ncu, C1 fp32 mode: layer-2 DRAM reads 7.8 -> 3.9 GB, layer time
// -7%, against running a group's feature tiles back to back on one pair, whose re-reads
// were evicted by the output writes in between). Returns false past the pair's last tile.
__device__ __forceinline__ bool tile_of(int64_t k, int pair, int npairs, int m_pairs, int64_t n_tiles, int64_t& n,
                                        int& m) {
  const int64_t tile = pair + k * npairs;
  n = tile / m_pairs;
  m = (int)(tile % m_pairs);
  return n < n_tiles;
}

// Persistent CTA PAIRS (cluster of 2, cta_group::2): each pair owns an M = 256 feature tile
// (CTA rank r holds features m0 + 128 r .. +127 of A = W and, in its TMEM, the matching
// accumulator lanes) and the N slots of pts_per_tile points (CTA rank r holds B rows
// r*N/2 .. +N/2-1). The pair's leader issues tcgen05.mma.cta_group::2; the tensor cores
// of both SMs read the two B halves from both CTAs' smem, so each SM stages half of B
// (less L2 -> SM traffic and fewer smem operand reads per useful FLOP than one CTA per tile).
// Pairs loop over tiles in the order of tile_of(). Warp roles, in BOTH CTAs:
//   warp 0   TMA producer: its A half and B half of each (K block, plane) into a kSlots-deep
//            ring of plane slots; the transaction bytes of both CTAs are counted on the
//            LEADER's full_bar (schedule: for_each_group below);
//   warp 1   leader only: MMA issuer (one thread), the bf16 plane products of the
//            precision mode into one of two TMEM accumulators; commits multicast to both
//            CTAs (empty_bar per slot, tmem_full);
//   warps 2-9 epilogue on this CTA's 128 accumulator lanes; releases a buffer with a
//            remote arrive on the leader's tmem_empty (8 warps x 2 CTAs).
// The operand schedule of one tile, as groups of consecutive ring slots:
//   fast mode (2 planes):  K block kb -> slots {p0, p1}; per 16-K step p1*p0, p0*p1, p0*p0;
//   fp32 mode (3 planes):  phase 1, K block kb -> slots {p0, p1, p2}; per 16-K step
//                          p2*p0, p1*p1, p0*p2, p1*p0, p0*p1 (the corrections, ~2^-8 of the
//                          result); phase 2, K block kb -> slot {p0}; per 16-K step p0*p0.
// The whole-K correction pass first keeps the accumulator small while the ~5K/16 correction
// MMAs round into it, so the round-toward-zero accumulation of the tensor cores costs what
// K/16 plain MMAs cost (scripts/emulate_schemes.py). f(phase, kb, nslots) per group.
// fp16x3 mode (2 planes, two phases): phase 1 {p0, p1} with p1*p0, p0*p1; phase 2 {p0}, p0*p0.
template <class F>
__device__ __forceinline__ void for_each_group(int nplanes, bool two_phase, int k_iters, F&& f) {
  for (int kb = 0; kb < k_iters; ++kb) f(0, kb, nplanes);
  if (nplanes == 3 || two_phase)
    for (int kb = 0; kb < k_iters; ++kb) f(1, kb, 1);
}

// Epilogue warp groups (4 warps each, one per TMEM lane quadrant) of a kernel instance. The
// plain K=2 rule is light enough to run with 4 groups (576 threads within the 113-register
// budget), which doubles the epilogue's point throughput when many small points share a
// tile (randomized S=8: +15%); with 4 points per tile (C1) 2 groups are faster.
template <int KORD, int FLAGS>
__host__ __device__ constexpr int epi_groups() {
  // the adjoint epilogue is latency-bound on its saved-Z loads: 4 groups (8-slot batches,
  // 96 registers, no spills) take 8% less time than 2 (measured)
  if (KORD == kBwd2) return 4;
  return (FLAGS & kFlagWide) ? 4 : 2;
}
template <int KORD, int FLAGS>
__host__ __device__ constexpr int layer_threads() {
  return 64 + 128 * epi_groups<KORD, FLAGS>();
}

template <int KORD, int FLAGS = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(layer_threads<KORD, FLAGS>(), 1)
    jet_layer_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const LayerParams p, const F16Args f16) {
  constexpr int NS = (FLAGS & kFlagRing7) ? kSlots7 : kSlots;        // ring slots
  constexpr int SB = (FLAGS & kFlagRing7) ? kSlotBytes7 : kSlotBytes;  // bytes per slot
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + NS * SB);
  uint64_t* empty_bar = full_bar + NS;
  uint64_t* tmem_full_bar = empty_bar + NS;    // [2]
  uint64_t* tmem_empty_bar = tmem_full_bar + 2;    // [2] (used in the leader)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty_bar + 2);
  float* red = reinterpret_cast<float*>(smem + NS * SB + 256);  // [4][kMaxPtsPerTile][2]
  float* jw = red + 4 * kMaxPtsPerTile * 2;                                    // [kMaxJets]
  float* xacc = jw + kMaxW;                                                 // [2][128] split-point partials

  constexpr int EG = epi_groups<KORD, FLAGS>();
  constexpr int NPL = planes_of<FLAGS>();  // operand planes read and written
  constexpr bool F16 = (FLAGS & kFlagF16) != 0;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int m_pairs = p.m_tiles >> 1;
  const int64_t n_tiles = (p.n_points + p.pts_per_tile - 1) / p.pts_per_tile;
  const int half_n = p.n_mma >> 1;
  const uint32_t b_bytes = (uint32_t)half_n * kBK * 2;  // this CTA's B half of one plane

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tmem_full_bar[b], 1);
      ptx::mbar_init(&tmem_empty_bar[b], 8 * EG);  // 4 EG epilogue warps in each CTA of the pair
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair<kTmemCols>(tmem_slot);
  if (KORD == 4 || KORD == kStd4 || p.weighted)  // all blocks' weights; a padded last block reads zeros
    for (int j = threadIdx.x; j < p.blocks * p.rb; j += blockDim.x) jw[j] = (j < p.J) ? p.jet_w[j] : 0.f;
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barrier inits and TMEM allocation visible to the pair
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: the prologue above overlaps the previous kernel's tail; everything below reads
  // its output (B operands via TMA) or overwrites the buffer it read, so wait for it here
  ptx::pdl_launch_dependents();
  ptx::pdl_wait_prior();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      uint32_t it = 0;
      int64_t nt;
      int mp;
      for (int64_t k = 0; tile_of(k, pair, npairs, m_pairs, n_tiles, nt, mp); ++k) {
        const int m0 = mp * (2 * kBM) + (int)rank * kBM;
        const int32_t row0 = (int32_t)(nt * p.pts_per_tile * p.P) + (int32_t)rank * half_n;
        for_each_group(NPL, F16, p.k_iters, [&](int phase, int kb, int nslots) {
          for (int pl = 0; pl < nslots; ++pl, ++it) {
            const uint32_t s = it % NS;
            const uint32_t ph = (it / NS) & 1u;
            {
              STAT_T0();
              ptx::mbar_wait(&empty_bar[s], ph ^ 1u);
              STAT_ADD(0);  // producer waits for a free slot
            }
            uint8_t* st = smem + s * SB;
            if (rank == 0) ptx::mbar_arrive_expect_tx(&full_bar[s], 2u * ((uint32_t)kATileBytes + b_bytes));
            const int k0 = kb * kBK;
            // fp16x3 phase 2: p0 of B with the weights' p0 * 2^11 (plane 2), the scale of the corrections
            ptx::tma_load_3d_pair(st, &tmA, &full_bar[s], k0, m0, (F16 && phase == 1) ? 2 : pl);
            ptx::tma_load_3d_pair(st + kATileBytes, &tmB, &full_bar[s], k0, row0, pl);
          }
        });
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader warp, one elected lane)
    // The whole warp runs the schedule (waits, descriptor arithmetic in uniform registers);
    // one elected lane issues. A lane-0-only branch made every MMA a divergent R2UR loop and
    // left the tensor pipe waiting on the issuing thread (STATS build: issuer busy 89%).
    if (rank == 0) {
#ifdef CTM_EXP_STATS
      const long long tstart = clock64();
#endif
      const uint32_t idesc = F16 ? ptx::idesc_f16(2 * kBM, (uint32_t)p.n_mma) : ptx::idesc_bf16(2 * kBM, (uint32_t)p.n_mma);
      // K-major SW128 descriptor of slot 0's A tile (slot s: + s * SB >> 4)
      const uint64_t desc0 = ptx::smem_desc_kmajor(ptx::smem_u32(smem), kSwSBO, kSwLayout);
      uint32_t it = 0, local = 0;
      int64_t nt;
      int mp;
      for (; tile_of(local, pair, npairs, m_pairs, n_tiles, nt, mp); ++local) {
        const uint32_t buf = local & 1u;
        const uint32_t use = local >> 1;
        {
          STAT_T0();
          ptx::mbar_wait(&tmem_empty_bar[buf], (use & 1u) ^ 1u);
          if (lane == 0) STAT_ADD(1);  // MMA waits for the epilogue to free an accumulator
        }
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * (kTmemCols / 2);
        uint32_t acc = 0;  // the tile's first MMA overwrites the accumulator
        for_each_group(NPL, F16, p.k_iters, [&](int phase, int, int nslots) {
          for (int pl = 0; pl < nslots; ++pl) {
            STAT_T0();
            ptx::mbar_wait(&full_bar[(it + pl) % NS], ((it + pl) / NS) & 1u);
            if (lane == 0) STAT_ADD(2);  // MMA waits for TMA
          }
          ptx::tc_fence_after();
          // descriptors of plane i of this group (A at the slot, B at +kATileBytes); the
          // start-address field is addr >> 4 in the low bits, so a K step of 32 bytes adds 2
          // (the single issuing thread must keep up with one MMA per ~100 tensor cycles)
          constexpr uint64_t kS = SB >> 4;
          const uint64_t dA0 = desc0 + (it % NS) * kS, dA1 = desc0 + ((it + 1) % NS) * kS,
                         dA2 = desc0 + ((it + 2) % NS) * kS;
          constexpr uint64_t kB = kATileBytes >> 4;
          if (ptx::elect_one()) {
#pragma unroll
          for (int ks = 0; ks < kBK / 16; ++ks) {  // bf16 MMA K = 16 (32 bytes)
            const uint64_t o = 2u * ks;
            if (nslots == 2) {  // fast mode: + p0*p0 here; fp16x3: p0*p0 in phase 2
              ptx::mma_bf16_pair(d_tmem, dA1 + o, dA0 + kB + o, idesc, acc);
              ptx::mma_bf16_pair(d_tmem, dA0 + o, dA1 + kB + o, idesc, 1u);
              if (!F16) ptx::mma_bf16_pair(d_tmem, dA0 + o, dA0 + kB + o, idesc, 1u);
            } else if (nslots == 3) {
              ptx::mma_bf16_pair(d_tmem, dA2 + o, dA0 + kB + o, idesc, acc);
              ptx::mma_bf16_pair(d_tmem, dA1 + o, dA1 + kB + o, idesc, 1u);
              ptx::mma_bf16_pair(d_tmem, dA0 + o, dA2 + kB + o, idesc, 1u);
              ptx::mma_bf16_pair(d_tmem, dA1 + o, dA0 + kB + o, idesc, 1u);
              ptx::mma_bf16_pair(d_tmem, dA0 + o, dA1 + kB + o, idesc, 1u);
            } else {
              ptx::mma_bf16_pair(d_tmem, dA0 + o, dA0 + kB + o, idesc, acc);
            }
            acc = 1u;
          }
          for (int pl = 0; pl < nslots; ++pl)  // both CTAs' slots are free once these retire
            ptx::mma_commit_pair(&empty_bar[(it + pl) % NS]);
          }
          __syncwarp();
          acc = 1u;
          it += nslots;
          (void)phase;
        });
        if (ptx::elect_one()) ptx::mma_commit_pair(&tmem_full_bar[buf]);  // both CTAs' accumulator halves complete
        __syncwarp();
      }
#ifdef CTM_EXP_STATS
      if (lane == 0) {
        g_stats[blockIdx.x][3] += clock64() - tstart;  // MMA issuer lifetime
        g_stats[blockIdx.x][7] += local;               // tiles
      }
#endif
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9, both CTAs)
    const int q = warp & 3;
    const int g = (warp - 2) >> 2;
    // split of a single point's middle slots between the groups, at a unit boundary
    const int unit = (KORD == 4) ? 3 : (KORD == kStd2) ? 2 : (KORD == kStd4) ? 4 : 1;
    const int nunits = ((KORD == kStd2 || KORD == kStd4) ? p.P - 1 : p.P - 2) / unit;
    const int split = 1 + (nunits / 2) * unit;
    const int m_local = q * 32 + lane;
    // fp16x3: the input block's unscale factors and this layer's output scales (every CTA
    // computes the same values from the same device data; CTA 0 publishes them)
    F16Ctx fcx{};
    if constexpr (F16) {
      const float wsi = f16.wsc[0];
#pragma unroll
      for (int t = 0; t < kF16Types; ++t) {
        fcx.us[t] = wsi / f16.in->scale[t];
        fcx.mx[t] = 0.f;
      }
      if (f16.out) {
        float rw = f16.rw;
        if (rw < 0.f) {  // weighted sums: the largest sum |w_r| over the direction blocks
          rw = 0.f;
          for (int b = 0; b < p.blocks; ++b) {
            float sb = 0.f;
            for (int j = 0; j < p.rb; ++j) sb += fabsf(jw[b * p.rb + j]);
            rw = fmaxf(rw, sb);
          }
        }
        if (KORD == 4)
          f16_out_scales4(f16, rw, fcx.os);
        else if (KORD == kBwd2)
          f16_bwd_scales(f16, p.P - 2, fcx.os);
        else if (KORD == kNest)
          f16_nest_scales(f16, p.J, fcx.os);
        else if (KORD == kStd2 || KORD == kStd4)
          f16_std_scales(f16, KORD == kStd4, fcx.os);
        else
          f16_out_scales(f16, rw, fcx.os);
        if (blockIdx.x == 0 && threadIdx.x == 64)
          for (int t = 0; t < kF16Types; ++t) f16.out->scale[t] = fcx.os[t];
      }
    }
    F16Ctx* const fc = F16 ? &fcx : nullptr;
    uint32_t local = 0;
    int64_t n_tile;
    int mp;
    for (; tile_of(local, pair, npairs, m_pairs, n_tiles, n_tile, mp); ++local) {
      const uint32_t buf = local & 1u;
      const uint32_t use = local >> 1;
      const int m_tile = mp * 2 + (int)rank;  // 128-feature tile of this CTA
      const int64_t row0 = n_tile * p.pts_per_tile * p.P;
      const int m = m_tile * kBM + m_local;
      const float bias = p.bias ? p.bias[m] : 0.f;
      const float wo = p.readout ? p.w_out[m] : 0.f;
      // direction block of the tile's first sub-point (weights offset jbase, see LayerParams)
      constexpr bool kW = (KORD == 4) || (KORD == kStd4) || (FLAGS & kFlagWeighted) != 0;  // instances reading jw
      const int blk0 = (kW && p.blocks > 1) ? (int)((n_tile * p.pts_per_tile) % p.blocks) : 0;
      const int64_t pts_left = p.n_points - n_tile * p.pts_per_tile;
      const int npts = (int)(pts_left < p.pts_per_tile ? pts_left : p.pts_per_tile);
      {
        STAT_T0();
        ptx::mbar_wait(&tmem_full_bar[buf], use & 1u);
        if (warp == 2 && lane == 0) STAT_ADD(4);  // epilogue waits for an accumulator
      }
#ifdef CTM_EXP_STATS
      const long long tw_ = clock64();
#endif
      ptx::tc_fence_after();
      const uint32_t tbase = tmem_base + buf * (kTmemCols / 2) + ((uint32_t)(q * 32) << 16);
      if (KORD == kBwd2) {
        for (int pt = g; pt < npts; pt += EG)
          epilogue_bwd2<EG == 4 ? 8 : 16, NPL, F16>(p, tbase + (uint32_t)(pt * p.P), row0 + (int64_t)pt * p.P, m, jw,
                                                    fc);
      } else if (KORD == kNest) {
        // nested biharmonic: a point is never split; with one point per tile (D >= 14)
        // only warp group 0 works on it
        for (int pt = g; pt < npts; pt += EG) {
          float fpart, opart;
          epilogue_nested_any<NPL, F16>(p, tbase + (uint32_t)(pt * p.P), row0 + (int64_t)pt * p.P, m, bias, wo,
                                        fpart, opart, fc);
          if (p.readout) {
            fpart = warp_sum(fpart);
            opart = warp_sum(opart);
            if (lane == 0) {
              red[(q * kMaxPtsPerTile + pt) * 2 + 0] = fpart;
              red[(q * kMaxPtsPerTile + pt) * 2 + 1] = opart;
            }
          }
        }
      } else if (p.pts_per_tile == 1) {
        // one point per tile: warp groups 0 and 1 share it (split at a jet / pair boundary)
        if (g < 2) {
          float fpart, opart;
          const int jbase = blk0 * p.rb;  // one sub-point per tile
          epilogue_point<KORD, FLAGS>(p, tbase, row0, m, bias, wo, jw + jbase, g + 1, split,
                                      xacc + (local & 1u) * kBM + m_local, 2 + q, fpart, opart, fc);
          if (p.readout) {
            const float v = warp_sum(g == 0 ? fpart : opart);
            if (lane == 0) red[(q * kMaxPtsPerTile + 0) * 2 + g] = v;
          }
        }
      } else {
        for (int pt = g; pt < npts; pt += EG) {
          float fpart, opart;
          const int jbase = (kW && p.blocks > 1) ? ((blk0 + pt) % p.blocks) * p.rb : 0;
          // (the plain K=2 instance runs only with < 8 points per tile, i.e. P > 28: no small path)
          constexpr bool kSmall = (KORD == 2) && ((FLAGS & ~kFlagNP2) != 0);
          if (kSmall && p.P <= 16 && pt * p.P + 16 <= kMaxN) {
            // P <= 12 as a compile-time constant: no runtime slot guards in the unrolled
            // loop (the epilogue is issue-bound there: S=4 +6%, S=8 +1.6%; P = 13..16 gained
            // nothing measurable and keep the runtime-P instance)
            const uint32_t tc = tbase + (uint32_t)(pt * p.P);
            const int64_t rw = row0 + (int64_t)pt * p.P;
            switch (p.P) {
#define CTM_SMALL_CASE(n) \
  case n: epilogue_point_small<FLAGS, n>(p, tc, rw, m, bias, wo, jw + jbase, fpart, opart, fc); break;
              CTM_SMALL_CASE(3) CTM_SMALL_CASE(4) CTM_SMALL_CASE(5) CTM_SMALL_CASE(6) CTM_SMALL_CASE(7)
              CTM_SMALL_CASE(8) CTM_SMALL_CASE(9) CTM_SMALL_CASE(10) CTM_SMALL_CASE(11) CTM_SMALL_CASE(12)
#undef CTM_SMALL_CASE
              default: epilogue_point_small<FLAGS>(p, tc, rw, m, bias, wo, jw + jbase, fpart, opart, fc); break;
            }
          } else
            epilogue_point<KORD, FLAGS>(p, tbase + (uint32_t)(pt * p.P), row0 + (int64_t)pt * p.P, m, bias, wo,
                                        jw + jbase, 0, 0, nullptr, 0, fpart, opart, fc);
          if (p.readout) {
            fpart = warp_sum(fpart);
            opart = warp_sum(opart);
            if (lane == 0) {
              red[(q * kMaxPtsPerTile + pt) * 2 + 0] = fpart;
              red[(q * kMaxPtsPerTile + pt) * 2 + 1] = opart;
            }
          }
        }
      }
      // every epilogue warp of both CTAs releases the buffer once per tile (leader's barrier)
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_remote(&tmem_empty_bar[buf], 0);
#ifdef CTM_EXP_STATS
      if (lane == 0) atomicAdd(&g_stats[blockIdx.x][5 + (warp == 2 ? 0 : 1)], (unsigned long long)(clock64() - tw_));
#endif
      if (p.readout) {
        asm volatile("bar.sync 1, %0;" ::"r"(128 * EG) : "memory");  // the epilogue warps only
        for (int j = threadIdx.x - 64; j < npts * 2; j += 128 * EG) {
          const int pj = j >> 1, comp = j & 1;
          const float s = red[(0 * kMaxPtsPerTile + pj) * 2 + comp] + red[(1 * kMaxPtsPerTile + pj) * 2 + comp] +
                          red[(2 * kMaxPtsPerTile + pj) * 2 + comp] + red[(3 * kMaxPtsPerTile + pj) * 2 + comp];
          const int64_t n = n_tile * p.pts_per_tile + pj;
          p.partial[(n * p.m_tiles + m_tile) * 2 + comp] = s;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(128 * EG) : "memory");  // red[] is reused by the next tile
      }
    }
    if constexpr (F16) {  // this thread's output maxima per slot type into the block's record
      if (f16.out) {
#pragma unroll
        for (int t = 0; t < ((KORD == 4 || KORD == kStd4) ? kF16Types : 3); ++t) {
          float v = fcx.mx[t];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
          if (lane == 0 && v > 0.f) atomicMax(&f16.out->maxabs[t], __float_as_uint(v));
        }
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // no CTA of the pair touches TMEM or the peer's barriers any more
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair<kTmemCols>(tmem_base);
  }
}

}  // namespace ctm
