// ctm.cu — libctm: the C ABI of include/ctm.h (collapsed Taylor mode on B200).
//
// Launch sequence of one operator call:
//   [prep]  per-call direction matrix (weighted / randomized with sigma only)
//   seed    layer 1: z0 = W1 x0 + b1, first-order coefficients, tanh Taylor rule  -> block B1
//   layer   l = 2..L-1: fused tcgen05 bf16-plane GEMM + tanh Taylor epilogue         -> block B_l
//           (the last hidden layer reduces straight against the output weights)
//   final   op = c * (w_L . sum h_K), f = w_L . h0 + b_L
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ctm.h"
#include "jet_layer.cuh"
#include "seed.cuh"
#include "backward.cuh"
#include "wgrad.cuh"

namespace {

thread_local std::string g_last_error;

ctm_status fail(ctm_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

#define CTM_CUDA(call)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(e_ == cudaErrorMemoryAllocation ? CTM_ENOMEM : CTM_ECUDA,                   \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                        \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 3D bf16 tensor map over the three planes of an operand: inner dim `cols` (contiguous),
// `rows`, plane (stride `pstride` elements); box {kBK, box_rows, 1} (128-byte rows);
// SWIZZLE_128B, matching the UMMA descriptors of jet_layer.cuh.
bool make_map3(CUtensorMap* m, const uint16_t* base, uint64_t cols, uint64_t rows, uint64_t pstride,
               uint32_t box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {cols, rows, 3};
  cuuint64_t strides[2] = {cols * sizeof(uint16_t), pstride * sizeof(uint16_t)};
  cuuint32_t box[3] = {(cuuint32_t)ctm::kBK, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// A plane-split operand block: three bf16 planes of `cap` elements each, contiguous
// (plane k at p + k * cap). cap is a multiple of 64 (TMA plane stride: 16-byte multiple).
struct Planes {
  uint16_t* p = nullptr;
  size_t cap = 0;
};

int round_up(int x, int m) { return (x + m - 1) / m * m; }

constexpr int kMaxD = 4096;  // input dimension (and Rv) cap: layer-1 K, seed staging chunks

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

struct ctm_mlp {
  int device = 0;
  int act = ctm::kActTanh;    // hidden-layer activation (ctm_set_activation)
  int sm_count = 148;
  bool seed_fixed_attr = false;  // max dynamic smem of the seed_fixed_kernel instances set
  bool seed_f16_attr = false;
  int L = 0;                  // affine layers
  std::vector<int> widths;    // L + 1
  std::vector<int> wpad;      // hidden widths padded to 128 (index = layer)
  // layer 1
  float* W1T = nullptr;       // [D, wpad[1]]
  float* b1 = nullptr;        // [wpad[1]]
  // operand precision (ctm_set_precision): 3 planes = fp32 mode, 2 planes = fast 3xBF16 or
  // (f16) the fp16x3 mode; nplanes is the plane count of the current call (an fp16x3 handle
  // runs the operators it does not cover in the fp32 mode, see f16_covers)
  int nplanes = 3;
  int prec = 0;               // ctm_precision of the handle
  bool cur_f16 = false;       // this call runs in the fp16x3 mode
  bool f16_stale = true;      // the fp16x3 weights do not match the bf16 planes (rebuilt on demand)
  // fp16x3 mode: fp16 weight planes [3][Mpad, Kpad] with per-layer power-of-two scales
  // (seed.cuh split_weights_f16_kernel), their statistics f16w[2 l] = 2^-(sa+11) (the
  // accumulator's weight factor), f16w[2 l + 1] = ||W_l||_inf (l = 1 .. L-1; layer 1 = W1p),
  // one scale record per slot block of a call (f16rec[l]: the output of layer l, [0] the
  // layer-1 input block of per-point directions), and bound scratch f16b[4]
  uint16_t* W1p16 = nullptr;
  CUtensorMap mapA1_16;
  std::vector<uint16_t*> Wp16;
  std::vector<CUtensorMap> mapA16;
  float* f16w = nullptr;
  ctm::F16Rec* f16rec = nullptr;
  unsigned* f16b = nullptr;
  // layer 1 as a tensor-core layer (randomized directions): bf16 planes [3][wpad[1], k1pad]
  int k1pad = 0;
  uint16_t* W1p = nullptr;
  CUtensorMap mapA1;
  // hidden GEMM layers l = 2..L-1 (index l-2)
  std::vector<uint16_t*> Wp;             // bf16 planes [3][Mpad, Kpad]
  std::vector<float*> bias;
  std::vector<CUtensorMap> mapA;
  // output layer
  float* w_out = nullptr;     // [wpad[L-1]]
  float* b_out = nullptr;     // [1] device (updated asynchronously by ctm_set_weights)
  float* bih_dirs = nullptr;  // [J_bih, D] biharmonic family directions
  // fixed direction sets
  float* U_lap = nullptr;     // [D, ld1]: z1 for e_d
  float* c_lap = nullptr;     // [ld1]
  float* U_bih = nullptr;     // [J, ld1]
  float* c_bih = nullptr;     // [ld1]
  float* w_bih = nullptr;     // [J] jet weights
  float* w_ones = nullptr;    // [kMaxW] unit weights (stochastic biharmonic: plain sum over samples)
  int J_bih = 0;
  // per-call scratch
  float* U_call = nullptr;
  float* c_call = nullptr;
  size_t U_call_elems = 0, c_call_elems = 0;
  float* c_blk = nullptr;     // [blocks, ld1] per-block constants of a fixed set split into blocks
  size_t c_blk_elems = 0;
  int forced_rb = 0;          // ctm_set_direction_block: directions per block (0 = planner)
  // workspace (bf16 planes): see ensure_workspace
  Planes blk[4];
  // ctm_gemm_probe scratch
  Planes probe_in, probe_out;
  float* probe_z = nullptr;
  size_t probe_z_elems = 0;
  float* partial = nullptr;
  size_t partial_elems = 0;
  // last plan
  int last_launches = 0, last_P = 0, last_ppt = 0, last_nmma = 0, last_nb = 1, last_rb = 0;
  bool smem_attr_set[512] = {};  // per (KORD, FLAGS) kernel instance
  // differentiable path (ctm_grad_enable / ctm_backward)
  bool grad = false;
  std::vector<uint16_t*> WTp;               // W_l^T bf16 planes [3][wpad[l-1], wpad[l]], l = 2..L-1
  std::vector<CUtensorMap> mapAT;
  // fp16x3 training (grad mode in CTM_PRECISION_FP16X3): W_l^T as the forward's fp16 planes
  // transposed, their statistics f16wT[2 l] = 2^-(sa+11), f16wT[2 l + 1] = ||W_l^T||_inf, the
  // scale records of the adjoint blocks Z_bar_l (f16zrec[l]), the backward seeds' bounds
  // f16bb[4] and the saved pre-activations' bounds f16zb[2 l], f16zb[2 l + 1] (backward.cuh)
  std::vector<uint16_t*> WTp16;
  std::vector<CUtensorMap> mapAT16;
  float* f16wT = nullptr;
  ctm::F16Rec* f16zrec = nullptr;
  float* f16bb = nullptr;
  float* f16zb = nullptr;
  unsigned* f16acc = nullptr;               // [3 (L+1)] weight-statistics accumulators (derive_f16_weights)
  float* eye = nullptr;                     // [256, 256] identity: fixed direction sets as shared V
  bool wgrad_attr[4] = {};                  // dynamic smem attribute set (wgrad_kernel<128|256, f16>)
  struct Tape {
    bool valid = false;
    int64_t N = 0;
    int P = 0, ppt = 0, nmma = 0;
    float scale = 1.f;
    int weighted = 0, J = 0;
    float* weights = nullptr;
    size_t weights_elems = 0;
    std::vector<Planes> B;                  // B_l, l = 0 .. L-1 (B_0 = layer-1 input block)
    int nplanes = 3;                        // precision the tape was recorded in
    bool f16 = false;                       // recorded in the fp16x3 mode (uniform block scales)
    bool random = false;                    // per-point directions (layer 1 on the tensor cores)
    std::vector<float*> Z;                  // Z_l, l = 1 .. L-1 (fp32 pre-activations)
    std::vector<size_t> Z_elems;
    Planes Zb[2];
    float* part = nullptr;
    size_t part_elems = 0;
    float* wpart = nullptr;                 // weight-gradient split partials
    size_t wpart_elems = 0;
  } tape;
  // profiling (events around launches)
  bool profiling = false;
  struct Rec {
    int kind;
    cudaEvent_t a, b;
    double work;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> event_pool;
};

namespace {

ctm_status free_all(ctm_mlp* h) {
  DeviceGuard g(h->device);
  auto F = [](auto*& p) {
    if (p) cudaFree(p);
    p = nullptr;
  };
  F(h->W1T); F(h->b1); F(h->w_out); F(h->W1p); F(h->b_out); F(h->bih_dirs);
  for (auto& p : h->Wp) F(p);
  for (auto& p : h->bias) F(p);
  F(h->U_lap); F(h->c_lap); F(h->w_ones); F(h->U_bih); F(h->c_bih); F(h->w_bih);
  F(h->U_call); F(h->c_call); F(h->c_blk);
  for (int i = 0; i < 4; ++i) F(h->blk[i].p);
  F(h->probe_in.p); F(h->probe_out.p); F(h->probe_z);
  F(h->partial);
  for (auto& p : h->WTp) F(p);
  F(h->W1p16); F(h->f16w); F(h->f16rec); F(h->f16b);
  for (auto& p : h->Wp16) F(p);
  for (auto& p : h->WTp16) F(p);
  F(h->f16wT); F(h->f16zrec); F(h->f16bb); F(h->f16zb); F(h->f16acc);
  F(h->eye);
  F(h->tape.weights); F(h->tape.part); F(h->tape.wpart);
  for (auto& p : h->tape.B) F(p.p);
  for (auto& p : h->tape.Z) F(p);
  for (int i = 0; i < 2; ++i) F(h->tape.Zb[i].p);
  for (auto& r : h->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  h->recs.clear();
  for (auto e : h->event_pool) cudaEventDestroy(e);
  h->event_pool.clear();
  return CTM_OK;
}

ctm_status ensure(float*& p, size_t& have, size_t need) {
  if (need <= have && p) return CTM_OK;
  if (p) cudaFree(p);
  p = nullptr;
  have = 0;
  CTM_CUDA(cudaMalloc(&p, std::max<size_t>(need, 1) * sizeof(float)));
  have = need;
  return CTM_OK;
}

// three planes of >= need elements each (grow-only)
ctm_status ensure_planes(Planes& b, size_t need) {
  if (need <= b.cap && b.p) return CTM_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  const size_t cap = (std::max<size_t>(need, 1) + 63) / 64 * 64;
  CTM_CUDA(cudaMalloc(&b.p, 3 * cap * sizeof(uint16_t)));
  b.cap = cap;
  return CTM_OK;
}

// blk[0], blk[1]: layer ping-pong blocks [rows, ldmax over hidden layers 1..L-1]; blk[2] (and blk[3] if nseed > 1):
// layer-1 blocks (seed output or random input block) [rows, max(ld1, k1pad)].
ctm_status ensure_workspace(ctm_mlp* h, int64_t rows, int nseed) {
  // the ping-pong blocks hold every tensor-core layer's output, including layer 1's when
  // per-point directions run layer 1 on the tensor cores (ld = wpad[1])
  int ldmax = 0;
  for (int l = 1; l < h->L; ++l) ldmax = std::max(ldmax, h->wpad[l]);
  const int ld_seed = std::max(h->wpad[1], h->k1pad);
  const size_t need[4] = {(size_t)rows * ldmax, (size_t)rows * ldmax, (size_t)rows * ld_seed,
                          nseed > 1 ? (size_t)rows * ld_seed : 0};
  for (int i = 0; i < 4; ++i) {
    if (need[i] == 0) continue;
    ctm_status s = ensure_planes(h->blk[i], need[i]);
    if (s != CTM_OK) return s;
  }
  return CTM_OK;
}


// The biharmonic direction family of Eq. `ttc_for_biharm_final` with the
// gamma of Fig. 3 (g40 = 13/192, g31 = -1/3, g22 = 5/8), rescaled so the
// directions are small integers:
//   A: e_d           weight 4^4 (2D g40 + 2 g31 + g22)/24 = (13D - 4)/9
//   B: 3 e_a + e_b   weight 2 g31 / 24               = -1/36      (a != b, a-major)
//   C: e_a + e_b     weight 2^4 * 2 g22 / 24         = 5/6        (a < b,  a-major)
void biharmonic_family(int D, std::vector<float>& dirs, std::vector<float>& w) {
  const double g40 = 13.0 / 192.0, g31 = -1.0 / 3.0, g22 = 5.0 / 8.0;
  const double wA = 256.0 * (2.0 * D * g40 + 2.0 * g31 + g22) / 24.0;
  const double wB = 2.0 * g31 / 24.0;
  const double wC = 16.0 * 2.0 * g22 / 24.0;
  dirs.clear();
  w.clear();
  auto push = [&](int a, float va, int b, float vb, double wt) {
    std::vector<float> v(D, 0.f);
    v[a] += va;
    if (b >= 0) v[b] += vb;
    dirs.insert(dirs.end(), v.begin(), v.end());
    w.push_back((float)wt);
  };
  for (int d = 0; d < D; ++d) push(d, 1.f, -1, 0.f, wA);
  for (int a = 0; a < D; ++a)
    for (int b = 0; b < D; ++b)
      if (a != b) push(a, 3.f, b, 1.f, wB);
  for (int a = 0; a < D; ++a)
    for (int b = a + 1; b < D; ++b) push(a, 1.f, b, 1.f, wC);
}

cudaEvent_t take_event(ctm_mlp* h) {
  if (!h->event_pool.empty()) {
    cudaEvent_t e = h->event_pool.back();
    h->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Brackets one launch with events when profiling is on.
struct ProfScope {
  ctm_mlp* h;
  int kind;
  double work;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(ctm_mlp* h_, int kind_, double work_, cudaStream_t st_) : h(h_), kind(kind_), work(work_), st(st_) {
    if (h->profiling) {
      a = take_event(h);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (h->profiling) {
      cudaEvent_t b = take_event(h);
      cudaEventRecord(b, st);
      h->recs.push_back({kind, a, b, work});
    }
  }
};

// cudaFuncSetAttribute is per device: tracked per handle (a handle lives on one device)
template <int KORD, int FLAGS = 0>
ctm_status set_layer_attr(ctm_mlp* h) {
  static_assert(KORD < 8 && FLAGS < 64, "smem_attr_set index");
  if (!h->smem_attr_set[KORD * 64 + FLAGS]) {
    CTM_CUDA(cudaFuncSetAttribute(ctm::jet_layer_kernel<KORD, FLAGS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  ctm::kLayerSmem));
    h->smem_attr_set[KORD * 64 + FLAGS] = true;
  }
  return CTM_OK;
}

template <int KORD, int FLAGS>
ctm_status launch_layer_instance(ctm_mlp* h, int64_t grid, const CUtensorMap& amap, const CUtensorMap& bmap,
                                 const ctm::LayerParams& lp, cudaStream_t st, const ctm::F16Args& fa) {
  ctm_status s = set_layer_attr<KORD, FLAGS>(h);
  if (s != CTM_OK) return s;
  // programmatic dependent launch: the prologue (barriers, TMEM allocation, descriptor
  // prefetch) overlaps the previous kernel's tail; the kernel waits before reading its input
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(ctm::layer_threads<KORD, FLAGS>());
  cfg.dynamicSmemBytes = ctm::kLayerSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CTM_CUDA(cudaLaunchKernelEx(&cfg, ctm::jet_layer_kernel<KORD, FLAGS>, amap, bmap, lp, fa));
  return CTM_OK;
}

// the instance with the handle's plane count (lp.nplanes) as a compile-time constant
// (fa.wsc set: the fp16x3 instance, K=2 forward only)
template <int KORD, int FLAGS>
ctm_status launch_layer_kernel(ctm_mlp* h, int64_t grid, const CUtensorMap& amap, const CUtensorMap& bmap,
                               const ctm::LayerParams& lp, cudaStream_t st, const ctm::F16Args& fa = {}) {
  if constexpr (KORD == 2 || (KORD == 4 && FLAGS == 0) || (KORD == ctm::kBwd2 && FLAGS == 0) ||
                (KORD == ctm::kNest && FLAGS == 0) || (KORD == ctm::kStd2 && FLAGS == 0) ||
                (KORD == ctm::kStd4 && FLAGS == 0)) {
    if (fa.wsc) return launch_layer_instance<KORD, FLAGS | ctm::kFlagF16>(h, grid, amap, bmap, lp, st, fa);
  }
  if (fa.wsc) return fail(CTM_EUNSUPPORTED, "fp16x3: collapsed K=2 / K=4 layers and the K=2 adjoint only");
  if (lp.nplanes == 2) return launch_layer_instance<KORD, FLAGS | ctm::kFlagNP2>(h, grid, amap, bmap, lp, st, fa);
  return launch_layer_instance<KORD, FLAGS>(h, grid, amap, bmap, lp, st, fa);
}

// Tile plan of one operator call. A point's R directions (K=4: jets) are split into nb
// blocks of rb (the last one zero padded); each block is a sub-point of P slots
// [x0; its directions; its partial collapsed top]. The collapsed top enters the Taylor rule
// of Eq. 7 linearly and the direction sum is additive, so the partial tops of
// the blocks sum to the point's top at every layer ("direction blocks");
// each block repeats the primal. ppt sub-points share one MMA N tile of nmma columns.
struct Plan {
  int P = 0, ppt = 0, nmma = 0;
  int nb = 1, rb = 0;
  int useful_P = 0;  // slots of the point with all its directions in one block (roofline work)
};

void tile_plan(Plan& pl) {
  int k = 1;
  while (round_up((k + 1) * pl.P, 16) <= ctm::kMaxN && k + 1 <= ctm::kMaxPtsPerTile) ++k;
  pl.ppt = k;
  pl.nmma = round_up(k * pl.P, 16);
}

// slots of a block of rb directions: K=2 rb + 2, K=4 3 rb + 2 (jets of 3), standard 1 + 2 rb,
// standard K=4 1 + 4 rb
int block_slots(int KORD, int rb) {
  return KORD == 4 ? 3 * rb + 2 : KORD == ctm::kStd2 ? 1 + 2 * rb : KORD == ctm::kStd4 ? 1 + 4 * rb : rb + 2;
}

// Modelled cost per point (relative units), from the round-1 sweep of the layer kernel over
// N: a tile of N columns runs at eff(N) = min(1, 2N / (256 + N)) of the
// tensor-pipe ceiling (the W tile is re-staged per N tile: N = 144 -> 0.72, 208 -> 0.90,
// >= 240 -> 0.97-1), plus the HBM write of the layer-1 block (0.17 per slot row, C1 ratio).
double plan_cost(const Plan& pl) {
  const double eff = std::min(1.0, 2.0 * pl.nmma / (256.0 + pl.nmma));
  return (double)pl.nb * pl.nmma / pl.ppt / eff + 0.17 * pl.nb * pl.P;
}

// R directions (jets): forced_rb > 0 fixes the block size; otherwise the cheapest split by
// plan_cost, keeping one block unless a split is modelled > 3% cheaper. P_fixed > 0 (nested
// biharmonic): no blocks. Returns P = 0 if no block fits a tile (P <= 256).
Plan make_plan_blocks(int KORD, int R, int forced_rb, bool allow_blocks, int P_fixed);
Plan make_plan(int KORD, int R, int forced_rb, bool allow_blocks, int P_fixed = 0) {
  Plan pl = make_plan_blocks(KORD, R, forced_rb, allow_blocks, P_fixed);
  pl.useful_P = P_fixed > 0 ? P_fixed : block_slots(KORD, std::max(R, 0));
  return pl;
}
Plan make_plan_blocks(int KORD, int R, int forced_rb, bool allow_blocks, int P_fixed) {
  Plan best;
  if (P_fixed > 0 || R < 1) {
    best.P = P_fixed > 0 ? P_fixed : block_slots(KORD, std::max(R, 0));
    best.rb = std::max(R, 0);
    if (best.P > ctm::kMaxN) best.P = 0;
    else tile_plan(best);
    return best;
  }
  auto make = [&](int rb) {
    Plan pl;
    pl.rb = rb;
    pl.nb = (R + rb - 1) / rb;
    pl.P = block_slots(KORD, rb);
    if (pl.P > ctm::kMaxN) pl.P = 0;
    else tile_plan(pl);
    return pl;
  };
  if (!allow_blocks) return make(R);
  if (forced_rb > 0) return make(std::min(forced_rb, R));
  const Plan one = make(R);
  double best_cost = 1e300;
  for (int nb = 1; nb <= R; ++nb) {
    const int rb = (R + nb - 1) / nb;
    if (nb > 1 && (R + rb - 1) / rb != nb) continue;  // same rb as a smaller nb
    const Plan pl = make(rb);
    if (pl.P == 0) continue;
    const double c = plan_cost(pl);
    if (c < best_cost) best_cost = c, best = pl;
    if (pl.P <= 8) break;                              // smaller blocks only add primal copies
  }
  if (one.P > 0 && plan_cost(one) <= 1.03 * best_cost) return one;
  return best;
}

enum Op { OP_LAP, OP_WLAP, OP_RLAP, OP_BIH, OP_LAP_STD, OP_SBIH, OP_BIH_NEST, OP_DSUM, OP_WLAP_X, OP_BIH_STD,
          OP_RLAP_STD, OP_SBIH_STD };

struct CallArgs {
  Op op;
  const float* X;
  int64_t N;
  const float* sigma;
  int R;
  int S;
  const float* V;
  uint64_t seed;
  int64_t point_offset;
  int Rv;
  int gaussian;
  float* op_out;
  float* f_out;
  cudaStream_t stream;
  // OP_DSUM: sum_j w_j <d^K f, u_j^K>; dirs [J, D] (shared) or [N, J, D] (per point)
  int K = 0;
  int J = 0;
  const float* dirs = nullptr;
  int per_point = 0;
  const float* weights = nullptr;
  int v_trans = 0;  // OP_WLAP_X: V = sigma(x) stored [N, D, R]
};

// per-point K=2 directions: the input block [x0; u; 0] and layer 1 on the tensor cores
bool random_k2(const CallArgs& a) {
  return a.op == OP_RLAP || a.op == OP_RLAP_STD || a.op == OP_WLAP_X || (a.op == OP_DSUM && a.per_point && a.K == 2);
}
// per-point K=4 directions: layer 1 in fp32 on the CUDA cores (seed_stoch_biharmonic_kernel)
bool stoch_k4(const CallArgs& a) {
  return a.op == OP_SBIH || a.op == OP_SBIH_STD || (a.op == OP_DSUM && a.per_point && a.K == 4);
}

struct GemmLayer {
  const CUtensorMap* amap;
  const float* bias;
  int kpad, mpad, w_in, w_out;
  const CUtensorMap* amap16;  // fp16x3 weight planes
  int lidx;                   // network layer index (1 .. L-1)
};

// grad mode: where a layer writes its output block and its pre-activations
struct LayerIO {
  Planes* out;
  float* z;
};

// sups of |s| and its first four derivatives for the activations the fp16x3 mode covers
// (tanh: |tanh''| <= 4/(3 sqrt 3) = 0.7698, |tanh'''| <= 2 (at 0), |tanh''''| <= 4.0859; sin: 1)
void f16_act_sups(int act, float& s0, float& s1, float& s2, float& s3, float& s4) {
  const bool th = (act == ctm::kActTanh);
  s0 = 1.f;
  s1 = 1.f;
  s2 = th ? 0.7699f : 1.f;
  s3 = th ? 2.0001f : 1.f;
  s4 = th ? 4.0860f : 1.f;
}

// max |a| over n floats into the bound record out (zeroed at the start of the call)
void launch_maxabs(const float* a, int64_t n, unsigned* out, cudaStream_t st) {
  const int64_t blocks = std::min<int64_t>(1184, (n + 255) / 256);
  if (blocks > 0) ctm::maxabs_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, n, out);
}

void launch_seed_random(int nplanes, int64_t N, const ctm::SeedRandomParams& rp, cudaStream_t st) {
  if (rp.f16_out) {
    ctm::seed_random_kernel<2, true><<<(unsigned)N, ctm::kSeedThreads, 0, st>>>(rp);
    return;
  }
  if (nplanes == 3)
    ctm::seed_random_kernel<3><<<(unsigned)N, ctm::kSeedThreads, 0, st>>>(rp);
  else
    ctm::seed_random_kernel<2><<<(unsigned)N, ctm::kSeedThreads, 0, st>>>(rp);
}

// Layer 1 for fixed direction sets (and the stochastic biharmonic) for points
// [p0, p0 + n): writes the layer-1 output block into buf.
ctm_status launch_seed(ctm_mlp* h, const CallArgs& a, int KORD, const Plan& pl, int64_t p0, int64_t n,
                       const Planes& buf, const float* UT, const float* csum, int R, cudaStream_t st, int& launches,
                       float* z_out = nullptr) {
  const int P = pl.P;
  const int D = h->widths[0], ld1 = h->wpad[1];
  const int threads = std::min(ctm::kSeedThreads, ld1 / 4);
  const int mchunks = (ld1 + 4 * threads - 1) / (4 * threads);
  const int64_t blocks = n * mchunks;
  if (blocks > INT32_MAX) return fail(CTM_EUNSUPPORTED, "batch too large for one call");
  // bytes written: the layer-1 block, every slot row of every direction block, bf16 planes
  ProfScope ps(h, CTM_KIND_SEED, (double)n * pl.nb * P * ld1 * 2.0 * h->nplanes, st);
  if (stoch_k4(a)) {
    ctm::SeedStochParams bp{};
    bp.X = a.X + p0 * D;
    bp.D = D;
    bp.W1T = h->W1T;
    bp.b1 = h->b1;
    bp.ld = ld1;
    bp.S = a.S;
    bp.V = a.V ? a.V + p0 * a.S * D : nullptr;
    bp.w = (a.op == OP_DSUM) ? a.weights : nullptr;
    bp.seed = a.seed;
    bp.point_offset = a.point_offset + p0;
    bp.blocks = pl.nb;
    bp.rb = pl.rb;
    bp.standard = (a.op == OP_SBIH_STD);
    bp.out = buf.p;
    bp.pstride = (int64_t)buf.cap;
    bp.nplanes = h->nplanes;
    bp.act = h->act;
    if (h->cur_f16) {  // fp16x3: bounds from ||W1||_inf and max |v| (explicit V: f16b[7]; generated: 6)
      ctm::SeedStochF16 sf{};
      if (a.V) {
        launch_maxabs(a.V + p0 * a.S * D, n * (int64_t)a.S * D, h->f16b + 7, st);
        ++launches;
        sf.vmax = h->f16b + 7;
      }
      sf.g1 = h->f16w + 2;
      sf.vgen = 6.f;  // |Box-Muller draw| <= sqrt(-2 ln 2^-25) = 5.9
      f16_act_sups(h->act, sf.s0, sf.s1, sf.s2, sf.s3, sf.s4);
      sf.out = h->f16rec + 1;
      ctm::seed_stoch_biharmonic_kernel<2, true><<<(unsigned)blocks, threads, sizeof(float) * a.S * D, st>>>(bp, sf);
    } else if (h->nplanes == 3) {
      ctm::seed_stoch_biharmonic_kernel<3><<<(unsigned)blocks, threads, sizeof(float) * a.S * D, st>>>(bp);
    } else {
      ctm::seed_stoch_biharmonic_kernel<2><<<(unsigned)blocks, threads, sizeof(float) * a.S * D, st>>>(bp);
    }
  } else {
    ctm::SeedParams sp{};
    sp.X = a.X + p0 * D;
    sp.D = D;
    sp.n_points = n;
    sp.W1T = h->W1T;
    sp.b1 = h->b1;
    sp.ld = ld1;
    sp.P = P;
    sp.UT = UT;
    sp.csum = csum;
    sp.R = R;
    sp.blocks = pl.nb;
    sp.rb = (KORD == ctm::kNest) ? R : pl.rb;
    sp.out = buf.p;
    sp.pstride = (int64_t)buf.cap;
    sp.nplanes = h->nplanes;
    sp.act = h->act;
    sp.z_out = z_out;
    // forward K=2 fixed sets: the streaming seed (tables in shared memory) when its slice of
    // W1^T and U^T fits (C1 seed 0.93 -> 0.83 ms in the bench step). Grad mode (z_out) and the
    // other rules keep seed_layer_kernel; the K=4 instance of the streaming seed was 6% slower
    // than it in the power-capped C4 step (1.70-1.75 vs 1.61-1.65 ms), so K=4 stays there too.
    const size_t fsm = ctm::seed_fixed_smem(D, R, pl.nb);
    constexpr size_t kFixedSmemMax = 200 * 1024;
    // (the fp16x3 mode's K=4 seed is the streaming kernel too: seed_layer_kernel has no fp16 planes)
    // (grad mode z_out: the fp16x3 mode's seed writes the pre-activations too, seed_layer_kernel
    // has no fp16 planes; the fp32 mode keeps seed_layer_kernel there)
    if ((KORD == 2 || (KORD == 4 && h->cur_f16)) && (!z_out || h->cur_f16) && fsm <= kFixedSmemMax &&
        ld1 % ctm::kSeedFixedFeats == 0 && n > 0) {
      if (!h->seed_fixed_attr) {
        CTM_CUDA(cudaFuncSetAttribute(ctm::seed_fixed_kernel<2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kFixedSmemMax));
        CTM_CUDA(cudaFuncSetAttribute(ctm::seed_fixed_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kFixedSmemMax));
        h->seed_fixed_attr = true;
      }
      ctm::SeedF16 sf{};
      if (h->cur_f16) {  // fp16x3: bounds of this call's direction images, output record of layer 1
        if (!h->seed_f16_attr) {
          CTM_CUDA(cudaFuncSetAttribute(ctm::seed_fixed_kernel<2, 2, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFixedSmemMax));
          CTM_CUDA(cudaFuncSetAttribute(ctm::seed_fixed_kernel<4, 2, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFixedSmemMax));
          h->seed_f16_attr = true;
        }
        launch_maxabs(UT, (int64_t)R * ld1, h->f16b, st);
        launch_maxabs(csum, (int64_t)pl.nb * ld1, h->f16b + 1, st);
        launches += 2;
        sf.bounds = h->f16b;
        f16_act_sups(h->act, sf.s0, sf.s1, sf.s2, sf.s3, sf.s4);
        sf.out = h->f16rec + 1;
        sf.uniform = z_out != nullptr;  // grad mode: one scale per block (the weight gradients)
      }
      // one wave: as many blocks as are resident at once (registers, shared memory)
      const int slices = ld1 / ctm::kSeedFixedFeats;
      const int thr = ctm::kSeedFixedWarps * 32;
      int per_sm = 1;
      CTM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm,
          h->cur_f16 ? (KORD == 4 ? ctm::seed_fixed_kernel<4, 2, true> : ctm::seed_fixed_kernel<2, 2, true>)
                     : (h->nplanes == 3 ? ctm::seed_fixed_kernel<2, 3> : ctm::seed_fixed_kernel<2, 2>),
          thr, fsm));
      const int64_t want = std::max<int64_t>(1, (int64_t)h->sm_count * std::max(per_sm, 1) / slices);
      const int64_t groups0 = std::min<int64_t>(want, (n + ctm::kSeedFixedWarps - 1) / ctm::kSeedFixedWarps);
      const int64_t ppg = (n + groups0 - 1) / groups0;
      const int64_t groups = (n + ppg - 1) / ppg;
      if (groups > 65535) return fail(CTM_EUNSUPPORTED, "batch too large for one call");
      const dim3 grid((unsigned)slices, (unsigned)groups);
      if (h->cur_f16 && KORD == 4)
        ctm::seed_fixed_kernel<4, 2, true><<<grid, thr, fsm, st>>>(sp, ppg, sf);
      else if (h->cur_f16)
        ctm::seed_fixed_kernel<2, 2, true><<<grid, thr, fsm, st>>>(sp, ppg, sf);
      else
        (h->nplanes == 3 ? ctm::seed_fixed_kernel<2, 3><<<grid, thr, fsm, st>>>(sp, ppg, sf)
                         : ctm::seed_fixed_kernel<2, 2><<<grid, thr, fsm, st>>>(sp, ppg, sf));
      ++launches;
      return CTM_OK;
    }
#define CTM_SEED(K)                                                            \
  (h->nplanes == 3 ? ctm::seed_layer_kernel<K, 3><<<(unsigned)blocks, threads, 0, st>>>(sp) \
                   : ctm::seed_layer_kernel<K, 2><<<(unsigned)blocks, threads, 0, st>>>(sp))
    if (KORD == 2)
      CTM_SEED(2);
    else if (KORD == 4)
      CTM_SEED(4);
    else if (KORD == ctm::kNest && h->cur_f16) {  // fp16x3: bounds max|U|, max|csum| of this call
      launch_maxabs(UT, (int64_t)R * ld1, h->f16b, st);
      launch_maxabs(csum, (int64_t)ld1, h->f16b + 1, st);
      launches += 2;
      ctm::SeedF16 sf{};
      sf.bounds = h->f16b;
      f16_act_sups(h->act, sf.s0, sf.s1, sf.s2, sf.s3, sf.s4);
      sf.out = h->f16rec + 1;
      ctm::seed_layer_kernel<ctm::kNest, 2, true><<<(unsigned)blocks, threads, 0, st>>>(sp, sf);
    } else if (KORD == ctm::kNest)
      CTM_SEED(ctm::kNest);
    else if ((KORD == ctm::kStd4 || KORD == ctm::kStd2) && h->cur_f16) {  // fp16x3: bound max|U| of this call
      launch_maxabs(UT, (int64_t)R * ld1, h->f16b, st);
      ++launches;
      ctm::SeedF16 sf{};
      sf.bounds = h->f16b;
      f16_act_sups(h->act, sf.s0, sf.s1, sf.s2, sf.s3, sf.s4);
      sf.out = h->f16rec + 1;
      if (KORD == ctm::kStd4)
        ctm::seed_layer_kernel<ctm::kStd4, 2, true><<<(unsigned)blocks, threads, 0, st>>>(sp, sf);
      else
        ctm::seed_layer_kernel<ctm::kStd2, 2, true><<<(unsigned)blocks, threads, 0, st>>>(sp, sf);
    } else if (KORD == ctm::kStd4)
      CTM_SEED(ctm::kStd4);
    else
      CTM_SEED(ctm::kStd2);
#undef CTM_SEED
  }
  ++launches;
  return CTM_OK;
}

// The tensor-core layers for points [p0, p0 + n), whose first GEMM reads `in`;
// ping-pongs through blk[0] / blk[1] and ends in the readout of op/f. `after_first`
// (optional) is recorded on st once the first GEMM (the reader of `in`) is enqueued.
ctm_status launch_layers(ctm_mlp* h, const CallArgs& a, int KORD, const Plan& pl, const std::vector<GemmLayer>& layers,
                         int64_t p0, int64_t n, const Planes* in, float scale, cudaStream_t st,
                         cudaEvent_t after_first, int& launches, const std::vector<LayerIO>* io = nullptr) {
  const int P = pl.P;
  const int64_t nsub = n * pl.nb;  // sub-points (direction blocks) = the kernel's points
  const int64_t rows = nsub * (int64_t)P;
  if (layers.empty()) {  // a single hidden layer: read the layer-1 block
    const int threads = 256, ppb = threads / 32;
    ProfScope ps(h, CTM_KIND_FINAL, 0.0, st);
    ctm::readout_block_kernel<<<(unsigned)((n + ppb - 1) / ppb), threads, 0, st>>>(
        in->p, (int64_t)in->cap, h->nplanes, h->wpad[1], P, pl.nb, h->widths[1], h->w_out, h->b_out, scale, n,
        a.op_out + p0,
        a.f_out ? a.f_out + p0 : nullptr,
        (a.op == OP_LAP_STD || a.op == OP_RLAP_STD) ? 2 : (a.op == OP_BIH_STD || a.op == OP_SBIH_STD) ? 4 : 0,
        a.op == OP_SBIH_STD ? h->w_ones : h->w_bih, std::max(pl.rb, 1), a.op == OP_SBIH_STD ? a.S : h->J_bih);
    ++launches;
    if (after_first) CTM_CUDA(cudaEventRecord(after_first, st));
    return CTM_OK;
  }
  const int64_t n_tiles = (nsub + pl.ppt - 1) / pl.ppt;
  const Planes* src = in;
  int dst = 0;
  for (size_t li = 0; li < layers.size(); ++li) {
    const GemmLayer& gl = layers[li];
    const int m_tiles = gl.mpad / ctm::kBM;
    const bool last = (li + 1 == layers.size());
    CUtensorMap mb;  // a CTA stages half of B
    if (!make_map3(&mb, src->p, (uint64_t)gl.kpad, (uint64_t)rows, src->cap, (uint32_t)pl.nmma / 2))
      return fail(CTM_ECUDA, "cuTensorMapEncodeTiled failed for the activation block");
    ctm::LayerParams lp{};
    lp.bias = gl.bias;
    lp.act = h->act;
    const Planes* outp = io ? (*io)[li].out : &h->blk[dst];
    lp.out = outp ? outp->p : nullptr;
    lp.pstride = outp ? (int64_t)outp->cap : 0;
    lp.nplanes = (int16_t)h->nplanes;
    lp.ldo = gl.mpad;
    lp.z_out = io ? (*io)[li].z : nullptr;
    lp.ldz = gl.mpad;
    lp.m_tiles = m_tiles;
    lp.n_points = nsub;
    lp.P = P;
    lp.pts_per_tile = pl.ppt;
    lp.n_mma = pl.nmma;
    lp.k_iters = gl.kpad / ctm::kBK;
    lp.blocks = pl.nb;
    lp.rb = std::max(pl.rb, 1);
    switch (a.op) {
      case OP_SBIH: case OP_SBIH_STD: lp.jet_w = h->w_ones; lp.J = a.S; break;
      case OP_BIH: case OP_BIH_STD: lp.jet_w = h->w_bih; lp.J = h->J_bih; break;
      case OP_BIH_NEST: lp.J = h->widths[0]; break;
      case OP_DSUM: lp.jet_w = a.weights; lp.J = a.J; lp.weighted = (a.K == 2); break;
      default: break;
    }
    if (last) {
      ctm_status s = ensure(h->partial, h->partial_elems, (size_t)nsub * m_tiles * 2);
      if (s != CTM_OK) return s;
      lp.readout = 1;
      lp.w_out = h->w_out;
      lp.partial = h->partial;
    }
    // persistent CTA pairs: an even grid, at most one CTA per SM
    const int64_t grid = 2 * std::min<int64_t>(n_tiles * (m_tiles / 2), h->sm_count / 2);
    {
      // useful FLOP: the point's slots with all directions in one block (the duplicated
      // primal / top rows and zero padding of direction blocks are not counted)
      ProfScope ps(h, CTM_KIND_LAYER, 2.0 * n * pl.useful_P * gl.w_in * gl.w_out, st);
      ctm_status s;
      int flags = (lp.weighted ? ctm::kFlagWeighted : 0) | (lp.z_out ? ctm::kFlagSaveZ : 0);
      if (KORD == 2 && flags == 0 && pl.ppt >= 8) flags = ctm::kFlagWide;
      // a 7-slot ring when the B half-tile fits 104 rows (C1 / C2: 4 points of 52 slots)
      if (KORD == 2 && flags == 0 && pl.nmma <= 208) flags = ctm::kFlagRing7;
      ctm::F16Args fa{};
      const CUtensorMap* am = gl.amap;
      if (h->cur_f16) {  // fp16x3: this layer's weight planes, its input and output block records
        fa.in = h->f16rec + (gl.lidx - 1);
        fa.out = last ? nullptr : h->f16rec + gl.lidx;
        fa.wsc = h->f16w + 2 * gl.lidx;
        f16_act_sups(h->act, fa.s0, fa.s1, fa.s2, fa.s3, fa.s4);
        // K=2: sum |w_r| = rb (unit weights) unless weighted; K=4: the jets' weights (from smem)
        fa.rw = (lp.weighted || KORD == 4) ? -1.f : (float)std::max(pl.rb, 1);
        fa.uniform = io != nullptr;
        am = gl.amap16;
      }
      if (KORD == 2) {
        switch (flags) {
          case ctm::kFlagWide:
            s = launch_layer_kernel<2, ctm::kFlagWide>(h, grid, *am, mb, lp, st, fa);
            break;
          case ctm::kFlagRing7:
            s = launch_layer_kernel<2, ctm::kFlagRing7>(h, grid, *am, mb, lp, st, fa);
            break;
          case 0: s = launch_layer_kernel<2, 0>(h, grid, *am, mb, lp, st, fa); break;
          case 1: s = launch_layer_kernel<2, 1>(h, grid, *am, mb, lp, st, fa); break;
          case 2: s = launch_layer_kernel<2, 2>(h, grid, *am, mb, lp, st, fa); break;
          default: s = launch_layer_kernel<2, 3>(h, grid, *am, mb, lp, st, fa); break;
        }
      } else if (KORD == 4) {
        s = launch_layer_kernel<4, 0>(h, grid, *am, mb, lp, st, fa);
      } else if (KORD == ctm::kNest) {
        s = launch_layer_kernel<ctm::kNest, 0>(h, grid, *am, mb, lp, st, fa);
      } else if (KORD == ctm::kStd4) {
        s = launch_layer_kernel<ctm::kStd4, 0>(h, grid, *am, mb, lp, st, fa);
      } else {
        s = launch_layer_kernel<ctm::kStd2, 0>(h, grid, *am, mb, lp, st, fa);
      }
      if (s != CTM_OK) return s;
    }
    ++launches;
    if (li == 0 && after_first) CTM_CUDA(cudaEventRecord(after_first, st));
    if (last) {
      ProfScope ps(h, CTM_KIND_FINAL, 0.0, st);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)((n + 255) / 256));
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CTM_CUDA(cudaLaunchKernelEx(&cfg, ctm::finalize_kernel, (const float*)h->partial, m_tiles, pl.nb, n,
                                  (const float*)h->b_out, scale, a.op_out + p0, a.f_out ? a.f_out + p0 : nullptr));
      ++launches;
    }
    src = io ? (*io)[li].out : &h->blk[dst];
    dst ^= 1;
  }
  return CTM_OK;
}

// the K=2 operators have a backward (ctm_backward)
bool differentiable(const CallArgs& a) {
  return a.op == OP_LAP || a.op == OP_WLAP || a.op == OP_RLAP || a.op == OP_WLAP_X || (a.op == OP_DSUM && a.K == 2);
}

// grad mode: per-layer tape buffers for `rows` slot rows
ctm_status prepare_tape(ctm_mlp* h, int64_t rows) {
  auto& T = h->tape;
  const int L = h->L;
  T.B.resize(L);
  T.Z.resize(L, nullptr);
  T.Z_elems.resize(L, 0);
  ctm_status s = ensure_planes(T.B[0], (size_t)rows * h->k1pad);
  if (s != CTM_OK) return s;
  for (int l = 1; l <= std::max(1, L - 2); ++l) {
    s = ensure_planes(T.B[l], (size_t)rows * h->wpad[l]);
    if (s != CTM_OK) return s;
  }
  for (int l = 1; l <= L - 1; ++l) {
    s = ensure(T.Z[l], T.Z_elems[l], (size_t)rows * h->wpad[l]);
    if (s != CTM_OK) return s;
  }
  return CTM_OK;
}

// the calls the fp16x3 mode covers (include/ctm.h ctm_set_precision): K=2 collapsed forward
// operators of tanh / sin nets, random directions without sigma, >= 2 points per tile (no
// split point), the streaming seed for fixed sets, and at least one tensor-core layer
bool f16_covers(const ctm_mlp* h, const CallArgs& a, int KORD, const Plan& pl, bool grad, int R) {
  if (h->prec != CTM_PRECISION_FP16X3 || pl.ppt < 2) return false;
  // grad mode (fp16x3 training): the K=2 operators (uniform block scales)
  if (grad && (KORD != 2 || h->WTp16.empty())) return false;
  if (h->act != ctm::kActTanh && h->act != ctm::kActSin) return false;
  const bool k2op = a.op == OP_LAP || a.op == OP_WLAP || a.op == OP_RLAP || a.op == OP_WLAP_X ||
                    (a.op == OP_DSUM && a.K == 2);
  // K=4: the fixed interpolation family, and (session 3) per-point K=4 directions -- the
  // stochastic biharmonic and per-point K=4 sums, whose layer 1 stays fp32 on the CUDA cores
  // and writes the fp16x3 planes of its output block
  const bool k4op = a.op == OP_BIH || a.op == OP_SBIH || (a.op == OP_DSUM && a.K == 4);
  // the nested biharmonic (session 3): one scale per block (seed_layer_kernel<kNest, 2, true>)
  if (KORD == ctm::kNest) return a.op == OP_BIH_NEST && h->L >= 3;
  // the standard-mode baselines (session 3): the seeds' and epilogues' standard layouts
  if (KORD == ctm::kStd2 || KORD == ctm::kStd4) {
    if (h->L < 3) return false;
    return a.op == OP_LAP_STD || a.op == OP_RLAP_STD || a.op == OP_BIH_STD || a.op == OP_SBIH_STD;
  }
  if (!(KORD == 2 ? k2op : k4op)) return false;
  if (random_k2(a)) return true;
  if (stoch_k4(a)) return h->L >= 3;
  const int D = h->widths[0], ld1 = h->wpad[1];
  return h->L >= 3 && ctm::seed_fixed_smem(D, R, pl.nb) <= 200 * 1024 && ld1 % ctm::kSeedFixedFeats == 0;
}

ctm_status run(ctm_mlp* h, const CallArgs& a) {
  const int D = h->widths[0];
  const int ld1 = h->wpad[1];
  const int KORD = (a.op == OP_BIH || a.op == OP_SBIH || (a.op == OP_DSUM && a.K == 4)) ? 4
                   : (a.op == OP_LAP_STD || a.op == OP_RLAP_STD)                      ? ctm::kStd2
                   : (a.op == OP_BIH_STD || a.op == OP_SBIH_STD)                      ? ctm::kStd4
                   : (a.op == OP_BIH_NEST)                                            ? ctm::kNest
                                                                                      : 2;
  int R = 0;  // directions (K=4: jets) of the operator
  switch (a.op) {
    case OP_LAP: case OP_LAP_STD: R = D; break;
    case OP_WLAP: R = a.R; break;
    case OP_RLAP: case OP_SBIH: case OP_WLAP_X: case OP_RLAP_STD: case OP_SBIH_STD: R = a.S; break;
    case OP_BIH: case OP_BIH_STD: R = h->J_bih; break;
    case OP_DSUM: R = a.J; break;
    case OP_BIH_NEST: break;
  }
  h->tape.valid = false;  // whatever happens below, an earlier call's tape is stale now
  // grad mode records one block per point (the backward kernels have no block structure)
  const bool grad = h->grad && differentiable(a);
  const Plan pl = make_plan(KORD, R, h->forced_rb, !grad,
                            a.op == OP_BIH_NEST ? 2 + 2 * D + D * (D + 1) / 2 : 0);
  if (pl.P == 0)
    return fail(CTM_EUNSUPPORTED, grad ? "grad mode: slots per point exceed the cap of 256 (one block per point)"
                                       : "direction block does not fit one tile (slots per block > 256)");
  if (stoch_k4(a) && (int64_t)a.S * D > 12288)
    return fail(CTM_EUNSUPPORTED, "S * D > 12288 for per-point K=4 directions");
  if ((KORD == 4 || KORD == ctm::kStd4 || a.op == OP_DSUM) && (int64_t)pl.nb * pl.rb > ctm::kMaxW)
    return fail(CTM_EUNSUPPORTED, "more than 2048 weighted directions (jets) per point");
  // arithmetic of this call: an fp16x3 handle runs what the mode does not cover in fp32 mode
  h->cur_f16 = f16_covers(h, a, KORD, pl, grad, R);
  h->nplanes = (h->prec == CTM_PRECISION_BF16X3 || h->cur_f16) ? 2 : 3;
  const int P = pl.P;
  h->last_P = pl.P;
  h->last_ppt = pl.ppt;
  h->last_nmma = pl.nmma;
  h->last_nb = pl.nb;
  h->last_rb = pl.rb;
  h->last_launches = 0;
  if (a.N == 0) {
    if (grad) {  // an empty tape: ctm_backward gives zero gradients
      h->tape.N = 0;
      h->tape.P = P;
      h->tape.nplanes = h->nplanes;
      h->tape.valid = true;
    }
    return CTM_OK;
  }
  const int64_t rows_total = a.N * pl.nb * (int64_t)P;
  if (rows_total > (int64_t)INT32_MAX) return fail(CTM_EUNSUPPORTED, "N * slots exceeds 2^31 rows");

  DeviceGuard g(h->device);
  cudaStream_t st = a.stream;
  int launches = 0;
  ctm_status s;
  if (h->cur_f16) {  // fresh scale records and bound scratch for this call
    CTM_CUDA(cudaMemsetAsync(h->f16rec, 0, sizeof(ctm::F16Rec) * (h->L + 1), st));
    CTM_CUDA(cudaMemsetAsync(h->f16b, 0, sizeof(unsigned) * 8, st));
  }
  // grad mode: record the tape of this call (differentiable operators only)
  std::vector<LayerIO> io;
  if (grad) {
    s = prepare_tape(h, a.N * (int64_t)P);
    if (s != CTM_OK) return s;
    const int first = random_k2(a) ? 1 : 2;
    for (int l = first; l <= h->L - 1; ++l) io.push_back({l < h->L - 1 ? &h->tape.B[l] : nullptr, h->tape.Z[l]});
  }
  const Planes* tapeB0 = grad ? &h->tape.B[0] : nullptr;
  const Planes* tapeB1 = grad ? &h->tape.B[1] : nullptr;

  // GEMM layers: layer 1 for per-point K=2 directions, then the hidden layers 2..L-1
  std::vector<GemmLayer> layers;
  if (random_k2(a)) layers.push_back({&h->mapA1, h->b1, h->k1pad, ld1, D, h->widths[1], &h->mapA1_16, 1});
  for (int l = 2; l <= h->L - 1; ++l)
    layers.push_back({&h->mapA[l - 2], h->bias[l - 2], h->wpad[l - 1], h->wpad[l], h->widths[l - 1], h->widths[l],
                      &h->mapA16[l - 2], l});

  if (random_k2(a)) {
    // per-point K=2 directions: the input block [x0; u_1..u_S; 0], then layer 1 on the
    // tensor cores like every other layer
    s = ensure_workspace(h, rows_total, 1);
    if (s != CTM_OK) return s;
    ctm::SeedRandomParams rp{};
    rp.X = a.X;
    rp.D = D;
    rp.ldk = h->k1pad;
    rp.S = a.S;
    rp.Rv = a.Rv;
    rp.V = a.V;
    rp.sigma = a.sigma;
    rp.seed = a.seed;
    rp.point_offset = a.point_offset;
    rp.gaussian = a.gaussian;
    rp.v_trans = a.v_trans;
    rp.blocks = pl.nb;
    rp.rb = pl.rb;
    rp.standard = (a.op == OP_RLAP_STD);
    const Planes& b0 = grad ? *tapeB0 : h->blk[2];
    rp.out = b0.p;
    rp.pstride = (int64_t)b0.cap;
    rp.nplanes = h->nplanes;
    if (h->cur_f16) {  // fp16x3: bounds of x0 and of explicit directions; the input block's record
      launch_maxabs(a.X, a.N * (int64_t)D, h->f16b + 2, st);
      ++launches;
      if (a.V) {
        launch_maxabs(a.V, a.N * (int64_t)a.S * a.Rv, h->f16b + 3, st);
        ++launches;
      }
      if (a.sigma) {  // u = sigma v: |u| <= Rv max|sigma| max|v| (seed_random_kernel)
        launch_maxabs(a.sigma, (int64_t)D * a.Rv, h->f16b + 4, st);
        ++launches;
      }
      rp.f16_bounds = h->f16b + 2;
      rp.vgen = a.gaussian ? 6.f : 1.f;  // |Box-Muller draw| <= sqrt(-2 ln 2^-25) = 5.9
      rp.f16_out = h->f16rec;
      rp.f16_uniform = grad ? 1 : 0;  // fp16x3 training: B_0 feeds the layer-1 weight gradient
    }
    {
      ProfScope ps(h, CTM_KIND_SEED, (double)rows_total * h->k1pad * 2.0 * h->nplanes, st);
      launch_seed_random(h->nplanes, a.N, rp, st);
    }
    ++launches;
    const float scale = (a.op == OP_RLAP || a.op == OP_RLAP_STD) ? 1.f / (float)a.S : 1.f;  // Eq. 8/10 stochastic
    s = launch_layers(h, a, KORD, pl, layers, 0, a.N, grad ? tapeB0 : &h->blk[2], scale, st, nullptr, launches,
                      grad ? &io : nullptr);
    if (s != CTM_OK) return s;
  } else {
    // fixed direction sets (or the K=4 stochastic seed): U and the per-feature constant
    const float* UT = h->U_lap;
    const float* csum = h->c_lap;
    if (a.op == OP_BIH || a.op == OP_BIH_STD) {
      UT = h->U_bih;
      csum = h->c_bih;
    } else if (a.op == OP_DSUM && !a.per_point) {  // U = W1 u_j, c = sum_j w_j (W1 u_j)^K for this call
      s = ensure(h->U_call, h->U_call_elems, (size_t)a.J * ld1);
      if (s != CTM_OK) return s;
      s = ensure(h->c_call, h->c_call_elems, (size_t)ld1);
      if (s != CTM_OK) return s;
      {
        ProfScope ps(h, CTM_KIND_PREP, 0.0, st);
        ctm::prep_directions_kernel<<<(ld1 + 127) / 128, 128, 0, st>>>(h->W1T, D, ld1, a.dirs, a.J, a.weights, a.K,
                                                                       h->U_call, h->c_call);
      }
      ++launches;
      UT = h->U_call;
      csum = h->c_call;
    } else if (a.op == OP_WLAP) {  // U = W1 sigma for this call
      s = ensure(h->U_call, h->U_call_elems, (size_t)a.R * ld1);
      if (s != CTM_OK) return s;
      s = ensure(h->c_call, h->c_call_elems, (size_t)ld1);
      if (s != CTM_OK) return s;
      {
        ProfScope ps(h, CTM_KIND_PREP, 0.0, st);
        ctm::prep_sigma_kernel<<<(ld1 + 127) / 128, 128, 0, st>>>(h->W1T, D, ld1, a.sigma, a.R, h->U_call,
                                                                  h->c_call);
      }
      ++launches;
      UT = h->U_call;
      csum = h->c_call;
    }
    const float scale = (a.op == OP_SBIH || a.op == OP_SBIH_STD) ? 1.f / (3.f * (float)a.S) : 1.f;  // Eq. 12: 1/(3S), Q1
    // Sequential: running the HBM-write-bound seed of one chunk beside the power-capped
    // tensor-core layers of another was measured slower (2.58-2.65 M vs 2.68 M points/s at
    // C1): the two compete for the 1 kW budget rather than for SMs.
    s = ensure_workspace(h, rows_total, 1);
    if (s != CTM_OK) return s;
    if (pl.nb > 1 && !stoch_k4(a)) {  // per-block constants of the fixed set (UT has R rows)
      s = ensure(h->c_blk, h->c_blk_elems, (size_t)pl.nb * ld1);
      if (s != CTM_OK) return s;
      {
        ProfScope ps(h, CTM_KIND_PREP, 0.0, st);
        const float* w = (a.op == OP_BIH || a.op == OP_BIH_STD) ? h->w_bih : (a.op == OP_DSUM) ? a.weights : nullptr;
        ctm::block_csum_kernel<<<(ld1 + 127) / 128, 128, 0, st>>>(UT, R, ld1, w, KORD == 4 ? 4 : 2, pl.nb, pl.rb,
                                                                  h->c_blk);
      }
      ++launches;
      csum = h->c_blk;
    }
    if (grad) {
      // the layer-1 input block B_0 = [x0; u_r; 0] for dW_1 (directions shared by all points)
      ctm::SeedRandomParams rp{};
      rp.X = a.X;
      rp.D = D;
      rp.ldk = h->k1pad;
      rp.v_shared = 1;
      if (a.op == OP_LAP) {
        rp.S = D, rp.Rv = D, rp.V = h->eye, rp.ldv = 256;
      } else if (a.op == OP_WLAP) {
        rp.S = a.R, rp.Rv = a.R, rp.V = h->eye, rp.ldv = 256, rp.sigma = a.sigma;
      } else {
        rp.S = a.J, rp.Rv = D, rp.V = a.dirs, rp.ldv = D;
      }
      rp.blocks = 1;
      rp.rb = rp.S;
      rp.out = tapeB0->p;
      rp.pstride = (int64_t)tapeB0->cap;
      rp.nplanes = h->nplanes;
      if (h->cur_f16) {  // fp16x3: B_0 with one scale (bounds max|x|, max|v|, max|sigma| at f16b[2..4])
        launch_maxabs(a.X, a.N * (int64_t)D, h->f16b + 2, st);
        launch_maxabs(rp.V, (int64_t)rp.S * rp.ldv, h->f16b + 3, st);
        launches += 2;
        if (rp.sigma) {
          launch_maxabs(rp.sigma, (int64_t)D * a.R, h->f16b + 4, st);
          ++launches;
        }
        rp.f16_bounds = h->f16b + 2;
        rp.vgen = 1.f;
        rp.f16_out = h->f16rec;
        rp.f16_uniform = 1;
      }
      launch_seed_random(h->nplanes, a.N, rp, st);
      ++launches;
    }
    s = launch_seed(h, a, KORD, pl, 0, a.N, grad ? *tapeB1 : h->blk[2], UT, csum, a.op == OP_BIH_NEST ? D : R, st,
                    launches, grad ? h->tape.Z[1] : nullptr);
    if (s != CTM_OK) return s;
    s = launch_layers(h, a, KORD, pl, layers, 0, a.N, grad ? tapeB1 : &h->blk[2], scale, st, nullptr, launches,
                      grad ? &io : nullptr);
    if (s != CTM_OK) return s;
  }
  if (grad) {
    auto& T = h->tape;
    T.N = a.N;
    T.P = P;
    T.ppt = pl.ppt;
    T.nmma = pl.nmma;
    T.scale = (a.op == OP_RLAP) ? 1.f / (float)a.S : 1.f;
    T.weighted = (a.op == OP_DSUM);
    T.J = (a.op == OP_DSUM) ? a.J : 0;
    T.nplanes = h->nplanes;
    T.f16 = h->cur_f16;
    T.random = random_k2(a);
    if (T.weighted) {  // the caller's weights may not outlive the call
      s = ensure(T.weights, T.weights_elems, (size_t)a.J);
      if (s != CTM_OK) return s;
      CTM_CUDA(cudaMemcpyAsync(T.weights, a.weights, sizeof(float) * a.J, cudaMemcpyDeviceToDevice, st));
    }
    T.valid = true;
  }
  CTM_CUDA(cudaGetLastError());
  h->last_launches = launches;
  return CTM_OK;
}

// dW[o, i] (o < rows_out, i < cols_in, caller's layout; = or +=) = sum over the slot rows
// of Z[row, o] B[row, i] (Z [rows, Mout], B [rows, Kin], both bf16 planes): wgrad_kernel
// (tcgen05, MN-major operands, fixed K splits, chunked TMEM accumulation) and
// wgrad_reduce_kernel (the splits summed in order, cropped into dW). Deterministic.
ctm_status weight_grad(ctm_mlp* h, const Planes& B, int Kin, const Planes& Z, int Mout, int64_t rows, int rows_out,
                       int cols_in, float* dW, int acc, cudaStream_t st, const ctm::F16Rec* zrec = nullptr,
                       const ctm::F16Rec* brec = nullptr) {
  auto& T = h->tape;
  const bool f16 = zrec != nullptr;  // fp16x3 operands (uniform scales zrec / brec)
  const int N = (Kin % 256 == 0) ? 256 : 128;
  ctm::WgradParams wp{};
  wp.rows = rows;
  wp.k_blocks = (int)((rows + 63) / 64);
  wp.m_pairs = Mout / 256;
  wp.n_tiles = (Kin + N - 1) / N;
  const int tiles = wp.m_pairs * wp.n_tiles;
  const int npairs = h->sm_count / 2;
  wp.splits = std::max(1, std::min(npairs / tiles, wp.k_blocks));
  wp.kb_per_split = (wp.k_blocks + wp.splits - 1) / wp.splits;
  wp.nplanes = T.nplanes;
  const int units = tiles * wp.splits;
  ctm_status s = ensure(T.wpart, T.wpart_elems, (size_t)units * 256 * N);
  if (s != CTM_OK) return s;
  wp.part = T.wpart;
  CUtensorMap mz, mb;
  if (!make_map3(&mz, Z.p, (uint64_t)Mout, (uint64_t)rows, Z.cap, 64) ||
      !make_map3(&mb, B.p, (uint64_t)Kin, (uint64_t)rows, B.cap, 64))
    return fail(CTM_ECUDA, "cuTensorMapEncodeTiled failed for the weight-gradient operands");
  const int grid = 2 * std::min(units, npairs);
  {
    ProfScope ps(h, CTM_KIND_WGRAD, 2.0 * (double)T.N * T.P * rows_out * cols_in, st);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = ctm::kWgradSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto* kern = N == 256 ? (f16 ? ctm::wgrad_kernel<256, true> : ctm::wgrad_kernel<256, false>)
                          : (f16 ? ctm::wgrad_kernel<128, true> : ctm::wgrad_kernel<128, false>);
    const int ai = (N == 256 ? 1 : 0) + (f16 ? 2 : 0);
    if (!h->wgrad_attr[ai]) {
      CTM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ctm::kWgradSmem));
      h->wgrad_attr[ai] = true;
    }
    CTM_CUDA(cudaLaunchKernelEx(&cfg, kern, mz, mb, wp));
  }
  {
    const int64_t n = (int64_t)rows_out * cols_in;
    ProfScope ps(h, CTM_KIND_BAUX, 0.0, st);
    ctm::wgrad_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(T.wpart, N, wp.n_tiles, wp.splits, rows_out,
                                                                        cols_in, dW, acc, zrec, brec);
  }
  h->last_launches += 2;
  return CTM_OK;
}

// out[m] (=|+=) sum_n Zb[n * P + 0, m] for m < ncols (the bias gradient: bias on slot 0 only)
ctm_status bias_grad(ctm_mlp* h, const Planes& Z, int ld, int ncols, float* out, int acc, cudaStream_t st,
                     const ctm::F16Rec* zrec = nullptr) {
  const int G = 1024;  // point groups: enough independent rows in flight per column
  ctm_status s = ensure(h->tape.part, h->tape.part_elems, (size_t)G * std::max(ncols, 1));
  if (s != CTM_OK) return s;
  ProfScope ps(h, CTM_KIND_BAUX, 0.0, st);
  h->last_launches += 2;
  ctm::colsum_kernel<<<dim3((ncols + 127) / 128, G), 128, 0, st>>>(Z.p, (int64_t)Z.cap, h->tape.nplanes, nullptr,
                                                                   h->tape.N, h->tape.P, ld, ncols, G, h->tape.part,
                                                                   zrec);
  ctm::reduce_groups_kernel<<<(ncols + 31) / 32, dim3(32, 32), 0, st>>>(h->tape.part, G, ncols, ncols, out, acc);
  return CTM_OK;
}

ctm_status backward(ctm_mlp* h, const float* gop, const float* gf, float* const* dW, float* const* db, int acc,
                    cudaStream_t st) {
  auto& T = h->tape;
  const int L = h->L, P = T.P;
  const int64_t N = T.N, rows = N * (int64_t)P;
  int ldmax = 0;
  for (int l = 1; l <= L - 1; ++l) ldmax = std::max(ldmax, h->wpad[l]);
  ctm_status s;
  for (int i = 0; i < 2; ++i) {
    s = ensure_planes(T.Zb[i], (size_t)rows * ldmax);
    if (s != CTM_OK) return s;
  }
  const float* jw = T.weighted ? T.weights : nullptr;
  h->last_launches = 0;
  const bool f16 = T.f16;
  // fp16x3 records: the adjoint blocks' scales (f16zrec), the bounds of the backward seeds and
  // of the saved pre-activations (backward.cuh f16_bwd_prep_kernel)
  float s0 = 1.f, s1 = 1.f, s2 = 1.f, s3 = 1.f, s4 = 1.f;
  if (f16) {
    f16_act_sups(h->act, s0, s1, s2, s3, s4);
    ProfScope ps(h, CTM_KIND_BAUX, 0.0, st);
    CTM_CUDA(cudaMemsetAsync(h->f16zrec, 0, sizeof(ctm::F16Rec) * (L + 1), st));
    CTM_CUDA(cudaMemsetAsync(h->f16b + 5, 0, sizeof(unsigned) * 2, st));  // max |gop|, max |gf|
    launch_maxabs(gop, N, h->f16b + 5, st);
    if (gf) launch_maxabs(gf, N, h->f16b + 6, st);
    ctm::f16_bwd_prep_kernel<<<1, 1024, 0, st>>>(h->f16b + 5, gf != nullptr, h->w_out, h->wpad[L - 1], T.scale, jw,
                                                 P - 2, h->f16b, T.random ? 1 : 0, h->f16w, h->f16rec, L, h->f16bb,
                                                 h->f16zb);
    h->last_launches += gf ? 3 : 2;
  }
  auto zrec = [&](int l) -> const ctm::F16Rec* { return f16 ? h->f16zrec + l : nullptr; };
  auto brec = [&](int l) -> const ctm::F16Rec* { return f16 ? h->f16rec + l : nullptr; };
  // ---- readout and the last hidden rule, transposed
  {
    ProfScope ps(h, CTM_KIND_BAUX, 0.0, st);
    h->last_launches += 3;
    const int G = 2048, w = h->wpad[L - 1];  // point groups of top_bwd_kernel (dW_L partial rows)
    s = ensure(T.part, T.part_elems, (size_t)G * w);
    if (s != CTM_OK) return s;
    ctm::TopBwdParams tp{};
    tp.Z = T.Z[L - 1];
    tp.ldz = w;
    tp.P = P;
    tp.N = N;
    tp.width = w;
    tp.w_out = h->w_out;
    tp.c = T.scale;
    tp.gop = gop;
    tp.gf = gf;
    tp.jw = jw;
    tp.act = h->act;
    tp.out = T.Zb[0].p;
    tp.pstride = (int64_t)T.Zb[0].cap;
    tp.nplanes = T.nplanes;
    tp.ldo = w;
    tp.dw_part = T.part;
    tp.G = G;
    if (f16) {
      tp.zb = h->f16zb + 2 * (L - 1);
      tp.bb = h->f16bb;
      tp.s1 = s1, tp.s2 = s2, tp.s3 = s3;
      tp.f16_out = h->f16zrec + (L - 1);
      ctm::top_bwd_kernel<true><<<dim3((w + 511) / 512, G), 128, 0, st>>>(tp);
    } else {
      ctm::top_bwd_kernel<false><<<dim3((w + 511) / 512, G), 128, 0, st>>>(tp);
    }
    // part rows have stride w (padded); only the widths[L-1] real columns reach dW_L
    ctm::reduce_groups_kernel<<<(h->widths[L - 1] + 31) / 32, dim3(32, 32), 0, st>>>(T.part, G, w, h->widths[L - 1],
                                                                                    dW[L - 1], acc);
    if (gf)
      ctm::vector_sum_kernel<<<1, 256, 0, st>>>(gf, N, db[L - 1], acc);
    else if (!acc)
      CTM_CUDA(cudaMemsetAsync(db[L - 1], 0, sizeof(float), st));
  }
  // ---- hidden layers L-1 .. 2: weight gradients, then the adjoint of the previous layer
  int cur = 0;
  for (int l = L - 1; l >= 2; --l) {
    const int Mout = h->wpad[l], Kin = h->wpad[l - 1];
    s = weight_grad(h, T.B[l - 1], Kin, T.Zb[cur], Mout, rows, h->widths[l], h->widths[l - 1], dW[l - 1], acc, st,
                    zrec(l), brec(l - 1));
    if (s != CTM_OK) return s;
    s = bias_grad(h, T.Zb[cur], Mout, h->widths[l], db[l - 1], acc, st, zrec(l));
    if (s != CTM_OK) return s;
    // Z_bar_{l-1} = rule^T( (Z_bar_l W_l)^T ) on the tensor cores (jet_layer_kernel<kBwd2>)
    CUtensorMap mb;
    if (!make_map3(&mb, T.Zb[cur].p, (uint64_t)Mout, (uint64_t)rows, T.Zb[cur].cap, (uint32_t)T.nmma / 2))
      return fail(CTM_ECUDA, "cuTensorMapEncodeTiled failed for the adjoint block");
    ctm::LayerParams lp{};
    lp.bias = nullptr;
    lp.act = h->act;
    lp.out = T.Zb[cur ^ 1].p;
    lp.pstride = (int64_t)T.Zb[cur ^ 1].cap;
    lp.nplanes = (int16_t)T.nplanes;
    lp.ldo = Kin;
    lp.m_tiles = Kin / ctm::kBM;
    lp.n_points = N;
    lp.P = P;
    lp.pts_per_tile = T.ppt;
    lp.n_mma = T.nmma;
    lp.k_iters = Mout / ctm::kBK;
    lp.jet_w = jw;
    lp.J = T.J;
    lp.blocks = 1;
    lp.rb = std::max(T.J, 1);
    lp.weighted = T.weighted;
    lp.z_in = T.Z[l - 1];
    lp.ldzi = Kin;
    const int64_t n_tiles = (N + T.ppt - 1) / T.ppt;
    const int64_t grid = 2 * std::min<int64_t>(n_tiles * (lp.m_tiles / 2), h->sm_count / 2);
    {
      ProfScope ps(h, CTM_KIND_BWD, 2.0 * N * P * h->widths[l - 1] * h->widths[l], st);
      ++h->last_launches;
      if (f16) {  // fp16x3: W_l^T fp16 planes, Z_bar_l's record in, Z_bar_{l-1}'s out (one scale)
        ctm::F16Args fa{};
        fa.in = h->f16zrec + l;
        fa.out = h->f16zrec + (l - 1);
        fa.wsc = h->f16wT + 2 * l;
        fa.s0 = s0, fa.s1 = s1, fa.s2 = s2, fa.s3 = s3, fa.s4 = s4;
        fa.uniform = 1;
        fa.zb = h->f16zb + 2 * (l - 1);
        fa.bb = h->f16bb;
        s = launch_layer_kernel<ctm::kBwd2, 0>(h, grid, h->mapAT16[l - 2], mb, lp, st, fa);
      } else {
        s = launch_layer_kernel<ctm::kBwd2, 0>(h, grid, h->mapAT[l - 2], mb, lp, st);
      }
      if (s != CTM_OK) return s;
    }
    cur ^= 1;
  }
  // ---- layer 1: dW_1 = Z_bar_1^T B_0 (B_0 = [x0; u_r; 0]), db_1
  s = weight_grad(h, T.B[0], h->k1pad, T.Zb[cur], h->wpad[1], rows, h->widths[1], h->widths[0], dW[0], acc, st,
                  zrec(1), brec(0));
  if (s != CTM_OK) return s;
  s = bias_grad(h, T.Zb[cur], h->wpad[1], h->widths[1], db[0], acc, st, zrec(1));
  if (s != CTM_OK) return s;
  CTM_CUDA(cudaGetLastError());
  return CTM_OK;
}

// Every array derived from the weights, written on `st` (load and ctm_set_weights):
// fp16x3 weight planes and statistics of every tensor-core layer (layer 1's W1p and the
// hidden GEMM layers), from their bf16 planes (seed.cuh split_weights_f16_kernel)
// grad mode: W_l^T of the fp16x3 planes (the adjoint's A operand) and ||W_l^T||_inf
void derive_f16_transposed(ctm_mlp* h, cudaStream_t st) {
  for (size_t i = 0; i < h->WTp16.size(); ++i) {
    const int l = (int)i + 2, mpad = h->wpad[l], kpad = h->wpad[l - 1];
    const int64_t n = (int64_t)mpad * kpad;
    ctm::transpose_planes_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(h->Wp16[i], mpad, kpad, h->WTp16[i]);
  }
}
void derive_f16_weights(ctm_mlp* h, cudaStream_t st) {
  const int L = h->L, ld1 = h->wpad[1];
  {
    const int64_t n = (int64_t)ld1 * h->k1pad;
    cudaMemsetAsync(h->f16acc, 0, sizeof(unsigned) * 3 * (L + 1), st);
    ctm::f16_weight_norms_kernel<<<(unsigned)((ld1 * 32 + 255) / 256), 256, 0, st>>>(h->W1p, ld1, h->k1pad, 0,
                                                                                    h->f16acc + 3);
    ctm::f16_weight_stats_kernel<<<1, 1, 0, st>>>(h->f16acc + 3, h->f16w + 2, nullptr);
    ctm::split_weights_f16_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(h->W1p, n, h->f16w + 2, h->W1p16);
  }
  for (int l = 2; l <= L - 1; ++l) {
    const int mpad = h->wpad[l], kpad = h->wpad[l - 1];
    const int64_t n = (int64_t)mpad * kpad;
    const bool tr = !h->WTp16.empty();  // grad mode: ||W^T||_inf for the adjoint too
    const int thr = std::max(mpad * 32, tr ? kpad : 0);
    ctm::f16_weight_norms_kernel<<<(unsigned)((thr + 255) / 256), 256, 0, st>>>(h->Wp[l - 2], mpad, kpad, tr ? 1 : 0,
                                                                               h->f16acc + 3 * l);
    ctm::f16_weight_stats_kernel<<<1, 1, 0, st>>>(h->f16acc + 3 * l, h->f16w + 2 * l,
                                                  tr ? h->f16wT + 2 * l : nullptr);
    ctm::split_weights_f16_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(h->Wp[l - 2], n, h->f16w + 2 * l,
                                                                               h->Wp16[l - 2]);
  }
  derive_f16_transposed(h, st);
  h->f16_stale = false;
}

// W1^T and b1, the bf16 pairs of every tensor-core layer (and W_l^T in grad mode), the
// padded output weights, and the fixed direction sets' U = W1 V, c = sum w (W1 v)^K.
void derive_weights(ctm_mlp* h, const float* const* W, const float* const* b, cudaStream_t st) {
  const int L = h->L, D = h->widths[0], ld1 = h->wpad[1];
  {
    const int64_t n = (int64_t)D * ld1;
    ctm::transpose_w1_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(W[0], b[0], h->widths[1], D, ld1, h->W1T,
                                                                          h->b1);
  }
  {
    const int64_t n = (int64_t)ld1 * h->k1pad;
    ctm::split_weights_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(W[0], b[0], h->widths[1], D, ld1, h->k1pad,
                                                                           h->W1p, h->b1);
  }
  for (int l = 2; l <= L - 1; ++l) {
    const int mpad = h->wpad[l], kpad = h->wpad[l - 1];
    const int64_t n = (int64_t)mpad * kpad;
    ctm::split_weights_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        W[l - 1], b[l - 1], h->widths[l], h->widths[l - 1], mpad, kpad, h->Wp[l - 2], h->bias[l - 2]);
    if (!h->WTp.empty())
      ctm::transpose_planes_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(h->Wp[l - 2], mpad, kpad,
                                                                                h->WTp[l - 2]);
  }
  {
    const int lpad = h->wpad[L - 1];
    ctm::pad_vector_kernel<<<(lpad + 255) / 256, 256, 0, st>>>(W[L - 1], h->widths[L - 1], lpad, h->w_out);
    cudaMemcpyAsync(h->b_out, b[L - 1], sizeof(float), cudaMemcpyDeviceToDevice, st);
  }
  ctm::prep_laplacian_kernel<<<(ld1 + 127) / 128, 128, 0, st>>>(h->W1T, D, ld1, h->U_lap, h->c_lap);
  if (h->J_bih)
    ctm::prep_directions_kernel<<<(ld1 + 127) / 128, 128, 0, st>>>(h->W1T, D, ld1, h->bih_dirs, h->J_bih, h->w_bih, 4,
                                                                   h->U_bih, h->c_bih);
  h->last_launches = 4 + (L - 2) * (h->WTp.empty() ? 1 : 2) + (h->J_bih ? 1 : 0);
  // the fp16x3 weights follow (after the bf16 planes, from which they are derived) only if
  // the handle is in that mode; otherwise they are rebuilt when it switches to it
  if (h->prec == CTM_PRECISION_FP16X3) {
    derive_f16_weights(h, st);
    h->last_launches += 3 * (L - 1) + (int)h->WTp16.size();
  } else {
    h->f16_stale = true;
  }
  h->tape.valid = false;
}

ctm_status check_common(ctm_mlp* h, const float* X, int64_t N, float* op_out, float* f_out) {
  if (!h) return fail(CTM_EINVAL, "NULL handle");
  if (N < 0) return fail(CTM_EINVAL, "N < 0");
  if (N > 0 && (!X || !op_out)) return fail(CTM_EINVAL, "NULL X or op_out");
  if ((X && !aligned16(X)) || (op_out && !aligned16(op_out)) || (f_out && !aligned16(f_out)))
    return fail(CTM_ESHAPE, "pointers must be 16-byte aligned");
  return CTM_OK;
}

}  // namespace

extern "C" {

const char* ctm_status_str(ctm_status s) {
  switch (s) {
    case CTM_OK: return "CTM_OK";
    case CTM_EINVAL: return "CTM_EINVAL";
    case CTM_ESHAPE: return "CTM_ESHAPE";
    case CTM_ENOMEM: return "CTM_ENOMEM";
    case CTM_ECUDA: return "CTM_ECUDA";
    case CTM_EUNSUPPORTED: return "CTM_EUNSUPPORTED";
  }
  return "CTM_UNKNOWN";
}

const char* ctm_last_error(void) { return g_last_error.c_str(); }

ctm_status ctm_load_mlp(int32_t n_layers, const int32_t* widths, const float* const* W, const float* const* b,
                        int32_t device, ctm_mlp_t* out) {
  g_last_error.clear();
  if (!out) return fail(CTM_EINVAL, "NULL out");
  *out = nullptr;
  if (n_layers < 2 || !widths || !W || !b) return fail(CTM_EINVAL, "need n_layers >= 2 and non-NULL widths/W/b");
  for (int l = 0; l <= n_layers; ++l)
    if (widths[l] < 1) return fail(CTM_EINVAL, "width < 1");
  if (widths[n_layers] != 1) return fail(CTM_EUNSUPPORTED, "only scalar-output MLPs (widths[L] == 1)");
  if (widths[0] > kMaxD) return fail(CTM_EUNSUPPORTED, "input dimension D > 4096");
  for (int l = 1; l < n_layers; ++l)
    if (widths[l] > 8192) return fail(CTM_EUNSUPPORTED, "hidden width > 8192");
  for (int l = 0; l < n_layers; ++l)
    if (!W[l] || !b[l] || !aligned16(W[l]) || !aligned16(b[l]))
      return fail(W[l] && b[l] ? CTM_ESHAPE : CTM_EINVAL, "weights must be non-NULL and 16-byte aligned");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(CTM_ECUDA, "no such CUDA device");
  if (!get_encode()) return fail(CTM_ECUDA, "cuTensorMapEncodeTiled unavailable");

  ctm_mlp* h = new ctm_mlp();
  h->device = device;
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device);
  h->L = n_layers;
  h->widths.assign(widths, widths + n_layers + 1);
  h->wpad.assign(n_layers + 1, 0);
  for (int l = 1; l < n_layers; ++l) h->wpad[l] = round_up(widths[l], 2 * ctm::kBM);  // CTA-pair M tile
  DeviceGuard g(device);
  const int D = widths[0], ld1 = h->wpad[1];
  auto bail = [&](ctm_status s) {
    free_all(h);
    delete h;
    return s;
  };
#define LOAD_CUDA(call)                                                                       \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      fail(e_ == cudaErrorMemoryAllocation ? CTM_ENOMEM : CTM_ECUDA,                          \
           std::string(#call) + ": " + cudaGetErrorString(e_));                               \
      return bail(e_ == cudaErrorMemoryAllocation ? CTM_ENOMEM : CTM_ECUDA);                  \
    }                                                                                         \
  } while (0)

  // ---- allocations and tensor maps (the values are written by derive_weights)
  h->k1pad = round_up(D, ctm::kBK);
  LOAD_CUDA(cudaMalloc(&h->W1T, sizeof(float) * (size_t)D * ld1));
  LOAD_CUDA(cudaMalloc(&h->b1, sizeof(float) * ld1));
  LOAD_CUDA(cudaMalloc(&h->W1p, 3 * sizeof(uint16_t) * (size_t)ld1 * h->k1pad));
  if (!make_map3(&h->mapA1, h->W1p, h->k1pad, ld1, (uint64_t)ld1 * h->k1pad, ctm::kBM)) {
    fail(CTM_ECUDA, "cuTensorMapEncodeTiled failed for W1");
    return bail(CTM_ECUDA);
  }
  for (int l = 2; l <= n_layers - 1; ++l) {
    const int mpad = h->wpad[l], kpad = h->wpad[l - 1];
    uint16_t* wp;
    float* bp;
    LOAD_CUDA(cudaMalloc(&wp, 3 * sizeof(uint16_t) * (size_t)mpad * kpad));
    h->Wp.push_back(wp);
    LOAD_CUDA(cudaMalloc(&bp, sizeof(float) * mpad));
    h->bias.push_back(bp);
    CUtensorMap mw;
    if (!make_map3(&mw, wp, kpad, mpad, (uint64_t)mpad * kpad, ctm::kBM)) {
      fail(CTM_ECUDA, "cuTensorMapEncodeTiled failed for weights");
      return bail(CTM_ECUDA);
    }
    h->mapA.push_back(mw);
  }
  {  // fp16x3 mode: fp16 weight planes, their statistics, the per-call scale records
    LOAD_CUDA(cudaMalloc(&h->W1p16, 3 * sizeof(uint16_t) * (size_t)ld1 * h->k1pad));
    if (!make_map3(&h->mapA1_16, h->W1p16, h->k1pad, ld1, (uint64_t)ld1 * h->k1pad, ctm::kBM)) {
      fail(CTM_ECUDA, "cuTensorMapEncodeTiled failed for W1 (fp16)");
      return bail(CTM_ECUDA);
    }
    for (int l = 2; l <= n_layers - 1; ++l) {
      const int mpad = h->wpad[l], kpad = h->wpad[l - 1];
      uint16_t* wp;
      LOAD_CUDA(cudaMalloc(&wp, 3 * sizeof(uint16_t) * (size_t)mpad * kpad));
      h->Wp16.push_back(wp);
      CUtensorMap mw;
      if (!make_map3(&mw, wp, kpad, mpad, (uint64_t)mpad * kpad, ctm::kBM)) {
        fail(CTM_ECUDA, "cuTensorMapEncodeTiled failed for weights (fp16)");
        return bail(CTM_ECUDA);
      }
      h->mapA16.push_back(mw);
    }
    LOAD_CUDA(cudaMalloc(&h->f16w, sizeof(float) * 2 * (n_layers + 1)));
    LOAD_CUDA(cudaMalloc(&h->f16rec, sizeof(ctm::F16Rec) * (n_layers + 1)));
    LOAD_CUDA(cudaMalloc(&h->f16b, sizeof(unsigned) * 8));
    LOAD_CUDA(cudaMalloc(&h->f16wT, sizeof(float) * 2 * (n_layers + 1)));
    LOAD_CUDA(cudaMalloc(&h->f16zrec, sizeof(ctm::F16Rec) * (n_layers + 1)));
    LOAD_CUDA(cudaMalloc(&h->f16bb, sizeof(float) * 4));
    LOAD_CUDA(cudaMalloc(&h->f16zb, sizeof(float) * 2 * (n_layers + 1)));
    LOAD_CUDA(cudaMalloc(&h->f16acc, sizeof(unsigned) * 3 * (n_layers + 1)));
  }
  LOAD_CUDA(cudaMalloc(&h->w_out, sizeof(float) * h->wpad[n_layers - 1]));
  LOAD_CUDA(cudaMalloc(&h->b_out, sizeof(float)));
  {  // fixed direction sets: the Laplacian's e_d and, for D <= 36, the biharmonic family
    LOAD_CUDA(cudaMalloc(&h->U_lap, sizeof(float) * (size_t)D * ld1));
    LOAD_CUDA(cudaMalloc(&h->c_lap, sizeof(float) * ld1));
    if (D * (3 * D - 1) / 2 <= ctm::kMaxW) {  // the jet weights of all blocks live in smem
      std::vector<float> dirs, w;
      biharmonic_family(D, dirs, w);
      h->J_bih = (int)w.size();
      LOAD_CUDA(cudaMalloc(&h->bih_dirs, sizeof(float) * dirs.size()));
      LOAD_CUDA(cudaMemcpy(h->bih_dirs, dirs.data(), sizeof(float) * dirs.size(), cudaMemcpyHostToDevice));
      LOAD_CUDA(cudaMalloc(&h->w_bih, sizeof(float) * w.size()));
      LOAD_CUDA(cudaMemcpy(h->w_bih, w.data(), sizeof(float) * w.size(), cudaMemcpyHostToDevice));
      LOAD_CUDA(cudaMalloc(&h->U_bih, sizeof(float) * (size_t)h->J_bih * ld1));
      LOAD_CUDA(cudaMalloc(&h->c_bih, sizeof(float) * ld1));
    }
  }
  {
    std::vector<float> ones(ctm::kMaxW, 1.f);
    LOAD_CUDA(cudaMalloc(&h->w_ones, sizeof(float) * ones.size()));
    LOAD_CUDA(cudaMemcpy(h->w_ones, ones.data(), sizeof(float) * ones.size(), cudaMemcpyHostToDevice));
  }
  derive_weights(h, W, b, 0);
  LOAD_CUDA(cudaGetLastError());
  LOAD_CUDA(cudaDeviceSynchronize());
#undef LOAD_CUDA
  *out = h;
  return CTM_OK;
}

ctm_status ctm_free_mlp(ctm_mlp_t mlp) {
  if (!mlp) return CTM_OK;
  {
    DeviceGuard g(mlp->device);
    cudaDeviceSynchronize();
  }
  free_all(mlp);
  delete mlp;
  return CTM_OK;
}

ctm_status ctm_laplacian(ctm_mlp_t mlp, const float* X, int64_t N, float* op_out, float* f_out, void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  CallArgs a{OP_LAP, X, N, nullptr, 0, 0, nullptr, 0, 0, 0, 0, op_out, f_out, (cudaStream_t)stream};
  return run(mlp, a);
}

ctm_status ctm_laplacian_standard(ctm_mlp_t mlp, const float* X, int64_t N, float* op_out, float* f_out,
                                  void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  CallArgs a{OP_LAP_STD, X, N, nullptr, 0, 0, nullptr, 0, 0, 0, 0, op_out, f_out, (cudaStream_t)stream};
  return run(mlp, a);
}

ctm_status ctm_weighted_laplacian(ctm_mlp_t mlp, const float* X, int64_t N, const float* sigma, int32_t R,
                                  float* op_out, float* f_out, void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  if (R < 1 || !sigma) return fail(CTM_EINVAL, "need sigma and R >= 1");
  if (!aligned16(sigma)) return fail(CTM_ESHAPE, "sigma must be 16-byte aligned");
  CallArgs a{OP_WLAP, X, N, sigma, R, 0, nullptr, 0, 0, 0, 0, op_out, f_out, (cudaStream_t)stream};
  return run(mlp, a);
}

ctm_status ctm_randomized_laplacian(ctm_mlp_t mlp, const float* X, int64_t N, int32_t S, const float* V,
                                    ctm_dist dist, uint64_t seed, int64_t point_offset, const float* sigma,
                                    int32_t Rv, float* op_out, float* f_out, void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  if (S < 1 || Rv < 1 || point_offset < 0) return fail(CTM_EINVAL, "need S >= 1, Rv >= 1, point_offset >= 0");
  if (dist != CTM_RADEMACHER && dist != CTM_GAUSSIAN) return fail(CTM_EINVAL, "bad dist");
  if (!sigma && Rv != mlp->widths[0]) return fail(CTM_ESHAPE, "Rv must equal D when sigma is NULL");
  if ((V && !aligned16(V)) || (sigma && !aligned16(sigma))) return fail(CTM_ESHAPE, "V/sigma must be 16-byte aligned");
  if (Rv > kMaxD) return fail(CTM_EUNSUPPORTED, "Rv > 4096");
  CallArgs a{OP_RLAP, X, N, sigma, 0, S, V, seed, point_offset, Rv, dist == CTM_GAUSSIAN, op_out, f_out,
             (cudaStream_t)stream};
  return run(mlp, a);
}

ctm_status ctm_randomized_laplacian_standard(ctm_mlp_t mlp, const float* X, int64_t N, int32_t S, const float* V,
                                             ctm_dist dist, uint64_t seed, int64_t point_offset, const float* sigma,
                                             int32_t Rv, float* op_out, float* f_out, void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  if (S < 1 || Rv < 1 || point_offset < 0) return fail(CTM_EINVAL, "need S >= 1, Rv >= 1, point_offset >= 0");
  if (dist != CTM_RADEMACHER && dist != CTM_GAUSSIAN) return fail(CTM_EINVAL, "bad dist");
  if (!sigma && Rv != mlp->widths[0]) return fail(CTM_ESHAPE, "Rv must equal D when sigma is NULL");
  if ((V && !aligned16(V)) || (sigma && !aligned16(sigma))) return fail(CTM_ESHAPE, "V/sigma must be 16-byte aligned");
  if (Rv > kMaxD) return fail(CTM_EUNSUPPORTED, "Rv > 4096");
  CallArgs a{OP_RLAP_STD, X, N, sigma, 0, S, V, seed, point_offset, Rv, dist == CTM_GAUSSIAN, op_out, f_out,
             (cudaStream_t)stream};
  return run(mlp, a);
}

ctm_status ctm_stochastic_biharmonic_standard(ctm_mlp_t mlp, const float* X, int64_t N, int32_t S, const float* V,
                                              ctm_dist dist, uint64_t seed, int64_t point_offset, float* op_out,
                                              float* f_out, void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  if (S < 1 || point_offset < 0) return fail(CTM_EINVAL, "need S >= 1 and point_offset >= 0");
  if (dist != CTM_GAUSSIAN)
    return fail(CTM_EINVAL, "the stochastic biharmonic needs standard normal directions (CTM_GAUSSIAN)");
  if (V && !aligned16(V)) return fail(CTM_ESHAPE, "V must be 16-byte aligned");
  if (mlp->widths[0] > kMaxD) return fail(CTM_EUNSUPPORTED, "D > 4096");
  CallArgs a{OP_SBIH_STD, X, N, nullptr, 0, S, V, seed, point_offset, mlp->widths[0], 1, op_out, f_out,
             (cudaStream_t)stream};
  return run(mlp, a);
}

ctm_status ctm_biharmonic(ctm_mlp_t mlp, const float* X, int64_t N, float* op_out, float* f_out, void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  if (mlp->J_bih == 0)
    return fail(CTM_EUNSUPPORTED, "biharmonic needs J = D(3D-1)/2 <= 2048 jets, i.e. D <= 36");
  CallArgs a{OP_BIH, X, N, nullptr, 0, 0, nullptr, 0, 0, 0, 0, op_out, f_out, (cudaStream_t)stream};
  return run(mlp, a);
}

ctm_status ctm_biharmonic_standard(ctm_mlp_t mlp, const float* X, int64_t N, float* op_out, float* f_out,
                                   void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  if (mlp->J_bih == 0)
    return fail(CTM_EUNSUPPORTED, "biharmonic needs J = D(3D-1)/2 <= 2048 jets, i.e. D <= 36");
  CallArgs a{OP_BIH_STD, X, N, nullptr, 0, 0, nullptr, 0, 0, 0, 0, op_out, f_out, (cudaStream_t)stream};
  return run(mlp, a);
}

ctm_status ctm_biharmonic_nested(ctm_mlp_t mlp, const float* X, int64_t N, float* op_out, float* f_out,
                                 void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  if (mlp->widths[0] > ctm::kNestMaxD)
    return fail(CTM_EUNSUPPORTED, "nested biharmonic needs 2 + 2D + D(D+1)/2 <= 256 slots, i.e. D <= 20");
  CallArgs a{OP_BIH_NEST, X, N, nullptr, 0, 0, nullptr, 0, 0, 0, 0, op_out, f_out, (cudaStream_t)stream};
  return run(mlp, a);
}

ctm_status ctm_directional_sum(ctm_mlp_t mlp, const float* X, int64_t N, int32_t K, int32_t J, const float* dirs,
                               int32_t per_point, const float* weights, float* op_out, float* f_out, void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  if (K != 2 && K != 4) return fail(CTM_EUNSUPPORTED, "K must be 2 or 4");
  if (J < 1 || !weights || (!dirs && !(per_point && N == 0))) return fail(CTM_EINVAL, "need J >= 1, dirs and weights");
  if (!aligned16(dirs) || !aligned16(weights)) return fail(CTM_ESHAPE, "dirs/weights must be 16-byte aligned");
  if (mlp->widths[0] > kMaxD) return fail(CTM_EUNSUPPORTED, "D > 4096");
  CallArgs a{OP_DSUM, X, N, nullptr, 0, per_point ? J : 0, per_point ? dirs : nullptr, 0, 0, mlp->widths[0], 0,
             op_out, f_out, (cudaStream_t)stream};
  a.K = K;
  a.J = J;
  a.dirs = dirs;
  a.per_point = per_point != 0;
  a.weights = weights;
  return run(mlp, a);
}

ctm_status ctm_weighted_laplacian_pointwise(ctm_mlp_t mlp, const float* X, int64_t N, const float* sigma_x, int32_t R,
                                            float* op_out, float* f_out, void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  if (R < 1 || (!sigma_x && N > 0)) return fail(CTM_EINVAL, "need sigma_x and R >= 1");
  if (!aligned16(sigma_x)) return fail(CTM_ESHAPE, "sigma_x must be 16-byte aligned");
  if (mlp->widths[0] > kMaxD) return fail(CTM_EUNSUPPORTED, "D > 4096");
  CallArgs a{OP_WLAP_X, X, N, nullptr, 0, R, sigma_x, 0, 0, mlp->widths[0], 0, op_out, f_out, (cudaStream_t)stream};
  a.v_trans = 1;
  return run(mlp, a);
}

ctm_status ctm_set_activation(ctm_mlp_t mlp, ctm_activation act) {
  g_last_error.clear();
  if (!mlp) return fail(CTM_EINVAL, "NULL handle");
  if (act != CTM_ACT_TANH && act != CTM_ACT_IDENTITY && act != CTM_ACT_SQUARE && act != CTM_ACT_SIN &&
      act != CTM_ACT_EXP)
    return fail(CTM_EINVAL, "unknown activation");
  static_assert(CTM_ACT_TANH == ctm::kActTanh && CTM_ACT_IDENTITY == ctm::kActIdentity &&
                    CTM_ACT_SQUARE == ctm::kActSquare && CTM_ACT_SIN == ctm::kActSin && CTM_ACT_EXP == ctm::kActExp,
                "ABI activation codes");
  mlp->act = (int)act;
  mlp->tape.valid = false;  // the backward reads the activation: a tape of another one is stale
  return CTM_OK;
}

ctm_status ctm_set_precision(ctm_mlp_t mlp, ctm_precision prec) {
  g_last_error.clear();
  if (!mlp) return fail(CTM_EINVAL, "NULL handle");
  if (prec != CTM_PRECISION_FP32 && prec != CTM_PRECISION_BF16X3 && prec != CTM_PRECISION_FP16X3)
    return fail(CTM_EINVAL, "unknown precision");
  mlp->prec = prec;
  mlp->nplanes = (prec == CTM_PRECISION_FP32) ? 3 : 2;
  if (prec == CTM_PRECISION_FP16X3 && mlp->f16_stale) {  // host-side call: build and wait
    DeviceGuard g(mlp->device);
    derive_f16_weights(mlp, 0);
    CTM_CUDA(cudaDeviceSynchronize());
  }
  mlp->tape.valid = false;
  return CTM_OK;
}

ctm_status ctm_set_weights(ctm_mlp_t mlp, const float* const* W, const float* const* b, void* stream) {
  g_last_error.clear();
  if (!mlp) return fail(CTM_EINVAL, "NULL handle");
  if (!W || !b) return fail(CTM_EINVAL, "NULL W/b arrays");
  for (int l = 0; l < mlp->L; ++l)
    if (!W[l] || !b[l] || !aligned16(W[l]) || !aligned16(b[l]))
      return fail(W[l] && b[l] ? CTM_ESHAPE : CTM_EINVAL, "weights must be non-NULL and 16-byte aligned");
  DeviceGuard g(mlp->device);
  derive_weights(mlp, W, b, (cudaStream_t)stream);
  CTM_CUDA(cudaGetLastError());
  return CTM_OK;
}

ctm_status ctm_grad_enable(ctm_mlp_t mlp, int32_t enable) {
  g_last_error.clear();
  if (!mlp) return fail(CTM_EINVAL, "NULL handle");
  DeviceGuard g(mlp->device);
  mlp->tape.valid = false;
  mlp->grad = enable != 0;
  if (!mlp->grad || !mlp->WTp.empty()) return CTM_OK;
  // W_l^T as bf16 planes (the A operand of the adjoint GEMMs), from the split weights
  for (int l = 2; l <= mlp->L - 1; ++l) {
    const int mpad = mlp->wpad[l], kpad = mlp->wpad[l - 1];
    uint16_t* tp = nullptr;
    CTM_CUDA(cudaMalloc(&tp, 3 * sizeof(uint16_t) * (size_t)mpad * kpad));
    mlp->WTp.push_back(tp);
    const int64_t n = (int64_t)mpad * kpad;
    ctm::transpose_planes_kernel<<<(unsigned)((n + 255) / 256), 256>>>(mlp->Wp[l - 2], mpad, kpad, tp);
    CUtensorMap mt;
    if (!make_map3(&mt, tp, mpad, kpad, (uint64_t)n, ctm::kBM))
      return fail(CTM_ECUDA, "cuTensorMapEncodeTiled failed for W^T");
    mlp->mapAT.push_back(mt);
    uint16_t* tp16 = nullptr;  // fp16x3 training: the same for the fp16 planes
    CTM_CUDA(cudaMalloc(&tp16, 3 * sizeof(uint16_t) * (size_t)mpad * kpad));
    mlp->WTp16.push_back(tp16);
    if (!make_map3(&mt, tp16, mpad, kpad, (uint64_t)n, ctm::kBM))
      return fail(CTM_ECUDA, "cuTensorMapEncodeTiled failed for W^T (fp16)");
    mlp->mapAT16.push_back(mt);
  }
  if (!mlp->f16_stale) derive_f16_weights(mlp, 0);  // (||W^T||_inf and the transposed fp16 planes too)
  {
    std::vector<float> eye(256 * 256, 0.f);
    for (int i = 0; i < 256; ++i) eye[i * 257] = 1.f;
    CTM_CUDA(cudaMalloc(&mlp->eye, sizeof(float) * eye.size()));
    CTM_CUDA(cudaMemcpy(mlp->eye, eye.data(), sizeof(float) * eye.size(), cudaMemcpyHostToDevice));
  }
  CTM_CUDA(cudaDeviceSynchronize());
  return CTM_OK;
}

ctm_status ctm_backward(ctm_mlp_t mlp, const float* gop, const float* gf, float* const* dW, float* const* db,
                        int32_t accumulate, void* stream) {
  g_last_error.clear();
  if (!mlp) return fail(CTM_EINVAL, "NULL handle");
  if (!mlp->grad || !mlp->tape.valid)
    return fail(CTM_EUNSUPPORTED, "no differentiable call recorded (ctm_grad_enable, then a K=2 operator call)");
  if (!dW || !db) return fail(CTM_EINVAL, "NULL gradient arrays");
  for (int l = 0; l < mlp->L; ++l)
    if (!dW[l] || !db[l]) return fail(CTM_EINVAL, "NULL gradient pointer");
  if (mlp->tape.N > 0 && !gop) return fail(CTM_EINVAL, "NULL gop");
  if ((gop && !aligned16(gop)) || (gf && !aligned16(gf))) return fail(CTM_ESHAPE, "gop/gf must be 16-byte aligned");
  DeviceGuard g(mlp->device);
  if (mlp->tape.N == 0) {
    if (!accumulate)
      for (int l = 0; l < mlp->L; ++l) {
        CTM_CUDA(cudaMemsetAsync(dW[l], 0, sizeof(float) * mlp->widths[l] * mlp->widths[l + 1], (cudaStream_t)stream));
        CTM_CUDA(cudaMemsetAsync(db[l], 0, sizeof(float) * mlp->widths[l + 1], (cudaStream_t)stream));
      }
    return CTM_OK;
  }
  return backward(mlp, gop, gf, dW, db, accumulate != 0, (cudaStream_t)stream);
}

ctm_status ctm_gemm_probe(ctm_mlp_t mlp, int32_t layer, const float* B, int64_t rows, float* Z, void* stream) {
  g_last_error.clear();
  if (!mlp) return fail(CTM_EINVAL, "NULL handle");
  if (layer < 2 || layer > mlp->L - 1) return fail(CTM_EINVAL, "layer must be a hidden GEMM layer (2 .. L-1)");
  if (rows < 0 || (rows > 0 && (!B || !Z))) return fail(CTM_EINVAL, "need B, Z and rows >= 0");
  if ((B && !aligned16(B)) || (Z && !aligned16(Z))) return fail(CTM_ESHAPE, "B/Z must be 16-byte aligned");
  if (rows == 0) return CTM_OK;
  ctm_mlp* h = mlp;
  DeviceGuard g(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int w_in = h->widths[layer - 1], w_out = h->widths[layer];
  const int kpad = h->wpad[layer - 1], mpad = h->wpad[layer];
  constexpr int P = 16;  // slot rows per "point": 16 points fill an N = 256 tile
  const int64_t rows_pad = (rows + P - 1) / P * P;
  if (rows_pad > (int64_t)INT32_MAX) return fail(CTM_EUNSUPPORTED, "too many rows");
  ctm_status s = ensure_planes(h->probe_in, (size_t)rows_pad * kpad);
  if (s != CTM_OK) return s;
  s = ensure_planes(h->probe_out, (size_t)rows_pad * mpad);
  if (s != CTM_OK) return s;
  s = ensure(h->probe_z, h->probe_z_elems, (size_t)rows_pad * mpad);
  if (s != CTM_OK) return s;
  // the handle's precision (not the plane count of its last call)
  const bool f16 = (h->prec == CTM_PRECISION_FP16X3);
  h->nplanes = (h->prec == CTM_PRECISION_FP32) ? 3 : 2;
  ctm::F16Args fa{};
  {
    const int64_t n = rows_pad * kpad;
    if (f16) {  // one scale for every slot type: that of the measured max |B|
      CTM_CUDA(cudaMemsetAsync(h->f16rec, 0, sizeof(ctm::F16Rec) * 2, st));
      CTM_CUDA(cudaMemsetAsync(h->f16b, 0, sizeof(unsigned) * 8, st));
      launch_maxabs(B, rows * (int64_t)w_in, h->f16b, st);
      ctm::probe_f16_record_kernel<<<1, 1, 0, st>>>(h->f16b, h->f16rec);
      ctm::split_rows_f16_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
          B, rows, w_in, rows_pad, kpad, h->f16rec, h->probe_in.p, (int64_t)h->probe_in.cap);
      fa.in = h->f16rec;
      fa.out = h->f16rec + 1;
      fa.wsc = h->f16w + 2 * layer;
      f16_act_sups(h->act, fa.s0, fa.s1, fa.s2, fa.s3, fa.s4);
      fa.rw = (float)(P - 2);
    } else if (h->nplanes == 3) {
      ctm::split_rows_kernel<3><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(B, rows, w_in, rows_pad, kpad,
                                                                            h->probe_in.p, (int64_t)h->probe_in.cap);
    } else {
      ctm::split_rows_kernel<2><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(B, rows, w_in, rows_pad, kpad,
                                                                            h->probe_in.p, (int64_t)h->probe_in.cap);
    }
  }
  CUtensorMap mb;
  if (!make_map3(&mb, h->probe_in.p, (uint64_t)kpad, (uint64_t)rows_pad, h->probe_in.cap, 128))
    return fail(CTM_ECUDA, "cuTensorMapEncodeTiled failed for the probe block");
  ctm::LayerParams lp{};
  lp.bias = nullptr;
  lp.act = h->act;
  lp.out = h->probe_out.p;
  lp.pstride = (int64_t)h->probe_out.cap;
  lp.nplanes = (int16_t)h->nplanes;
  lp.ldo = mpad;
  lp.z_out = h->probe_z;
  lp.ldz = mpad;
  lp.m_tiles = mpad / ctm::kBM;
  lp.n_points = rows_pad / P;
  lp.P = P;
  lp.pts_per_tile = 256 / P;
  lp.n_mma = 256;
  lp.k_iters = kpad / ctm::kBK;
  lp.blocks = 1;
  lp.rb = P - 2;
  const int64_t n_tiles = (lp.n_points + lp.pts_per_tile - 1) / lp.pts_per_tile;
  const int64_t grid = 2 * std::min<int64_t>(n_tiles * (lp.m_tiles / 2), h->sm_count / 2);
  s = f16 ? launch_layer_instance<2, ctm::kFlagSaveZ | ctm::kFlagF16>(h, grid, h->mapA16[layer - 2], mb, lp, st, fa)
          : launch_layer_kernel<2, ctm::kFlagSaveZ>(h, grid, h->mapA[layer - 2], mb, lp, st);
  if (s != CTM_OK) return s;
  {
    const int64_t n = rows * (int64_t)w_out;
    ctm::crop_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(h->probe_z, mpad, (int)rows, w_out, Z, 0);
  }
  CTM_CUDA(cudaGetLastError());
  return CTM_OK;
}

ctm_status ctm_profile_enable(ctm_mlp_t mlp, int32_t enable) {
  if (!mlp) return fail(CTM_EINVAL, "NULL handle");
  DeviceGuard g(mlp->device);
  for (auto& r : mlp->recs) {
    cudaEventSynchronize(r.b);
    mlp->event_pool.push_back(r.a);
    mlp->event_pool.push_back(r.b);
  }
  mlp->recs.clear();
  mlp->profiling = enable != 0;
  return CTM_OK;
}

ctm_status ctm_profile_read(ctm_mlp_t mlp, double* ms, int64_t* launches, double* work) {
  if (!mlp) return fail(CTM_EINVAL, "NULL handle");
  DeviceGuard g(mlp->device);
  for (int k = 0; k < CTM_KIND_COUNT; ++k) {
    if (ms) ms[k] = 0.0;
    if (launches) launches[k] = 0;
    if (work) work[k] = 0.0;
  }
  for (auto& r : mlp->recs) {
    CTM_CUDA(cudaEventSynchronize(r.b));
    float t = 0.f;
    CTM_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    if (ms) ms[r.kind] += t;
    if (launches) launches[r.kind] += 1;
    if (work) work[r.kind] += r.work;
    mlp->event_pool.push_back(r.a);
    mlp->event_pool.push_back(r.b);
  }
  mlp->recs.clear();
  return CTM_OK;
}

ctm_status ctm_stochastic_biharmonic(ctm_mlp_t mlp, const float* X, int64_t N, int32_t S, const float* V,
                                     ctm_dist dist, uint64_t seed, int64_t point_offset, float* op_out, float* f_out,
                                     void* stream) {
  g_last_error.clear();
  ctm_status s = check_common(mlp, X, N, op_out, f_out);
  if (s != CTM_OK) return s;
  if (S < 1 || point_offset < 0) return fail(CTM_EINVAL, "need S >= 1 and point_offset >= 0");
  if (dist != CTM_GAUSSIAN)
    return fail(CTM_EINVAL, "the stochastic biharmonic needs standard normal directions (CTM_GAUSSIAN)");
  if (V && !aligned16(V)) return fail(CTM_ESHAPE, "V must be 16-byte aligned");
  if (mlp->widths[0] > kMaxD) return fail(CTM_EUNSUPPORTED, "D > 4096");
  CallArgs a{OP_SBIH, X, N, nullptr, 0, S, V, seed, point_offset, mlp->widths[0], 1, op_out, f_out,
             (cudaStream_t)stream};
  return run(mlp, a);
}

ctm_status ctm_set_direction_block(ctm_mlp_t mlp, int32_t rb) {
  g_last_error.clear();
  if (!mlp) return fail(CTM_EINVAL, "NULL handle");
  if (rb < 0) return fail(CTM_EINVAL, "rb < 0");
  mlp->forced_rb = rb;
  return CTM_OK;
}

ctm_status ctm_last_blocks(ctm_mlp_t mlp, int32_t* blocks, int32_t* per_block) {
  if (!mlp) return fail(CTM_EINVAL, "NULL handle");
  if (blocks) *blocks = mlp->last_nb;
  if (per_block) *per_block = mlp->last_rb;
  return CTM_OK;
}

ctm_status ctm_plan_blocks(int32_t order, int32_t R, int32_t forced_rb, int32_t* blocks, int32_t* per_block,
                           int32_t* slots_per_block, int32_t* points_per_tile, int32_t* mma_n) {
  g_last_error.clear();
  if ((order != 2 && order != 3 && order != 4 && order != 5) || R < 1 || forced_rb < 0)
    return fail(CTM_EINVAL, "need order 2, 3, 4 or 5, R >= 1 and forced_rb >= 0");
  const int KORD = (order == 3) ? ctm::kStd2 : (order == 5) ? ctm::kStd4 : order;
  const Plan pl = make_plan(KORD, R, forced_rb, true);
  if (pl.P == 0) return fail(CTM_EUNSUPPORTED, "no direction block fits a tile");
  if (blocks) *blocks = pl.nb;
  if (per_block) *per_block = pl.rb;
  if (slots_per_block) *slots_per_block = pl.P;
  if (points_per_tile) *points_per_tile = pl.ppt;
  if (mma_n) *mma_n = pl.nmma;
  return CTM_OK;
}

#ifdef CTM_EXP_STATS
int ctm_debug_stats(unsigned long long* out, int reset) {  // experiment build only
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, ctm::g_stats, sizeof(ctm::g_stats));
  if (reset) {
    static unsigned long long zero[256][8];
    cudaMemcpyToSymbol(ctm::g_stats, zero, sizeof(zero));
  }
  return 0;
}
#endif

ctm_status ctm_last_precision(ctm_mlp_t mlp, int32_t* precision) {
  if (!mlp || !precision) return fail(CTM_EINVAL, "NULL handle or output");
  *precision = mlp->cur_f16 ? CTM_PRECISION_FP16X3 : (mlp->nplanes == 3 ? CTM_PRECISION_FP32 : CTM_PRECISION_BF16X3);
  return CTM_OK;
}

ctm_status ctm_last_plan(ctm_mlp_t mlp, int32_t* launches, int32_t* slots_per_point, int32_t* points_per_tile,
                         int32_t* mma_n) {
  if (!mlp) return fail(CTM_EINVAL, "NULL handle");
  if (launches) *launches = mlp->last_launches;
  if (slots_per_point) *slots_per_point = mlp->last_P;
  if (points_per_tile) *points_per_tile = mlp->last_ppt;
  if (mma_n) *mma_n = mlp->last_nmma;
  return CTM_OK;
}

}  // extern "C"
