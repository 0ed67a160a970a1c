// nb200 engine: contexts, sessions, lowering and the Fisher / forward
// pipelines behind the C ABI (include/nb200.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "engine.hpp"

namespace nb {

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();  // clear sticky-free errors
  nb_status s = NB_ERR_CUDA;
  if (e == cudaErrorMemoryAllocation) s = NB_ERR_OUT_OF_MEMORY;
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ||
      e == cudaErrorNoKernelImageForDevice)
    s = NB_ERR_NO_DEVICE;
  fail(s, std::string(what) + ": " + cudaGetErrorString(e));
}

void DevBuf::ensure(size_t n) {
  if (n <= bytes) return;
  // grow by at least half (a reallocation synchronizes the whole device)
  n = std::max(n, bytes + bytes / 2);
  if (p) {
    NB_CUDA(cudaDeviceSynchronize());
    NB_CUDA(cudaFree(p));
    p = nullptr;
    bytes = 0;
  }
  n = std::max<size_t>(n, 256);
  NB_CUDA(cudaMalloc(&p, n));
  bytes = n;
}

DevBuf::~DevBuf() {
  if (p) cudaFree(p);
}

void PinnedBuf::ensure(size_t n) {
  if (n <= bytes) return;
  if (p) {
    NB_CUDA(cudaDeviceSynchronize());
    cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
  n = std::max<size_t>(n, 4096);
  NB_CUDA(cudaMallocHost(&p, n));
  bytes = n;
}

PinnedBuf::~PinnedBuf() {
  if (p) cudaFreeHost(p);
}

cudaEvent_t Profiler::get() {
  if (!pool_.empty()) {
    cudaEvent_t e = pool_.back();
    pool_.pop_back();
    return e;
  }
  cudaEvent_t e;
  NB_CUDA(cudaEventCreate(&e));
  return e;
}

void Profiler::begin(cudaStream_t st) {
  if (!active) return;
  cur_ = get();
  NB_CUDA(cudaEventRecord(cur_, st));
}

void Profiler::end(cudaStream_t st, const char* fam, double flops, double bytes) {
  if (!active || !cur_) return;
  cudaEvent_t b = get();
  NB_CUDA(cudaEventRecord(b, st));
  pending_.push_back({cur_, b, fam, flops, bytes});
  cur_ = nullptr;
}

void Profiler::resolve() {
  for (auto& p : pending_) {
    float ms = 0.f;
    NB_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    KStat& k = stats[p.fam];
    k.launches += 1;
    k.ms += ms;
    k.flops += p.flops;
    k.bytes += p.bytes;
    pool_.push_back(p.a);
    pool_.push_back(p.b);
  }
  pending_.clear();
}

Profiler::~Profiler() {
  for (auto e : pool_) cudaEventDestroy(e);
  for (auto& p : pending_) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
}

namespace {
int64_t align64(int64_t v) { return (v + 63) & ~int64_t(63); }

// N tile of a range: the largest that divides the per-group width.  A wider
// tile re-reads each A (activation) stage for more output channels, which
// is what bounds the kernel (shared-memory operand traffic, profiles/);
// SMs left idle by a small tile count are filled by the other candidates
// the scheduler runs concurrently on the same GPU.
// The fp32-accurate tier's tensor-core split (NB_TC_SPLIT): 2 = 3xFP16
// (default: kind::f16 with per-image / per-layer power-of-two scaling -- half
// the MMA time and B bytes of 3xTF32 at its 22 significand bits,
// profiles/r02_precision.md), 1 = 3xBF16 (16 bits, no scaling; "bf16"),
// 0 = 3xTF32 ("tf32").
int split_h16() {
  static const int m = [] {
    const char* e = std::getenv("NB_TC_SPLIT");
    if (e && std::string(e) == "tf32") return 0;
    if (e && std::string(e) == "bf16") return 1;
    return 2;
  }();
  return m;
}
bool split_bf16() { return split_h16() != 0; }

// fp16 weight scale 2^k for a layer whose largest |w| is maxabs: |w 2^k| < 2^15
int weight_shift(double maxabs) {
  if (!(maxabs > 0.0) || !std::isfinite(maxabs)) return 0;
  int ex = 0;
  std::frexp(maxabs, &ex);  // maxabs < 2^ex
  const int k = 15 - ex;
  return k < -126 ? -126 : (k > 126 ? 126 : k);
}

int pick_bn(int n_per_group, bool split3) {
  // NB_TC_BN3=256: the 256-wide single-accumulator 3xTF32 tile (experiment)
  static const bool wide3 = [] {
    const char* e = std::getenv("NB_TC_BN3");
    return e && std::atoi(e) >= 256;
  }();
  if (split3 && wide3 && split_h16() != 1 && n_per_group % 256 == 0) return 256;
  static const int o3[] = {128, 64, 32};
  static const int o1[] = {256, 128, 64, 32};
  const int* o = split3 ? o3 : o1;
  const int no = split3 ? 3 : 4;
  for (int i = 0; i < no; ++i)
    if (n_per_group % o[i] == 0) return o[i];
  return 0;
}

// N tile of a padded plan (one group, width a multiple of `gran` that no
// tile divides): the last tile's extra columns are zero weight rows (TMA
// out-of-bounds fill) the epilogue does not store -- fprop stores stop at 4
// columns (gran 4), the fused dgrad epilogue at 16.
int pick_bn_padded(int n, bool split3, int gran = 16) {
  if (n % gran) return 0;
  return n <= 32 ? 32 : n <= 64 ? 64 : split3 ? 128 : (n <= 128 ? 128 : 256);
}

// A grouped range whose slices miss the 32-channel K chunk runs as one dense
// GEMM over block-diagonal weights when it has at most 8 groups (NB_TC_DENSE
// sets the cap; 0 = never): G x the MACs on the tensor pipe still beat the
// FFMA kernels' 5-15 TFLOP/s.
int dense_cap() {
  static const int cap = [] {
    const char* e = std::getenv("NB_TC_DENSE");
    return e ? std::atoi(e) : 8;
  }();
  return cap;
}
bool use_dense(const RangeDesc& r, int64_t Ci) {
  return r.groups > 1 && r.groups <= dense_cap() && r.slice_ci % 32 != 0 && Ci % 4 == 0 &&
         r.len % 16 == 0;
}

// Images per M tile of a tensor-core launch over `nimg` images.
int plan_bni(int OH, int OW, int64_t nimg, int S) {
  tc::TcArgs t{};
  tc::plan_tiles(OH, OW, int(nimg), S, t);
  return t.BNI;
}

// M tiles of a tensor-core launch over `nimg` images (plan_tiles' count).
int m_tiles_at(int OH, int OW, int64_t nimg, int S) {
  tc::TcArgs t{};
  tc::plan_tiles(OH, OW, int(nimg), S, t);
  return t.m_tiles;
}

// Split-K factor of a tensor-core launch: when its output tiles cannot fill
// one wave of SMs, divide the K blocks (taps x 32-channel chunks, at least 4
// per split) so that tiles x splits still fits in one wave.
int choose_ksplit(const tc::TcArgs& t, int m_tiles, int num_sms, bool pair) {
  static const int mode = [] {  // NB_TC_KSPLIT=0: never split K (experiments)
    const char* e = std::getenv("NB_TC_KSPLIT");
    return e ? std::atoi(e) : 1;
  }();
  if (!mode) return 1;
  const int tiles = t.nphase * (pair ? (m_tiles + 1) / 2 : m_tiles) * t.n_tiles;
  if (pair) num_sms /= 2;
  int mink = 1 << 30;
  for (int p = 0; p < t.nphase; ++p) mink = std::min(mink, t.ntaps[p] * t.a_cblocks);
  if (tiles * 2 > num_sms || mink < 8) return 1;
  int ks = std::min({num_sms / tiles, mink / 4, 8});
  return ks >= 2 ? ks : 1;
}

// CTA-pair N tile for a range whose per-group width is n: the pair runs
// M = 256 and each CTA stages half of B, halving the weight-operand traffic
// per SM.  Measured slower than single-CTA tiles on the R34 layers (fprop
// 128@16x16: 88 us vs 61 us, tensor pipe 39% vs 56%, profiles/): the
// single-CTA kernel is not shared-memory or L2 bound at BN=128, and the
// pair adds a cross-SM handshake per stage.  Off by default; NB_TC_PAIR=1
// enables it (NB_TC_PAIR_BN=256 allows the single-accumulator 256-wide
// 3xTF32 pair).  0 = no pair.
int pick_pair_bn(int n, int m_tiles, bool split3, bool bf3 = false) {
  if (bf3) return 0;  // (3xBF16 runs single-CTA plans only)
  static const int mode = [] {
    const char* e = std::getenv("NB_TC_PAIR");
    return e ? std::atoi(e) : 0;
  }();
  static const char* cap_env = std::getenv("NB_TC_PAIR_BN");
  // 3xTF32 at 256 keeps a single TMEM accumulator (no epilogue overlap)
  const int cap = cap_env ? std::atoi(cap_env) : (split3 ? 128 : 256);
  if (!mode || m_tiles < 2) return 0;
  if (mode == 2) return n % 64 == 0 && n < 128 ? 64 : 0;  // pairs only for 64-wide groups
  if (n % 256 == 0 && cap >= 256) return 256;
  if (n % 128 == 0 && cap >= 128) return 128;
  if (n % 64 == 0) return 64;
  return 0;
}

// Multicast cluster for a single-CTA tile plan: two CTAs on two M tiles of
// one N tile share every B stage (each loads half, multicast to both), which
// halves the weight operand's L2 -> SM traffic.  NB_TC_MC=0 disables it.
bool use_mc(int bn, int m_tiles, bool pair, bool kwf = false, bool bf3 = false) {
  if (bf3 && split_h16() != 2) return false;  // (16-bit multicast: fp16 only)
  // NB_TC_MC: 0 (default) off, 1 every single-CTA plan, 2 kw-fused plans only
  // (their B stage is 3x wider, 48 KB, the same for every CTA; measured: the
  // stage period drops 7% but the evaluation time does not)
  static const int mode = [] {
    const char* e = std::getenv("NB_TC_MC");
    return e ? std::atoi(e) : 0;
  }();
  if (mode == 0 || pair || m_tiles < 2) return false;
  if (kwf) return true;
  return mode == 1 && (bn == 64 || bn == 128);
}

// kw-fused plan (Cfg KWF in kernels_tc.cu) for a 64-wide single-group GEMM
// over 32-pixel rows: 3-wide, stride 1, pad 1 -- the R34 CIFAR stage-1
// layers.  NB_TC_KWF=0 disables it.
bool use_kwf(const ConvGeom& g, int width, int rows_w) {
  static const int mode = [] {
    const char* e = std::getenv("NB_TC_KWF");
    return e ? std::atoi(e) : 1;
  }();
  // image rows of 4..32 pixels that tile a warp exactly (tile rows = image
  // rows: lane segments of rows_w lanes hold one image row each)
  return mode != 0 && width == 64 && g.KW == 3 && g.S == 1 && g.P == 1 && rows_w == g.OW &&
         g.W == g.OW && g.OW >= 4 && g.OW <= 32 && 32 % g.OW == 0;
}

// the kh taps of a kw-fused plan: A shifted in h only, B K chunk kh
void kwf_taps(const ConvGeom& g, tc::TcArgs& t, int sgn) {
  t.ntaps[0] = g.KH;
  for (int kh = 0; kh < g.KH; ++kh)
    t.taps[0][kh] = tc::pack_tap(kh, sgn > 0 ? kh - g.P : g.P - kh, 0);
  t.kwf_sgn = sgn;
  t.kwf_w = g.OW;
}

// fprop: one phase over the OH x OW output, every tap, A box at
// (S*oy - P + kh, S*ox - P + kw) (the element stride S is in the tensor map).
void fprop_phase(const ConvGeom& g, tc::TcArgs& t) {
  t.nphase = 1;
  t.PS = 1;
  t.OHp[0] = g.OH;
  t.OWp[0] = g.OW;
  t.py[0] = t.px[0] = 0;
  t.OutH = g.OH;
  t.OutW = g.OW;
  int n = 0;
  for (int kh = 0; kh < g.KH; ++kh)
    for (int kw = 0; kw < g.KW; ++kw) t.taps[0][n++] = tc::pack_tap(kh * g.KW + kw, kh - g.P, kw - g.P);
  t.ntaps[0] = n;
}

// dgrad (I/nnet.hpp:235-243 as a gather): g[ih,iw] = sum over taps with
// (ih + P - kh) % S == 0 of W * dY[(ih + P - kh)/S, ...].  With ih = S*oy + py
// the dY row is oy + (py + P - kh)/S, so each phase (py, px) is a stride-1
// correlation over the taps of matching parity; out-of-range dY rows (the
// border and the output crop, I/ir.hpp:47-50) are TMA zero fill.
void dgrad_phases(const ConvGeom& g, tc::TcArgs& t) {
  const int S = g.S;
  t.nphase = S * S;
  t.PS = S;
  t.OutH = g.H;
  t.OutW = g.W;
  for (int py = 0; py < S; ++py)
    for (int px = 0; px < S; ++px) {
      const int ph = py * S + px;
      t.py[ph] = py;
      t.px[ph] = px;
      t.OHp[ph] = (g.H - py + S - 1) / S;
      t.OWp[ph] = (g.W - px + S - 1) / S;
      int n = 0;
      for (int kh = 0; kh < g.KH; ++kh) {
        const int th = py + g.P - kh;
        if (((th % S) + S) % S) continue;
        for (int kw = 0; kw < g.KW; ++kw) {
          const int tw = px + g.P - kw;
          if (((tw % S) + S) % S) continue;
          // floor division of the (exact) multiples of S
          t.taps[ph][n++] = tc::pack_tap(kh * g.KW + kw, (th - ((th % S) + S) % S) / S,
                                         (tw - ((tw % S) + S) % S) / S);
        }
      }
      t.ntaps[ph] = n;
    }
}
}  // namespace

// Lowering of a (derived, repaired) network to kernel plans (SURVEY 7
// "Lowering design"): per layer the ConvSpec ranges (I/ir.hpp:54-57) become
// RangeDescs; each range's fprop and the layer's dgrad get a kernel family --
// tcgen05 implicit GEMM when the range is tensor-core shaped (32-channel K
// chunks, 16-aligned N), the direct FFMA kernels otherwise -- plus packed-
// weight, activation and Fisher-partial arena offsets.
NetPlan lower(const NetDesc& net, int64_t n, nb_precision prec, int num_sms, int64_t plan_n,
              bool stem_col) {
  if (plan_n <= 0) plan_n = n;
  NetPlan P;
  const bool tc_on = prec != NB_PREC_SIMT;
  P.split3 = prec == NB_PREC_FP32;
  P.h16 = P.split3 ? split_h16() : 0;
  const int64_t L = net.L();
  for (int64_t l = 0; l < L; ++l) {
    const Spec& s = net.specs[l];
    LayerPlan lp;
    ConvGeom& g = lp.geom;
    g.N = int(n);
    g.H = int(s.h);
    g.W = int(s.w);
    g.Ci = int(s.ci);
    g.OH = int(s.oh());
    g.OW = int(s.ow());
    g.Co = int(s.co_eff());
    g.KH = int(s.kh);
    g.KW = int(s.kw);
    g.S = int(s.stride);
    g.P = int(s.pad);
    auto rs = s.ranges();
    if (int(rs.size()) > kMaxRanges)
      fail(NB_ERR_UNSUPPORTED, "more than 16 channel ranges in one layer");
    g.nranges = int(rs.size());
    lp.tcf.resize(size_t(g.nranges));
    int64_t off = 0;
    const int taps = int(s.kh * s.kw);
    for (int i = 0; i < g.nranges; ++i) {
      RangeDesc& r = g.r[i];
      r.b = int(rs[i].begin);
      r.len = int(rs[i].end - rs[i].begin);
      r.groups = int(rs[i].groups);
      r.slice_co = r.len / r.groups;
      r.slice_ci = int(s.ci / rs[i].groups);
      const int64_t used = int64_t(r.len) * r.slice_ci * taps;
      r.wf_off = off;
      off += align64(used);
      r.wd_off = off;
      off += align64(used);
      lp.family[i] = Family::Direct;
      // channel counts off the 32-channel K chunk (e.g. DenseNet's 48-wide
      // growth) run as padded plans when the layer is one group; a few groups
      // of narrow slices run as one dense GEMM over block-diagonal weights
      // (G x the MACs, on the tensor pipe instead of FFMA)
      const bool dense = use_dense(r, g.Ci);
      const int G = dense ? 1 : r.groups;
      const int sci = dense ? int(g.Ci) : r.slice_ci;
      const int sco = dense ? r.len : r.slice_co;
      const bool pad_ok = G == 1 && g.Ci % 4 == 0;
      if (tc_on && (g.S == 1 || g.S == 2) && (sci % 32 == 0 || pad_ok) &&
          r.b % 16 == 0 && g.Co % 4 == 0 && taps <= tc::kMaxPhaseTaps) {
        tc::TcArgs t{};
        if (tc::plan_tiles(g.OH, g.OW, g.N, g.S, t)) {
          // launch-shape decisions are made at the planning batch size, so an
          // example shard runs the whole batch's kernels (same split-K, so
          // the same summation order per output)
          const int mt = m_tiles_at(g.OH, g.OW, plan_n, g.S);
          // (kw-fused B layouts are [kw][co][kh][ci] with K = KH x sci: no
          // K padding, so a padded K runs the plain tap-major plan)
          const bool kwf = G == 1 && !dense && sci % 32 == 0 && use_kwf(g, sco, t.BW);
          const int pbn = kwf ? 0 : pick_pair_bn(sco, mt, P.split3, P.h16 != 0);
          int bn = pbn ? pbn : pick_bn(sco, P.split3);
          static const int gran = [] {  // NB_TC_PADG: fprop padded-width granularity
            const char* e = std::getenv("NB_TC_PADG");
            return e ? std::atoi(e) : 4;
          }();
          if (!bn && pad_ok) bn = pick_bn_padded(sco, P.split3, gran);
          const int kp = (sci + 31) / 32 * 32;
          if (bn) {
            t.mode = 0;
            t.n_tiles_per_group = (sco + bn - 1) / bn;
            t.n_tiles = G * t.n_tiles_per_group;
            t.S = g.S;
            fprop_phase(g, t);
            if (kwf) kwf_taps(g, t, +1);
            t.a_cblocks = kp / 32;
            t.a_c_base = 0;
            t.a_c_per_group = sci;
            t.b_k_per_tap = kp;
            t.b_row_base = 0;
            t.b_row_per_group = sco;
            t.out_ld = g.Co;
            t.out_c_base = r.b;
            t.out_c_per_group = sco;
            const bool mc = use_mc(bn, mt, pbn != 0, kwf, P.h16 != 0);
            t.ksplit = choose_ksplit(t, mt, num_sms, pbn != 0 || mc);
            if (t.ksplit > 1)
              P.ws_floats = std::max(P.ws_floats, int64_t(t.ksplit) * n * g.OH * g.OW * g.Co);
            TcPlan& tp = lp.tcf[i];
            tp.bn = bn;
            tp.plan_bni = plan_bni(g.OH, g.OW, plan_n, g.S);
            tp.pair = pbn != 0;
            tp.mc = mc;
            tp.kwf = kwf;
            tp.tile = t;
            tp.kp = kp != sci ? kp : 0;
            tp.dense = dense ? r.groups : 0;
            tp.hw_chunks = t.ksplit > 1 ? splitk_hw_chunks(plan_n, g.OH * g.OW, r.len) : 1;
            tp.w_n = align64(int64_t(r.len) * taps * kp);
            tp.w_off = off;
            tp.b_rows = kwf ? g.KW * r.len : r.len;
            tp.b_k = kwf ? g.KH * sci : taps * kp;
            off += 2 * tp.w_n;
            lp.family[i] = Family::TensorCore;
          }
        }
      }
      // a narrow stem (Ci*KH*KW <= 32, e.g. the 3-channel 3x3 input layer)
      // reading the session batch: a 1x1 GEMM over its im2col copy, K = 32
      static const bool col_on = [] {  // NB_TC_COL=0: FFMA stem (experiments)
        const char* e = std::getenv("NB_TC_COL");
        return !e || std::atoi(e) != 0;
      }();
      if (lp.family[i] == Family::Direct && stem_col && col_on && l == 0 && g.nranges == 1 &&
          r.groups == 1 && tc_on && g.Ci * taps <= 32 && r.len % 4 == 0 && g.Co % 4 == 0) {
        ConvGeom g1 = g;
        g1.H = g.OH;
        g1.W = g.OW;
        g1.Ci = 32;
        g1.KH = g1.KW = 1;
        g1.S = 1;
        g1.P = 0;
        tc::TcArgs t{};
        int bn = pick_bn(r.len, P.split3);
        if (!bn) bn = pick_bn_padded(r.len, P.split3, 4);
        if (bn && tc::plan_tiles(g.OH, g.OW, g.N, 1, t)) {
          const int mt = m_tiles_at(g.OH, g.OW, plan_n, 1);
          t.mode = 0;
          t.n_tiles_per_group = (r.len + bn - 1) / bn;
          t.n_tiles = t.n_tiles_per_group;
          t.S = 1;
          fprop_phase(g1, t);
          t.a_cblocks = 1;
          t.a_c_base = 0;
          t.a_c_per_group = 32;
          t.b_k_per_tap = 32;
          t.b_row_base = 0;
          t.b_row_per_group = r.len;
          t.out_ld = g.Co;
          t.out_c_base = r.b;
          t.out_c_per_group = r.len;
          t.ksplit = choose_ksplit(t, mt, num_sms, false);
          TcPlan& tp = lp.tcf[i];
          tp.bn = bn;
          tp.tile = t;
          tp.kp = 32;
          tp.col = true;
          tp.hw_chunks = t.ksplit > 1 ? splitk_hw_chunks(plan_n, g.OH * g.OW, r.len) : 1;
          if (t.ksplit > 1)
            P.ws_floats = std::max(P.ws_floats, int64_t(t.ksplit) * n * g.OH * g.OW * g.Co);
          tp.w_n = align64(int64_t(r.len) * 32);
          tp.w_off = off;
          tp.b_rows = r.len;
          tp.b_k = 32;
          off += 2 * tp.w_n;
          lp.family[i] = Family::TensorCore;
        }
      }
    }
    // dgrad on the tensor cores: stride 1 as one phase, stride 2 as the four
    // sub-pixel phases (a phase grid of ceil(H/2) x ceil(W/2)).
    // (a grouped layer whose slices do not tile the GEMM densifies as in fprop)
    const RangeDesc& r0 = g.r[0];
    const bool ddense = g.nranges == 1 && r0.groups > 1 && r0.groups <= dense_cap() &&
                        (r0.slice_co % 32 != 0 || !pick_bn(r0.slice_ci, P.split3)) &&
                        g.Co % 4 == 0 && g.Ci % 16 == 0;
    const int DG = ddense ? 1 : r0.groups;
    const int dsci = ddense ? int(g.Ci) : r0.slice_ci;
    const int dsco = ddense ? r0.len : r0.slice_co;
    const bool dpad_ok = DG == 1 && g.Co % 4 == 0;
    if (l >= 1 && tc_on && g.nranges == 1 && (g.S == 1 || g.S == 2) &&
        (dsco % 32 == 0 || dpad_ok) && g.Ci % 4 == 0 && taps <= tc::kMaxPhaseTaps) {
      const RangeDesc& r = g.r[0];
      tc::TcArgs t{};
      const int gh = (g.H + g.S - 1) / g.S, gw = (g.W + g.S - 1) / g.S;
      if (tc::plan_tiles(gh, gw, g.N, 1, t)) {
        const int mt = m_tiles_at(gh, gw, plan_n, 1);
        const bool kwf = DG == 1 && !ddense && dsco % 32 == 0 && use_kwf(g, dsci, t.BW);
        const int pbn = kwf ? 0 : pick_pair_bn(dsci, mt * t.nphase, P.split3, P.h16 != 0);
        int bn = pbn ? pbn : pick_bn(dsci, P.split3);
        if (!bn && dpad_ok) bn = pick_bn_padded(dsci, P.split3);
        const int kp = (dsco + 31) / 32 * 32;
        if (bn) {
          t.mode = 1;
          t.n_tiles_per_group = (dsci + bn - 1) / bn;
          t.n_tiles = DG * t.n_tiles_per_group;
          t.S = 1;
          dgrad_phases(g, t);
          if (kwf) kwf_taps(g, t, -1);
          t.a_cblocks = kp / 32;
          t.a_c_base = r.b;
          t.a_c_per_group = dsco;
          t.b_k_per_tap = kp;
          t.b_row_base = 0;
          t.b_row_per_group = dsci;
          t.out_ld = g.Ci;
          t.out_c_base = 0;
          t.out_c_per_group = dsci;
          t.part_ld = g.Ci;
          const bool mc = use_mc(bn, mt, pbn != 0, kwf, P.h16 != 0);
          t.ksplit = choose_ksplit(t, mt, num_sms, pbn != 0 || mc);
          // split-K dgrad: k_splitk_epilogue writes one partial per (image, pixel chunk)
          const int hw_chunks = t.ksplit > 1 ? splitk_hw_chunks(plan_n, g.H * g.W, g.Ci) : 1;
          t.part_tiles_per_img =
              t.ksplit > 1 ? hw_chunks : t.nphase * (t.BNI == 1 ? t.tiles_h * t.tiles_w : 1);
          if (t.ksplit > 1)
            P.ws_floats = std::max(P.ws_floats, int64_t(t.ksplit) * n * g.H * g.W * g.Ci);
          TcPlan& tp = lp.tcd;
          tp.bn = bn;
          tp.plan_bni = plan_bni(gh, gw, plan_n, 1);
          tp.pair = pbn != 0;
          tp.mc = mc;
          tp.kwf = kwf;
          tp.tile = t;
          tp.kp = kp != dsco ? kp : 0;
          tp.dense = ddense ? r.groups : 0;
          tp.hw_chunks = hw_chunks;
          tp.w_n = align64(int64_t(g.Ci) * taps * kp);
          tp.w_off = off;
          tp.b_rows = kwf ? g.KW * g.Ci : g.Ci;
          tp.b_k = kwf ? g.KH * dsco : taps * kp;
          off += 2 * tp.w_n;
          lp.dgrad_family = Family::TensorCore;
        }
      }
    }
    lp.wpack_floats = off;
    lp.h16 = P.h16;
    lp.w_off = P.w_total;
    P.w_total += off;
    lp.act_floats = n * s.co_eff() * s.oh() * s.ow();
    lp.act_off = P.act_total;
    P.act_total += align64(lp.act_floats);
    P.dpre_floats = std::max(P.dpre_floats, lp.act_floats);
    P.ch_total += s.co_eff();
    lp.fprop_flops = 2.0 * double(n) * double(s.macs());
    lp.dgrad_flops = l > 0 ? 2.0 * double(n) * double(s.macs()) : 0.0;
    P.layers.push_back(lp);
  }
  // Fisher partials of layer l are produced by the dgrad of layer l+1 (or the
  // head for the last layer); their tiling follows that kernel.
  for (int64_t l = 0; l < L; ++l) {
    LayerPlan& lp = P.layers[l];
    if (l == L - 1) {
      lp.tiles = 1;
    } else {
      const LayerPlan& nx = P.layers[l + 1];
      lp.tiles = nx.dgrad_family == Family::TensorCore ? nx.tcd.tile.part_tiles_per_img
                                                       : direct_dgrad_tiles(nx.geom);
    }
    lp.part_off = P.part_total;
    P.part_total += align64(n * lp.tiles * lp.geom.Co);
  }
  return P;
}

void ctx_activate(nb_ctx* c) { NB_CUDA(cudaSetDevice(c->device)); }

namespace {

const double* ensure_z(nb_ctx* c, uint64_t seed, int64_t stream, int64_t count) {
  auto key = std::make_pair(seed, stream);
  auto& buf = c->zdev[key];
  if (!buf) buf = std::make_unique<DevBuf>();
  int64_t& have = c->zlen[key];
  if (have < count) {
    // The host stream is cached for the process lifetime, so the copy can be
    // stream-ordered with the pack kernels that read it (a plain cudaMemcpy
    // from pageable memory may return before its DMA lands, and the context
    // stream does not synchronise with the legacy stream).
    const std::vector<double>& z = z_stream(seed, stream, count);
    buf->ensure(size_t(count) * 8);
    NB_CUDA(cudaMemcpyAsync(buf->p, z.data(), size_t(count) * 8, cudaMemcpyHostToDevice,
                            c->stream));
    have = count;
  }
  return buf->as<double>();
}

// max |z| of the z-stream prefix (seed, stream, count) -- the scale of the
// fp16 split's packed weights -- cached per context
double zmax_of(nb_ctx* c, uint64_t seed, int64_t stream, int64_t count) {
  const auto key = std::make_tuple(seed, stream, count);
  auto it = c->zmax.find(key);
  if (it != c->zmax.end()) return it->second;
  const std::vector<double>& z = z_stream(seed, stream, count);
  double m = 0.0;
  for (int64_t i = 0; i < count; ++i) m = std::max(m, std::fabs(z[size_t(i)]));
  c->zmax.emplace(key, m);
  return m;
}

// Identity of a layer's packed init_weights weights: the z-stream (seed,
// layer), the fan-in scale and every offset/family the lowering chose.
std::string wkey(uint64_t seed, int64_t l, const Spec& sp, const LayerPlan& lp) {
  std::string k = std::to_string(seed) + "/" + std::to_string(l) + "/" + std::to_string(sp.ci) +
                  "x" + std::to_string(sp.kh) + "x" + std::to_string(sp.kw) + "/" +
                  std::to_string(lp.wpack_floats) + "/h" + std::to_string(lp.h16) + "," +
                  std::to_string(lp.b_shift);
  const ConvGeom& g = lp.geom;
  for (int r = 0; r < g.nranges; ++r) {
    const RangeDesc& d = g.r[r];
    k += "|" + std::to_string(d.b) + "," + std::to_string(d.len) + "," + std::to_string(d.groups) +
         "," + std::to_string(d.wf_off) + "," + std::to_string(d.wd_off) + "," +
         std::to_string(int(lp.family[r]));
    if (lp.family[r] == Family::TensorCore)
      k += "," + std::to_string(lp.tcf[r].w_off) + "," + std::to_string(lp.tcf[r].w_n) +
           (lp.tcf[r].kwf ? "k" : "") + (lp.tcf[r].dense ? "D" : "") +
           (lp.tcf[r].kp ? "p" : "") + (lp.tcf[r].col ? "c" : "");
  }
  if (lp.dgrad_family == Family::TensorCore)
    k += "|d" + std::to_string(lp.tcd.w_off) + "," + std::to_string(lp.tcd.w_n) +
         (lp.tcd.kwf ? "k" : "") + (lp.tcd.dense ? "D" : "") + (lp.tcd.kp ? "p" : "");
  return k;
}

// packed-weight slab bytes per context: a search's distinct layers of one
// pool stay resident (a full slab is reset between runs, repacking every
// layer of the next candidates), at a few GB of the 180 GB per GPU
constexpr size_t kWCacheCap = size_t(6) << 30;

void pack_layer(nb_ctx* c, const LayerPlan& lp, const double* src, double scale,
                cudaStream_t st) {
  float* base = lp.wbase;
  for (int r = 0; r < lp.geom.nranges; ++r) {
    // the direct-kernel layouts only where a direct kernel reads them
    const bool need_wf = lp.family[r] != Family::TensorCore;
    const bool need_wd = lp.dgrad_family != Family::TensorCore;
    PackDst d{need_wf ? base : nullptr, need_wd ? base : nullptr, nullptr, nullptr, nullptr,
              nullptr};
    d.KW = lp.geom.KW;
    d.h16 = lp.h16;
    d.h16_scale = float(std::ldexp(1.0, lp.b_shift));
    if (lp.family[r] == Family::TensorCore) {
      d.tcf_hi = base + lp.tcf[r].w_off;
      d.tcf_lo = d.tcf_hi + lp.tcf[r].w_n;
      d.kwf_f = lp.tcf[r].kwf ? 1 : 0;
      d.kpf = lp.tcf[r].tile.b_k_per_tap;  // K per tap of the layout (padded / dense)
      d.dense_f = lp.tcf[r].dense ? 1 : 0;
      d.col_f = lp.tcf[r].col ? 1 : 0;
      if (d.kpf || d.dense_f)  // the padded K columns / off-diagonal blocks stay zero
        NB_CUDA(cudaMemsetAsync(d.tcf_hi, 0, size_t(2 * lp.tcf[r].w_n) * 4, st));
    }
    if (r == 0 && lp.dgrad_family == Family::TensorCore) {
      d.tcd_hi = base + lp.tcd.w_off;
      d.tcd_lo = d.tcd_hi + lp.tcd.w_n;
      d.kwf_d = lp.tcd.kwf ? 1 : 0;
      d.kpd = lp.tcd.tile.b_k_per_tap;
      d.dense_d = lp.tcd.dense ? 1 : 0;
      if (d.kpd || d.dense_d) NB_CUDA(cudaMemsetAsync(d.tcd_hi, 0, size_t(2 * lp.tcd.w_n) * 4, st));
    }
    launch_pack_weights(src, scale, lp.geom, r, d, st);
    c->launches++;
  }
}

void launch_tc(nb_ctx* c, const TcPlan& tp, const tc::TcArgs& args, bool split3, bool bf3,
               const float* A, int AC, int AW, int AH, int AN, const float* whi,
               cudaStream_t st) {
  tc::TcLaunch L;
  L.args = args;
  static const int dbg = [] {
    const char* e = std::getenv("NB_TC_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  L.args.debug = dbg;
  // NB_TC_TRACE=<launch index>: record CTA 0's stage timeline of that TC
  // launch of this context and dump it to nb_tc_trace.txt (experiments)
  static const int trace_at = [] {
    const char* e = std::getenv("NB_TC_TRACE");
    return e ? std::atoi(e) : -1;
  }();
  static int tc_launch_no = 0;
  const bool tracing = trace_at >= 0 && tc_launch_no++ == trace_at;
  if (tracing) {
    c->trace.ensure((tc::kTraceRoles * tc::kTraceStages + 4 * 1024) * 8);
    NB_CUDA(cudaMemsetAsync(c->trace.p, 0, (tc::kTraceRoles * tc::kTraceStages + 4 * 1024) * 8, st));
    L.args.trace = c->trace.as<long long>();
  }
  L.bn = tp.bn;
  L.split3 = split3;
  L.bf = bf3;
  L.pair = tp.pair;
  L.mc = tp.mc;
  L.kwf = tp.kwf;
  // NB_TC_CONVH: 1 = both converter groups split every stage by channel
  // halves, 0 = groups alternate stages, 2 = halves for kw-fused only.
  // Default: halves for 3xTF32 (its kw-fused plans have two TMEM A slots, so
  // per-stage latency counts), alternate stages for the 16-bit splits (four
  // or more slots; alternating halves the per-stage barrier overhead:
  // 3xF16 bench 576 vs 561 candidates/s)
  static const int convh = [] {
    const char* e = std::getenv("NB_TC_CONVH");
    return e ? std::atoi(e) : -1;
  }();
  const int ch = convh >= 0 ? convh : (bf3 ? 0 : 1);
  L.args.conv_halves = ch == 1 || (ch == 2 && tp.kwf) ? 1 : 0;
  L.num_sms = c->num_sms;
  // Halo mode (default; NB_TC_HALO=0 turns it off): a split-converter launch
  // over a stride-1 A operand with several taps per phase loads one halo box
  // per 32-channel chunk (tile + the taps' offsets) and its converters form
  // the shifted rows of every tap from it, when the box fits the kernel's
  // halo buffers.  A's L2 -> SM bytes per 3x3 stage drop from 16 KB to ~3 KB.
  // It tied with the row-per-tap A operand while the converters were slower;
  // after the late-round-2 epilogue work it is ahead (origin Fisher 2.79 ->
  // 2.62 ms, same-box A/B, profiles/r02_kernels.md section 6).
  static const bool halo_on = [] {
    const char* e = std::getenv("NB_TC_HALO");
    return !e || std::atoi(e) != 0;
  }();
  L.args.halo = 0;
  if (halo_on && split3 && !tp.pair && args.S == 1) {
    int span_h = 0, span_w = 0, most = 0;
    for (int ph = 0; ph < args.nphase; ++ph) {
      int h0 = 0, h1 = 0, w0 = 0, w1 = 0;
      for (int t = 0; t < args.ntaps[ph]; ++t) {
        const int dh = tc::tap_dh(args.taps[ph][t]), dw = tc::tap_dw(args.taps[ph][t]);
        h0 = t ? std::min(h0, dh) : dh;
        h1 = t ? std::max(h1, dh) : dh;
        w0 = t ? std::min(w0, dw) : dw;
        w1 = t ? std::max(w1, dw) : dw;
      }
      L.args.halo_dh0[ph] = h0;
      L.args.halo_dw0[ph] = w0;
      span_h = std::max(span_h, h1 - h0);
      span_w = std::max(span_w, w1 - w0);
      most = std::max(most, args.ntaps[ph]);
    }
    const int hh = args.BH + span_h, hw = args.BW + span_w;
    const int64_t bytes = int64_t(hh) * hw * std::max(args.BNI, tp.plan_bni) * 128;
    if (most >= 2 && hh <= 256 && hw <= 256 && bytes <= tc::halo_capacity(L)) {
      L.args.halo = 1;
      L.args.halo_h = hh;
      L.args.halo_w = hw;
    }
  }
  static const bool halo_log = std::getenv("NB_TC_HALO_LOG") != nullptr;  // (experiments)
  if (halo_log)
    std::fprintf(stderr, "tc mode %d n %d BW %d BH %d BNI %d mt %d nt %d ks %d taps %d halo %d %dx%d\n",
                 args.mode, args.nimg, args.BW, args.BH, args.BNI, args.m_tiles, args.n_tiles,
                 args.ksplit, args.ntaps[0], L.args.halo, L.args.halo_w, L.args.halo_h);
  if (!tc::make_maps(L, A, AC, AW, AH, AN, whi, whi + tp.w_n, tp.b_k, tp.b_rows))
    fail(NB_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  NB_CUDA(tc::launch(L, st));
  c->launches++;
  if (tracing) {
    std::vector<long long> h(tc::kTraceRoles * tc::kTraceStages + 4 * 1024);
    NB_CUDA(cudaMemcpyAsync(h.data(), c->trace.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaStreamSynchronize(st));
    FILE* f = std::fopen("nb_tc_trace.txt", "w");
    if (f) {
      std::fprintf(f, "# bn=%d split3=%d stages tiles=%d kblocks/tile=%d\n", L.bn, int(L.split3),
                   args.m_tiles * args.n_tiles, args.ntaps[0] * args.a_cblocks);
      for (int i = 0; i < tc::kTraceStages; ++i)
      {
        std::fprintf(f, "%d", i);
        for (int role = 0; role < tc::kTraceRoles; ++role)
          std::fprintf(f, " %lld", h[role * tc::kTraceStages + i]);
        std::fprintf(f, "\n");
      }
      std::fclose(f);
    }
    // per CTA: entry, after the grid dependency, MMA issue done, epilogue done (ns)
    FILE* g = std::fopen("nb_tc_ctas.txt", "w");
    if (g) {
      for (int i = 0; i < 1024; ++i) {
        const long long* e = &h[tc::kTraceRoles * tc::kTraceStages + 4 * i];
        if (e[0]) std::fprintf(g, "%d %lld %lld %lld %lld\n", i, e[0], e[1], e[2], e[3]);
      }
      std::fclose(g);
    }
  }
}

// One layer's fprop (all ranges): y = relu?(conv(x)).
// The profiler name of a tensor-core launch (fprop, or dgrad with the Fisher
// epilogue) for the plan's arithmetic.
const char* split_name(const NetPlan& P, bool dgrad) {
  static const char* const f[] = {"conv_fprop_tc_tf32", "conv_fprop_tc_3xtf32",
                                  "conv_fprop_tc_3xbf16", "conv_fprop_tc_3xf16"};
  static const char* const d[] = {"conv_dgrad_tc_tf32_fisher", "conv_dgrad_tc_3xtf32_fisher",
                                  "conv_dgrad_tc_3xbf16_fisher", "conv_dgrad_tc_3xf16_fisher"};
  const int i = P.h16 ? 1 + P.h16 : (P.split3 ? 1 : 0);
  return dgrad ? d[i] : f[i];
}

// fp16-split scaling of a tensor-core launch (TcArgs::h16_f16): the per-image
// max of its A operand (in_amax) and of what it writes for the next GEMM
// (out_amax), the layer's weight scale
void set_scaling(const NetPlan& P, const LayerPlan& lp, tc::TcArgs& a, const uint32_t* in_amax,
                 uint32_t* out_amax) {
  const bool f16 = P.h16 == 2;
  a.h16_f16 = f16 ? 1 : 0;
  a.a_amax = f16 ? in_amax : nullptr;
  a.out_amax = f16 ? out_amax : nullptr;
  a.b_inv = f16 ? float(std::ldexp(1.0, -lp.b_shift)) : 1.f;
}

// One layer's fprop (all ranges): y = relu?(conv(x)).  fp16 split: in_amax =
// per-image max |x|; out_amax (nullable) receives per-image max |y|.
void fprop_layer(nb_ctx* c, const NetPlan& P, const LayerPlan& lp, const float* x, float* y,
                 bool relu, cudaStream_t st, const uint32_t* in_amax, uint32_t* out_amax) {
  Range range("conv_fprop");
  const ConvGeom& g = lp.geom;
  float* base = lp.wbase;
  bool direct = false;
  for (int r = 0; r < g.nranges; ++r) {
    const RangeDesc& rd = g.r[r];
    const double fl =
        2.0 * double(g.N) * rd.len * g.OH * g.OW * rd.slice_ci * g.KH * g.KW;
    const double by = 4.0 * (double(g.N) * g.H * g.W * g.Ci +
                             double(rd.len) * rd.slice_ci * g.KH * g.KW +
                             double(g.N) * g.OH * g.OW * rd.len);
    c->prof.begin(st);
    if (lp.family[r] == Family::TensorCore) {
      tc::TcArgs a = lp.tcf[r].tile;
      a.out = y;
      a.relu = relu ? 1 : 0;
      a.ws = c->ws.as<float>();
      a.ws_stride = int64_t(g.N) * g.OH * g.OW * g.Co;
      set_scaling(P, lp, a, in_amax, out_amax);
      // (a col stem reads the session's im2col copy: 32 columns per output pixel)
      const bool col = lp.tcf[r].col;
      launch_tc(c, lp.tcf[r], a, P.split3, P.h16 != 0, x, col ? 32 : g.Ci, col ? g.OW : g.W,
                col ? g.OH : g.H, g.N, base + lp.tcf[r].w_off, st);
      if (a.ksplit > 1) {
        SplitEpi e{};
        e.ws = a.ws;
        e.ws_stride = a.ws_stride;
        e.ksplit = a.ksplit;
        e.mode = 0;
        e.N = g.N;
        e.HW = g.OH * g.OW;
        e.ld = g.Co;
        e.c0 = rd.b;
        e.C = rd.len;
        e.out = y;
        e.relu = relu ? 1 : 0;
        e.hw_chunks = lp.tcf[r].hw_chunks;
        e.out_amax = a.out_amax;
        launch_splitk_epilogue(e, st);
        c->launches++;
      }
      c->prof.end(st, split_name(P, false), fl, by);
    } else {
      launch_fprop_direct(g, r, x, base, y, relu, st);
      c->launches++;
      c->prof.end(st, "conv_fprop_direct", fl, by);
      direct = true;
    }
  }
  // a direct range does not record its output's max: scan the output
  if (direct && out_amax && P.h16 == 2) {
    launch_amax(y, g.N, int64_t(g.OH) * g.OW * g.Co, out_amax, st);
    c->launches++;
  }
}

// One layer's dgrad with the fused epilogue on the previous layer's output.
// fp16 split: in_amax = per-image max |dpre|; out_amax (nullable) receives
// per-image max |dpre_out|.
void dgrad_layer(nb_ctx* c, const NetPlan& P, const LayerPlan& lp, const float* dpre,
                 const float* a_prev, bool relu_prev, float* dpre_out, float* g_out,
                 double* partial, cudaStream_t st, const uint32_t* in_amax, uint32_t* out_amax) {
  Range range("conv_dgrad");
  const ConvGeom& g = lp.geom;
  float* base = lp.wbase;
  const double prev_floats = double(g.N) * g.H * g.W * g.Ci;
  const double by = 4.0 * (double(g.N) * g.OH * g.OW * g.Co + double(lp.wpack_floats) / 6.0 +
                           (a_prev ? prev_floats : 0.0) + (dpre_out ? prev_floats : 0.0) +
                           (g_out ? prev_floats : 0.0));
  c->prof.begin(st);
  if (lp.dgrad_family == Family::TensorCore) {
    tc::TcArgs a = lp.tcd.tile;
    a.out = g_out;
    a.g_out = g_out;
    a.a_prev = a_prev;
    a.dpre_out = dpre_out;
    a.partial = partial;
    a.relu_prev = relu_prev ? 1 : 0;
    a.ws = c->ws.as<float>();
    a.ws_stride = int64_t(g.N) * g.H * g.W * g.Ci;
    set_scaling(P, lp, a, in_amax, dpre_out ? out_amax : nullptr);
    launch_tc(c, lp.tcd, a, P.split3, P.h16 != 0, dpre, g.Co, g.OW, g.OH, g.N, base + lp.tcd.w_off, st);
    if (a.ksplit > 1) {
      SplitEpi e{};
      e.ws = a.ws;
      e.ws_stride = a.ws_stride;
      e.ksplit = a.ksplit;
      e.mode = 1;
      e.N = g.N;
      e.HW = g.H * g.W;
      e.ld = g.Ci;
      e.c0 = 0;
      e.C = g.Ci;
      e.a_prev = a_prev;
      e.dpre_out = dpre_out;
      e.g_out = g_out;
      e.partial = partial;
      e.relu_prev = relu_prev ? 1 : 0;
      e.hw_chunks = lp.tcd.hw_chunks;
      e.out_amax = a.out_amax;
      launch_splitk_epilogue(e, st);
      c->launches++;
    }
    c->prof.end(st, split_name(P, true),
                lp.dgrad_flops, by);
  } else {
    launch_dgrad_direct(g, dpre, base, a_prev, relu_prev, dpre_out, g_out, partial, st);
    c->launches++;
    c->prof.end(st, "conv_dgrad_direct_fisher", lp.dgrad_flops, by);
    if (dpre_out && out_amax && P.h16 == 2) {
      launch_amax(dpre_out, g.N, int64_t(g.H) * g.W * g.Ci, out_amax, st);
      c->launches++;
    }
  }
}

}  // namespace

// The smallest spare session buffer of the context that fits, else a new one
// (no cudaMalloc per session once the context has served a few).
std::unique_ptr<DevBuf> take_spare(nb_ctx* c, size_t bytes) {
  auto best = c->spare.end();
  for (auto it = c->spare.begin(); it != c->spare.end(); ++it)
    if ((*it)->bytes >= bytes && (best == c->spare.end() || (*it)->bytes < (*best)->bytes))
      best = it;
  std::unique_ptr<DevBuf> buf;
  if (best != c->spare.end()) {
    buf = std::move(*best);
    c->spare.erase(best);
  } else {
    buf = std::make_unique<DevBuf>();
    buf->ensure(bytes);
  }
  return buf;
}

// Per-image max |x| of the session batch (fp16 split of the first GEMM),
// computed once per session.
const uint32_t* session_xamax(nb_ctx* c, nb_session* s, cudaStream_t st) {
  if (!s->xamax) {
    s->xamax = take_spare(c, size_t(s->n) * 4);
    NB_CUDA(cudaMemsetAsync(s->xamax->p, 0, size_t(s->n) * 4, st));
    launch_amax(s->x->as<float>(), s->n, s->h * s->w * s->ci, s->xamax->as<uint32_t>(), st);
    c->launches++;
  }
  return s->xamax->as<uint32_t>();
}

// The session batch's im2col copy for a col stem (built once per geometry;
// stream-ordered before the stem launch that reads it).
const float* session_xcol(nb_ctx* c, nb_session* s, const ConvGeom& g, cudaStream_t st) {
  const std::string sig = std::to_string(g.KH) + "," + std::to_string(g.KW) + "," +
                          std::to_string(g.S) + "," + std::to_string(g.P) + "," +
                          std::to_string(g.OH) + "," + std::to_string(g.OW);
  if (s->xcol_sig != sig) {
    const size_t bytes = size_t(s->n) * g.OH * g.OW * 32 * 4;
    if (!s->xcol || s->xcol->bytes < bytes) {
      if (s->xcol) c->spare.push_back(std::move(s->xcol));
      s->xcol = take_spare(c, bytes);
    }
    launch_im2col32(s->x->as<float>(), s->n, int(s->h), int(s->w), int(s->ci), g.KH, g.KW, g.S,
                    g.P, g.OH, g.OW, s->xcol->as<float>(), st);
    c->launches++;
    s->xcol_sig = sig;
  }
  return s->xcol->as<float>();
}

// Sizes the context's run buffers for plan P over N examples (grow-only; a
// growth synchronizes the device, so nb_evaluate reserves for every
// candidate of a call before any runs).
void reserve_run(nb_ctx* c, const NetPlan& P, int64_t N, int64_t K, int64_t L, bool want_grads,
                 bool explicit_w) {
  c->act.ensure(size_t(P.act_total) * 4);
  if (explicit_w) c->wpack.ensure(size_t(P.w_total) * 4);
  c->part.ensure(size_t(P.part_total) * 8);
  if (P.ws_floats) c->ws.ensure(size_t(P.ws_floats) * 4);
  c->dpre[0].ensure(size_t(P.dpre_floats) * 4);
  c->dpre[1].ensure(size_t(P.dpre_floats) * 4);
  if (want_grads) c->gtmp.ensure(size_t(P.act_total) * 4);
  // misc: probs N*K | ex_loss N | per_channel sum C | fisher table L
  c->misc.ensure(size_t(align64(N * K) + align64(N) + align64(P.ch_total) +
                        align64(int64_t(L) * int64_t(sizeof(FisherLayer)) / 8 + 1)) *
                 8);
  if (P.h16 == 2) c->amax.ensure(size_t(2 * L * N) * 4);
  c->host_io.ensure(size_t(L) * sizeof(FisherLayer));
  c->host_out.ensure(size_t(N * K + N + P.ch_total) * 8);
}

void run_enqueue(nb_session* s, const NetDesc& net, const nb_weights* w, nb_precision prec,
                 bool backward, const RunOut& out, Pending& pend, NetPlan* pre) {
  Range range(backward ? "fisher_enqueue" : "forward_enqueue");
  nb_ctx* c = s->ctx;
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  ctx_activate(c);
  const Spec& s0 = net.specs.front();
  if (s0.ci != s->ci || s0.h != s->h || s0.w != s->w)
    fail(NB_ERR_SHAPE_MISMATCH, "network input shape does not match the session batch");
  if (net.num_classes != s->num_classes)
    fail(NB_ERR_CONFIG, "network class count does not match the session batch");
  const int64_t N = s->n, L = net.L(), K = net.num_classes;
  cudaStream_t st = c->stream;
  NB_CUDA(cudaEventRecord(c->ev_start, st));
  c->prof.start_eval();
  using clk = std::chrono::steady_clock;
  auto tp = clk::now();
  auto phase = [&](const char* name) {
    const auto now = clk::now();
    c->prof.host(name, std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  };
  // (a plan lowered ahead by the scheduler for this batch size and GPU)
  NetPlan own;
  if (!pre) own = lower(net, N, prec, c->num_sms, out.grad_n > 0 ? out.grad_n : N, true);
  NetPlan& P = pre ? *pre : own;
  const bool want_grads = out.grads != nullptr;
  phase("host_lower");

  const bool explicit_w = w && w->layer;
  reserve_run(c, P, N, K, L, want_grads, explicit_w);
  double* d_probs = c->misc.as<double>();
  double* d_exloss = d_probs + align64(N * K);
  double* d_perch = d_exloss + align64(N);
  FisherLayer* d_ftab = reinterpret_cast<FisherLayer*>(d_perch + align64(P.ch_total));
  float* act = c->act.as<float>();
  double* part = c->part.as<double>();

  phase("host_alloc");
  // ---- weights: z-stream prefix (init_weights) or explicit, packed on device
  int64_t wsrc_need = 0;
  if (w && w->layer)
    for (int64_t l = 0; l < L; ++l) wsrc_need += align64(net.specs[l].weight_count());
  if (w && w->head) wsrc_need += align64(K * net.c_last());
  if (wsrc_need) c->wsrc.ensure(size_t(wsrc_need) * 8);
  int64_t wsrc_off = 0;
  // init_weights draws: W_l = z_l * 1/sqrt(Ci*Kh*Kw) (I/nnet.hpp:64-68),
  // packed once per distinct (seed, layer, lowering) into the context's slab.
  // The slab is reset before (never during) a run whose misses do not fit,
  // so no pointer handed to this run is overwritten by it.
  // fp16 split: each layer's weight scale from its largest |w| (host data)
  if (P.h16 == 2)
    for (int64_t l = 0; l < L; ++l) {
      const Spec& sp = net.specs[l];
      const int64_t cnt = sp.weight_count();
      double m = 0.0;
      if (explicit_w) {
        for (int64_t i = 0; i < cnt; ++i) m = std::max(m, std::fabs(w->layer[l][i]));
      } else {
        m = zmax_of(c, net.seed, l, cnt) / std::sqrt(double(sp.ci * sp.kh * sp.kw));
      }
      P.layers[l].b_shift = weight_shift(m);
    }
  std::vector<std::string> keys;
  if (!explicit_w) {
    size_t miss = 0, all = 0;
    for (int64_t l = 0; l < L; ++l) {
      keys.push_back(wkey(net.seed, l, net.specs[l], P.layers[l]));
      const size_t bytes = (size_t(P.layers[l].wpack_floats) * 4 + 255) & ~size_t(255);
      all += bytes;
      if (!c->wcache.count(keys.back())) miss += bytes;
    }
    if (!c->wslab.p) c->wslab.ensure(std::max(kWCacheCap, all));
    if (c->wcache_bytes + miss > c->wslab.bytes) {
      NB_CUDA(cudaStreamSynchronize(st));
      c->wcache.clear();
      c->wcache_bytes = 0;
      if (all > c->wslab.bytes) c->wslab.ensure(all);
    }
  }
  for (int64_t l = 0; l < L; ++l) {
    const Spec& sp = net.specs[l];
    LayerPlan& lp = P.layers[l];
    if (explicit_w) {
      double* dst = c->wsrc.as<double>() + wsrc_off;
      NB_CUDA(cudaMemcpyAsync(dst, w->layer[l], size_t(sp.weight_count()) * 8,
                              cudaMemcpyHostToDevice, st));
      wsrc_off += align64(sp.weight_count());
      lp.wbase = c->wpack.as<float>() + lp.w_off;
      pack_layer(c, lp, dst, 1.0, st);
      continue;
    }
    auto it = c->wcache.find(keys[size_t(l)]);
    if (it != c->wcache.end()) {
      lp.wbase = it->second;
      continue;
    }
    lp.wbase = reinterpret_cast<float*>(static_cast<char*>(c->wslab.p) + c->wcache_bytes);
    c->wcache_bytes += (size_t(lp.wpack_floats) * 4 + 255) & ~size_t(255);
    const double* src = ensure_z(c, net.seed, l, sp.weight_count());
    pack_layer(c, lp, src, 1.0 / std::sqrt(double(sp.ci * sp.kh * sp.kw)), st);
    c->wcache.emplace(keys[size_t(l)], lp.wbase);
  }
  const double* head_src;
  double head_scale;
  if (w && w->head) {
    double* dst = c->wsrc.as<double>() + wsrc_off;
    NB_CUDA(cudaMemcpyAsync(dst, w->head, size_t(K * net.c_last()) * 8,
                            cudaMemcpyHostToDevice, st));
    head_src = dst;
    head_scale = 1.0;
  } else {
    head_src = ensure_z(c, net.seed, L, K * net.c_last());
    head_scale = 1.0 / std::sqrt(double(net.c_last()));  // I/nnet.hpp:72-73
  }

  phase("host_weights");
  // fp16 split: per-(layer, image) max slots of the activations (act_amax)
  // and masked gradients (dpre_amax) the GEMMs read, zeroed for this run
  uint32_t* act_amax = nullptr;
  uint32_t* dpre_amax = nullptr;
  const uint32_t* x_amax = nullptr;
  if (P.h16 == 2) {
    NB_CUDA(cudaMemsetAsync(c->amax.p, 0, size_t(2 * L * N) * 4, st));
    act_amax = c->amax.as<uint32_t>();
    dpre_amax = act_amax + L * N;
    x_amax = session_xamax(c, s, st);
  }
  // ---- forward (I/nnet.hpp:180-197)
  const float* x = s->x->as<float>();
  if (P.layers[0].family[0] == Family::TensorCore && P.layers[0].tcf[0].col)
    x = session_xcol(c, s, P.layers[0].geom, st);
  for (int64_t l = 0; l < L; ++l) {
    float* y = act + P.layers[l].act_off;
    fprop_layer(c, P, P.layers[l], x, y, net.relu[l], st,
                l == 0 ? x_amax : (act_amax ? act_amax + (l - 1) * N : nullptr),
                act_amax && l + 1 < L ? act_amax + l * N : nullptr);
    x = y;
  }

  // ---- head (+ backward start)
  const LayerPlan& last = P.layers[L - 1];
  HeadArgs ha{};
  ha.act = act + last.act_off;
  ha.N = int(N);
  ha.grad_n = double(out.grad_n > 0 ? out.grad_n : N);
  ha.HW = last.geom.OH * last.geom.OW;
  ha.C = last.geom.Co;
  ha.K = int(K);
  ha.head_src = head_src;
  ha.head_scale = head_scale;
  ha.labels = s->labels->as<int32_t>();
  ha.probs = d_probs;
  ha.ex_loss = d_exloss;
  ha.backward = backward;
  ha.relu_last = net.relu[L - 1];
  ha.partial = backward ? part + last.part_off : nullptr;
  ha.dpre = (backward && L > 1) ? c->dpre[0].as<float>() : nullptr;
  ha.g_out = (backward && want_grads) ? c->gtmp.as<float>() + last.act_off : nullptr;
  c->prof.begin(st);
  launch_head(ha, st);
  c->prof.end(st, "head", 0.0, 4.0 * double(last.act_floats) * (backward ? 3 : 1));
  c->launches++;
  if (ha.dpre && dpre_amax) {  // the head's masked gradient, read by the last dgrad
    launch_amax(ha.dpre, N, int64_t(ha.HW) * ha.C, dpre_amax + (L - 1) * N, st);
    c->launches++;
  }

  if (backward) {
    // ---- activation gradients with the fused Fisher epilogue (I/nnet.hpp:225-243)
    int cur = 0;
    for (int64_t l = L - 1; l >= 1; --l) {
      const LayerPlan& lp = P.layers[l];
      const LayerPlan& prev = P.layers[l - 1];
      float* dpre_out = (l - 1 >= 1) ? c->dpre[cur ^ 1].as<float>() : nullptr;
      float* g_out = want_grads ? c->gtmp.as<float>() + prev.act_off : nullptr;
      dgrad_layer(c, P, lp, c->dpre[cur].as<float>(), act + prev.act_off, net.relu[l - 1],
                  dpre_out, g_out, part + prev.part_off, st,
                  dpre_amax ? dpre_amax + l * N : nullptr,
                  dpre_amax ? dpre_amax + (l - 1) * N : nullptr);
      cur ^= 1;
    }
    // ---- Fisher reduction (I/nnet.hpp:330-350)
    FisherLayer* ht = c->host_io.as<FisherLayer>();
    int64_t off = 0;
    int max_c = 1;
    for (int64_t l = 0; l < L; ++l) {
      const LayerPlan& lp = P.layers[l];
      ht[l] = FisherLayer{part + lp.part_off, lp.geom.Co, lp.tiles, off,
                          int64_t(lp.tiles) * lp.geom.Co};
      off += lp.geom.Co;
      max_c = std::max(max_c, lp.geom.Co);
    }
    NB_CUDA(cudaMemcpyAsync(d_ftab, ht, size_t(L) * sizeof(FisherLayer),
                            cudaMemcpyHostToDevice, st));
    c->prof.begin(st);
    launch_fisher_reduce(d_ftab, int(L), max_c, int(N), d_perch, out.s_dev, P.ch_total, st);
    c->prof.end(st, "fisher_reduce", 0.0, 8.0 * double(P.part_total));
    c->launches++;
  }

  phase("host_launch");
  // ---- results back to the host (pinned staging; completed by run_finish)
  double* h_probs = c->host_out.as<double>();
  double* h_exl = h_probs + N * K;
  double* h_perch = h_exl + N;
  NB_CUDA(cudaMemcpyAsync(h_probs, d_probs, size_t(N * K) * 8, cudaMemcpyDeviceToHost, st));
  NB_CUDA(cudaMemcpyAsync(h_exl, d_exloss, size_t(N) * 8, cudaMemcpyDeviceToHost, st));
  if (backward)
    NB_CUDA(cudaMemcpyAsync(h_perch, d_perch, size_t(P.ch_total) * 8, cudaMemcpyDeviceToHost,
                            st));
  if (out.acts || out.grads) {
    c->io.ensure(size_t(P.dpre_floats) * 8);
    int64_t o = 0;
    for (int64_t l = 0; l < L; ++l) {
      const LayerPlan& lp = P.layers[l];
      const ConvGeom& g = lp.geom;
      for (int which = 0; which < 2; ++which) {
        double* dst = which == 0 ? out.acts : out.grads;
        if (!dst) continue;
        const float* src = (which == 0 ? act : c->gtmp.as<float>()) + lp.act_off;
        launch_nhwc32_to_nchw64(src, c->io.as<double>(), N, g.Co, g.OH, g.OW, st);
        c->launches++;
        NB_CUDA(cudaMemcpyAsync(dst + o, c->io.p, size_t(lp.act_floats) * 8,
                                cudaMemcpyDeviceToHost, st));
      }
      o += lp.act_floats;
    }
  }
  NB_CUDA(cudaGetLastError());
  NB_CUDA(cudaEventRecord(c->ev_done, st));
  pend.s = s;
  pend.out = out;
  pend.backward = backward;
  pend.active = true;
  pend.N = N;
  pend.K = K;
  pend.layer_co.clear();
  for (int64_t l = 0; l < L; ++l) pend.layer_co.push_back(P.layers[l].geom.Co);
  pend.ch_total = P.ch_total;
  pend.h_probs = h_probs;
  pend.h_exl = h_exl;
  pend.h_perch = h_perch;
}

void run_finish(Pending& pend) {
  if (!pend.active) return;
  pend.active = false;
  nb_ctx* c = pend.s->ctx;
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  ctx_activate(c);
  const auto t0 = std::chrono::steady_clock::now();
  NB_CUDA(cudaStreamSynchronize(c->stream));
  c->prof.host("host_wait_gpu",
               std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                   .count());
  c->prof.resolve();
  const RunOut& out = pend.out;
  const int64_t N = pend.N, K = pend.K;
  double lsum = 0.0;
  for (int64_t i = 0; i < N; ++i) lsum += pend.h_exl[i];
  if (out.loss) *out.loss = lsum / double(N);
  if (out.probs) std::memcpy(out.probs, pend.h_probs, size_t(N * K) * 8);
  if (out.ex_loss) std::memcpy(out.ex_loss, pend.h_exl, size_t(N) * 8);
  if (pend.backward) {
    // per_layer / total in the reference's order (I/nnet.hpp:345-349)
    double tot = 0.0;
    int64_t o = 0;
    for (size_t l = 0; l < pend.layer_co.size(); ++l) {
      double layer = 0.0;
      for (int64_t ch = 0; ch < pend.layer_co[l]; ++ch) layer += pend.h_perch[o + ch];
      if (out.per_layer) out.per_layer[l] = layer;
      o += pend.layer_co[l];
      tot += layer;
    }
    if (out.per_channel) std::memcpy(out.per_channel, pend.h_perch, size_t(pend.ch_total) * 8);
    if (out.total) *out.total = tot;
  }
}

bool run_ready(const Pending& pend) {
  if (!pend.active) return true;
  nb_ctx* c = pend.s->ctx;
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  ctx_activate(c);
  const cudaError_t e = cudaEventQuery(c->ev_done);
  if (e == cudaErrorNotReady) {
    (void)cudaGetLastError();  // not an error: clear it
    return false;
  }
  return true;  // done, or failed (run_finish reports it)
}

double run_device_ms(nb_ctx* c) {
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  ctx_activate(c);
  float ms = 0.f;
  NB_CUDA(cudaEventElapsedTime(&ms, c->ev_start, c->ev_done));
  return double(ms);
}

void run_network(nb_session* s, const NetDesc& net, const nb_weights* w, nb_precision prec,
                 bool backward, const RunOut& out) {
  Pending p;
  run_enqueue(s, net, w, prec, backward, out, p);
  run_finish(p);
}

// Single-layer entry points (reference_conv / the dgrad step) through the
// same per-layer executors as the network pipeline.
void conv_single(nb_ctx* ctx, const nb_conv_spec* spec, int64_t n, const double* in,
                 const double* w, double* out, int32_t relu, nb_precision prec, bool dgrad,
                 int oh_lo, int oh_hi) {
  nb_layer layer{*spec, relu, 0};
  nb_network one{1, &layer, 2, 0};
  NetDesc d = NetDesc::from(&one);
  if (dgrad) {
    // plan the layer as the second of a pair so the dgrad family is chosen
    NetDesc two = d;
    two.specs.insert(two.specs.begin(), d.specs[0]);
    two.relu.insert(two.relu.begin(), false);
    d = two;
  }
  const Spec& s = d.specs.back();
  std::lock_guard<std::recursive_mutex> lk(ctx->mu);
  ctx_activate(ctx);
  cudaStream_t st = ctx->stream;
  ctx->prof.start_eval();
  NetPlan P = lower(d, n, prec, ctx->num_sms);
  LayerPlan& lp = P.layers.back();
  const int64_t x_cnt = n * s.ci * s.h * s.w, y_cnt = lp.act_floats;
  ctx->io.ensure(size_t(std::max(x_cnt, y_cnt)) * 8);
  ctx->gtmp.ensure(size_t(align64(x_cnt) + align64(y_cnt)) * 4);
  ctx->wsrc.ensure(size_t(s.weight_count()) * 8);
  ctx->wpack.ensure(size_t(P.w_total) * 4);
  if (P.ws_floats) ctx->ws.ensure(size_t(P.ws_floats) * 4);
  P.layers.back().wbase = ctx->wpack.as<float>() + P.layers.back().w_off;
  float* xb = ctx->gtmp.as<float>();
  float* yb = xb + align64(x_cnt);
  NB_CUDA(cudaMemcpyAsync(ctx->wsrc.p, w, size_t(s.weight_count()) * 8, cudaMemcpyHostToDevice,
                          st));
  uint32_t* in_amax = nullptr;
  if (P.h16 == 2) {
    double m = 0.0;
    for (int64_t i = 0; i < s.weight_count(); ++i) m = std::max(m, std::fabs(w[i]));
    lp.b_shift = weight_shift(m);
    ctx->amax.ensure(size_t(n) * 4);
    in_amax = ctx->amax.as<uint32_t>();
    NB_CUDA(cudaMemsetAsync(in_amax, 0, size_t(n) * 4, st));
  }
  pack_layer(ctx, lp, ctx->wsrc.as<double>(), 1.0, st);
  if (!dgrad) {
    NB_CUDA(cudaMemcpyAsync(ctx->io.p, in, size_t(x_cnt) * 8, cudaMemcpyHostToDevice, st));
    launch_nchw64_to_nhwc32(ctx->io.as<double>(), xb, n, int(s.ci), int(s.h), int(s.w), st);
    if (in_amax) launch_amax(xb, n, s.ci * s.h * s.w, in_amax, st);
    if (oh_hi > oh_lo && (oh_lo > 0 || oh_hi < lp.geom.OH)) {
      // a band of output rows (nb_conv_band): tensor-core ranges tile only
      // the band's rows (the other rows of y are left undefined); direct
      // ranges compute every row
      for (int r = 0; r < lp.geom.nranges; ++r) {
        if (lp.family[r] != Family::TensorCore) continue;
        tc::TcArgs& t = lp.tcf[r].tile;
        tc::TcArgs b{};
        if (!tc::plan_tiles(oh_hi - oh_lo, t.OW, t.nimg, t.S, b)) continue;
        t.OH = b.OH;
        t.BW = b.BW;
        t.BH = b.BH;
        t.BNI = b.BNI;
        t.tiles_w = b.tiles_w;
        t.tiles_h = b.tiles_h;
        t.tiles_n = b.tiles_n;
        t.m_tiles = b.m_tiles;
        t.OHp[0] = oh_hi - oh_lo;
        t.oh_base = oh_lo;
        t.ksplit = 1;
      }
    }
    fprop_layer(ctx, P, lp, xb, yb, relu != 0, st, in_amax, nullptr);
    launch_nhwc32_to_nchw64(yb, ctx->io.as<double>(), n, lp.geom.Co, lp.geom.OH, lp.geom.OW, st);
    NB_CUDA(cudaMemcpyAsync(out, ctx->io.p, size_t(y_cnt) * 8, cudaMemcpyDeviceToHost, st));
  } else {
    NB_CUDA(cudaMemcpyAsync(ctx->io.p, in, size_t(y_cnt) * 8, cudaMemcpyHostToDevice, st));
    launch_nchw64_to_nhwc32(ctx->io.as<double>(), yb, n, lp.geom.Co, lp.geom.OH, lp.geom.OW, st);
    if (in_amax) launch_amax(yb, n, int64_t(lp.geom.Co) * lp.geom.OH * lp.geom.OW, in_amax, st);
    dgrad_layer(ctx, P, lp, yb, nullptr, false, nullptr, xb, nullptr, st, in_amax, nullptr);
    launch_nhwc32_to_nchw64(xb, ctx->io.as<double>(), n, int(s.ci), int(s.h), int(s.w), st);
    NB_CUDA(cudaMemcpyAsync(out, ctx->io.p, size_t(x_cnt) * 8, cudaMemcpyDeviceToHost, st));
  }
  NB_CUDA(cudaGetLastError());
  NB_CUDA(cudaStreamSynchronize(st));
  ctx->prof.resolve();
}

void warm_z(nb_ctx* c, const NetDesc& net) {
  std::vector<std::pair<int64_t, int64_t>> want;
  for (int64_t l = 0; l < net.L(); ++l) want.push_back({l, net.specs[l].weight_count()});
  want.push_back({net.L(), net.num_classes * net.c_last()});
  z_prefetch(net.seed, want);
  for (int64_t l = 0; l < net.L(); ++l) ensure_z(c, net.seed, l, net.specs[l].weight_count());
  ensure_z(c, net.seed, net.L(), net.num_classes * net.c_last());
}

}  // namespace nb

using namespace nb;

namespace {

nb_session* make_session(nb_ctx* c, const NetDesc& net, const nb_batch* b) {
  if (!b || b->n < 1) fail(NB_ERR_CONFIG, "batch must hold at least one example");
  const Spec& s0 = net.specs.front();
  const int64_t per = s0.ci * s0.h * s0.w;
  std::vector<double> xs;
  std::vector<int32_t> ls;
  const double* xp = b->inputs;
  const int32_t* lp = b->labels;
  if (!xp) {
    xs.resize(size_t(b->n * per));
    ls.resize(size_t(b->n));
    make_batch(net, b->n, b->seed, xs.data(), ls.data());
    xp = xs.data();
    lp = ls.data();
  } else {
    if (!lp) fail(NB_ERR_CONFIG, "explicit batch inputs need labels");
    for (int64_t i = 0; i < b->n; ++i)
      if (lp[i] < 0 || lp[i] >= net.num_classes) fail(NB_ERR_CONFIG, "label out of range");
  }
  auto s = std::make_unique<nb_session>();
  s->ctx = c;
  s->n = b->n;
  s->ci = s0.ci;
  s->h = s0.h;
  s->w = s0.w;
  s->num_classes = net.num_classes;
  s->seed = b->seed;
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  ctx_activate(c);
  auto take = [&](size_t bytes) { return take_spare(c, bytes); };
  s->x = take(size_t(b->n * per) * 4);
  s->labels = take(size_t(b->n) * 4);
  c->io.ensure(size_t(b->n * per) * 8);
  NB_CUDA(cudaMemcpyAsync(c->io.p, xp, size_t(b->n * per) * 8, cudaMemcpyHostToDevice,
                          c->stream));
  launch_nchw64_to_nhwc32(c->io.as<double>(), s->x->as<float>(), b->n, int(s0.ci), int(s0.h),
                          int(s0.w), c->stream);
  c->launches++;
  NB_CUDA(cudaMemcpyAsync(s->labels->p, lp, size_t(b->n) * 4, cudaMemcpyHostToDevice,
                          c->stream));
  NB_CUDA(cudaStreamSynchronize(c->stream));
  return s.release();
}

void need(const void* p, const char* what) {
  if (!p) fail(NB_ERR_CONFIG, std::string("null ") + what);
}

// A one-layer network around a bare ConvSpec (for nb_conv_forward/dgrad).
struct OneLayer {
  nb_layer layer;
  nb_network net;
  explicit OneLayer(const nb_conv_spec* spec, int relu) {
    layer.spec = *spec;
    layer.relu = relu;
    layer.reserved = 0;
    net = nb_network{1, &layer, 2, 0};
  }
};

}  // namespace

extern "C" {

int nb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

nb_status nb_ctx_create(int device, nb_ctx** out) {
  return guard([&] {
    need(out, "output pointer");
    int n = nb_device_count();
    if (n < 1) fail(NB_ERR_NO_DEVICE, "no CUDA device visible: nb200 has no CPU fallback");
    if (device < 0 || device >= n) fail(NB_ERR_NO_DEVICE, "device index out of range");
    cudaDeviceProp prop{};
    NB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
      fail(NB_ERR_NO_DEVICE, std::string("nb200 is built for sm_100a (B200); device is ") +
                                 prop.name);
    auto c = std::make_unique<nb_ctx>();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    NB_CUDA(cudaSetDevice(device));
    static const bool prefer_shared = [] {
      const char* e = std::getenv("NB_CARVEOUT");
      return e && std::atoi(e) == 1;
    }();
    if (prefer_shared) NB_CUDA(cudaDeviceSetCacheConfig(cudaFuncCachePreferShared));
    NB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    NB_CUDA(cudaEventCreate(&c->ev_start));
    NB_CUDA(cudaEventCreate(&c->ev_done));
    *out = c.release();
  });
}

int nb_ctx_device(const nb_ctx* ctx) { return ctx ? ctx->device : -1; }

nb_status nb_ctx_destroy(nb_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaStream_t st = ctx->stream;
    cudaEvent_t e0 = ctx->ev_start, e1 = ctx->ev_done;
    delete ctx;
    cudaStreamDestroy(st);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  });
}

void* nb_ctx_stream(nb_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

nb_status nb_ctx_set_profiling(nb_ctx* ctx, int enable) {
  return guard([&] {
    need(ctx, "context");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ctx->prof.on = enable != 0;
    ctx->prof.every = enable > 1 ? enable : 1;
    ctx->prof.calls = 0;
  });
}

nb_status nb_ctx_kernel_stats(nb_ctx* ctx, nb_kernel_stat* stats, int32_t cap, int32_t* count) {
  return guard([&] {
    need(ctx, "context");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    int32_t i = 0;
    for (const auto& [name, k] : ctx->prof.stats) {
      if (i < cap && stats) {
        nb_kernel_stat& o = stats[i];
        std::memset(&o, 0, sizeof(o));
        std::strncpy(o.name, name.c_str(), sizeof(o.name) - 1);
        o.launches = k.launches;
        o.ms = k.ms;
        o.flops = k.flops;
        o.bytes = k.bytes;
      }
      ++i;
    }
    if (count) *count = i;
  });
}

nb_status nb_ctx_reset_stats(nb_ctx* ctx) {
  return guard([&] {
    need(ctx, "context");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ctx->prof.stats.clear();
  });
}

nb_status nb_ctx_clear_caches(nb_ctx* ctx) {
  return guard([&] {
    need(ctx, "context");
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ctx_activate(ctx);
    NB_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->wcache.clear();
    ctx->wcache_bytes = 0;
    ctx->zdev.clear();
    ctx->zlen.clear();
  });
}

int64_t nb_ctx_launch_count(nb_ctx* ctx) { return ctx ? ctx->launches : 0; }

nb_status nb_session_create(nb_ctx* ctx, const nb_network* shape_net, const nb_batch* batch,
                            nb_session** out) {
  return guard([&] {
    need(ctx, "context");
    need(out, "output pointer");
    NetDesc d = NetDesc::from(shape_net);
    *out = make_session(ctx, d, batch);
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ctx_activate(ctx);
    warm_z(ctx, d);  // candidates draw prefixes of the origin's z-streams
  });
}

nb_status nb_session_destroy(nb_session* s) {
  return guard([&] {
    if (!s) return;
    std::lock_guard<std::recursive_mutex> lk(s->ctx->mu);
    ctx_activate(s->ctx);
    // keep the batch buffers for the context's next session (bounded)
    if (s->ctx->spare.size() < 12) {
      s->ctx->spare.push_back(std::move(s->x));
      s->ctx->spare.push_back(std::move(s->labels));
      if (s->xcol) s->ctx->spare.push_back(std::move(s->xcol));
      if (s->xamax) s->ctx->spare.push_back(std::move(s->xamax));
    }
    delete s;
  });
}

nb_ctx* nb_session_ctx(nb_session* s) { return s ? s->ctx : nullptr; }

nb_status nb_session_fisher(nb_session* s, const nb_network* net, const nb_weights* w,
                            nb_precision prec, nb_fisher_out* out) {
  return guard([&] {
    need(s, "session");
    need(out, "output");
    NetDesc d = NetDesc::from(net);
    RunOut ro;
    ro.per_channel = out->per_channel;
    ro.per_layer = out->per_layer;
    ro.total = &out->total;
    ro.loss = &out->loss;
    ro.probs = out->probs;
    run_network(s, d, w, prec, true, ro);
    out->seed = s->seed;
  });
}

// fisher_potential (I/nnet.hpp:321-350) of one network over a batch split
// into consecutive example shards, one session (normally one GPU) each --
// SURVEY 8(e)'s secondary axis, for when there are fewer networks than GPUs.
// Every shard plans its launches for the whole batch and divides dz by the
// whole batch's N, so its per-example sums s_nc are bitwise those of one
// session holding the whole batch.  They are gathered into shards[0]'s GPU
// (peer copies over NVLink) and reduced there by k_fisher_reduce in the same
// fixed order; loss and probabilities are concatenated in example order.
nb_status nb_fisher_sharded(nb_session* const* shards, int32_t count, const nb_network* net,
                            const nb_weights* w, nb_precision prec, nb_fisher_out* out) {
  return guard([&] {
    Range range("nb_fisher_sharded");
    need(shards, "shards");
    need(out, "output");
    if (count < 1) fail(NB_ERR_CONFIG, "need at least one shard");
    NetDesc d = NetDesc::from(net);
    int64_t n_all = 0;
    for (int32_t i = 0; i < count; ++i) {
      need(shards[i], "shard session");
      for (int32_t j = 0; j < i; ++j)
        if (shards[j]->ctx == shards[i]->ctx)
          fail(NB_ERR_CONFIG, "example shards must use distinct contexts");
      if (shards[i]->seed != shards[0]->seed)
        fail(NB_ERR_CONFIG, "example shards must hold slices of one batch (same seed)");
      n_all += shards[i]->n;
    }
    const int64_t L = d.L(), K = d.num_classes;
    int64_t ch_total = 0;
    for (int64_t l = 0; l < L; ++l) ch_total += d.specs[l].co_eff();
    nb_ctx* root = shards[0]->ctx;
    // Every shard context stays locked for the whole call (in one global
    // order, so concurrent sharded calls cannot deadlock): the gather
    // buffers are sized, written by the shards and read by the root's
    // reduction without another call resizing or overwriting them between.
    std::vector<nb_ctx*> held;
    for (int32_t i = 0; i < count; ++i) held.push_back(shards[i]->ctx);
    std::sort(held.begin(), held.end(), std::less<nb_ctx*>());
    std::vector<std::unique_lock<std::recursive_mutex>> locks;
    for (nb_ctx* c : held) locks.emplace_back(c->mu);
    ctx_activate(root);
    root->shard_s.ensure(size_t(n_all * ch_total) * 8);
    std::vector<double> ex_loss(static_cast<size_t>(n_all));
    std::vector<Pending> pend(static_cast<size_t>(count));
    std::vector<int64_t> first(static_cast<size_t>(count));
    int64_t n0 = 0;
    for (int32_t i = 0; i < count; ++i) {
      nb_session* sh = shards[i];
      first[size_t(i)] = n0;
      double* s_dev = root->shard_s.as<double>();
      if (i > 0) {
        ctx_activate(sh->ctx);
        sh->ctx->shard_s.ensure(size_t(sh->n * ch_total) * 8);
        s_dev = sh->ctx->shard_s.as<double>();
      }
      RunOut ro;
      ro.probs = out->probs ? out->probs + n0 * K : nullptr;
      ro.ex_loss = ex_loss.data() + n0;
      ro.grad_n = n_all;
      ro.s_dev = s_dev;
      run_enqueue(sh, d, w, prec, true, ro, pend[size_t(i)]);
      n0 += sh->n;
    }
    for (auto& p : pend) run_finish(p);
    double lsum = 0.0;
    for (double v : ex_loss) lsum += v;
    out->loss = lsum / double(n_all);
    out->seed = shards[0]->seed;

    ctx_activate(root);
    cudaStream_t st = root->stream;
    double* S = root->shard_s.as<double>();
    for (int32_t i = 1; i < count; ++i) {
      nb_ctx* c = shards[i]->ctx;
      NB_CUDA(cudaMemcpyPeerAsync(S + first[size_t(i)] * ch_total, root->device, c->shard_s.p,
                                  c->device, size_t(shards[i]->n * ch_total) * 8, st));
    }
    // the gathered s_nc as one-tile partials: s = 0 - (s_nc) per example,
    // squared exactly as the unsharded reduction squares s_nc
    root->shard_aux.ensure(size_t(L) * sizeof(FisherLayer) + size_t(ch_total) * 8);
    root->host_io.ensure(size_t(L) * sizeof(FisherLayer) + size_t(ch_total) * 8);
    FisherLayer* ht = root->host_io.as<FisherLayer>();
    int64_t off = 0;
    int max_c = 1;
    std::vector<int64_t> co(static_cast<size_t>(L));
    for (int64_t l = 0; l < L; ++l) {
      const int c = int(d.specs[l].co_eff());
      ht[l] = FisherLayer{S + off, c, 1, off, ch_total};
      co[size_t(l)] = c;
      off += c;
      max_c = std::max(max_c, c);
    }
    FisherLayer* d_tab = root->shard_aux.as<FisherLayer>();
    double* d_pc = reinterpret_cast<double*>(d_tab + L);
    NB_CUDA(cudaMemcpyAsync(d_tab, ht, size_t(L) * sizeof(FisherLayer), cudaMemcpyHostToDevice,
                            st));
    launch_fisher_reduce(d_tab, int(L), max_c, int(n_all), d_pc, nullptr, 0, st);
    root->launches++;
    double* h_pc = reinterpret_cast<double*>(ht + L);
    NB_CUDA(cudaMemcpyAsync(h_pc, d_pc, size_t(ch_total) * 8, cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaGetLastError());
    NB_CUDA(cudaStreamSynchronize(st));
    // per_layer / total in the reference's order (I/nnet.hpp:345-349)
    double tot = 0.0;
    int64_t o = 0;
    for (int64_t l = 0; l < L; ++l) {
      double layer = 0.0;
      for (int64_t ch = 0; ch < co[size_t(l)]; ++ch) layer += h_pc[o + ch];
      if (out->per_layer) out->per_layer[l] = layer;
      o += co[size_t(l)];
      tot += layer;
    }
    if (out->per_channel) std::memcpy(out->per_channel, h_pc, size_t(ch_total) * 8);
    out->total = tot;
  });
}

nb_status nb_session_forward(nb_session* s, const nb_network* net, const nb_weights* w,
                             nb_precision prec, double* probs, double* loss) {
  return guard([&] {
    need(s, "session");
    NetDesc d = NetDesc::from(net);
    RunOut ro;
    ro.probs = probs;
    ro.loss = loss;
    run_network(s, d, w, prec, false, ro);
  });
}

nb_status nb_fisher_potential(nb_ctx* ctx, const nb_network* net, const nb_weights* w,
                              const nb_batch* batch, nb_precision prec, nb_fisher_out* out) {
  return guard([&] {
    need(ctx, "context");
    need(out, "output");
    NetDesc d = NetDesc::from(net);
    std::unique_ptr<nb_session> s(make_session(ctx, d, batch));
    RunOut ro;
    ro.per_channel = out->per_channel;
    ro.per_layer = out->per_layer;
    ro.total = &out->total;
    ro.loss = &out->loss;
    ro.probs = out->probs;
    run_network(s.get(), d, w, prec, true, ro);
    out->seed = batch->seed;
  });
}

nb_status nb_forward(nb_ctx* ctx, const nb_network* net, const nb_weights* w,
                     const nb_batch* batch, nb_precision prec, double* probs,
                     double* example_loss, double* loss) {
  return guard([&] {
    need(ctx, "context");
    NetDesc d = NetDesc::from(net);
    std::unique_ptr<nb_session> s(make_session(ctx, d, batch));
    RunOut ro;
    ro.probs = probs;
    ro.ex_loss = example_loss;
    ro.loss = loss;
    run_network(s.get(), d, w, prec, false, ro);
  });
}

nb_status nb_activation_gradients(nb_ctx* ctx, const nb_network* net, const nb_weights* w,
                                  const nb_batch* batch, nb_precision prec, double* acts,
                                  double* grads) {
  return guard([&] {
    need(ctx, "context");
    NetDesc d = NetDesc::from(net);
    std::unique_ptr<nb_session> s(make_session(ctx, d, batch));
    RunOut ro;
    ro.acts = acts;
    ro.grads = grads;
    run_network(s.get(), d, w, prec, grads != nullptr, ro);
  });
}

// reference_conv / layer_forward over n images through the same fprop
// kernels the network pipeline uses.
nb_status nb_conv_forward(nb_ctx* ctx, const nb_conv_spec* spec, int64_t n, const double* x,
                          const double* w, double* y, int32_t relu, nb_precision prec) {
  return guard([&] {
    need(ctx, "context");
    need(spec, "spec");
    need(x, "input");
    need(w, "weights");
    need(y, "output");
    conv_single(ctx, spec, n, x, w, y, relu, prec, false);
  });
}

nb_status nb_conv_band(nb_ctx* ctx, const nb_conv_spec* spec, int64_t n, const double* x,
                       const double* w, int32_t oh_lo, int32_t oh_hi, double* y,
                       nb_precision prec) {
  return guard([&] {
    need(ctx, "context");
    need(spec, "spec");
    need(x, "input");
    need(w, "weights");
    need(y, "output");
    Spec s = Spec::from(*spec);
    s.validate();
    if (oh_lo < 0 || oh_hi > s.oh() || oh_lo >= oh_hi) fail(NB_ERR_CONFIG, "bad output row band");
    conv_single(ctx, spec, n, x, w, y, 0, prec, false, oh_lo, oh_hi);
  });
}

nb_status nb_conv_dgrad(nb_ctx* ctx, const nb_conv_spec* spec, int64_t n, const double* dy,
                        const double* w, double* dx, nb_precision prec) {
  return guard([&] {
    need(ctx, "context");
    need(spec, "spec");
    need(dy, "dy");
    need(w, "weights");
    need(dx, "dx");
    conv_single(ctx, spec, n, dy, w, dx, 0, prec, true);
  });
}

}  // extern "C"
