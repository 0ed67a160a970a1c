// The per-GPU engine: contexts, resident batches (sessions), the lowering of
// a network to kernel plans, and the Fisher / forward pipelines.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.hpp"
#include "kernels.cuh"
#include "kernels_tc.cuh"

namespace nb {

void cuda_check(cudaError_t e, const char* what);
#define NB_CUDA(x) ::nb::cuda_check((x), #x)

// Growable device buffer (grown only between launches on the owning stream).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n);
  ~DevBuf();
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n);
  ~PinnedBuf();
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// Kernel family of one output-channel range (the lowering of SURVEY 7:
// ConvSpec range -> family).
enum class Family { Direct = 0, TensorCore = 1 };

// Tensor-core lowering of one GEMM (a range's fprop or a layer's dgrad).
struct TcPlan {
  int bn = 0;
  bool pair = false;   // CTA-pair (cta_group::2) launch, bn = the pair's N tile
  bool mc = false;     // multicast cluster of 2 (B stage shared, cta_group::1 MMAs)
  bool kwf = false;    // kw-fused 64-channel plan (B rows kw*64 + c, K = kh x channels)
  tc::TcArgs tile{};   // M/N tiling and operand bases (pointers filled at launch)
  int64_t w_off = 0;   // hi at w_off, lo at w_off + w_n (floats, layer-relative)
  int64_t w_n = 0;
  int b_rows = 0, b_k = 0;
  // padded plan: K per tap rounded up to 32-channel chunks (0 = exact); the
  // packed weights' extra K columns are zero, the activations' extra
  // channels are TMA out-of-bounds zero fill
  int kp = 0;
  // densified grouped range: the original group count (0 = not densified);
  // the packed weights are block-diagonal over the full channel range
  int dense = 0;
  // split-K epilogue pixel chunks (splitk_hw_chunks at the planning batch)
  int hw_chunks = 1;
  // stem on the session's im2col copy of the batch: A = (N, OH, OW, 32) with
  // K = (tap, channel) in 32 columns, a 1x1 GEMM (session_xcol)
  bool col = false;
  // images per M tile at the planning batch size: the halo-mode decision
  // (launch_tc) is made on it, so an example shard (fewer images, possibly
  // fewer per tile) runs the whole batch's K order
  int plan_bni = 0;
};

// Lowered layer: geometry + per-range family + packed-weight offsets.
struct LayerPlan {
  ConvGeom geom{};
  Family family[kMaxRanges]{};
  // fprop tensor-core plans of ranges 0 .. nranges-1 (family == TensorCore);
  // sized per layer (a plan is lowered per candidate and copied around)
  std::vector<TcPlan> tcf;
  Family dgrad_family = Family::Direct;
  TcPlan tcd;                // dgrad tensor-core plan
  int64_t wpack_floats = 0;  // floats of all packings of this layer
  int64_t w_off = 0;         // offset of this layer's block in the weight arena
  float* wbase = nullptr;    // the layer's packed weights at run time (arena or cache)
  int64_t act_off = 0;       // offset (floats) of the layer's output activation
  int64_t act_floats = 0;
  int64_t part_off = 0;      // offset (doubles) of its Fisher partials
  int tiles = 0;
  double fprop_flops = 0, dgrad_flops = 0;
  int h16 = 0;      // tensor-core weights packed as 16-bit halves (NetPlan::h16)
  int b_shift = 0;  // fp16 halves: the weights were packed times 2^b_shift
};

struct NetPlan {
  std::vector<LayerPlan> layers;
  int64_t act_total = 0, w_total = 0, part_total = 0, dpre_floats = 0;
  int64_t ws_floats = 0;  // split-K workspace (floats)
  int64_t ch_total = 0;  // sum_l C_l
  bool split3 = false;    // split fp32 tensor-core numerics (NB_PREC_FP32)
  int h16 = 0;            // ... in 16-bit halves (kind::f16): 1 bf16, 2 fp16 (scaled); 0 = 3xTF32
};

// plan_n: the batch size launch shapes are chosen for (0 = n; an example
// shard passes the whole batch's size)
NetPlan lower(const NetDesc& net, int64_t n, nb_precision prec, int num_sms = 148,
              int64_t plan_n = 0, bool stem_col = false);

struct KStat {
  int64_t launches = 0;
  double ms = 0, flops = 0, bytes = 0;
};

// Event-timed launch records (profiling) resolved at the end of each call.
class Profiler {
 public:
  bool on = false;
  int every = 1;        // events on every `every`-th evaluation (sampling)
  int64_t calls = 0;
  bool active = false;  // this evaluation records kernel events
  void start_eval() { active = on && (calls++ % every == 0); }
  void begin(cudaStream_t st);
  void end(cudaStream_t st, const char* family, double flops, double bytes);
  void resolve();  // stream must be synchronized
  // host-side wall time of a pipeline phase (recorded while profiling)
  void host(const char* phase, double ms) {
    if (!on) return;
    KStat& k = stats[phase];
    k.launches += 1;
    k.ms += ms;
  }
  std::map<std::string, KStat> stats;
  ~Profiler();

 private:
  struct Pending {
    cudaEvent_t a, b;
    std::string fam;
    double flops, bytes;
  };
  std::vector<cudaEvent_t> pool_;
  std::vector<Pending> pending_;
  cudaEvent_t cur_ = nullptr;
  cudaEvent_t get();
};

}  // namespace nb

struct nb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::recursive_mutex mu;
  nb::DevBuf act, wpack, part, misc, wsrc, dpre[2], gtmp, io, ws, tilecnt, trace;
  nb::DevBuf legal;  // semantic-legality workspace (legality.cu)
  nb::DevBuf shard_s, shard_aux;  // example-sharded Fisher (nb_fisher_sharded)
  // fp16 split: per-(layer, image) max |value| of the activations and of the
  // masked gradients each GEMM reads (float bits), reset per run
  nb::DevBuf amax;
  // max |z| of a cached z-stream prefix (seed, stream, count): the fp16
  // weight scale of init_weights layers
  std::map<std::tuple<uint64_t, int64_t, int64_t>, double> zmax;
  int num_sms = 148;
  nb::PinnedBuf host_io, host_out;
  // bracket the evaluation in flight on this context's stream (one at a
  // time): its device duration and completion, for the scheduler
  cudaEvent_t ev_start = nullptr, ev_done = nullptr;
  // device copies of z streams keyed by (seed, stream index)
  std::map<std::pair<uint64_t, int64_t>, std::unique_ptr<nb::DevBuf>> zdev;
  std::map<std::pair<uint64_t, int64_t>, int64_t> zlen;
  // packed init_weights weights per (seed, layer, lowering) -- candidates of
  // one search share most layers with the origin, so each distinct layer is
  // packed once per context
  // (bump-allocated from one slab, so no cudaMalloc runs per candidate)
  std::map<std::string, float*> wcache;
  nb::DevBuf wslab;
  size_t wcache_bytes = 0;
  nb::Profiler prof;
  int64_t launches = 0;
  // batch buffers of destroyed sessions, reused by the next ones (no
  // cudaMalloc / cudaFree per session)
  std::vector<std::unique_ptr<nb::DevBuf>> spare;
};

struct nb_session {
  nb_ctx* ctx = nullptr;
  int64_t n = 0;
  int64_t ci = 0, h = 0, w = 0, num_classes = 0;
  uint64_t seed = 0;
  std::unique_ptr<nb::DevBuf> x;       // (N, H, W, Ci) fp32
  std::unique_ptr<nb::DevBuf> labels;  // N int32
  // im2col copy of x for a narrow stem (N, OH, OW, 32), built once per stem
  // geometry (xcol_sig) -- the batch is resident and fixed
  std::unique_ptr<nb::DevBuf> xcol;
  std::string xcol_sig;
  // per-image max |x| (float bits) for the fp16 split of the first GEMM,
  // computed once (the im2col copy holds the same values and zeros)
  std::unique_ptr<nb::DevBuf> xamax;
};

namespace nb {

// Outputs requested from one pipeline run (host pointers, nullable).
struct RunOut {
  double* per_channel = nullptr;
  double* per_layer = nullptr;
  double* total = nullptr;
  double* probs = nullptr;
  double* ex_loss = nullptr;
  double* loss = nullptr;
  double* acts = nullptr;   // reference layout, see nb_activation_gradients
  double* grads = nullptr;
  // example sharding (nb_fisher_sharded): the whole batch's size, which dz is
  // divided by and the lowering plans for (0 = this session's own N), and a
  // device buffer receiving s_nc as [n][ch_total] doubles (nullable)
  int64_t grad_n = 0;
  double* s_dev = nullptr;
};

// An evaluation enqueued on its session's stream, not yet collected.
struct Pending {
  nb_session* s = nullptr;
  RunOut out;
  bool backward = false, active = false;
  int64_t N = 0, K = 0, ch_total = 0;
  std::vector<int> layer_co;
  double *h_probs = nullptr, *h_exl = nullptr, *h_perch = nullptr;  // pinned staging
};

// Runs forward (and, when `backward`, activation gradients + Fisher) of `net`
// on the session's resident batch: run_enqueue issues every kernel and the
// result copies asynchronously on the session's stream, run_finish waits for
// them and fills `out`.  One evaluation per session may be in flight.
// `pre`: the network's plan lowered ahead for this session's batch size and
// GPU (nb_evaluate), used and updated in place; null = lower here.
void run_enqueue(nb_session* s, const NetDesc& net, const nb_weights* w, nb_precision prec,
                 bool backward, const RunOut& out, Pending& pend, NetPlan* pre = nullptr);
// Sizes a context's run buffers for plan P (grow-only).
void reserve_run(nb_ctx* c, const NetPlan& P, int64_t N, int64_t K, int64_t L, bool want_grads,
                 bool explicit_w);
void run_finish(Pending& pend);
// The evaluation's kernels and result copies have completed on the device
// (run_finish will not block).
bool run_ready(const Pending& pend);
// Device time of the last evaluation collected on the context (ms).
double run_device_ms(nb_ctx* c);
void run_network(nb_session* s, const NetDesc& net, const nb_weights* w, nb_precision prec,
                 bool backward, const RunOut& out);

void ctx_activate(nb_ctx* c);
// oh_lo < oh_hi: fprop of the output rows [oh_lo, oh_hi) only (the rest of
// out undefined; nb_conv_band)
void conv_single(nb_ctx* ctx, const nb_conv_spec* spec, int64_t n, const double* in,
                 const double* w, double* out, int32_t relu, nb_precision prec, bool dgrad,
                 int oh_lo = 0, int oh_hi = 0);
void warm_z(nb_ctx* c, const NetDesc& net);

}  // namespace nb
