// nestopt <-> nb200 bridge: the reference-side binding of the B200 hot path.
//
// This header is what a nestopt maintainer adds to the reference's C++ host
// (proj/include/nestopt stays intact and is used through the include path):
// it converts the reference's value types to the plain-C descriptors of
// include/nb200.h, calls the sm_100a library through that C ABI, and turns
// nb_status codes back into the *same* nestopt exception classes
// (I/errors.hpp), so callers written against the reference -- evaluate_
// candidate-style code catching `const nestopt::Error&` -- behave the same.
//
// Replaced reference functions (I/ = proj/include/nestopt/):
//   fisher_potential   I/nnet.hpp:321  -> nb200::fisher_potential
//   forward            I/nnet.hpp:180  -> nb200::forward (probs + loss)
//   layer_forward      I/nnet.hpp:130  -> nb200::layer_forward
//   reference_conv     I/interp.hpp:152 -> nb200::reference_conv
//   evaluate_all       I/search.hpp:315 -> nb200::evaluate_all_gpu
//   run_search         I/search.hpp:364 -> nb200::run_search_gpu
// Everything else (draw_candidates, apply, check_semantic_legality,
// derived_spec, rank_survivors, the report writers) is the reference's own
// code, called unchanged.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <tuple>
#include <type_traits>
#include <random>
#include <sstream>
#include <map>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "nb200.h"
#include "nestopt/nestopt.hpp"

namespace nb200 {

// A CUDA / device failure.  Deliberately NOT a nestopt::Error: the
// reference's evaluate_candidate turns nestopt::Error into a semantic
// rejection, and a device failure must end the search, not reject candidates.
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// A semantic run the GPU legality kernel cannot key (nb_semantic_legality
// NB_ERR_UNSUPPORTED, or a nest the bridge cannot compile).  There is no
// host fallback on the search path: the search fails loudly.
struct LegalityUnsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// A nest the masked box executor cannot decompose into dense boxes
// (execute_boxes); nb200::execute interprets any nest.
struct BoxUnsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Which implementation answered the semantic-legality checks of a gate pass.
struct LegalityCounts {
  std::atomic<long long> gpu{0}, host{0};
};

// nb_status -> the nestopt exception class it mirrors (include/nb200.h).
[[noreturn]] inline void rethrow(nb_status s) {
  const std::string m = nb_last_error();
  switch (s) {
    case NB_ERR_INVALID_SPEC: throw nestopt::InvalidSpec(m);
    case NB_ERR_CONFIG: throw nestopt::ConfigError(m);
    case NB_ERR_SHAPE_MISMATCH: throw nestopt::ShapeMismatch(m);
    case NB_ERR_CAP_EXCEEDED: throw nestopt::CapExceeded(m);
    case NB_ERR_TRANSFORM: throw nestopt::TransformError(m);
    case NB_ERR_PARSE: throw nestopt::ParseError(m);
    case NB_ERR_IO: throw nestopt::IoError(m);
    case NB_ERR_GENERIC: throw nestopt::Error(m);
    default: throw DeviceError("nb200 [" + std::to_string(int(s)) + "]: " + m);
  }
}

inline void check(nb_status s) {
  if (s != NB_OK) rethrow(s);
}

// ---- descriptors ----------------------------------------------------------

// ConvSpec (I/ir.hpp:26-87) -> nb_conv_spec; keeps the split array alive.
struct SpecDesc {
  std::vector<nb_channel_split> splits;
  nb_conv_spec c{};
  explicit SpecDesc(const nestopt::ConvSpec& s) {
    for (const auto& r : s.channel_splits) splits.push_back({r.begin, r.end, r.groups});
    c = nb_conv_spec{s.ci, s.co, s.h, s.w, s.kh, s.kw, s.stride, s.pad, s.groups,
                     s.bottleneck_out, s.spatial_div_h, s.spatial_div_w,
                     int64_t(splits.size()), splits.empty() ? nullptr : splits.data()};
  }
};

// Network (I/nnet.hpp:28-79) -> nb_network (+ explicit weights when the
// network carries them, else the device draws init_weights(seed) itself).
struct NetDesc {
  std::vector<SpecDesc> specs;
  std::vector<nb_layer> layers;
  std::vector<const double*> wptr;
  std::vector<double> head;
  nb_network c{};
  nb_weights w{};
  bool explicit_weights = false;
  explicit NetDesc(const nestopt::Network& n) {
    specs.reserve(n.layers.size());
    for (const auto& l : n.layers) specs.emplace_back(l.spec);
    for (size_t i = 0; i < n.layers.size(); ++i)
      layers.push_back(nb_layer{specs[i].c, n.layers[i].relu ? 1 : 0, 0});
    c = nb_network{int64_t(layers.size()), layers.data(), n.num_classes, n.seed};
    if (!n.weights.empty()) {
      explicit_weights = true;
      for (const auto& t : n.weights) wptr.push_back(t.data.data());
      for (const auto& row : n.head) head.insert(head.end(), row.begin(), row.end());
      w = nb_weights{wptr.data(), head.data()};
    }
  }
  const nb_weights* weights() const { return explicit_weights ? &w : nullptr; }
};

// Batch (I/nnet.hpp:81-85) -> nb_batch with the reference's own values.
struct BatchDesc {
  std::vector<double> x;
  std::vector<int32_t> y;
  nb_batch c{};
  explicit BatchDesc(const nestopt::Batch& b) {
    for (const auto& t : b.inputs) x.insert(x.end(), t.data.begin(), t.data.end());
    for (int v : b.labels) y.push_back(int32_t(v));
    c = nb_batch{int64_t(b.inputs.size()), x.data(), y.data(), b.seed};
  }
};

// ---- contexts and sessions ---------------------------------------------------

class Context {
 public:
  explicit Context(int device = 0) { check(nb_ctx_create(device, &p_)); }
  ~Context() { nb_ctx_destroy(p_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  nb_ctx* get() const { return p_; }

 private:
  nb_ctx* p_ = nullptr;
};

// A batch resident in one GPU's HBM (the search's fixed batch).
class Session {
 public:
  Session(Context& ctx, const nestopt::Network& shape, const nestopt::Batch& batch) {
    NetDesc nd(shape);
    BatchDesc bd(batch);
    check(nb_session_create(ctx.get(), &nd.c, &bd.c, &p_));
  }
  ~Session() { nb_session_destroy(p_); }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;
  nb_session* get() const { return p_; }

 private:
  nb_session* p_ = nullptr;
};

// ---- hot-path functions --------------------------------------------------

inline nestopt::FisherReport to_report(const nestopt::Network& net,
                                       const std::vector<double>& per_channel,
                                       const std::vector<double>& per_layer, double total,
                                       uint64_t seed) {
  nestopt::FisherReport r;
  r.per_layer = per_layer;
  r.total = total;
  r.seed = seed;
  size_t off = 0;
  for (const auto& l : net.layers) {
    const size_t c = size_t(l.spec.co_eff());
    r.per_channel.emplace_back(per_channel.begin() + long(off), per_channel.begin() + long(off + c));
    off += c;
  }
  return r;
}

inline size_t channel_total(const nestopt::Network& net) {
  size_t t = 0;
  for (const auto& l : net.layers) t += size_t(l.spec.co_eff());
  return t;
}

// fisher_potential, I/nnet.hpp:321-352.
inline nestopt::FisherReport fisher_potential(Context& ctx, const nestopt::Network& net,
                                              const nestopt::Batch& batch,
                                              nb_precision prec = NB_PREC_FP32) {
  NetDesc nd(net);
  BatchDesc bd(batch);
  std::vector<double> pc(channel_total(net)), pl(net.layers.size());
  nb_fisher_out out{pc.data(), pl.data(), 0.0, 0, 0.0, nullptr};
  check(nb_fisher_potential(ctx.get(), &nd.c, nd.weights(), &bd.c, prec, &out));
  return to_report(net, pc, pl, out.total, out.seed);
}

inline nestopt::FisherReport fisher_potential(Session& s, const nestopt::Network& net,
                                              nb_precision prec = NB_PREC_FP32) {
  NetDesc nd(net);
  std::vector<double> pc(channel_total(net)), pl(net.layers.size());
  nb_fisher_out out{pc.data(), pl.data(), 0.0, 0, 0.0, nullptr};
  check(nb_session_fisher(s.get(), &nd.c, nd.weights(), prec, &out));
  return to_report(net, pc, pl, out.total, out.seed);
}

// forward, I/nnet.hpp:180-197: the outputs ForwardCache exposes to callers
// (probs, example_loss, loss).
struct ForwardResult {
  std::vector<std::vector<double>> probs;
  std::vector<double> example_loss;
  double loss = 0.0;
};

inline ForwardResult forward(Context& ctx, const nestopt::Network& net, const nestopt::Batch& batch,
                             nb_precision prec = NB_PREC_FP32) {
  NetDesc nd(net);
  BatchDesc bd(batch);
  const size_t n = batch.inputs.size(), k = size_t(net.num_classes);
  std::vector<double> probs(n * k);
  ForwardResult r;
  r.example_loss.resize(n);
  check(nb_forward(ctx.get(), &nd.c, nd.weights(), &bd.c, prec, probs.data(),
                   r.example_loss.data(), &r.loss));
  for (size_t i = 0; i < n; ++i)
    r.probs.emplace_back(probs.begin() + long(i * k), probs.begin() + long((i + 1) * k));
  return r;
}

// reference_conv<double>, I/interp.hpp:151-186 (one image).
inline nestopt::TensorF reference_conv(Context& ctx, const nestopt::ConvSpec& spec,
                                       const nestopt::TensorF& input,
                                       const nestopt::TensorF& weights,
                                       nb_precision prec = NB_PREC_FP32, bool relu = false) {
  SpecDesc sd(spec);
  nestopt::TensorF out({spec.co_eff(), spec.out_h(), spec.out_w()});
  check(nb_conv_forward(ctx.get(), &sd.c, 1, input.data.data(), weights.data.data(),
                        out.data.data(), relu ? 1 : 0, prec));
  return out;
}

// layer_forward, I/nnet.hpp:130-141.
inline nestopt::TensorF layer_forward(Context& ctx, const nestopt::Layer& layer,
                                      const nestopt::TensorF& weights,
                                      const nestopt::TensorF& input,
                                      nb_precision prec = NB_PREC_FP32) {
  return reference_conv(ctx, layer.spec, input, weights, prec, layer.relu);
}

// ---- general loop nests (execute, I/interp.hpp:67-145) ----------------------

// A LoopNest in the executable form of nb_nest (include/nb200.h): per block
// of compute_blocks (I/ir.hpp:163-218), its multiply-accumulate statements
// with their coordinate programs over the block's loop values and their
// access programs over the statement's domain values.
namespace detail {

// AffineExpr (I/affine.hpp:17-72) -> postfix (op, arg) pairs over slots
inline void emit_into(const nestopt::AffineExpr& e, const std::map<std::string, int>& slots,
                      std::vector<int64_t>& out) {
  using K = nestopt::AffineExpr::Kind;
  switch (e.kind) {
    case K::Const: out.insert(out.end(), {0, e.k}); return;
    case K::Var: {
      auto it = slots.find(e.var);
      if (it == slots.end()) throw nestopt::Error("unbound iterator '" + e.var + "'");
      out.insert(out.end(), {1, it->second});
      return;
    }
    case K::Add:
      for (const auto& a : e.args) emit_into(a, slots, out);
      out.insert(out.end(), {2, int64_t(e.args.size())});
      return;
    case K::Mul: emit_into(e.args[0], slots, out); out.insert(out.end(), {3, e.k}); return;
    case K::Div: emit_into(e.args[0], slots, out); out.insert(out.end(), {4, e.k}); return;
    case K::Mod: emit_into(e.args[0], slots, out); out.insert(out.end(), {5, e.k}); return;
  }
}
inline std::vector<int64_t> emit(const nestopt::AffineExpr& e,
                                 const std::map<std::string, int>& slots) {
  std::vector<int64_t> out;
  emit_into(e, slots, out);
  return out;
}
}  // namespace detail

class NestProgram {
 public:
  NestProgram(const nestopt::LoopNest& nest, const std::string& out_name,
              const std::vector<long long>& out_shape, const std::vector<long long>& in_shape,
              const std::vector<long long>& w_shape) {
    using namespace nestopt;
    std::vector<StmtRec> recs;
    for (const Block& b : compute_blocks(nest)) {
      const NestPart& part = nest.parts[size_t(b.part)];
      std::map<std::string, int> slots;
      for (size_t i = 0; i < b.iters.size(); ++i) slots[b.iters[i].name] = int(i);
      for (auto [si, depth] : b.stmts) {
        const Statement& st = part.stmts[size_t(si)];
        if (st.kind != StmtKind::Mac) continue;  // the output starts at zero
        StmtRec r;
        for (int d = 0; d < depth; ++d) r.extents.push_back(b.iters[size_t(d)].extent);
        std::map<std::string, int> dslots;
        for (size_t i = 0; i < st.domain.size(); ++i) {
          dslots[st.domain[i]] = int(i);
          r.coord.push_back(detail::emit(st.coord.at(st.domain[i]), slots));
        }
        for (const AccessMap& acc : st.accesses) {
          AccRec ar;
          ar.tensor = acc.tensor == out_name ? 0 : acc.tensor == "I" ? 1 : acc.tensor == "K" ? 2 : -1;
          if (ar.tensor < 0) throw UnboundTensor("tensor '" + acc.tensor + "' is not bound");
          if (ar.tensor != 0 && acc.mode != AccessMode::Read)
            throw Error("nest writes more than one tensor");
          ar.zero_pad = acc.zero_pad ? 1 : 0;
          for (const auto& e : acc.indices) ar.idx.push_back(detail::emit(e, dslots));
          r.acc.push_back(std::move(ar));
        }
        recs.push_back(std::move(r));
      }
    }
    recs_ = std::move(recs);
    for (auto& r : recs_) {
      r.coord_c.clear();
      for (auto& c : r.coord) r.coord_c.push_back(nb_nest_expr{int32_t(c.size() / 2), c.data()});
      r.acc_c.clear();
      for (auto& a : r.acc) {
        a.idx_c.clear();
        for (auto& c : a.idx) a.idx_c.push_back(nb_nest_expr{int32_t(c.size() / 2), c.data()});
        r.acc_c.push_back(nb_nest_access{a.tensor, a.zero_pad, int32_t(a.idx_c.size()),
                                         a.idx_c.data()});
      }
      stmts_.push_back(nb_nest_stmt{int32_t(r.extents.size()), r.extents.data(),
                                    int32_t(r.coord_c.size()), r.coord_c.data(),
                                    int32_t(r.acc_c.size()), r.acc_c.data()});
    }
    c_ = nb_nest{};
    c_.num_stmts = int64_t(stmts_.size());
    c_.stmts = stmts_.data();
    auto fill = [](int64_t* d, int32_t& rank, const std::vector<long long>& s) {
      rank = int32_t(s.size());
      for (int i = 0; i < 4; ++i) d[i] = i < rank ? s[size_t(i)] : 1;
    };
    fill(c_.out_shape, c_.out_rank, out_shape);
    fill(c_.in_shape, c_.in_rank, in_shape);
    fill(c_.w_shape, c_.w_rank, w_shape);
  }
  const nb_nest* get() const { return &c_; }

 private:
  struct AccRec {
    int32_t tensor = 0, zero_pad = 0;
    std::vector<std::vector<int64_t>> idx;
    std::vector<nb_nest_expr> idx_c;
  };
  struct StmtRec {
    std::vector<int64_t> extents;
    std::vector<std::vector<int64_t>> coord;
    std::vector<nb_nest_expr> coord_c;
    std::vector<AccRec> acc;
    std::vector<nb_nest_access> acc_c;
  };
  std::vector<StmtRec> recs_;
  std::vector<nb_nest_stmt> stmts_;
  nb_nest c_{};
};

// execute<T> (I/interp.hpp:67-145) of any transformed conv nest on the GPU,
// with the bindings "I" (Ci,H,W) and "K" (Co_eff,Ci,Kh,Kw) of the reference
// and the output allocated from provenance.  T = long long (exact) or double.
template <typename T>
nestopt::Tensor<T> execute(Context& ctx, const nestopt::LoopNest& nest,
                           const nestopt::ExecEnv<T>& env) {
  using namespace nestopt;
  if (!nest.provenance) throw UnboundTensor("output tensor 'O' is not bound");
  std::string out_name;
  for (const auto& part : nest.parts)
    for (const auto& st : part.stmts)
      for (const auto& acc : st.accesses)
        if (acc.mode != AccessMode::Read) {
          if (!out_name.empty() && out_name != acc.tensor)
            throw Error("nest writes more than one tensor");
          out_name = acc.tensor;
        }
  if (out_name.empty()) throw Error("nest has no written tensor");
  const Tensor<T>& ti = env.bindings.at("I");
  const Tensor<T>& tk = env.bindings.at("K");
  Tensor<T> out(output_shape(*nest.provenance));
  NestProgram prog(nest, out_name, out.shape, ti.shape, tk.shape);
  check(nb_nest_execute(ctx.get(), prog.get(), std::is_integral<T>::value ? 1 : 0,
                        ti.data.data(), tk.data.data(), out.data.data()));
  return out;
}

// ---- the masked box executor (SURVEY 7 "Non-ConvSpec nests", 8(f) #2) -------

// What execute_boxes ran: the boxes (output channel range x output row band x
// input channel range, every column and tap) and their MACs against the
// nest's own instance count.
struct BoxReport {
  struct Box {
    long long co_lo, co_hi, oh_lo, oh_hi, ci_lo, ci_hi;
  };
  std::vector<Box> boxes;
  long long box_macs = 0, nest_macs = 0;
};

// execute<T> (I/interp.hpp:67-145) of a transformed conv nest -- one with
// no ConvSpec such as the paper's Sequence 1 included -- as tensor-core
// implicit GEMMs over boxes.  A GPU cell pass (nb_nest_cells) finds, per
// output cell, the input-channel range and the number of MAC instances
// adding into it.  Every covered cell must receive exactly its channel
// range x every tap (a dense box row); cells with the same range over whole
// output rows are grouped into (output-channel range x row band) boxes,
// and each box runs as a conv over its channel slices restricted to its row
// band (nb_conv_band: the tensor-core tiles cover only the band).  Cells no
// instance writes stay zero, as in execute.  The arithmetic is the
// requested precision tier's (FP32 default: exact for integer inputs whose
// sums stay below 2^22, within the tier's tolerance otherwise); a nest that
// does not decompose throws BoxUnsupported (nb200::execute interprets it).
template <typename T>
nestopt::Tensor<T> execute_boxes(Context& ctx, const nestopt::LoopNest& nest,
                                 const nestopt::ExecEnv<T>& env,
                                 nb_precision prec = NB_PREC_FP32, BoxReport* report = nullptr) {
  using namespace nestopt;
  if (!nest.provenance) throw UnboundTensor("output tensor 'O' is not bound");
  std::string out_name;
  for (const auto& part : nest.parts)
    for (const auto& st : part.stmts)
      for (const auto& acc : st.accesses)
        if (acc.mode != AccessMode::Read) out_name = acc.tensor;
  if (out_name.empty()) throw Error("nest has no written tensor");
  const Tensor<T>& ti = env.bindings.at("I");
  const Tensor<T>& tk = env.bindings.at("K");
  const ConvSpec& ps = *nest.provenance;
  Tensor<T> out(output_shape(ps));
  NestProgram prog(nest, out_name, out.shape, ti.shape, tk.shape);
  const long long Co = out.shape[0], OH = out.shape[1], OW = out.shape[2];
  const long long Ci = ti.shape[0], H = ti.shape[1], W = ti.shape[2];
  const long long taps = ps.kh * ps.kw;
  const size_t cells = size_t(Co * OH * OW);
  std::vector<int32_t> lo(cells), hi(cells);
  std::vector<int64_t> cnt(cells);
  check(nb_nest_cells(ctx.get(), prog.get(), lo.data(), hi.data(), cnt.data()));
  long long nest_macs = 0;
  for (size_t i = 0; i < cells; ++i) {
    nest_macs += cnt[i];
    if (cnt[i] && cnt[i] != (long long)(hi[i] - lo[i] + 1) * taps)
      throw BoxUnsupported("execute_boxes: an output cell is not a dense channel-range box");
  }
  // (channel range, row band) -> the output channels computing it over whole rows
  std::map<std::tuple<int, int, long long, long long>, std::vector<long long>> runs;
  for (long long co = 0; co < Co; ++co) {
    long long oh = 0;
    while (oh < OH) {
      const size_t c0 = size_t((co * OH + oh) * OW);
      for (long long ow = 1; ow < OW; ++ow)
        if ((cnt[c0 + size_t(ow)] != 0) != (cnt[c0] != 0) ||
            (cnt[c0] && (lo[c0 + size_t(ow)] != lo[c0] || hi[c0 + size_t(ow)] != hi[c0])))
          throw BoxUnsupported("execute_boxes: an output row mixes channel ranges");
      if (!cnt[c0]) {
        ++oh;
        continue;
      }
      long long end = oh + 1;
      while (end < OH) {
        const size_t c1 = size_t((co * OH + end) * OW);
        if (!cnt[c1] || lo[c1] != lo[c0] || hi[c1] != hi[c0]) break;
        ++end;
      }
      runs[{lo[c0], hi[c0], oh, end}].push_back(co);
      oh = end;
    }
  }
  BoxReport rep;
  rep.nest_macs = nest_macs;
  for (auto& [key, cos] : runs) {
    const auto [clo, chi, oh0, oh1] = key;
    for (size_t i = 0; i < cos.size();) {
      size_t j = i + 1;
      while (j < cos.size() && cos[j] == cos[j - 1] + 1) ++j;
      rep.boxes.push_back({cos[i], cos[j - 1] + 1, oh0, oh1, clo, chi + 1});
      i = j;
    }
  }
  for (const auto& b : rep.boxes) {
    const long long nci = b.ci_hi - b.ci_lo, nco = b.co_hi - b.co_lo;
    ConvSpec bs = ps;
    bs.ci = nci;
    bs.co = nco;
    bs.groups = 1;
    bs.bottleneck_out = 1;
    bs.channel_splits.clear();
    std::vector<double> xs(size_t(nci * H * W)), ws(size_t(nco * nci * taps)),
        ys(size_t(nco * OH * OW));
    for (long long c = 0; c < nci; ++c)
      for (long long k = 0; k < H * W; ++k)
        xs[size_t(c * H * W + k)] = double(ti.data[size_t((b.ci_lo + c) * H * W + k)]);
    for (long long o = 0; o < nco; ++o)
      for (long long c = 0; c < nci; ++c)
        for (long long t = 0; t < taps; ++t)
          ws[size_t((o * nci + c) * taps + t)] =
              double(tk.data[size_t(((b.co_lo + o) * Ci + b.ci_lo + c) * taps + t)]);
    SpecDesc d(bs);
    check(nb_conv_band(ctx.get(), &d.c, 1, xs.data(), ws.data(), int32_t(b.oh_lo),
                       int32_t(b.oh_hi), ys.data(), prec));
    for (long long o = 0; o < nco; ++o)
      for (long long oh = b.oh_lo; oh < b.oh_hi; ++oh)
        for (long long ow = 0; ow < OW; ++ow) {
          const double v = ys[size_t((o * OH + oh) * OW + ow)];
          T& dst = out.data[size_t(((b.co_lo + o) * OH + oh) * OW + ow)];
          if constexpr (std::is_integral<T>::value) dst += T(std::llround(v));
          else dst += T(v);
        }
    rep.box_macs += nco * (b.oh_hi - b.oh_lo) * OW * nci * taps;
  }
  if (report) *report = std::move(rep);
  return out;
}

// ---- semantic legality on the GPU -----------------------------------------

namespace detail {

// Interval of a postfix program over slot intervals (any enclosing box is a
// valid packing bound for nb_semantic_legality).
inline std::pair<int64_t, int64_t> interval(const std::vector<int64_t>& code,
                                            const std::vector<std::pair<int64_t, int64_t>>& slot) {
  auto fdiv = [](int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
  };
  std::vector<std::pair<int64_t, int64_t>> st;
  for (size_t i = 0; i + 1 < code.size(); i += 2) {
    const int64_t op = code[i], arg = code[i + 1];
    switch (op) {
      case 0: st.push_back({arg, arg}); break;
      case 1: st.push_back(slot.at(size_t(arg))); break;
      case 2: {
        std::pair<int64_t, int64_t> s{0, 0};
        for (int64_t k = 0; k < arg; ++k) {
          s.first += st.back().first;
          s.second += st.back().second;
          st.pop_back();
        }
        st.push_back(s);
        break;
      }
      case 3: {
        auto& t = st.back();
        t = arg >= 0 ? std::pair<int64_t, int64_t>{t.first * arg, t.second * arg}
                     : std::pair<int64_t, int64_t>{t.second * arg, t.first * arg};
        break;
      }
      case 4: {
        auto& t = st.back();
        t = arg > 0 ? std::pair<int64_t, int64_t>{fdiv(t.first, arg), fdiv(t.second, arg)}
                    : std::pair<int64_t, int64_t>{fdiv(t.second, arg), fdiv(t.first, arg)};
        break;
      }
      default: {
        auto& t = st.back();
        if (arg > 0 && fdiv(t.first, arg) == fdiv(t.second, arg)) {
          const int64_t q = fdiv(t.first, arg) * arg;
          t = {t.first - q, t.second - q};
        } else {
          t = arg > 0 ? std::pair<int64_t, int64_t>{0, arg - 1}
                      : std::pair<int64_t, int64_t>{arg + 1, 0};
        }
      }
    }
  }
  return st.back();
}

// One nest in nb_legal_nest form: an entry per statement of each block of
// compute_blocks (I/ir.hpp:169-204), with the schedule-rank formula of
// for_each_instance's walk (I/ir.hpp:262-292): at loop level k the walk
// first visits the n_k statements of that depth, then ext_k subtrees of
// T(k+1) instances each, so an instance at depth d with loop values v has
// rank block_base + sum_{k<d} (n_k + v_k T(k+1)) + its index among the
// depth-d statements.
class LegalNest {
 public:
  LegalNest(const nestopt::LoopNest& nest, std::map<std::string, int>& sid,
            const std::map<std::string, int>* tensor_ids,
            const std::vector<char>* written) {
    using namespace nestopt;
    std::map<std::string, int> gid_of;  // compute_dependences' interning, I/ir.hpp:343-346
    for (const auto& part : nest.parts)
      for (const auto& st : part.stmts) gid_of.emplace(st.id, int(gid_of.size()));
    int64_t block_base = 0;
    for (const Block& b : compute_blocks(nest)) {
      const NestPart& part = nest.parts[size_t(b.part)];
      const size_t D = b.iters.size();
      std::vector<int64_t> n_at(D + 1, 0), T(D + 2, 0);
      for (auto [si, depth] : b.stmts) n_at[size_t(depth)]++;
      T[D] = n_at[D];
      for (size_t k = D; k-- > 0;) T[k] = n_at[k] + b.iters[k].extent * T[k + 1];
      std::map<std::string, int> slots;
      std::vector<std::pair<int64_t, int64_t>> loop_rng;
      for (size_t i = 0; i < D; ++i) {
        slots[b.iters[i].name] = int(i);
        loop_rng.push_back({0, std::max<int64_t>(0, b.iters[i].extent - 1)});
      }
      std::vector<int64_t> seen(D + 1, 0);
      for (auto [si, depth] : b.stmts) {
        const Statement& st = part.stmts[size_t(si)];
        Rec r;
        r.id = st.id;
        r.sid = sid.emplace(st.id, int(sid.size())).first->second;
        r.gid = gid_of.at(st.id);
        r.rank_base = block_base + seen[size_t(depth)]++;
        for (int k = 0; k < depth; ++k) {
          r.rank_base += n_at[size_t(k)];
          r.extents.push_back(b.iters[size_t(k)].extent);
          r.stride.push_back(T[size_t(k) + 1]);
        }
        std::map<std::string, int> dslots;
        std::vector<std::pair<int64_t, int64_t>> dom_rng;
        for (size_t i = 0; i < st.domain.size(); ++i) {
          dslots[st.domain[i]] = int(i);
          r.coord.push_back(emit(st.coord.at(st.domain[i]), slots));
          const auto iv = interval(r.coord.back(), loop_rng);
          r.lo.push_back(iv.first);
          r.hi.push_back(iv.second);
          dom_rng.push_back(iv);
        }
        if (tensor_ids)
          for (const AccessMap& acc : st.accesses) {
            const int t = tensor_ids->at(acc.tensor);
            if (!(*written)[size_t(t)]) continue;  // read-only: never in a pair
            Acc a;
            a.tensor = t;
            a.mode = acc.mode == AccessMode::Read ? 0 : acc.mode == AccessMode::Write ? 1 : 2;
            for (const auto& e : acc.indices) {
              a.idx.push_back(emit(e, dslots));
              const auto iv = interval(a.idx.back(), dom_rng);
              a.lo.push_back(iv.first);
              a.hi.push_back(iv.second);
            }
            r.acc.push_back(std::move(a));
          }
        recs_.push_back(std::move(r));
      }
      block_base += T[0];
    }
    for (auto& r : recs_) {
      for (auto& c : r.coord) r.coord_c.push_back(nb_nest_expr{int32_t(c.size() / 2), c.data()});
      for (auto& a : r.acc) {
        for (auto& c : a.idx) a.idx_c.push_back(nb_nest_expr{int32_t(c.size() / 2), c.data()});
        r.acc_c.push_back(nb_legal_access{a.tensor, a.mode, int32_t(a.idx_c.size()),
                                          a.idx_c.data(), a.lo.data(), a.hi.data()});
      }
      stmts_.push_back(nb_legal_stmt{r.sid, r.gid, int32_t(r.extents.size()), r.extents.data(),
                                     r.rank_base, r.stride.data(), int32_t(r.coord_c.size()),
                                     r.coord_c.data(), r.lo.data(), r.hi.data(),
                                     int32_t(r.acc_c.size()), r.acc_c.data()});
    }
    c_ = nb_legal_nest{int64_t(stmts_.size()), stmts_.data()};
  }
  const nb_legal_nest* get() const { return &c_; }
  const std::string& id(int entry) const { return recs_.at(size_t(entry)).id; }
  size_t ndomain(int entry) const { return recs_.at(size_t(entry)).coord.size(); }

 private:
  struct Acc {
    int32_t tensor = 0, mode = 0;
    std::vector<std::vector<int64_t>> idx;
    std::vector<nb_nest_expr> idx_c;
    std::vector<int64_t> lo, hi;
  };
  struct Rec {
    std::string id;
    int32_t sid = 0, gid = 0;
    int64_t rank_base = 0;
    std::vector<int64_t> extents, stride, lo, hi;
    std::vector<std::vector<int64_t>> coord;
    std::vector<nb_nest_expr> coord_c;
    std::vector<Acc> acc;
    std::vector<nb_legal_access> acc_c;
  };
  std::vector<Rec> recs_;
  std::vector<nb_legal_stmt> stmts_;
  nb_legal_nest c_{};
};

}  // namespace detail

// check_semantic_legality (I/transforms.hpp:598-663) with the brute-force
// dependence check on the GPU (nb_semantic_legality): the same CapExceeded
// throws (checked on the host from instance counts, as the reference does
// first), verdicts and reasons.  Every check runs on the device -- there is
// no host fallback; a nest the kernel cannot key throws LegalityUnsupported.
inline nestopt::LegalityResult check_semantic_legality(
    Context& ctx, const nestopt::LoopNest& original, const nestopt::LoopNest& transformed,
    long long cap = nestopt::kDefaultInstanceCap) {
  using namespace nestopt;
  const long long nt = instance_count(transformed);
  if (nt > cap) throw CapExceeded("transformed nest exceeds brute-force cap");
  const long long no = instance_count(original);
  if (no > cap)
    throw CapExceeded("instance count exceeds brute-force cap of " + std::to_string(cap));
  std::map<std::string, int> tensor_ids;  // I/ir.hpp:347-352 interning order
  for (const auto& part : original.parts)
    for (const auto& st : part.stmts)
      for (const auto& a : st.accesses) tensor_ids.emplace(a.tensor, int(tensor_ids.size()));
  std::vector<char> written(tensor_ids.size(), 0);
  for (const auto& part : original.parts)
    for (const auto& st : part.stmts)
      for (const auto& a : st.accesses)
        if (a.mode != AccessMode::Read) written[size_t(tensor_ids.at(a.tensor))] = 1;
  std::map<std::string, int> sid;
  std::unique_ptr<detail::LegalNest> lo, lt;
  try {
    lo = std::make_unique<detail::LegalNest>(original, sid, &tensor_ids, &written);
    lt = std::make_unique<detail::LegalNest>(transformed, sid, nullptr, nullptr);
  } catch (const std::exception& e) {
    throw LegalityUnsupported(std::string("semantic legality: nest not compilable for the GPU "
                                          "check: ") + e.what());
  }
  nb_legal_out out{};
  const nb_status s = nb_semantic_legality(ctx.get(), lo->get(), lt->get(), &out);
  if (s == NB_ERR_UNSUPPORTED)
    throw LegalityUnsupported(std::string("semantic legality: ") + nb_last_error());
  check(s);
  switch (out.verdict) {
    case NB_LEGAL: return {Verdict::Legal, ""};
    case NB_ILLEGAL_DUPLICATE:
      return {Verdict::Illegal, "transformed schedule duplicates an instance"};
    case NB_NOT_APPLICABLE:
      return {Verdict::NotApplicable, "instance sets differ (neural rewrite changes the domain)"};
    default: break;
  }
  std::ostringstream os;
  os << "dependence " << lo->id(out.src_stmt) << "(";
  for (size_t i = 0; i < lo->ndomain(out.src_stmt); ++i) os << (i ? "," : "") << out.src_coord[i];
  os << ") -> " << lo->id(out.dst_stmt) << "(";
  for (size_t i = 0; i < lo->ndomain(out.dst_stmt); ++i) os << (i ? "," : "") << out.dst_coord[i];
  os << ") is reordered";
  return {Verdict::Illegal, os.str()};
}

// ---- the candidate scheduler -------------------------------------------

// The host half of evaluate_candidate (I/search.hpp:219-293): replays the
// per-layer steps, flushes semantic runs through the reference's brute-force
// legality check, lowers each layer with derived_spec, and repairs shapes.
// Returns false when the candidate is decided here (semantic rejection or
// a non-neural survivor); otherwise `net` is the network to score.
// Differences from the reference: repair_network's init_weights (0.8 s on
// the R34 chain) is skipped -- the device draws the same weights from the
// cached z-streams -- so only Network::validate() runs after propagation.
inline bool host_gates(nestopt::Candidate& cand, const nestopt::Network& origin,
                       const nestopt::SearchConfig& cfg,
                       const nestopt::FisherReport& origin_fisher, nestopt::Network& net,
                       Context* legal_ctx = nullptr, LegalityCounts* counts = nullptr) {
  using namespace nestopt;
  std::vector<ConvSpec> specs;
  for (size_t l = 0; l < origin.layers.size(); ++l) {
    LoopNest nest = conv_nest(origin.layers[l].spec);
    LoopNest run_origin = nest;
    bool pending_semantic = false;
    auto flush = [&](size_t s) {
      if (!pending_semantic) return true;
      LegalityResult lr =
          legal_ctx ? nb200::check_semantic_legality(*legal_ctx, run_origin, nest, cfg.cap)
                    : nestopt::check_semantic_legality(run_origin, nest, cfg.cap);
      if (counts) ++(legal_ctx ? counts->gpu : counts->host);
      pending_semantic = false;
      if (lr.verdict == Verdict::Illegal) {
        cand.status = CandidateStatus::RejectedSemantic;
        cand.reason = "layer " + std::to_string(l) + " steps up to " + std::to_string(s) +
                      ": " + lr.reason;
        return false;
      }
      return true;
    };
    for (size_t s = 0; s < cand.layer_seqs[l].steps.size(); ++s) {
      const Transform& t = cand.layer_seqs[l].steps[s];
      try {
        if (t.cls() == TransformClass::Semantic) {
          nest = apply(nest, t);
          pending_semantic = true;
        } else {
          if (!flush(s)) return false;
          nest = apply(nest, t);
          run_origin = nest;
        }
      } catch (const Error& e) {
        cand.status = CandidateStatus::RejectedSemantic;
        cand.reason = "layer " + std::to_string(l) + " step " + std::to_string(s + 1) + " (" +
                      to_dsl(t) + "): " + e.what();
        return false;
      }
    }
    try {
      if (!flush(cand.layer_seqs[l].steps.size())) return false;
    } catch (const Error& e) {
      cand.status = CandidateStatus::RejectedSemantic;
      cand.reason = "layer " + std::to_string(l) + ": " + e.what();
      return false;
    }
    std::optional<ConvSpec> spec = derived_spec(nest);
    if (!spec) {
      cand.status = CandidateStatus::RejectedSemantic;
      cand.reason = "layer " + std::to_string(l) + ": rewritten nest is not a convolution operator";
      return false;
    }
    specs.push_back(*spec);
  }
  net.layers = origin.layers;
  net.num_classes = origin.num_classes;
  net.seed = origin.seed;
  net.weights.clear();
  net.head.clear();
  for (size_t l = 0; l < specs.size(); ++l) net.layers[l].spec = specs[l];
  try {
    // repair_network's shape propagation (I/nnet.hpp:372-380)
    for (size_t l = 1; l < net.layers.size(); ++l) {
      const ConvSpec& prev = net.layers[l - 1].spec;
      ConvSpec& cur = net.layers[l].spec;
      cur.ci = prev.co_eff();
      cur.h = prev.out_h();
      cur.w = prev.out_w();
    }
    net.validate();
  } catch (const Error& e) {
    cand.status = CandidateStatus::RejectedSemantic;
    cand.reason = std::string("network repair failed: ") + e.what();
    return false;
  }
  const ConvSpec& in0 = origin.layers[0].spec;
  const ConvSpec& in1 = net.layers[0].spec;
  if (in0.ci != in1.ci || in0.h != in1.h || in0.w != in1.w) {
    cand.status = CandidateStatus::RejectedSemantic;
    cand.reason = "network input shape changed";
    return false;
  }
  cand.macs = network_macs(net);
  if (!cand.neural) {
    cand.status = CandidateStatus::Survivor;
    cand.fisher_total = origin_fisher.total;
    cand.fisher_per_layer = origin_fisher.per_layer;
    return false;
  }
  return true;
}

// Stated tolerance of each arithmetic mode on Fisher totals of deep chains
// (paper_2102_06599_b200/api.py TOLERANCE_DEEP: the
// 33-layer ResNet-34 chain at N=128).
inline double total_tolerance(nb_precision p) {
  return p == NB_PREC_FP32 ? 1.5e-3 : p == NB_PREC_TF32 ? 5e-2 : 3e-4;
}

// Near-threshold band of a throughput mode (api.py RECHECK_BAND): a
// candidate's score and the origin's may each be off by the mode's total
// tolerance in opposite directions, so a decision can only differ from the
// reference's when |cand - origin| <= 2 x tolerance; the band adds 25% on
// top.  Candidates inside it are re-scored, with the origin, in
// NB_PREC_SIMT (true fp32, totals within 3e-4 of the fp64 reference on the
// 33-layer chain) before the accept decision.  Only ties closer than SIMT's
// own 2 x 3e-4 can then differ from the reference (the documented
// near-threshold tie band, api.py TIE_BAND).
inline double recheck_band(nb_precision p) {
  return p == NB_PREC_SIMT ? 0.0 : 2.5 * total_tolerance(p);
}

// |cand - origin| <= band * |origin|: the decision needs the SIMT recheck.
inline bool near_threshold(double cand, double origin, nb_precision p) {
  const double band = recheck_band(p);
  return band > 0 && std::fabs(cand - origin) <= band * std::fabs(origin);
}

inline bool same_network(const nestopt::Network& a, const nestopt::Network& b) {
  if (a.layers.size() != b.layers.size() || a.num_classes != b.num_classes || a.seed != b.seed)
    return false;
  for (size_t l = 0; l < a.layers.size(); ++l) {
    const nestopt::ConvSpec &x = a.layers[l].spec, &y = b.layers[l].spec;
    if (a.layers[l].relu != b.layers[l].relu || x.ci != y.ci || x.co != y.co || x.h != y.h ||
        x.w != y.w || x.kh != y.kh || x.kw != y.kw || x.stride != y.stride || x.pad != y.pad ||
        x.bottleneck_out != y.bottleneck_out || x.spatial_div_h != y.spatial_div_h ||
        x.spatial_div_w != y.spatial_div_w)
      return false;
    auto rx = x.ranges(), ry = y.ranges();
    if (rx.size() != ry.size()) return false;
    for (size_t i = 0; i < rx.size(); ++i)
      if (rx[i].begin != ry[i].begin || rx[i].end != ry[i].end || rx[i].groups != ry[i].groups)
        return false;
  }
  return true;
}

// draw_candidates (I/search.hpp:188-214) with the candidate indices spread
// over `threads` host threads.  Every index seeds its own
// mt19937_64 from detail::mix_seed(seed, idx) and draws through the
// reference's own detail::draw_step, so the candidates are identical to the
// serial loop's; only the per-layer conv_nest of the origin is built once.
inline std::vector<nestopt::Candidate> draw_candidates(const nestopt::Network& origin,
                                                       const nestopt::SearchConfig& cfg,
                                                       int threads) {
  using namespace nestopt;
  cfg.validate();
  std::vector<LoopNest> base(origin.layers.size());
  for (size_t l = 0; l < origin.layers.size(); ++l)
    if (cfg.layer_allowed(l)) base[l] = conv_nest(origin.layers[l].spec);
  std::vector<Candidate> out(size_t(std::max(cfg.candidate_count, 0)));
  std::atomic<size_t> next{0};
  auto worker = [&]() {
    for (size_t idx; (idx = next.fetch_add(1)) < out.size();) {
      std::mt19937_64 rng(nestopt::detail::mix_seed(cfg.seed, uint64_t(idx)));
      Candidate cand;
      for (size_t l = 0; l < origin.layers.size(); ++l) {
        TransformSequence seq;
        if (cfg.layer_allowed(l)) {
          const int len = std::uniform_int_distribution<int>(0, cfg.max_seq_len)(rng);
          LoopNest nest = base[l];
          for (int st = 0; st < len; ++st) {
            LoopNest nxt;
            auto t = nestopt::detail::draw_step(rng, nest, cfg, nxt);
            if (!t) break;
            seq.steps.push_back(*t);
            nest = std::move(nxt);
            if (t->cls() == TransformClass::Neural) cand.neural = true;
          }
        }
        cand.layer_seqs.push_back(std::move(seq));
      }
      out[idx] = std::move(cand);
    }
  };
  const int nt = std::max(1, std::min<int>(threads, int(out.size())));
  if (nt == 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
  }
  return out;
}

// Scheduler statistics of one evaluate_all_gpu call.
struct GpuStats {
  int64_t scored = 0, evaluated = 0, deduplicated = 0, origin_equal = 0, rechecked = 0;
  int64_t legality_gpu = 0, legality_host = 0;  // semantic runs checked on each side
  int64_t rank_rechecked = 0, requeued = 0;
  std::vector<double> est_flops, busy_ms;
  std::vector<int64_t> evaluations;
  double gates_ms = 0, gpu_ms = 0;
};

// evaluate_all, I/search.hpp:315-334, on GPU sessions: host gates on
// cfg.jobs threads (same per-index result slots as the reference), then
// every neural candidate that passed them is scored by nb_evaluate (dedupe +
// LPT over the sessions, one worker per GPU), then the reference's accept
// rule and rejection message are applied.
inline GpuStats evaluate_all_gpu(std::vector<nestopt::Candidate>& cands,
                                 const nestopt::Network& origin,
                                 const nestopt::SearchConfig& cfg,
                                 const nestopt::FisherReport& origin_fisher,
                                 const std::vector<Session*>& sessions,
                                 nb_precision prec = NB_PREC_FP32) {
  using namespace nestopt;
  GpuStats st;
  auto t0 = std::chrono::steady_clock::now();
  std::vector<Network> nets(cands.size());
  std::vector<char> pending(cands.size(), 0);
  {
    const int jobs = std::max(1, std::min<int>(cfg.jobs, int(cands.size())));
    std::atomic<size_t> next{0};
    LegalityCounts counts;
    std::exception_ptr err;
    std::mutex err_mu;
    // each gate thread checks its semantic runs on its own context of a
    // session's GPU (every check on the device, none on the host)
    auto worker = [&](int j) {
      try {
        std::unique_ptr<Context> lctx;
        for (;;) {
          const size_t i = next.fetch_add(1);
          if (i >= cands.size()) return;
          if (!lctx && !sessions.empty())
            lctx = std::make_unique<Context>(
                nb_ctx_device(nb_session_ctx(sessions[size_t(j) % sessions.size()]->get())));
          pending[i] =
              host_gates(cands[i], origin, cfg, origin_fisher, nets[i], lctx.get(), &counts) ? 1
                                                                                             : 0;
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(err_mu);
        if (!err) err = std::current_exception();
        next = cands.size();  // the other gate threads stop too
      }
    };
    if (jobs == 1) {
      worker(0);
    } else {
      std::vector<std::thread> pool;
      for (int j = 0; j < jobs; ++j) pool.emplace_back(worker, j);
      for (auto& t : pool) t.join();
    }
    if (err) std::rethrow_exception(err);
    st.legality_gpu = counts.gpu.load();
    st.legality_host = counts.host.load();
  }
  auto t1 = std::chrono::steady_clock::now();
  // A candidate whose network is the origin's (e.g. bottleneck(ci) undone by
  // repair, I/nnet.hpp:376) scores exactly the origin: an exact tie.
  std::vector<size_t> idx;
  for (size_t i = 0; i < cands.size(); ++i) {
    if (!pending[i]) continue;
    if (same_network(nets[i], origin)) {
      cands[i].fisher_total = origin_fisher.total;
      cands[i].fisher_per_layer = origin_fisher.per_layer;
      cands[i].status = CandidateStatus::Survivor;  // fisher_accepts: ties accepted
      ++st.origin_equal;
      continue;
    }
    idx.push_back(i);
  }
  st.scored = int64_t(idx.size());
  std::vector<nb_session*> sp;
  for (auto* s : sessions) sp.push_back(s->get());
  // scores `which` (candidate indices) in mode p into totals / per-layer values
  auto score = [&](const std::vector<size_t>& which, nb_precision p, std::vector<double>& tot,
                   std::vector<std::vector<double>>& pl) {
    std::vector<NetDesc> descs;
    descs.reserve(which.size());
    for (size_t i : which) descs.emplace_back(nets[i]);
    std::vector<nb_network> cnets;
    for (auto& d : descs) cnets.push_back(d.c);
    pl.assign(which.size(), {});
    std::vector<nb_fisher_out> outs(which.size());
    for (size_t k = 0; k < which.size(); ++k) {
      pl[k].resize(nets[which[k]].layers.size());
      outs[k] = nb_fisher_out{nullptr, pl[k].data(), 0.0, 0, 0.0, nullptr};
    }
    std::vector<double> est(sp.size()), busy(sp.size());
    std::vector<int64_t> done(sp.size());
    nb_eval_stats es{};
    es.est_flops = est.data();
    es.busy_ms = busy.data();
    es.evaluations = done.data();
    check(nb_evaluate(sp.data(), int32_t(sp.size()), cnets.data(), int64_t(cnets.size()), p,
                      outs.data(), &es));
    tot.resize(which.size());
    for (size_t k = 0; k < which.size(); ++k) tot[k] = outs[k].total;
    if (p == prec) {
      st.evaluated += es.evaluated;
      st.deduplicated += es.deduplicated;
      st.requeued += es.requeued;
      st.est_flops.resize(sp.size());
      st.busy_ms.resize(sp.size());
      st.evaluations.resize(sp.size());
      for (size_t k = 0; k < sp.size(); ++k) {
        st.est_flops[k] += est[k];
        st.busy_ms[k] += busy[k];
        st.evaluations[k] += done[k];
      }
    }
  };
  // the origin's SIMT score, computed once when a recheck needs it
  bool have_simt_origin = false;
  double simt_origin = 0.0;
  auto origin_simt = [&]() {
    if (!have_simt_origin) {
      simt_origin = fisher_potential(*sessions[0], origin, NB_PREC_SIMT).total;
      have_simt_origin = true;
    }
    return simt_origin;
  };
  std::vector<char> simt_scored(cands.size(), 0);
  if (!idx.empty()) {
    std::vector<double> tot;
    std::vector<std::vector<double>> pl;
    score(idx, prec, tot, pl);
    // near-threshold candidates: re-score them and the origin in SIMT mode
    std::vector<size_t> near, near_k;
    for (size_t k = 0; k < idx.size(); ++k)
      if (near_threshold(tot[k], origin_fisher.total, prec)) {
        near.push_back(idx[k]);
        near_k.push_back(k);
      }
    if (!near.empty()) {
      origin_simt();
      std::vector<double> t2;
      std::vector<std::vector<double>> pl2;
      score(near, NB_PREC_SIMT, t2, pl2);
      for (size_t j = 0; j < near.size(); ++j) {
        tot[near_k[j]] = t2[j];
        pl[near_k[j]] = pl2[j];
        simt_scored[near[j]] = 1;
      }
      st.rechecked = int64_t(near.size());
    }
    for (size_t k = 0; k < idx.size(); ++k) {
      Candidate& cand = cands[idx[k]];
      cand.fisher_total = tot[k];
      cand.fisher_per_layer = pl[k];
      // a rechecked candidate is compared with the origin's SIMT score
      const double ref = simt_scored[idx[k]] ? simt_origin : origin_fisher.total;
      // fisher_accepts (I/nnet.hpp:356-359) and the message of
      // I/search.hpp:303-309, printing the value actually compared
      if (!(tot[k] >= ref)) {
        cand.status = CandidateStatus::RejectedFisher;
        std::ostringstream os;
        os << "fisher potential dropped: " << tot[k] << " < " << ref;
        cand.reason = os.str();
      } else {
        cand.status = CandidateStatus::Survivor;
      }
    }
    // rank_survivors (I/search.hpp:338-349) orders equal-MAC survivors by
    // their totals.  An equal-MAC group holding two different totals within
    // the mode's band of each other is re-scored entirely in SIMT (its scored
    // members; members carrying the origin's score -- non-neural survivors
    // and networks equal to the origin -- take the origin's SIMT score), so
    // the group's order is the reference's except for ties inside SIMT's own
    // tolerance.  Identical networks keep identical totals (dedupe).
    if (recheck_band(prec) > 0) {
      std::vector<char> scored(cands.size(), 0);
      for (size_t i : idx) scored[i] = 1;
      std::map<long long, std::vector<size_t>> by_macs;
      for (size_t i = 0; i < cands.size(); ++i)
        if (cands[i].status == CandidateStatus::Survivor) by_macs[cands[i].macs].push_back(i);
      std::vector<size_t> more, origin_valued;
      for (auto& kv : by_macs) {
        auto g = kv.second;
        if (g.size() < 2) continue;
        std::sort(g.begin(), g.end(), [&](size_t a, size_t b) {
          return cands[a].fisher_total < cands[b].fisher_total;
        });
        bool close = false;
        for (size_t j = 1; j < g.size() && !close; ++j) {
          const double a = cands[g[j - 1]].fisher_total, b = cands[g[j]].fisher_total;
          close = a != b && near_threshold(a, b, prec);
        }
        if (!close) continue;
        for (size_t i : g) {
          if (scored[i] && !simt_scored[i]) more.push_back(i);
          if (!scored[i]) origin_valued.push_back(i);
        }
      }
      if (!more.empty()) {
        std::sort(more.begin(), more.end());
        std::vector<double> t3;
        std::vector<std::vector<double>> pl3;
        score(more, NB_PREC_SIMT, t3, pl3);
        for (size_t j = 0; j < more.size(); ++j) {
          cands[more[j]].fisher_total = t3[j];
          cands[more[j]].fisher_per_layer = pl3[j];
          simt_scored[more[j]] = 1;
        }
        st.rank_rechecked = int64_t(more.size());
      }
      if (!origin_valued.empty()) {
        const double o = origin_simt();
        for (size_t i : origin_valued) cands[i].fisher_total = o;
      }
    }
  }
  auto t2 = std::chrono::steady_clock::now();
  st.gates_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  st.gpu_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
  return st;
}

// run_search, I/search.hpp:364-393, with the origin score and the candidate
// evaluation on the GPU sessions (one per entry of `devices`).
inline nestopt::SearchReport run_search_gpu(const nestopt::Network& origin,
                                            const nestopt::SearchConfig& cfg,
                                            const std::vector<int>& devices,
                                            nb_precision prec = NB_PREC_FP32,
                                            GpuStats* stats = nullptr) {
  using namespace nestopt;
  cfg.validate();
  origin.validate();
  if (devices.empty()) throw ConfigError("need at least one device");
  auto t0 = std::chrono::steady_clock::now();
  SearchReport rep;
  rep.config = cfg;
  rep.origin_macs = network_macs(origin);
  Batch batch = make_batch(origin, cfg.batch_n, cfg.batch_seed);
  std::vector<std::unique_ptr<Context>> ctxs;
  std::vector<std::unique_ptr<Session>> sess;
  std::vector<Session*> sp;
  for (int d : devices) {
    ctxs.push_back(std::make_unique<Context>(d));
    sess.push_back(std::make_unique<Session>(*ctxs.back(), origin, batch));
    sp.push_back(sess.back().get());
  }
  FisherReport origin_fisher = fisher_potential(*sess[0], origin, prec);
  rep.origin_fisher = origin_fisher.total;

  auto t1 = std::chrono::steady_clock::now();
  rep.candidates = nb200::draw_candidates(origin, cfg, cfg.jobs);
  auto t2 = std::chrono::steady_clock::now();
  GpuStats st = evaluate_all_gpu(rep.candidates, origin, cfg, origin_fisher, sp, prec);
  auto t3 = std::chrono::steady_clock::now();

  rep.survivors_ranked = rank_survivors(rep.candidates);
  for (const auto& c : rep.candidates) {
    switch (c.status) {
      case CandidateStatus::Survivor: ++rep.survivors; break;
      case CandidateStatus::RejectedSemantic: ++rep.rejected_semantic; break;
      case CandidateStatus::RejectedFisher: ++rep.rejected_fisher; break;
    }
  }
  rep.draw_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
  rep.eval_ms = std::chrono::duration<double, std::milli>(t3 - t2).count();
  rep.total_ms = std::chrono::duration<double, std::milli>(t3 - t0).count();
  if (stats) *stats = st;
  return rep;
}

}  // namespace nb200
