// extern "C" entry points over nestopt_b200.hpp, so the GPU search driver can
// be driven from Python tests and from the CLI: JSON in (the reference's
// search-config schema v1 with an embedded "network", as in
// P/samples/search_toy.json), the reference's search report JSON out
// (search_report_to_json, I/search.hpp:461-496) plus a "gpu" block.
#include <chrono>
#include <cstdlib>
#include <memory>
#include <limits>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "nestopt_b200.hpp"

namespace {
thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

std::vector<int> parse_devices(const char* devs) {
  std::vector<int> out;
  std::stringstream ss(devs ? devs : "0");
  std::string tok;
  while (std::getline(ss, tok, ',')) out.push_back(std::stoi(tok));
  return out;
}

// LoopNest <-> JSON (the reference has no nest serializer; this one lets
// tests hand-build nests the DSL cannot express, as the reference's own
// legality tests do, P/tests/test_transforms.cpp:311-408).  Expressions are
// nested arrays: ["c", k] | ["v", name] | ["add", e...] | ["mul"|"div"|"mod", e, k].
nlohmann::json expr_to_json(const nestopt::AffineExpr& e) {
  using K = nestopt::AffineExpr::Kind;
  switch (e.kind) {
    case K::Const: return nlohmann::json::array({"c", e.k});
    case K::Var: return nlohmann::json::array({"v", e.var});
    case K::Add: {
      nlohmann::json j = nlohmann::json::array({"add"});
      for (const auto& a : e.args) j.push_back(expr_to_json(a));
      return j;
    }
    case K::Mul: return nlohmann::json::array({"mul", expr_to_json(e.args[0]), e.k});
    case K::Div: return nlohmann::json::array({"div", expr_to_json(e.args[0]), e.k});
    case K::Mod: return nlohmann::json::array({"mod", expr_to_json(e.args[0]), e.k});
  }
  return {};
}

nestopt::AffineExpr expr_from_json(const nlohmann::json& j) {
  using K = nestopt::AffineExpr::Kind;
  nestopt::AffineExpr e;
  const std::string op = j.at(0).get<std::string>();
  if (op == "c") {
    e.kind = K::Const;
    e.k = j.at(1).get<long long>();
  } else if (op == "v") {
    e.kind = K::Var;
    e.var = j.at(1).get<std::string>();
  } else if (op == "add") {
    e.kind = K::Add;
    for (size_t i = 1; i < j.size(); ++i) e.args.push_back(expr_from_json(j[i]));
  } else {
    e.kind = op == "mul" ? K::Mul : op == "div" ? K::Div : op == "mod" ? K::Mod
                                                                       : throw nestopt::ParseError("bad expression op " + op);
    e.args.push_back(expr_from_json(j.at(1)));
    e.k = j.at(2).get<long long>();
  }
  return e;
}

nlohmann::json nest_to_json(const nestopt::LoopNest& n) {
  nlohmann::json parts = nlohmann::json::array();
  for (const auto& p : n.parts) {
    nlohmann::json spine = nlohmann::json::array(), stmts = nlohmann::json::array();
    for (const auto& iv : p.spine) spine.push_back({iv.name, iv.extent, iv.unroll, iv.kernel});
    for (const auto& st : p.stmts) {
      nlohmann::json coord = nlohmann::json::object(), acc = nlohmann::json::array();
      for (const auto& [k, e] : st.coord) coord[k] = expr_to_json(e);
      for (const auto& a : st.accesses) {
        nlohmann::json idx = nlohmann::json::array();
        for (const auto& e : a.indices) idx.push_back(expr_to_json(e));
        acc.push_back({{"tensor", a.tensor},
                       {"mode", a.mode == nestopt::AccessMode::Read    ? "r"
                                : a.mode == nestopt::AccessMode::Write ? "w"
                                                                       : "rmw"},
                       {"indices", idx},
                       {"zero_pad", a.zero_pad}});
      }
      stmts.push_back({{"id", st.id},
                       {"kind", st.kind == nestopt::StmtKind::Init ? "init" : "mac"},
                       {"domain", st.domain},
                       {"coord", coord},
                       {"accesses", acc}});
    }
    parts.push_back({{"spine", spine}, {"stmts", stmts}});
  }
  return {{"parts", parts}};
}

nestopt::LoopNest nest_from_json(const nlohmann::json& j) {
  nestopt::LoopNest n;
  for (const auto& pj : j.at("parts")) {
    nestopt::NestPart p;
    for (const auto& iv : pj.at("spine"))
      p.spine.push_back({iv.at(0).get<std::string>(), iv.at(1).get<long long>(),
                         iv.size() > 2 ? iv.at(2).get<long long>() : 1,
                         iv.size() > 3 ? iv.at(3).get<bool>() : false});
    for (const auto& sj : pj.at("stmts")) {
      nestopt::Statement st;
      st.id = sj.at("id").get<std::string>();
      st.kind = sj.at("kind").get<std::string>() == "init" ? nestopt::StmtKind::Init
                                                            : nestopt::StmtKind::Mac;
      st.domain = sj.at("domain").get<std::vector<std::string>>();
      for (const auto& [k, e] : sj.at("coord").items()) st.coord[k] = expr_from_json(e);
      for (const auto& aj : sj.at("accesses")) {
        nestopt::AccessMap a;
        a.tensor = aj.at("tensor").get<std::string>();
        const std::string m = aj.at("mode").get<std::string>();
        a.mode = m == "r" ? nestopt::AccessMode::Read
                 : m == "w" ? nestopt::AccessMode::Write
                            : nestopt::AccessMode::ReadModifyWrite;
        for (const auto& e : aj.at("indices")) a.indices.push_back(expr_from_json(e));
        a.zero_pad = aj.value("zero_pad", false);
        st.accesses.push_back(std::move(a));
      }
      p.stmts.push_back(std::move(st));
    }
    n.parts.push_back(std::move(p));
  }
  return n;
}

nlohmann::json legality_json(const nestopt::LoopNest& orig, const nestopt::LoopNest& tr,
                             long long cap, int device, double* ms) {
  std::unique_ptr<nb200::Context> ctx;
  if (device >= 0) ctx = std::make_unique<nb200::Context>(device);
  nlohmann::json out;
  const auto t0 = std::chrono::steady_clock::now();
  try {
    nestopt::LegalityResult r = ctx ? nb200::check_semantic_legality(*ctx, orig, tr, cap)
                                    : nestopt::check_semantic_legality(orig, tr, cap);
    out["path"] = ctx ? "gpu" : "host";
    out["verdict"] = r.verdict == nestopt::Verdict::Legal     ? "legal"
                     : r.verdict == nestopt::Verdict::Illegal ? "illegal"
                                                              : "not_applicable";
    out["reason"] = r.reason;
  } catch (const nestopt::CapExceeded& e) {
    out["error"] = "CapExceeded";
    out["what"] = e.what();
  }
  if (ms) *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return out;
}
}  // namespace

extern "C" {

const char* nbi_last_error(void) { return g_err.c_str(); }
void nbi_free(char* p) { std::free(p); }

// nb200::near_threshold: whether the search driver re-scores a candidate
// with this total against this origin total in SIMT before deciding.
int nbi_near_threshold(double cand, double origin, int precision) {
  return nb200::near_threshold(cand, origin, static_cast<nb_precision>(precision)) ? 1 : 0;
}

// Runs the search of `cfg_json` with candidate scoring on the GPU sessions
// listed in `devices` ("0,1,2,3"; a device may repeat: several sessions on
// one GPU exercise the multi-worker scheduler).  jobs > 0 overrides the
// config's host-gate thread count.  Returns 0 or an nb_status-style code.
int nbi_run_search(const char* cfg_json, const char* devices, int precision, int jobs,
                   char** report_json) {
  try {
    nlohmann::json j = nlohmann::json::parse(cfg_json);
    nestopt::Network net = nestopt::network_from_json(j.at("network"));
    nestopt::SearchConfig cfg = nestopt::search_config_from_json(j);
    if (jobs > 0) cfg.jobs = jobs;
    nb200::GpuStats st;
    nestopt::SearchReport rep =
        nb200::run_search_gpu(net, cfg, parse_devices(devices), nb_precision(precision), &st);
    nlohmann::json out = nestopt::search_report_to_json(rep);
    out["gpu"] = {{"devices", parse_devices(devices)},
                  {"precision", precision},
                  {"scored", st.scored},
                  {"evaluated", st.evaluated},
                  {"deduplicated", st.deduplicated},
                  {"origin_equal", st.origin_equal},
                  {"rechecked", st.rechecked},
                  {"legality_gpu", st.legality_gpu},
                  {"legality_host", st.legality_host},
                  {"rank_rechecked", st.rank_rechecked},
                  {"requeued", st.requeued},
                  {"est_flops", st.est_flops},
                  {"busy_ms", st.busy_ms},
                  {"evaluations", st.evaluations},
                  {"gates_ms", st.gates_ms},
                  {"gpu_ms", st.gpu_ms}};
    *report_json = dup(out.dump());
    return 0;
  } catch (const nestopt::ConfigError& e) {
    g_err = e.what();
    return NB_ERR_CONFIG;
  } catch (const nb200::DeviceError& e) {
    g_err = e.what();
    return NB_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NB_ERR_GENERIC;
  }
}

// execute<T> (I/interp.hpp:67-145) on the GPU of conv_nest(spec) rewritten
// by a DSL sequence (parse_sequence, I/transforms.hpp:756): any nest,
// including the ones with no ConvSpec (Sequence 1).  in (Ci,H,W), w
// (Co_eff,Ci,Kh,Kw), out (Co_eff,out_h,out_w); int64 when is_int else double.
// execute_boxes: the masked box executor in precision `prec`; fills
// *nboxes, *box_macs, *nest_macs (nullable).  Returns NB_ERR_UNSUPPORTED
// (last error says why) for a nest that does not decompose into boxes.
int nbi_execute_boxes(const char* spec_json, const char* dsl, int is_int, const void* in,
                      const void* w, void* out, int prec, long long* nboxes, long long* box_macs,
                      long long* nest_macs) {
  try {
    nestopt::ConvSpec s = nestopt::conv_spec_from_json(nlohmann::json::parse(spec_json));
    nestopt::LoopNest nest = nestopt::apply(nestopt::conv_nest(s), nestopt::parse_sequence(dsl));
    nb200::Context ctx(0);
    nb200::BoxReport rep;
    auto run = [&](auto tag) {
      using T = decltype(tag);
      nestopt::ExecEnv<T> env;
      nestopt::Tensor<T> ti({s.ci, s.h, s.w}), tw({s.co_eff(), s.ci, s.kh, s.kw});
      std::memcpy(ti.data.data(), in, ti.data.size() * 8);
      std::memcpy(tw.data.data(), w, tw.data.size() * 8);
      env.bindings["I"] = ti;
      env.bindings["K"] = tw;
      nestopt::Tensor<T> to = nb200::execute_boxes(ctx, nest, env, nb_precision(prec), &rep);
      std::memcpy(out, to.data.data(), to.data.size() * 8);
    };
    if (is_int) run((long long)0);
    else run(0.0);
    if (nboxes) *nboxes = (long long)rep.boxes.size();
    if (box_macs) *box_macs = rep.box_macs;
    if (nest_macs) *nest_macs = rep.nest_macs;
    return 0;
  } catch (const nb200::BoxUnsupported& e) {
    g_err = e.what();
    return NB_ERR_UNSUPPORTED;
  } catch (const nb200::DeviceError& e) {
    g_err = e.what();
    return NB_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NB_ERR_GENERIC;
  }
}

int nbi_execute(const char* spec_json, const char* dsl, int is_int, const void* in, const void* w,
                void* out) {
  try {
    nestopt::ConvSpec s = nestopt::conv_spec_from_json(nlohmann::json::parse(spec_json));
    nestopt::LoopNest nest = nestopt::apply(nestopt::conv_nest(s), nestopt::parse_sequence(dsl));
    nb200::Context ctx(0);
    auto run = [&](auto tag) {
      using T = decltype(tag);
      nestopt::ExecEnv<T> env;
      nestopt::Tensor<T> ti({s.ci, s.h, s.w}), tw({s.co_eff(), s.ci, s.kh, s.kw});
      std::memcpy(ti.data.data(), in, ti.data.size() * 8);
      std::memcpy(tw.data.data(), w, tw.data.size() * 8);
      env.bindings["I"] = ti;
      env.bindings["K"] = tw;
      nestopt::Tensor<T> to = nb200::execute(ctx, nest, env);
      std::memcpy(out, to.data.data(), to.data.size() * 8);
    };
    if (is_int) run((long long)0);
    else run(0.0);
    return 0;
  } catch (const nb200::DeviceError& e) {
    g_err = e.what();
    return NB_ERR_CUDA;
  } catch (const nestopt::Error& e) {
    g_err = e.what();
    return NB_ERR_GENERIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NB_ERR_GENERIC;
  }
}

// Host half of a search without a GPU: the reference's draw_candidates and
// the gates of evaluate_candidate (nb200::host_gates).  Per candidate the
// output holds its status after the gates ("fisher" = a neural candidate the
// GPU must score), reason, macs, and for "fisher" candidates the repaired
// network (network_to_json, I/nnet.hpp:444-454).  legal_device >= 0 checks
// semantic runs on that GPU (nb200::check_semantic_legality, one context per
// gate thread); -1 runs the reference's host check.
int nbi_gate_candidates(const char* cfg_json, int legal_device, char** out_json) {
  try {
    nlohmann::json j = nlohmann::json::parse(cfg_json);
    nestopt::Network origin = nestopt::network_from_json(j.at("network"));
    nestopt::SearchConfig cfg = nestopt::search_config_from_json(j);
    cfg.validate();
    origin.validate();
    std::vector<nestopt::Candidate> cands =
        nb200::draw_candidates(origin, cfg, int(std::max(1u, std::thread::hardware_concurrency())));
    nestopt::FisherReport dummy;
    dummy.total = std::numeric_limits<double>::quiet_NaN();
    std::vector<nestopt::Network> nets(cands.size());
    std::vector<char> pend(cands.size(), 0);
    nb200::LegalityCounts counts;
    {
      std::atomic<size_t> next{0};
      std::exception_ptr err;
      std::mutex err_mu;
      auto worker = [&]() {
        try {
          std::unique_ptr<nb200::Context> lctx;
          if (legal_device >= 0) lctx = std::make_unique<nb200::Context>(legal_device);
          for (size_t i; (i = next.fetch_add(1)) < cands.size();)
            pend[i] =
                nb200::host_gates(cands[i], origin, cfg, dummy, nets[i], lctx.get(), &counts) ? 1
                                                                                               : 0;
        } catch (...) {
          std::lock_guard<std::mutex> lk(err_mu);
          if (!err) err = std::current_exception();
          next = cands.size();
        }
      };
      std::vector<std::thread> pool;
      const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
      for (unsigned t = 0; t < nt; ++t) pool.emplace_back(worker);
      for (auto& t : pool) t.join();
      if (err) std::rethrow_exception(err);
    }
    nlohmann::json arr = nlohmann::json::array();
    for (size_t i = 0; i < cands.size(); ++i) {
      const nestopt::Candidate& c = cands[i];
      const nestopt::Network& net = nets[i];
      const bool pending = pend[i] != 0;
      nlohmann::json cj{{"status", pending ? "fisher" : nestopt::status_name(c.status)},
                        {"neural", c.neural},
                        {"macs", c.macs}};
      if (!c.reason.empty()) cj["reason"] = c.reason;
      if (pending) cj["network"] = nestopt::network_to_json(net);
      arr.push_back(std::move(cj));
    }
    *out_json = dup(nlohmann::json{{"candidates", arr},
                                   {"legality", {{"gpu", counts.gpu.load()},
                                                 {"host", counts.host.load()}}}}
                        .dump());
    return 0;
  } catch (const nestopt::ConfigError& e) {
    g_err = e.what();
    return NB_ERR_CONFIG;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NB_ERR_GENERIC;
  }
}

// check_semantic_legality (I/transforms.hpp:598-663) of one semantic run:
// original = conv_nest(spec) rewritten by `pre` (any steps, may be empty),
// transformed = original rewritten by `seq`.  device < 0 runs the
// reference's host function, else nb200::check_semantic_legality on that GPU
// (gpu_min_instances 0: always on the device).  Output JSON: {"verdict":
// "legal"|"illegal"|"not_applicable", "reason": ...} or {"error": class,
// "what": message} when the check throws (CapExceeded).
int nbi_legality(const char* spec_json, const char* pre, const char* seq, long long cap,
                 int device, double* ms, char** out_json) {
  try {
    nestopt::ConvSpec s = nestopt::conv_spec_from_json(nlohmann::json::parse(spec_json));
    nestopt::LoopNest orig = nestopt::conv_nest(s);
    if (pre && *pre) orig = nestopt::apply(orig, nestopt::parse_sequence(pre));
    nestopt::LoopNest tr = nestopt::apply(orig, nestopt::parse_sequence(seq));
    *out_json = dup(legality_json(orig, tr, cap, device, ms).dump());
    return 0;
  } catch (const nb200::DeviceError& e) {
    g_err = e.what();
    return NB_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NB_ERR_GENERIC;
  }
}

// The same check on two explicit nests (nest JSON above).
int nbi_legality_nests(const char* orig_json, const char* tr_json, long long cap, int device,
                       double* ms, char** out_json) {
  try {
    nestopt::LoopNest orig = nest_from_json(nlohmann::json::parse(orig_json));
    nestopt::LoopNest tr = nest_from_json(nlohmann::json::parse(tr_json));
    *out_json = dup(legality_json(orig, tr, cap, device, ms).dump());
    return 0;
  } catch (const nb200::DeviceError& e) {
    g_err = e.what();
    return NB_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NB_ERR_GENERIC;
  }
}

// The candidates of a search config as DSL per layer: threads == 0 runs the
// reference's serial draw_candidates, else nb200::draw_candidates.
int nbi_draw_candidates(const char* cfg_json, int threads, char** out_json) {
  try {
    nlohmann::json j = nlohmann::json::parse(cfg_json);
    nestopt::Network origin = nestopt::network_from_json(j.at("network"));
    nestopt::SearchConfig cfg = nestopt::search_config_from_json(j);
    std::vector<nestopt::Candidate> c = threads == 0
                                            ? nestopt::draw_candidates(origin, cfg)
                                            : nb200::draw_candidates(origin, cfg, threads);
    nlohmann::json arr = nlohmann::json::array();
    for (const auto& cand : c) {
      nlohmann::json layers = nlohmann::json::array();
      for (const auto& seq : cand.layer_seqs) layers.push_back(nestopt::to_dsl(seq));
      arr.push_back({{"neural", cand.neural}, {"layers", layers}});
    }
    *out_json = dup(arr.dump());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NB_ERR_GENERIC;
  }
}

// conv_nest(spec) rewritten by `dsl` (may be empty), as nest JSON.
int nbi_nest_json(const char* spec_json, const char* dsl, char** out_json) {
  try {
    nestopt::ConvSpec s = nestopt::conv_spec_from_json(nlohmann::json::parse(spec_json));
    nestopt::LoopNest n = nestopt::conv_nest(s);
    if (dsl && *dsl) n = nestopt::apply(n, nestopt::parse_sequence(dsl));
    *out_json = dup(nest_to_json(n).dump());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NB_ERR_GENERIC;
  }
}

}  // extern "C"
