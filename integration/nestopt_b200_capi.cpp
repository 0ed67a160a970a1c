// extern "C" entry points over nestopt_b200.hpp, so the GPU search driver can
// be driven from Python tests and from the CLI: JSON in (the reference's
// search-config schema v1 with an embedded "network", as in
// P/samples/search_toy.json), the reference's search report JSON out
// (search_report_to_json, I/search.hpp:461-496) plus a "gpu" block.
#include <cstdlib>
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
}  // namespace

extern "C" {

const char* nbi_last_error(void) { return g_err.c_str(); }
void nbi_free(char* p) { std::free(p); }

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
                  {"est_flops", st.est_flops},
                  {"busy_ms", st.busy_ms},
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
// network (network_to_json, I/nnet.hpp:444-454).
int nbi_gate_candidates(const char* cfg_json, char** out_json) {
  try {
    nlohmann::json j = nlohmann::json::parse(cfg_json);
    nestopt::Network origin = nestopt::network_from_json(j.at("network"));
    nestopt::SearchConfig cfg = nestopt::search_config_from_json(j);
    cfg.validate();
    origin.validate();
    std::vector<nestopt::Candidate> cands = nestopt::draw_candidates(origin, cfg);
    nestopt::FisherReport dummy;
    dummy.total = std::numeric_limits<double>::quiet_NaN();
    std::vector<nestopt::Network> nets(cands.size());
    std::vector<char> pend(cands.size(), 0);
    {
      std::atomic<size_t> next{0};
      auto worker = [&]() {
        for (size_t i; (i = next.fetch_add(1)) < cands.size();)
          pend[i] = nb200::host_gates(cands[i], origin, cfg, dummy, nets[i]) ? 1 : 0;
      };
      std::vector<std::thread> pool;
      const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
      for (unsigned t = 0; t < nt; ++t) pool.emplace_back(worker);
      for (auto& t : pool) t.join();
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
    *out_json = dup(nlohmann::json{{"candidates", arr}}.dump());
    return 0;
  } catch (const nestopt::ConfigError& e) {
    g_err = e.what();
    return NB_ERR_CONFIG;
  } catch (const std::exception& e) {
    g_err = e.what();
    return NB_ERR_GENERIC;
  }
}

}  // extern "C"
