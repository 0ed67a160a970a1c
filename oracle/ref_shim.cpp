// TEST INFRASTRUCTURE ONLY -- never linked into the product path.
//
// extern "C" shim over the UNMODIFIED reference library (nestopt, header-only
// C++20 under /root/reference/proj/include).  It is compiled in place from the
// reference headers by oracle/Makefile into oracle/_ref/libnestopt_ref.so and
// is used by tests/ (parity checker), oracle/gen_golden.py (fixture
// generator) and bench.py --impl reference (the reference CPU arm).
//
// Every entry point forwards to the reference function named in its comment;
// no reference logic is restated here.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "nestopt/nestopt.hpp"

using namespace nestopt;

namespace {
thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

// Error classes -> small ints (same numbering as include/nb200.h nb_status).
int code_of(const std::exception& e) {
  if (dynamic_cast<const InvalidSpec*>(&e)) return 1;
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const ShapeMismatch*>(&e)) return 3;
  if (dynamic_cast<const CapExceeded*>(&e)) return 4;
  if (dynamic_cast<const TransformError*>(&e)) return 5;
  if (dynamic_cast<const ParseError*>(&e)) return 6;
  if (dynamic_cast<const IoError*>(&e)) return 7;
  if (dynamic_cast<const Error*>(&e)) return 8;
  return 99;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

Network load_net(const char* net_json) {
  return network_from_json(nlohmann::json::parse(net_json));  // I/nnet.hpp:427
}

void override_weights(Network& net, const double* weights, const double* head) {
  if (weights) {
    size_t off = 0;
    for (auto& w : net.weights) {
      std::memcpy(w.data.data(), weights + off, w.data.size() * sizeof(double));
      off += w.data.size();
    }
  }
  if (head) {
    size_t off = 0;
    for (auto& row : net.head) {
      std::memcpy(row.data(), head + off, row.size() * sizeof(double));
      off += row.size();
    }
  }
}

Batch load_batch(const Network& net, int64_t n, const double* inputs,
                 const int32_t* labels, uint64_t seed) {
  if (!inputs) return make_batch(net, static_cast<size_t>(n), seed);  // I/nnet.hpp:87
  const ConvSpec& s0 = net.layers.front().spec;
  Batch b;
  b.seed = seed;
  size_t per = static_cast<size_t>(s0.ci * s0.h * s0.w);
  for (int64_t i = 0; i < n; ++i) {
    TensorF x({s0.ci, s0.h, s0.w});
    std::memcpy(x.data.data(), inputs + i * per, per * sizeof(double));
    b.inputs.push_back(std::move(x));
    b.labels.push_back(labels[i]);
  }
  return b;
}

ConvSpec load_spec(const char* spec_json) {
  return conv_spec_from_json(nlohmann::json::parse(spec_json));  // I/nnet.hpp:387
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

// Network::init_weights (I/nnet.hpp:58-79): flat per-layer (Co_eff,Ci,Kh,Kw)
// weights followed by nothing; head is [num_classes][C_last].
int ref_init_weights(const char* net_json, double* weights, double* head) {
  return guard([&] {
    Network net = load_net(net_json);
    size_t off = 0;
    for (auto& w : net.weights) {
      if (weights) std::memcpy(weights + off, w.data.data(), w.data.size() * 8);
      off += w.data.size();
    }
    off = 0;
    for (auto& row : net.head) {
      if (head) std::memcpy(head + off, row.data(), row.size() * 8);
      off += row.size();
    }
  });
}

// make_batch (I/nnet.hpp:87-101).
int ref_make_batch(const char* net_json, int64_t n, uint64_t seed, double* inputs,
                   int32_t* labels) {
  return guard([&] {
    Network net = load_net(net_json);
    Batch b = make_batch(net, static_cast<size_t>(n), seed);
    size_t off = 0;
    for (size_t i = 0; i < b.inputs.size(); ++i) {
      std::memcpy(inputs + off, b.inputs[i].data.data(), b.inputs[i].data.size() * 8);
      off += b.inputs[i].data.size();
      labels[i] = b.labels[i];
    }
  });
}

// fisher_potential (I/nnet.hpp:321-352) plus, optionally, the forward cache
// (I/nnet.hpp:180-197) and activation_gradients (I/nnet.hpp:201-247).
// per_channel: concatenation over layers of Co_eff values.
// acts/grads: for l in [0,L): for n in [0,N): (C,H,W) of layer l's output.
int ref_fisher(const char* net_json, const double* weights, const double* head,
               int64_t n, const double* inputs, const int32_t* labels,
               uint64_t batch_seed, double* per_channel, double* per_layer,
               double* total, double* loss, double* probs, double* acts,
               double* grads) {
  return guard([&] {
    Network net = load_net(net_json);
    override_weights(net, weights, head);
    Batch batch = load_batch(net, n, inputs, labels, batch_seed);
    FisherReport rep = fisher_potential(net, batch);
    size_t off = 0;
    for (size_t l = 0; l < rep.per_channel.size(); ++l) {
      if (per_channel)
        std::memcpy(per_channel + off, rep.per_channel[l].data(),
                    rep.per_channel[l].size() * 8);
      off += rep.per_channel[l].size();
      if (per_layer) per_layer[l] = rep.per_layer[l];
    }
    if (total) *total = rep.total;
    if (loss || probs || acts || grads) {
      ForwardCache fc = forward(net, batch);
      if (loss) *loss = fc.loss;
      if (probs)
        for (size_t i = 0; i < fc.probs.size(); ++i)
          std::memcpy(probs + i * net.num_classes, fc.probs[i].data(),
                      net.num_classes * 8);
      if (acts || grads) {
        auto g = activation_gradients(net, batch, fc);
        size_t o = 0;
        for (size_t l = 0; l < net.layers.size(); ++l)
          for (size_t i = 0; i < batch.inputs.size(); ++i) {
            const TensorF& a = fc.acts[i][l + 1];
            if (acts) std::memcpy(acts + o, a.data.data(), a.data.size() * 8);
            if (grads) std::memcpy(grads + o, g[i][l].data.data(), a.data.size() * 8);
            o += a.data.size();
          }
      }
    }
  });
}

// forward (I/nnet.hpp:180-197): probs [N][classes], per-example loss, mean loss.
int ref_forward(const char* net_json, int64_t n, uint64_t batch_seed, double* probs,
                double* example_loss, double* loss) {
  return guard([&] {
    Network net = load_net(net_json);
    Batch batch = make_batch(net, static_cast<size_t>(n), batch_seed);
    ForwardCache fc = forward(net, batch);
    for (size_t i = 0; i < fc.probs.size(); ++i) {
      if (probs)
        std::memcpy(probs + i * net.num_classes, fc.probs[i].data(),
                    net.num_classes * 8);
      if (example_loss) example_loss[i] = fc.example_loss[i];
    }
    if (loss) *loss = fc.loss;
  });
}

// reference_conv<T> (I/interp.hpp:151-186) on one image.  is_int selects
// TensorI (int64) vs TensorF (fp64).
int ref_conv(const char* spec_json, int is_int, const void* in, const void* w,
             void* out) {
  return guard([&] {
    ConvSpec s = load_spec(spec_json);
    auto run = [&](auto tag) {
      using T = decltype(tag);
      Tensor<T> ti({s.ci, s.h, s.w}), tw({s.co_eff(), s.ci, s.kh, s.kw});
      std::memcpy(ti.data.data(), in, ti.data.size() * 8);
      std::memcpy(tw.data.data(), w, tw.data.size() * 8);
      Tensor<T> to = reference_conv(s, ti, tw);
      std::memcpy(out, to.data.data(), to.data.size() * 8);
    };
    if (is_int) run((long long)0);
    else run(0.0);
  });
}

// layer_forward (I/nnet.hpp:130-141) on one image, fp64.
int ref_layer_forward(const char* spec_json, int relu, const double* in,
                      const double* w, double* out) {
  return guard([&] {
    Layer layer;
    layer.spec = load_spec(spec_json);
    layer.relu = relu != 0;
    const ConvSpec& s = layer.spec;
    TensorF ti({s.ci, s.h, s.w}), tw({s.co_eff(), s.ci, s.kh, s.kw});
    std::memcpy(ti.data.data(), in, ti.data.size() * 8);
    std::memcpy(tw.data.data(), w, tw.data.size() * 8);
    TensorF to = layer_forward(layer, tw, ti);
    std::memcpy(out, to.data.data(), to.data.size() * 8);
  });
}

// execute<T> (I/interp.hpp:67-145) of conv_nest(spec) rewritten by the DSL
// sequence (parse_sequence I/transforms.hpp:756, apply :474).  out_shape
// receives the (Co_eff, out_h, out_w) of the provenance spec.
int ref_execute(const char* spec_json, const char* dsl, int is_int, const void* in,
                const void* w, void* out) {
  return guard([&] {
    ConvSpec s = load_spec(spec_json);
    LoopNest nest = apply(conv_nest(s), parse_sequence(dsl));
    auto run = [&](auto tag) {
      using T = decltype(tag);
      ExecEnv<T> env;
      Tensor<T> ti({s.ci, s.h, s.w}), tw({s.co_eff(), s.ci, s.kh, s.kw});
      std::memcpy(ti.data.data(), in, ti.data.size() * 8);
      std::memcpy(tw.data.data(), w, tw.data.size() * 8);
      env.bindings["I"] = ti;
      env.bindings["K"] = tw;
      Tensor<T> to = execute(nest, env);
      std::memcpy(out, to.data.data(), to.data.size() * 8);
    };
    if (is_int) run((long long)0);
    else run(0.0);
  });
}

// count_macs (I/interp.hpp:190-202) of the rewritten nest.
int ref_count_macs(const char* spec_json, const char* dsl, int64_t* macs) {
  return guard([&] {
    ConvSpec s = load_spec(spec_json);
    *macs = count_macs(apply(conv_nest(s), parse_sequence(dsl)));
  });
}

// derived_spec (I/ir.hpp:524-545) of the rewritten nest, as JSON ("null" if
// the nest is not a convolution).
int ref_derived_spec(const char* spec_json, const char* dsl, char** out) {
  return guard([&] {
    ConvSpec s = load_spec(spec_json);
    auto d = derived_spec(apply(conv_nest(s), parse_sequence(dsl)));
    *out = dup(d ? conv_spec_to_json(*d).dump() : std::string("null"));
  });
}

// run_search (I/search.hpp:364-393) -> search_report_to_json (:461).
// cfg_json is a search config with an inline "network" object (the CLI's
// format, P/tools/main.cpp:160-170).  jobs > 0 overrides cfg.jobs.
int ref_search(const char* cfg_json, int jobs, char** out) {
  return guard([&] {
    nlohmann::json j = nlohmann::json::parse(cfg_json);
    Network net = network_from_json(j.at("network"));
    SearchConfig cfg = search_config_from_json(j);
    if (jobs > 0) cfg.jobs = jobs;
    SearchReport rep = run_search(net, cfg);
    *out = dup(search_report_to_json(rep).dump());
  });
}

// The reference CPU arm of bench.py: fisher_potential (I/nnet.hpp:321) of
// `count` networks, each scored on its own make_batch(net, n, batch_seed)
// (I/nnet.hpp:87), scheduled exactly as evaluate_all does (I/search.hpp:
// 315-334): `jobs` std::threads self-scheduling through next.fetch_add(1).
// Every job pays what evaluate_candidate pays for a neural candidate's
// score: network_from_json -> init_weights (the re-init repair_network
// performs, I/nnet.hpp:372-381), make_batch and fisher_potential.
// job_seconds[i] = that job's own duration, *wall_seconds = the whole pool.
int ref_fisher_jobs(const char* const* net_jsons, int count, int64_t n,
                    uint64_t batch_seed, int jobs, double* totals,
                    double* job_seconds, double* wall_seconds) {
  return guard([&] {
    using clock = std::chrono::steady_clock;
    std::atomic<int> next{0};
    std::atomic<int> failed{0};
    std::vector<std::string> errs(static_cast<size_t>(count));
    auto worker = [&]() {
      for (;;) {
        const int i = next.fetch_add(1);
        if (i >= count) return;
        const auto t0 = clock::now();
        try {
          Network net = load_net(net_jsons[i]);
          Batch batch = make_batch(net, static_cast<size_t>(n), batch_seed);
          FisherReport rep = fisher_potential(net, batch);
          if (totals) totals[i] = rep.total;
        } catch (const std::exception& e) {
          errs[static_cast<size_t>(i)] = e.what();
          failed.fetch_add(1);
        }
        if (job_seconds)
          job_seconds[i] = std::chrono::duration<double>(clock::now() - t0).count();
      }
    };
    const auto t0 = clock::now();
    std::vector<std::thread> pool;
    for (int j = 0; j < std::max(1, jobs); ++j) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    if (wall_seconds) *wall_seconds = std::chrono::duration<double>(clock::now() - t0).count();
    if (failed.load())
      for (const auto& e : errs)
        if (!e.empty()) throw Error(e);
  });
}

}  // extern "C"
