// nb200_search: the GPU counterpart of `nestopt search` (P/tools/main.cpp:160):
//   nb200_search <config.json> [--devices 0,1,..] [--precision fp32|tf32|simt]
//                [--jobs N] [--out report.json]
// Prints the reference's summary lines and writes the report JSON.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "nestopt_b200.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s config.json [--devices 0,..] [--precision fp32|tf32|simt]"
                         " [--jobs N] [--out report.json]\n", argv[0]);
    return 2;
  }
  std::string devices = "0", out_path, prec_s = "fp32";
  int jobs = 0;
  for (int i = 2; i + 1 < argc; i += 2) {
    if (!std::strcmp(argv[i], "--devices")) devices = argv[i + 1];
    else if (!std::strcmp(argv[i], "--precision")) prec_s = argv[i + 1];
    else if (!std::strcmp(argv[i], "--jobs")) jobs = std::atoi(argv[i + 1]);
    else if (!std::strcmp(argv[i], "--out")) out_path = argv[i + 1];
  }
  const nb_precision prec = prec_s == "tf32" ? NB_PREC_TF32 : prec_s == "simt" ? NB_PREC_SIMT
                                                                               : NB_PREC_FP32;
  try {
    std::ifstream in(argv[1]);
    if (!in) throw nestopt::IoError(std::string("cannot read '") + argv[1] + "'");
    nlohmann::json j = nlohmann::json::parse(in);
    nestopt::Network net = nestopt::network_from_json(j.at("network"));
    nestopt::SearchConfig cfg = nestopt::search_config_from_json(j);
    if (jobs > 0) cfg.jobs = jobs;
    std::vector<int> devs;
    std::stringstream ss(devices);
    std::string tok;
    while (std::getline(ss, tok, ',')) devs.push_back(std::stoi(tok));
    nb200::GpuStats st;
    nestopt::SearchReport rep = nb200::run_search_gpu(net, cfg, devs, prec, &st);
    std::cout << "candidates: " << rep.candidates.size() << "\n"
              << "survivors: " << rep.survivors << "\n"
              << "rejected_semantic: " << rep.rejected_semantic << "\n"
              << "rejected_fisher: " << rep.rejected_fisher << "\n"
              << "origin macs: " << rep.origin_macs << " fisher: " << rep.origin_fisher << "\n";
    if (!rep.survivors_ranked.empty())
      std::cout << "best: " << rep.survivors_ranked.front() << "\n";
    std::cout << "gpu: scored " << st.scored << " evaluated " << st.evaluated << " dedup "
              << st.deduplicated << " gates_ms " << st.gates_ms << " gpu_ms " << st.gpu_ms
              << "\n";
    if (!out_path.empty()) {
      std::ofstream o(out_path);
      o << nestopt::search_report_to_json(rep).dump(2) << "\n";
    }
    std::cout << "RESULT ok 0\n";
    return 0;
  } catch (const nestopt::Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    std::cout << "RESULT fail 1\n";
    return 1;
  }
}
