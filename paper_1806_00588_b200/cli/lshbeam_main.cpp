// lshbeam_main.cpp -- the `lshbeam` command-line front-end (build / decode /
// grid) over the C++ drop-in API, so the reference's CLI-level tests
// (/root/reference/proj/tests/test_cli.cpp, acceptance criterion 9) and
// users of its CLI can drive the GPU build. Same subcommands, flags, report
// schema (/root/reference/proj/README.md:91-113, tools/main.cpp:84-168),
// CSV layout and exit codes (0 ok, 1 runtime error, 2 usage error) as the
// reference CLI; the argument parser is a small hand-written one (the
// reference's CLI11 dependency is not vendored).
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "json.hpp"
#include "lshbeam/beam_decoder.hpp"
#include "lshbeam/rng.hpp"

using json = nlohmann::json;
using namespace lshbeam;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --name value / --flag parsing against a declared option set.
class Args {
 public:
  Args(int argc, char** argv, int first, const std::map<std::string, bool>& spec) {
    for (int i = first; i < argc; ++i) {
      const std::string a = argv[i];
      if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + a);
      const std::string name = a.substr(2);
      const auto it = spec.find(name);
      if (it == spec.end()) throw UsageError("unknown option: " + a);
      if (!it->second) {  // flag
        vals_[name] = "1";
        continue;
      }
      if (i + 1 >= argc) throw UsageError("option " + a + " needs a value");
      vals_[name] = argv[++i];
    }
  }
  bool has(const std::string& k) const { return vals_.count(k) != 0; }
  std::string str(const std::string& k, const std::string& def) const {
    return has(k) ? vals_.at(k) : def;
  }
  template <class T>
  T num(const std::string& k, T def) const {
    if (!has(k)) return def;
    std::istringstream is(vals_.at(k));
    T v{};
    if (!(is >> v) || !is.eof()) throw UsageError("--" + k + ": not a number: " + vals_.at(k));
    return v;
  }
  template <class T>
  std::vector<T> list(const std::string& k, std::vector<T> def) const {
    if (!has(k)) return def;
    std::vector<T> out;
    std::stringstream ss(vals_.at(k));
    std::string item;
    while (std::getline(ss, item, ',')) {
      if (item.empty()) continue;
      std::istringstream is(item);
      T v{};
      if (!(is >> v) || !is.eof()) throw UsageError("--" + k + ": not a number: " + item);
      out.push_back(v);
    }
    return out;
  }

 private:
  std::map<std::string, std::string> vals_;
};

const std::map<std::string, bool> kModelOpts = {{"vocab", true}, {"dim", true}, {"seed", true},
                                                {"bias", true},  {"synth", true}, {"emb", true}};

std::map<std::string, bool> with(std::map<std::string, bool> m,
                                 std::initializer_list<std::pair<const std::string, bool>> more) {
  m.insert(more);
  return m;
}

struct Model {
  SynthModel m;
  uint64_t seed = 0;
};

// --synth V,D,SEED | --emb FILE | --vocab/--dim/--seed; --bias for all
Model make_model(const Args& a) {
  const float bias = static_cast<float>(a.num<double>("bias", 0.0));
  if (a.has("synth")) {
    unsigned V = 0;
    int d = 0;
    unsigned long long s = 0;
    if (std::sscanf(a.str("synth", "").c_str(), "%u,%d,%llu", &V, &d, &s) != 3)
      throw UsageError("--synth expects V,D,SEED");
    return {synth_model(V, d, s, bias), s};
  }
  const uint64_t seed = a.num<unsigned long long>("seed", 1);
  if (a.has("emb")) {
    const std::string p = a.str("emb", "");
    if (!std::filesystem::exists(p)) throw UsageError("embedding file not found: " + p);
    return {synth_model_with_embeddings(load_embeddings(p), seed, bias), seed};
  }
  return {synth_model(a.num<uint32_t>("vocab", 1000), a.num<int>("dim", 64), seed, bias), seed};
}

// WTA and cuckoo seeds derived from the model seed (tools/main.cpp:79-82)
uint64_t wta_seed(uint64_t s) { return mix_seed(s, 1); }
uint64_t cuckoo_seed(uint64_t s) { return mix_seed(s, 2); }

json stages_json(const StageTimes& st) {
  return {{"wta_hash", st.wta_hash},
          {"cuckoo_lookup", st.cuckoo_lookup},
          {"construct_candidate_list", st.construct_candidate_list},
          {"construct_e_lsh", st.construct_e_lsh},
          {"matrix_multiply", st.matrix_multiply},
          {"normalization", st.normalization},
          {"softmax_path_total", st.softmax_path()},
          {"beam_expansion", st.beam_expansion},
          {"recurrence", st.recurrence},
          {"oracle", st.oracle}};
}

void write_text(const std::string& path, const std::string& text) {
  if (path.empty()) {
    std::cout << text;
    return;
  }
  std::ofstream f(path);
  if (!f) throw std::runtime_error("cannot open for write: " + path);
  f << text;
}

int cmd_build(const Args& a) {
  const Model mo = make_model(a);
  WtaParams p(a.num<int>("K", 8), a.num<int>("u", 3), a.num<int>("W", 100), wta_seed(mo.seed));
  const std::string out = a.str("out", "index.wtaidx");
  const LshIndex idx = build_lsh_index(mo.m.embeddings, p, cuckoo_seed(mo.seed));
  save_lsh_index(idx, out);
  std::printf("index: vocab=%u dim=%d K=%d u=%d W=%d -> %s\n", idx.bands.vocab_size(), idx.dim,
              p.K, p.u, p.W, out.c_str());
  std::printf("band distinct-code counts:");
  for (uint32_t c : idx.bands.distinct_codes_per_band()) std::printf(" %u", c);
  std::printf("\nmax span length: %u\n", idx.bands.max_span_length());
  return 0;
}

int cmd_decode(const Args& a) {
  const DecodeMode mode = parse_mode(a.str("mode", "full"));
  const Model mo = make_model(a);
  std::optional<LshIndex> idx;
  if (mode == DecodeMode::kLsh) {
    if (a.has("index")) {
      const std::string p = a.str("index", "");
      if (!std::filesystem::exists(p)) throw UsageError("index file not found: " + p);
      idx = load_lsh_index(p);
      if (idx->bands.vocab_size() != mo.m.vocab || idx->dim != mo.m.dim)
        throw UsageError("index shape does not match the model");
    } else {
      idx = build_lsh_index(mo.m.embeddings,
                            WtaParams(a.num<int>("K", 8), a.num<int>("u", 3), a.num<int>("W", 100),
                                      wta_seed(mo.seed)),
                            cuckoo_seed(mo.seed));
    }
  }
  DecodeConfig cfg;
  cfg.beam = a.num<int>("beam", 4);
  cfg.top_merge = a.num<uint32_t>("T", 0);
  cfg.threshold = a.num<int>("t", 1);
  cfg.max_len = a.num<int>("steps", 16);
  const bool oracle = a.has("oracle");
  const DecodeResult res = decode(mo.m, cfg, mode, idx ? &*idx : nullptr, oracle);

  const StageTimes& st = res.stages;
  std::printf("mode %s  vocab %u  dim %d  beam %d  steps %d/%d\n", mode_name(mode), mo.m.vocab,
              mo.m.dim, cfg.beam, res.steps, cfg.max_len);
  std::printf("  %-29s %10.2f ms\n", "Softmax path", st.softmax_path());
  std::printf("  %-29s %10.2f ms\n", "Beam expansion", st.beam_expansion);
  std::printf("  mean |V_LSH| %.1f\n", res.mean_vlsh());
  if (oracle) std::printf("  recall@%d %.4f\n", cfg.beam, res.mean_recall());

  bool covers = true;
  for (uint32_t v : res.per_step_vlsh) covers = covers && v == mo.m.vocab;
  json seqs = json::array(), scores = json::array(), fin = json::array();
  for (const auto& h : res.hypotheses) {
    seqs.push_back(h.tokens);
    scores.push_back(h.score);
    fin.push_back(h.finished);
  }
  json params{{"K", nullptr}, {"u", nullptr}, {"W", nullptr}};
  if (idx) {
    params["K"] = idx->params.K;
    params["u"] = idx->params.u;
    params["W"] = idx->params.W;
  }
  params["T"] = cfg.top_merge;
  params["t"] = cfg.threshold;
  params["seed"] = mo.seed;
  params["bias"] = mo.m.bias_strength;
  params["workers"] = a.num<int>("workers", 0);
  const json report{{"command", "decode"},
                    {"mode", mode_name(mode)},
                    {"vocab", mo.m.vocab},
                    {"dim", mo.m.dim},
                    {"beam", cfg.beam},
                    {"steps_requested", cfg.max_len},
                    {"steps_run", res.steps},
                    {"params", params},
                    {"full_vocabulary_equivalent", covers},
                    {"mean_vlsh", res.mean_vlsh()},
                    {"per_step_vlsh", res.per_step_vlsh},
                    {"recall_at_b", oracle ? json(res.mean_recall()) : json()},
                    {"per_step_recall", oracle ? json(res.per_step_recall) : json()},
                    {"provenance",
                     {{"threshold_survivors", res.threshold_survivors},
                      {"top_added", res.top_added},
                      {"specials_added", res.specials_added}}},
                    {"sequences", seqs},
                    {"scores", scores},
                    {"finished", fin},
                    {"stage_ms", stages_json(st)}};
  write_text(a.str("out", ""), report.dump(2) + "\n");
  return 0;
}

int cmd_grid(const Args& a) {
  const auto Ks = a.list<int>("K", {8}), us = a.list<int>("u", {3}), Ws = a.list<int>("W", {500});
  const auto Ts = a.list<uint32_t>("T", {0});
  const auto ts = a.list<int>("t", {1});
  if (Ks.empty() || us.empty() || Ws.empty() || Ts.empty() || ts.empty())
    throw UsageError("empty grid");
  const Model mo = make_model(a);
  const int beam = a.num<int>("beam", 12), steps = a.num<int>("steps", 16);
  std::string csv = "K,u,W,T,t,B,mean_vlsh,recall_at_b,softmax_ms,speedup\n";
  char line[256];
  DecodeConfig base;
  base.beam = beam;
  base.max_len = steps;
  base.threshold = 0;
  const double base_ms = decode(mo.m, base, DecodeMode::kFull, nullptr, false).stages.softmax_path();
  std::snprintf(line, sizeof(line), ",,,,,%d,%.1f,%.6f,%.3f,%.4f\n", beam,
                static_cast<double>(mo.m.vocab), 1.0, base_ms, 1.0);
  csv += line;
  for (int K : Ks)
    for (int u : us)
      for (int W : Ws) {
        const LshIndex idx = build_lsh_index(mo.m.embeddings, WtaParams(K, u, W, wta_seed(mo.seed)),
                                             cuckoo_seed(mo.seed));
        for (uint32_t T : Ts)
          for (int t : ts) {
            DecodeConfig cfg;
            cfg.beam = beam;
            cfg.top_merge = T;
            cfg.threshold = t;
            cfg.max_len = steps;
            const DecodeResult r = decode(mo.m, cfg, DecodeMode::kLsh, &idx, true);
            const double ms = r.stages.softmax_path();
            std::snprintf(line, sizeof(line), "%d,%d,%d,%u,%d,%d,%.1f,%.6f,%.3f,%.4f\n", K, u, W,
                          T, t, beam, r.mean_vlsh(), r.mean_recall(), ms,
                          ms > 0 ? base_ms / ms : 0.0);
            csv += line;
            std::fprintf(stderr, "grid K=%d u=%d W=%d T=%u t=%d: |V_LSH|=%.0f recall=%.4f speedup=%.2f\n",
                         K, u, W, T, t, r.mean_vlsh(), r.mean_recall(), ms > 0 ? base_ms / ms : 0.0);
          }
      }
  write_text(a.str("out", ""), csv);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw UsageError("a subcommand is required: build | decode | grid");
    const std::string sub = argv[1];
    if (sub == "build")
      return cmd_build(Args(argc, argv, 2,
                            with(kModelOpts, {{"K", true}, {"u", true}, {"W", true},
                                              {"workers", true}, {"out", true}})));
    if (sub == "decode")
      return cmd_decode(Args(argc, argv, 2,
                             with(kModelOpts, {{"index", true}, {"K", true}, {"u", true},
                                               {"W", true}, {"beam", true}, {"T", true},
                                               {"t", true}, {"steps", true}, {"mode", true},
                                               {"oracle", false}, {"workers", true},
                                               {"out", true}})));
    if (sub == "grid")
      return cmd_grid(Args(argc, argv, 2,
                           with(kModelOpts, {{"K", true}, {"u", true}, {"W", true}, {"T", true},
                                             {"t", true}, {"beam", true}, {"steps", true},
                                             {"workers", true}, {"out", true}})));
    throw UsageError("unknown subcommand: " + sub);
  } catch (const UsageError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
