// dropin_decode.cpp -- lshbeam/beam_decoder.hpp over the C ABI.
// compute_logits / softmax_rows / expand_beams are the K4 / K5 stage entry
// points (PARITY arithmetic). decode() follows the control flow of
// /root/reference/proj/src/beam_decoder.cpp:143-329 but keeps the hot path
// and the hidden states on the GPU: each step is one fused lsb_step (K1..K5,
// including the parent-row reorder of the hidden states) followed by one
// batched recurrence launch; the host only keeps tokens, scores and flags.
#include <algorithm>
#include <chrono>
#include <cstddef>
#include <stdexcept>

#include "dropin_runtime.hpp"
#include "lshbeam/beam_decoder.hpp"

namespace lshbeam {

using detail::check;
using detail::Guard;

static_assert(sizeof(BeamChoice) == sizeof(lsb_choice), "BeamChoice layout");
static_assert(offsetof(BeamChoice, score) == offsetof(lsb_choice, score), "BeamChoice layout");
static_assert(offsetof(BeamChoice, beam) == offsetof(lsb_choice, beam), "BeamChoice layout");
static_assert(offsetof(BeamChoice, word) == offsetof(lsb_choice, word), "BeamChoice layout");

MatF compute_logits(const MatF& H, const MatF& E_sub) {
  if (H.cols() != E_sub.cols())
    throw std::invalid_argument("compute_logits: inner dimensions disagree");
  MatF out(H.rows(), E_sub.rows());
  if (out.empty()) return out;
  Guard g(detail::api_mutex());
  check(lsb_compute_logits(detail::ctx(), H.data(), static_cast<int>(H.rows()), E_sub.data(),
                           static_cast<int64_t>(E_sub.rows()), static_cast<int>(H.cols()),
                           LSB_MODE_PARITY, out.data()),
        "compute_logits");
  return out;
}

MatF softmax_rows(const MatF& logits) {
  MatF out(logits.rows(), logits.cols());
  if (logits.rows() == 0) return out;
  Guard g(detail::api_mutex());
  check(lsb_softmax_rows(detail::ctx(), logits.data(), static_cast<int>(logits.rows()),
                         static_cast<int64_t>(logits.cols()), out.data()),
        "softmax_rows");
  return out;
}

std::vector<BeamChoice> expand_beams(const MatF& probs, std::span<const double> cum_scores,
                                     std::span<const uint32_t> live_beam_ids,
                                     std::span<const BeamChoice> frozen, int B,
                                     std::span<const uint32_t> id_map) {
  const size_t rows = probs.rows(), n = probs.cols();
  if (cum_scores.size() != rows || live_beam_ids.size() != rows)
    throw std::invalid_argument("expand_beams: row metadata mismatch");
  if (!id_map.empty() && id_map.size() != n)
    throw std::invalid_argument("expand_beams: id_map size mismatch");
  std::vector<BeamChoice> out(std::max(B, 0));
  if (B <= 0) return {};
  int count = 0;
  Guard g(detail::api_mutex());
  check(lsb_expand_beams(detail::ctx(), probs.data(), static_cast<int>(rows),
                         static_cast<int64_t>(n), cum_scores.data(), live_beam_ids.data(),
                         reinterpret_cast<const lsb_choice*>(frozen.data()),
                         static_cast<int>(frozen.size()), B,
                         id_map.empty() ? nullptr : id_map.data(),
                         reinterpret_cast<lsb_choice*>(out.data()), &count),
        "expand_beams");
  out.resize(count);
  return out;
}

DecodeMode parse_mode(const std::string& s) {
  if (s == "full") return DecodeMode::kFull;
  if (s == "lsh") return DecodeMode::kLsh;
  if (s == "top") return DecodeMode::kTopOnly;
  throw std::invalid_argument("unknown mode: " + s);
}

const char* mode_name(DecodeMode mode) {
  switch (mode) {
    case DecodeMode::kFull: return "full";
    case DecodeMode::kLsh: return "lsh";
    case DecodeMode::kTopOnly: return "top";
  }
  return "?";
}

double DecodeResult::mean_vlsh() const {
  if (per_step_vlsh.empty()) return 0.0;
  double s = 0.0;
  for (uint32_t v : per_step_vlsh) s += v;
  return s / per_step_vlsh.size();
}

double DecodeResult::mean_recall() const {
  if (per_step_recall.empty()) return 0.0;
  double s = 0.0;
  for (double v : per_step_recall) s += v;
  return s / per_step_recall.size();
}

namespace {

struct HostHyp {
  std::vector<uint32_t> tokens;
  double score = 0.0;
  bool finished = false;
};

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

DecodeResult decode(const SynthModel& model, const DecodeConfig& config, DecodeMode mode,
                    const LshIndex* lsh, bool with_oracle) {
  if (mode == DecodeMode::kLsh) {
    if (lsh == nullptr) throw std::invalid_argument("decode: lsh mode requires an index");
    if (lsh->bands.vocab_size() != model.vocab || lsh->dim != model.dim)
      throw std::invalid_argument("decode: index does not match the model");
    config.validate(model.vocab, lsh->params.W);
  } else {
    config.validate(model.vocab, std::max(config.threshold, 0));
  }
  std::vector<uint32_t> specials = config.specials;
  specials.push_back(model.eos_id);  // EOS is always a candidate

  Guard guard(detail::api_mutex());
  lsb_ctx* c = detail::ctx();
  const int d = model.dim, B = config.beam;
  const uint32_t V = model.vocab;
  // device copies cached across decode() calls on the same model (the
  // acceptance grid decodes one model 32 times)
  auto dm = detail::cached_model(model.embeddings.data(), V, d, model.freq_bias.data());
  auto rec = detail::cached_recurrent(model.w_hidden.data(), model.w_embed.data(), d);
  lsb_index* ix = mode == DecodeMode::kLsh
                      ? lsh->bands.device_with_perms(lsh->perms, lsh->params.u)
                      : nullptr;
  const bool full = mode == DecodeMode::kFull;
  lsb_step_config cfg{};
  cfg.S = 1;
  cfg.B = B;
  cfg.top_merge = config.top_merge;
  cfg.threshold = config.threshold;
  cfg.specials = specials.data();
  cfg.nspec = static_cast<int>(specials.size());
  cfg.mode = LSB_MODE_PARITY;
  cfg.full_vocab = full ? 1 : 0;
  cfg.top_only = mode == DecodeMode::kTopOnly ? 1 : 0;
  lsb_batch* braw = nullptr;
  check(lsb_batch_create(c, dm.get(), ix, &cfg, &braw), "decode");
  detail::BatchPtr batch(braw);
  check(lsb_batch_profile(braw, 1), "decode: profiling");

  detail::DevMem hid(sizeof(float) * B * d), tmp(sizeof(float) * B * d);
  detail::DevMem sc(sizeof(double) * B), fin(B), nh(sizeof(int32_t)), ch(sizeof(lsb_choice) * B),
      nch(sizeof(int32_t)), tok(sizeof(int64_t) * B);
  detail::h2d(hid.p, model.h0.data(), sizeof(float) * d);

  DecodeResult res;
  std::vector<HostHyp> hyps(1);
  std::vector<double> scores(B);
  std::vector<uint8_t> flags(B);
  std::vector<lsb_choice> chosen(B);
  std::vector<int64_t> tokens(B);
  std::vector<uint32_t> cand_ids(full ? 0 : V);
  std::vector<uint32_t> exact;

  for (int step = 0; step < config.max_len; ++step) {
    bool any_live = false;
    for (const auto& h : hyps) any_live = any_live || !h.finished;
    if (!any_live) break;
    const int n = static_cast<int>(hyps.size());
    for (int i = 0; i < n; ++i) {
      scores[i] = hyps[i].score;
      flags[i] = hyps[i].finished ? 1 : 0;
    }
    const int32_t n32 = n;
    detail::h2d(sc.p, scores.data(), sizeof(double) * n);
    detail::h2d(fin.p, flags.data(), n);
    detail::h2d(nh.p, &n32, sizeof(n32));
    lsb_state_dev in{hid.as<float>(), sc.as<double>(), fin.as<uint8_t>(), nh.as<int32_t>()};
    lsb_out_dev out{ch.as<lsb_choice>(), nch.as<int32_t>(), tmp.as<float>()};
    check(lsb_step(braw, &in, &out), "decode: step");
    int32_t count = 0;
    detail::d2h(&count, nch.p, sizeof(count));  // synchronises, surfaces errors
    float ms5[5];
    check(lsb_batch_stage_ms(braw, ms5), "decode: stage times");
    res.stages.cuckoo_lookup += ms5[0];
    res.stages.construct_candidate_list += ms5[1];
    res.stages.matrix_multiply += ms5[2];
    res.stages.normalization += ms5[3];
    res.stages.beam_expansion += ms5[4];

    uint32_t ncand = V, prov[3] = {0, 0, 0};
    if (!full) {
      check(lsb_batch_candidates(braw, 0, cand_ids.data(), &ncand, prov), "decode: candidates");
      res.threshold_survivors += prov[0];
      res.top_added += prov[1];
      res.specials_added += prov[2];
    }
    res.per_step_vlsh.push_back(ncand);

    if (with_oracle) {  // recall@B of the candidate set, outside the softmax path
      const auto t0 = std::chrono::steady_clock::now();
      if (full) {
        res.per_step_recall.push_back(1.0);
      } else {
        exact.assign(static_cast<size_t>(n) * B, 0);
        check(lsb_exact_topb(c, dm.get(), hid.as<float>(), n, 1, B, 1, exact.data(), nullptr),
              "decode: oracle");
        double total = 0.0;
        int live = 0;
        for (int i = 0; i < n; ++i) {
          if (hyps[i].finished) continue;
          int hit = 0;
          for (int k = 0; k < B; ++k)
            hit += std::binary_search(cand_ids.begin(), cand_ids.begin() + ncand,
                                      exact[static_cast<size_t>(i) * B + k]);
          total += static_cast<double>(hit) / B;
          ++live;
        }
        res.per_step_recall.push_back(live ? total / live : 0.0);
      }
      res.stages.oracle += ms_since(t0);
    }

    detail::d2h(chosen.data(), ch.p, sizeof(lsb_choice) * count);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<HostHyp> next;
    next.reserve(count);
    for (int k = 0; k < count; ++k) {
      const lsb_choice& cc = chosen[k];
      const HostHyp& parent = hyps[cc.beam];
      if (cc.word < 0) {  // frozen hypothesis carried over
        next.push_back(parent);
        tokens[k] = -1;
        continue;
      }
      HostHyp h;
      h.tokens = parent.tokens;
      h.tokens.push_back(static_cast<uint32_t>(cc.word));
      h.score = cc.score;
      h.finished = static_cast<uint32_t>(cc.word) == model.eos_id;
      tokens[k] = h.finished ? -1 : cc.word;  // EOS children keep the parent state
      next.push_back(std::move(h));
    }
    detail::h2d(tok.p, tokens.data(), sizeof(int64_t) * count);
    check(lsb_recurrence(c, dm.get(), rec.get(), tmp.as<float>(), tok.as<int64_t>(), count,
                         hid.as<float>()),
          "decode: recurrence");
    check(lsb_ctx_sync(c), "decode: recurrence");
    res.stages.recurrence += ms_since(t0);
    hyps = std::move(next);
    ++res.steps;
    bool done = true;
    for (const auto& h : hyps) done = done && h.finished;
    if (done) break;
  }

  std::vector<float> hidden(static_cast<size_t>(hyps.size()) * d);
  detail::d2h(hidden.data(), hid.p, sizeof(float) * hidden.size());
  res.hypotheses.reserve(hyps.size());
  for (size_t i = 0; i < hyps.size(); ++i) {
    Hypothesis h;
    h.tokens = std::move(hyps[i].tokens);
    h.score = hyps[i].score;
    h.finished = hyps[i].finished;
    h.hidden.assign(hidden.begin() + i * d, hidden.begin() + (i + 1) * d);
    res.hypotheses.push_back(std::move(h));
  }
  std::stable_sort(res.hypotheses.begin(), res.hypotheses.end(),
                   [](const Hypothesis& a, const Hypothesis& b) { return a.score > b.score; });
  return res;
}

}  // namespace lshbeam
