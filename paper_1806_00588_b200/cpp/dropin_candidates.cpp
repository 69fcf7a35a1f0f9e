// dropin_candidates.cpp -- lshbeam/candidate_selector.hpp over the C ABI
// (K3 bitmap/ballot compaction and the row-gather kernel). Config validation
// mirrors /root/reference/proj/src/candidate_selector.cpp:121-132.
#include <algorithm>
#include <stdexcept>
#include <string>

#include "dropin_runtime.hpp"
#include "lshbeam/candidate_selector.hpp"

namespace lshbeam {

using detail::check;
using detail::Guard;

bool CandidateSet::contains(uint32_t id) const {
  return std::binary_search(word_ids.begin(), word_ids.end(), id);
}

CandidateSet select_candidates(const HitMatrix& L, int threshold) {
  if (threshold < 0) throw std::invalid_argument("select_candidates: negative threshold");
  const uint32_t V = static_cast<uint32_t>(L.cols());
  CandidateSet out;
  out.word_ids.resize(V);
  uint32_t n = 0, ft = 0;
  Guard g(detail::api_mutex());
  check(lsb_select_candidates(detail::ctx(), L.data(), static_cast<int>(L.rows()), V, threshold,
                              out.word_ids.data(), &n, &ft),
        "select_candidates");
  out.word_ids.resize(n);
  out.from_threshold = ft;
  return out;
}

CandidateSet merge_top_frequent(CandidateSet cands, uint32_t top_merge,
                                std::span<const uint32_t> specials, uint32_t vocab) {
  std::vector<uint32_t> out(cands.word_ids.size() + top_merge + specials.size() + 1);
  uint32_t n = 0, prov[3] = {0, 0, 0};
  Guard g(detail::api_mutex());
  check(lsb_merge_top_frequent(detail::ctx(), cands.word_ids.data(),
                               static_cast<uint32_t>(cands.word_ids.size()), cands.from_threshold,
                               top_merge, specials.data(), static_cast<uint32_t>(specials.size()),
                               vocab, out.data(), &n, prov),
        "merge_top_frequent");
  out.resize(n);
  CandidateSet r;
  r.word_ids = std::move(out);
  r.from_threshold = prov[0];
  r.from_top = prov[1];
  r.from_specials = prov[2];
  return r;
}

GatheredEmbeddings gather_embeddings(const MatF& E, const CandidateSet& cands) {
  const uint32_t n = static_cast<uint32_t>(cands.size());
  GatheredEmbeddings g{MatF(n, E.cols()), cands.word_ids};
  if (n == 0 || E.cols() == 0) return g;
  for (uint32_t id : cands.word_ids)
    if (id >= E.rows()) throw std::invalid_argument("gather_embeddings: id out of range");
  Guard lock(detail::api_mutex());
  auto model = detail::cached_model(E.data(), static_cast<uint32_t>(E.rows()),
                                    static_cast<int>(E.cols()), nullptr);
  check(lsb_gather_embeddings(detail::ctx(), model.get(), cands.word_ids.data(), n, g.rows.data()),
        "gather_embeddings");
  return g;
}

void DecodeConfig::validate(uint32_t vocab, int num_bands) const {
  if (beam < 1) throw std::invalid_argument("config: beam must be >= 1");
  if (top_merge > vocab) throw std::invalid_argument("config: T exceeds vocabulary size");
  if (threshold < 0 || threshold > num_bands)
    throw std::invalid_argument("config: t must be in [0, W]");
  if (max_len < 1) throw std::invalid_argument("config: steps must be >= 1");
  for (uint32_t id : specials)
    if (id >= vocab) throw std::invalid_argument("config: special id out of range");
}

}  // namespace lshbeam
