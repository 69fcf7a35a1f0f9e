// dropin_index.cpp -- lshbeam/band_index.hpp over the C ABI.
//  * CuckooTable::build -> lsb_cuckoo_build (device build, reference slot
//    placement; /root/reference/proj/src/band_index.cpp:32-71);
//  * CuckooTable::find -> lsb_index_find on a lazily uploaded 1-band table;
//  * BandIndex::build -> lsb_index_build_codes (K2-build); lookup_hits_into
//    -> lsb_lookup_hits (K2-lookup);
//  * build_lsh_index -> lsb_index_build (K1 on E + K2-build);
//  * WTAIDX1 save/load (src/band_index.cpp:198-289): host file I/O; a loaded
//    index is uploaded on first device use (lsb_index_import).
#include <algorithm>
#include <cstring>
#include <fstream>
#include <stdexcept>

#include "dropin_runtime.hpp"
#include "lshbeam/band_index.hpp"

namespace lshbeam {

using detail::check;
using detail::Guard;

namespace {

void flatten_slots(const std::vector<CuckooTable::Slot>& slots, std::vector<uint32_t>& out) {
  for (const auto& s : slots) {
    out.push_back(s.key);
    out.push_back(s.start);
    out.push_back(s.length);
  }
}

std::vector<CuckooTable::Slot> unflatten_slots(const uint32_t* p, size_t n) {
  std::vector<CuckooTable::Slot> out(n);
  for (size_t i = 0; i < n; ++i) out[i] = CuckooTable::Slot{p[3 * i], p[3 * i + 1], p[3 * i + 2]};
  return out;
}

// Host mirror of band w of a device index.
CuckooTable mirror_table(lsb_index* idx, int w, uint32_t* words) {
  uint32_t lg = 0;
  check(lsb_index_band(idx, w, nullptr, &lg, nullptr, nullptr), "index band");
  uint64_t mul[2];
  std::vector<uint32_t> flat(3ull * (2ull << lg));
  check(lsb_index_band(idx, w, words, &lg, mul, flat.data()), "index band");
  return CuckooTable(lg, mul[0], mul[1], unflatten_slots(flat.data(), 2ull << lg));
}

detail::DeviceIndex import_tables(uint32_t vocab, const std::vector<uint32_t>* words,
                                  const std::vector<CuckooTable>& tables,
                                  const PermutationSet* perms, int u) {
  const int W = static_cast<int>(tables.size());
  std::vector<uint32_t> lgs(W), flat;
  std::vector<uint64_t> muls(2 * W);
  for (int w = 0; w < W; ++w) {
    lgs[w] = tables[w].log2_capacity();
    muls[2 * w] = tables[w].multiplier(0);
    muls[2 * w + 1] = tables[w].multiplier(1);
    flatten_slots(tables[w].slots(), flat);
  }
  lsb_index* idx = nullptr;
  check(lsb_index_import(detail::ctx(), vocab, W, words ? words->data() : nullptr, lgs.data(),
                         muls.data(), flat.data(), perms ? perms->prefixes().data() : nullptr,
                         perms ? perms->window() : 0, u, perms ? perms->dim() : 0, 0, &idx),
        "index upload");
  return detail::share(idx);
}

}  // namespace

// ------------------------------------------------------------ CuckooTable
CuckooTable::CuckooTable(uint32_t lg, uint64_t mul0, uint64_t mul1, std::vector<Slot> slots)
    : lg_(lg), slots_(std::move(slots)) {
  mul_[0] = mul0;
  mul_[1] = mul1;
  if (slots_.size() != 2ull * capacity())
    throw std::invalid_argument("CuckooTable: slot array size mismatch");
}

CuckooTable CuckooTable::build(const std::vector<std::pair<uint32_t, Span>>& entries,
                               uint64_t seed) {
  const uint32_t n = static_cast<uint32_t>(entries.size());
  std::vector<uint32_t> keys(n), starts(n), lens(n);
  for (uint32_t i = 0; i < n; ++i) {
    keys[i] = entries[i].first;
    starts[i] = entries[i].second.start;
    lens[i] = entries[i].second.length;
    if (keys[i] >= kEmptyCode) throw std::invalid_argument("CuckooTable: key collides with sentinel");
  }
  Guard g(detail::api_mutex());
  const uint32_t lg = lsb_cuckoo_log2_capacity(n);
  std::vector<uint32_t> flat(3ull * (2ull << lg));
  uint64_t mul[2];
  uint32_t lg_out = 0;
  check(lsb_cuckoo_build(detail::ctx(), keys.data(), starts.data(), lens.data(), n, seed, &lg_out,
                         mul, flat.data(), nullptr),
        "CuckooTable: build failed after rebuild budget");
  return CuckooTable(lg_out, mul[0], mul[1], unflatten_slots(flat.data(), 2ull << lg_out));
}

std::optional<CuckooTable::Span> CuckooTable::find_counted(uint32_t key, int& probes) const {
  Guard g(detail::api_mutex());
  if (!dev_) dev_ = import_tables(0, nullptr, std::vector<CuckooTable>{*this}, nullptr, 0);
  const int32_t band = 0;
  uint32_t start = 0, len = 0;
  uint8_t found = 0;
  check(lsb_index_find(detail::ctx(), dev_.get(), &band, &key, 1, &start, &len, &found),
        "CuckooTable::find");
  // the device probes table 0 then table 1 (band_index.cpp:73-83); report
  // how many slots that inspected
  const uint32_t s0 = static_cast<uint32_t>((mul_[0] * key) >> (64 - lg_));
  probes = slots_[s0].key == key ? 1 : 2;
  if (!found) return std::nullopt;
  return Span{start, len};
}

std::optional<CuckooTable::Span> CuckooTable::find(uint32_t key) const {
  int probes = 0;
  return find_counted(key, probes);
}

// -------------------------------------------------------------- BandIndex
BandIndex::BandIndex(uint32_t vocab, int W, std::vector<uint32_t> word_ids,
                     std::vector<CuckooTable> tables)
    : vocab_(vocab), W_(W), words_(std::move(word_ids)), tables_(std::move(tables)) {}

BandIndex BandIndex::build(const MatU32& band_codes, uint64_t seed) {
  const uint32_t V = static_cast<uint32_t>(band_codes.rows());
  const int W = static_cast<int>(band_codes.cols());
  for (size_t i = 0; i < static_cast<size_t>(V) * W; ++i)
    if (band_codes.data()[i] >= kEmptyCode)
      throw std::invalid_argument("CuckooTable: key collides with sentinel");
  Guard g(detail::api_mutex());
  lsb_index* idx = nullptr;
  const lsb_status st = lsb_index_build_codes(detail::ctx(), band_codes.data(), V, W, seed, &idx);
  if (st == LSB_ERUNTIME) throw std::runtime_error("BandIndex: cuckoo build failed");
  check(st, "BandIndex::build");
  auto dev = detail::share(idx);
  std::vector<uint32_t> words(static_cast<size_t>(W) * V);
  std::vector<CuckooTable> tables;
  tables.reserve(W);
  for (int w = 0; w < W; ++w)
    tables.push_back(mirror_table(idx, w, words.data() + static_cast<size_t>(w) * V));
  BandIndex out(V, W, std::move(words), std::move(tables));
  out.dev_ = std::move(dev);
  return out;
}

lsb_index* BandIndex::device() const {
  Guard g(detail::api_mutex());
  if (!dev_) {
    dev_ = import_tables(vocab_, &words_, tables_, nullptr, 0);
    dev_has_perms_ = false;
  }
  return dev_.get();
}

lsb_index* BandIndex::device_with_perms(const PermutationSet& perms, int u) const {
  Guard g(detail::api_mutex());
  if (!dev_ || !dev_has_perms_) {
    dev_ = import_tables(vocab_, &words_, tables_, &perms, u);
    dev_has_perms_ = true;
  }
  return dev_.get();
}

void BandIndex::lookup_hits_into(const MatU32& query_codes, HitMatrix& L) const {
  if (static_cast<int>(query_codes.cols()) != W_)
    throw std::invalid_argument("lookup_hits: band count mismatch");
  const int B = static_cast<int>(query_codes.rows());
  if (L.rows() != static_cast<size_t>(B) || L.cols() != vocab_) L = HitMatrix(B, vocab_);
  else L.fill(0);
  if (B == 0 || vocab_ == 0) return;
  Guard g(detail::api_mutex());
  check(lsb_lookup_hits(detail::ctx(), device(), query_codes.data(), B, L.data()),
        "lookup_hits");
}

HitMatrix BandIndex::lookup_hits(const MatU32& query_codes) const {
  HitMatrix L;
  lookup_hits_into(query_codes, L);
  return L;
}

std::vector<uint32_t> BandIndex::distinct_codes_per_band() const {
  std::vector<uint32_t> out(W_, 0);
  for (int w = 0; w < W_; ++w)
    for (const auto& s : tables_[w].slots()) out[w] += s.key != kEmptyCode;
  return out;
}

uint32_t BandIndex::max_span_length() const {
  uint32_t m = 0;
  for (const auto& t : tables_)
    for (const auto& s : t.slots())
      if (s.key != kEmptyCode) m = std::max(m, s.length);
  return m;
}

// ----------------------------------------------------------------- LshIndex
struct LshIndexBuilder {
  static LshIndex make(const WtaParams& params, int dim, PermutationSet perms, lsb_index* idx) {
    auto dev = detail::share(idx);
    lsb_index_info info{};
    check(lsb_index_info_get(idx, &info), "index info");
    const uint32_t V = info.vocab;
    const int W = info.W;
    std::vector<uint32_t> words(static_cast<size_t>(W) * V);
    std::vector<CuckooTable> tables;
    tables.reserve(W);
    for (int w = 0; w < W; ++w)
      tables.push_back(mirror_table(idx, w, words.data() + static_cast<size_t>(w) * V));
    BandIndex bands(V, W, std::move(words), std::move(tables));
    bands.dev_ = std::move(dev);
    bands.dev_has_perms_ = true;
    return LshIndex{params, dim, std::move(perms), std::move(bands)};
  }
};

LshIndex build_lsh_index(const MatF& embeddings, const WtaParams& params, uint64_t index_seed) {
  const int d = static_cast<int>(embeddings.cols());
  PermutationSet perms = generate_permutations(d, params);  // validates d >= K
  Guard g(detail::api_mutex());
  auto model = detail::cached_model(embeddings.data(), static_cast<uint32_t>(embeddings.rows()),
                                    d, nullptr);
  lsb_index* idx = nullptr;
  const lsb_status st = lsb_index_build(detail::ctx(), model.get(), params.K, params.u, params.W,
                                        params.seed, index_seed, &idx);
  if (st == LSB_ERUNTIME) throw std::runtime_error("BandIndex: cuckoo build failed");
  check(st, "build_lsh_index");
  return LshIndexBuilder::make(params, d, std::move(perms), idx);
}

// ------------------------------------------------------------- WTAIDX1 I/O
namespace {
constexpr char kMagic[7] = {'W', 'T', 'A', 'I', 'D', 'X', '1'};

template <typename T>
void wr(std::ofstream& f, T v) {
  f.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
T rd(std::ifstream& f) {
  T v{};
  f.read(reinterpret_cast<char*>(&v), sizeof(T));
  if (!f) throw std::runtime_error("index file: truncated");
  return v;
}
}  // namespace

void save_lsh_index(const LshIndex& index, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open for write: " + path);
  f.write(kMagic, sizeof(kMagic));
  const WtaParams& p = index.params;
  for (uint32_t v : {index.bands.vocab_size(), static_cast<uint32_t>(p.W),
                     static_cast<uint32_t>(p.K), static_cast<uint32_t>(p.u),
                     static_cast<uint32_t>(p.bits_per_index()), static_cast<uint32_t>(index.dim)})
    wr<uint32_t>(f, v);
  wr<uint64_t>(f, p.seed);
  for (int w = 0; w < p.W; ++w) {
    const CuckooTable& t = index.bands.table(w);
    wr<uint32_t>(f, t.log2_capacity());
    wr<uint64_t>(f, t.multiplier(0));
    wr<uint64_t>(f, t.multiplier(1));
    for (const auto& s : t.slots()) {
      wr<uint32_t>(f, s.key);
      wr<uint32_t>(f, s.start);
      wr<uint32_t>(f, s.length);
    }
    const auto ids = index.bands.band_words(w);
    f.write(reinterpret_cast<const char*>(ids.data()),
            static_cast<std::streamsize>(ids.size() * sizeof(uint32_t)));
  }
  if (!f) throw std::runtime_error("write failed: " + path);
}

LshIndex load_lsh_index(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open: " + path);
  char magic[sizeof(kMagic)];
  f.read(magic, sizeof(magic));
  if (!f || std::memcmp(magic, kMagic, sizeof(kMagic)) != 0)
    throw std::runtime_error("index file: bad magic");
  const uint32_t vocab = rd<uint32_t>(f), W = rd<uint32_t>(f), K = rd<uint32_t>(f);
  const uint32_t u = rd<uint32_t>(f), bits = rd<uint32_t>(f), dim = rd<uint32_t>(f);
  const uint64_t seed = rd<uint64_t>(f);
  WtaParams params(static_cast<int>(K), static_cast<int>(u), static_cast<int>(W), seed);
  if (bits != static_cast<uint32_t>(params.bits_per_index()))
    throw std::runtime_error("index file: inconsistent bits_per_index");
  std::vector<uint32_t> words(static_cast<size_t>(W) * vocab);
  std::vector<CuckooTable> tables;
  tables.reserve(W);
  for (uint32_t w = 0; w < W; ++w) {
    const uint32_t lg = rd<uint32_t>(f);
    const uint64_t m0 = rd<uint64_t>(f), m1 = rd<uint64_t>(f);
    if (lg > 30) throw std::runtime_error("index file: table size out of range");
    std::vector<CuckooTable::Slot> slots(2ull << lg);
    for (auto& s : slots) {
      s.key = rd<uint32_t>(f);
      s.start = rd<uint32_t>(f);
      s.length = rd<uint32_t>(f);
    }
    tables.emplace_back(lg, m0, m1, std::move(slots));
    f.read(reinterpret_cast<char*>(words.data() + static_cast<size_t>(w) * vocab),
           static_cast<std::streamsize>(vocab * sizeof(uint32_t)));
    if (!f) throw std::runtime_error("index file: truncated");
  }
  PermutationSet perms = PermutationSet::generate(static_cast<int>(dim), params.num_hashes(),
                                                  params.K, params.seed);
  return LshIndex{params, static_cast<int>(dim), std::move(perms),
                  BandIndex(vocab, static_cast<int>(W), std::move(words), std::move(tables))};
}

}  // namespace lshbeam
