// WTAIDX1 interop between the reference library and the GPU drop-in.
//
// The same source is compiled twice against the same public API
// (include/lshbeam/*.hpp):
//   * against the reference (oracle/_ref/libref_lshbeam.so, headers from
//     /root/reference/proj/include) by tests/golden/make_wtaidx.sh, in
//     `write` mode: build_lsh_index + save_lsh_index (src/band_index.cpp:189-243)
//     and the reference's lookup_hits for fixed queries -> tests/golden/;
//   * against the drop-in (paper_1806_00588_b200/liblshbeam.so) by
//     tests/test_gpu_interop.py, in `check` mode: load_lsh_index of the
//     reference-written file into device tables (src/band_index.cpp:245-289),
//     device lookups == the reference's hit counts, save_lsh_index of the
//     loaded index == the reference's bytes, and a GPU build_lsh_index of the
//     same embeddings saved == the reference's bytes (reference slot placement).
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "lshbeam/band_index.hpp"
#include "lshbeam/model_provider.hpp"
#include "lshbeam/rng.hpp"
#include "lshbeam/wta_hash.hpp"

using namespace lshbeam;

static constexpr uint32_t kV = 1500;
static constexpr int kD = 48, kK = 4, kU = 2, kW = 8, kRows = 6;
static constexpr uint64_t kSeed = 7;

static std::vector<char> slurp(const std::string& p) {
  std::ifstream f(p, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open " + p);
  return std::vector<char>(std::istreambuf_iterator<char>(f), {});
}

static MatF queries() {
  MatF H(kRows, kD);
  SplitMix64 g(mix_seed(kSeed, 3));
  for (size_t i = 0; i < H.rows(); ++i)
    for (size_t c = 0; c < H.cols(); ++c) H(i, c) = static_cast<float>(g.gaussian());
  return H;
}

static LshIndex build() {
  const SynthModel m = synth_model(kV, kD, kSeed, 0.0f);
  return build_lsh_index(m.embeddings, WtaParams(kK, kU, kW, mix_seed(kSeed, 1)),
                         mix_seed(kSeed, 2));
}

int main(int argc, char** argv) {
  if (argc < 3) {
    fprintf(stderr, "usage: %s write <dir> | check <dir> <tmpdir>\n", argv[0]);
    return 2;
  }
  const std::string mode = argv[1], dir = argv[2];
  const std::string idx_path = dir + "/ref_index.wtaidx", hits_path = dir + "/ref_hits.bin";
  try {
    if (mode == "write") {
      const LshIndex idx = build();
      save_lsh_index(idx, idx_path);
      const MatU32 q = hash_matrix(queries(), idx.perms, idx.params);
      const HitMatrix L = idx.bands.lookup_hits(q);
      std::ofstream f(hits_path, std::ios::binary);
      f.write(reinterpret_cast<const char*>(q.data()), (q.rows() * q.cols()) * 4);
      f.write(reinterpret_cast<const char*>(L.data()), (L.rows() * L.cols()) * 4);
      printf("wrote %s and %s\n", idx_path.c_str(), hits_path.c_str());
      return 0;
    }
    if (mode != "check" || argc < 4) return 2;
    const std::string tmp = argv[3];
    int bad = 0;
    const std::vector<char> ref_bytes = slurp(idx_path), hits = slurp(hits_path);
    // 1. load the reference-written file into device tables; lookups match
    const LshIndex loaded = load_lsh_index(idx_path);
    MatU32 q(kRows, kW);
    std::memcpy(q.data(), hits.data(), (q.rows() * q.cols()) * 4);
    const HitMatrix L = loaded.bands.lookup_hits(q);
    if ((L.rows() * L.cols()) != static_cast<size_t>(kRows) * kV ||
        std::memcmp(L.data(), hits.data() + (q.rows() * q.cols()) * 4, (L.rows() * L.cols()) * 4) != 0) {
      printf("FAIL lookup_hits of the loaded index differs from the reference's\n");
      ++bad;
    }
    // query codes recomputed from the loaded permutations match too
    const MatU32 q2 = hash_matrix(queries(), loaded.perms, loaded.params);
    if (std::memcmp(q2.data(), q.data(), (q.rows() * q.cols()) * 4) != 0) {
      printf("FAIL hash_matrix with the loaded permutations differs\n");
      ++bad;
    }
    // 2. re-export of the loaded index is byte-identical
    save_lsh_index(loaded, tmp + "/reexport.wtaidx");
    if (slurp(tmp + "/reexport.wtaidx") != ref_bytes) {
      printf("FAIL re-exported WTAIDX1 differs from the reference-written bytes\n");
      ++bad;
    }
    // 3. a GPU build of the same embeddings exports the reference's bytes
    save_lsh_index(build(), tmp + "/gpu_build.wtaidx");
    if (slurp(tmp + "/gpu_build.wtaidx") != ref_bytes) {
      printf("FAIL GPU-built WTAIDX1 differs from the reference-written bytes\n");
      ++bad;
    }
    printf("%s (%zu bytes)\n", bad ? "FAILED" : "ok", ref_bytes.size());
    return bad ? 1 : 0;
  } catch (const std::exception& e) {
    printf("exception: %s\n", e.what());
    return 1;
  }
}
