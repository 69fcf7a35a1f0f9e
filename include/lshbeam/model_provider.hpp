// lshbeam/model_provider.hpp -- drop-in for the reference's synthetic scorer
// (/root/reference/proj/include/lshbeam/model_provider.hpp). The tensors are
// drawn on the host from one SplitMix64 stream in the reference's order
// (embeddings, W_h, W_e, h0, then the Zipf bias; src/model_provider.cpp:21-65)
// so both sides see identical inputs. The recurrence step_hidden runs on the
// GPU (FP32 in the reference's 4-lane order, tanh in double then rounded);
// WTAEMB1 I/O is host file handling.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "lshbeam/matrix.hpp"

namespace lshbeam {

struct SynthModel {
  uint32_t vocab = 0;
  int dim = 0;
  uint64_t seed = 0;
  float bias_strength = 0.0f;
  uint32_t eos_id = 0;  // vocab - 1

  MatF embeddings;  // |V| x d
  MatF w_hidden;    // d x d, scale 1/sqrt(d)
  MatF w_embed;     // d x d, scale 0.02/sqrt(d)
  std::vector<float> h0;
  std::vector<float> freq_bias;
};

SynthModel synth_model(uint32_t vocab, int dim, uint64_t seed, float bias_strength);
SynthModel synth_model_with_embeddings(MatF embeddings, uint64_t seed, float bias_strength);

// h' = tanh(W_h h + W_e emb(token)); throws on an out-of-range token or a
// dimension mismatch.
void step_hidden(const SynthModel& model, std::span<const float> h, uint32_t token,
                 std::span<float> out);
std::vector<float> step_hidden(const SynthModel& model, std::span<const float> h,
                               uint32_t token);

// WTAEMB1: magic | version 0x01 | u32 vocab | u32 dim | vocab*dim f32.
void save_embeddings(const MatF& E, const std::string& path);
MatF load_embeddings(const std::string& path);

}  // namespace lshbeam
