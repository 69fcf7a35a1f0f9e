// batch.cuh -- host state of one lsb_batch (per-step scratch for S
// sentences), shared by the fused step (capi_step.cu) and the vocabulary-
// sharded step (capi_shard.cu).
#pragma once

#include <vector>

#include "k_step.cuh"

struct lsb_batch {
  lsb_ctx* ctx = nullptr;
  const lsb_model* model = nullptr;
  const lsb_index* idx = nullptr;
  int S = 0, B = 0, d = 0, t = 0;
  uint32_t V = 0, T = 0;
  lsb_mode mode = LSB_MODE_PARITY;
  int cmode = 0;  // 0 threshold, 1 all words (t == 0), 2 full vocabulary
  uint32_t n_shared = 0;
  size_t ncap = 0;
  uint32_t nwords = 0, slice_len = 0;
  int counter_bytes = 1;
  int levels = -1;  // bit-sliced hit counting when 1 <= t <= 8
  int nspec = 0;
  int keep_probs = 0;
  int seq_denom = 0;  // test hook: LSB_SEQ_DENOM=1 at create (SoftmaxArgs::seq_denominator)
  // device scratch
  uint32_t* specials = nullptr;
  uint32_t* qcodes = nullptr;
  uint32_t* bitmap = nullptr;
  uint32_t* ids = nullptr;
  uint32_t* n_cand = nullptr;
  uint32_t* prov = nullptr;
  float* logits = nullptr;
  lsb::TopEntry* top = nullptr;
  int32_t* top_n = nullptr;
  uint32_t* arrive = nullptr;   // fused K5: per-sentence arrival counters (zeroed)
  float* tc_A = nullptr;        // FAST: pre-tiled E[0, n_shared) for tcgen05
  float* tc_H = nullptr;        // FAST: per-step tiled H
  int tc_N = 0;
  // few rows: band-split K1+K2 (probe_G > 0) with 16-bit hit counters
  int probe_G = 0;
  uint32_t* split_cnt = nullptr;     // [S*B][split_words], self-cleaning
  uint32_t split_words = 0;
  uint32_t* split_arrive = nullptr;  // [S*B]
  // long rows (full vocabulary / t = 0): segmented K5a scratch
  int seg_P = 0;
  float* seg_max = nullptr;
  double* seg_sum = nullptr;
  double* seg_c = nullptr;
  double* seg_b = nullptr;
  lsb::TopEntry* seg_top = nullptr;
  int32_t* seg_n = nullptr;
  uint32_t* seg_count = nullptr;
  float* seg_e = nullptr;            // [S*B][ncap] float(e): the logits stay intact
  float* seg_inv = nullptr;          // [S*B] float(1/denom), the reference's
  lsb::TopEntry* sh_top = nullptr;   // vocabulary-sharded step: local top-B'
  int32_t* sh_topn = nullptr;
  // small batches: the whole step as one cooperative launch (k_step_fused.cu)
  int fused = -1;               // -1 undecided, 0 no, 1 yes
  int fused_grid = 0, fused_rb = 0;
  uint32_t fused_slice_len = 0;  // probe slices: enough to cover the grid
  size_t fused_smem = 0;
  int fused_timing = -1;                    // LSB_FUSED_TIMING (debug), read once
  unsigned long long* fused_stamps = nullptr;  // mapped host memory [8]
  double fused_acc[5] = {};
  int fused_nacc = 0;
  // staging for lsb_step_host
  float* h_hidden = nullptr;
  double* h_scores = nullptr;
  uint8_t* h_finished = nullptr;
  int32_t* h_nhyp = nullptr;
  lsb_choice* h_choices = nullptr;
  int32_t* h_nchoices = nullptr;
  float* h_hidden_out = nullptr;
  // pipelined host-buffer steps (lsb_step_host_async): three staging slots, a
  // copy stream for the uploads, events ordering uploads and kernels
  struct AsyncSlot {
    float* hidden = nullptr;
    double* scores = nullptr;
    uint8_t* finished = nullptr;
    int32_t* n_hyp = nullptr;
    lsb_choice* choices = nullptr;
    int32_t* n_choices = nullptr;
    cudaEvent_t uploaded = nullptr, computed = nullptr, consumed = nullptr;
    cudaEvent_t uploaded2 = nullptr;  // second half of the hidden states
    bool used = false;
  } slot[3];
  static constexpr int kSlots = 3;  // an upload waits on the step three calls back
  cudaStream_t copy_stream = nullptr;   // uploads
  cudaStream_t copy_stream2 = nullptr;  // second copy engine: half of each hidden upload
  cudaStream_t down_stream = nullptr;   // read-backs
  int next_slot = 0;
  // CUDA graph of one lsb_step on fixed device buffers (lsb_batch_graph_*)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  uint64_t graph_kernels = 0;   // kernel launches recorded in the graph
  // last step (for the per-sentence views)
  lsb_state_dev last{};
  bool has_last = false;
  // profiling: one set of 6 events per step in a ring, summed on demand
  bool profile = false;
  int profile_every = 1;   // record stage events on every n-th step
  uint64_t step_count = 0;
  bool rec = false;        // this step records stage events
  std::vector<cudaEvent_t> ring;  // kRing * 6
  int ring_next = 0, ring_used = 0;
  cudaEvent_t* ev = nullptr;       // current step's 6 events
};


namespace lsb {
// K1+K2 -> K3 -> K4 of one step (profiling events 0..3): candidate sets in
// b->ids / b->n_cand, logits in b->logits.
lsb_status step_front(lsb_batch* b, const lsb_state_dev* in, int empty_is_error);
// The per-kernel arguments of one step on b's scratch (capi_step.cu).
ProbeArgs probe_args(const lsb_batch* b, const lsb_state_dev* in);
CompactArgs compact_args(const lsb_batch* b, const lsb_state_dev* in, int empty_is_error);
LogitsArgs logits_args(const lsb_batch* b, const lsb_state_dev* in);
SoftmaxArgs softmax_args(const lsb_batch* b, const lsb_state_dev* in);
ExpandArgs expand_args(const lsb_batch* b, const lsb_state_dev* in, const lsb_out_dev* out);
// Small batches: the whole lsb_step (K1..K5b) as ONE cooperative launch
// (k_step_fused.cu). *done = false (and nothing launched) when it does not
// apply to this batch / step; the caller then runs the separate kernels.
lsb_status launch_step_fused(lsb_batch* b, const lsb_state_dev* in, const lsb_out_dev* out,
                             bool* done);
// Vocabulary-sharded step: phase-2 scratch (capi_shard.cu).
lsb_status ensure_shard_scratch(lsb_batch* b, int G);
}  // namespace lsb
