// k_step.cuh -- kernel argument blocks and launch helpers shared by the
// fused step (capi_step.cu) and the per-stage entry points (capi_stages.cu).
#pragma once

#include "lsb_internal.cuh"

namespace lsb {

struct TopEntry {
  float p;     // probability
  uint32_t r;  // candidate column
};

// K1+K2: hash + probe + threshold hit counting.
struct ProbeArgs {
  IndexView ix;
  const float* hidden;      // [S*B][d]
  const uint8_t* finished;  // [S*B] or null (all live)
  const int32_t* n_hyp;     // [S] or null (all B)
  int S, B, t;
  uint32_t slice_len;       // counters per CTA (multiple of 64)
  int counter_bytes;        // 1 or 2 (byte counters)
  int levels;               // >= 0: bit-sliced counting with t-1 levels (t <= 8); -1: counters
  uint32_t* qcodes;         // [S*B][W]
  uint32_t* bitmap;         // [S][nwords]
  uint32_t nwords;
  uint32_t* err;
};

// K3: bitmap (threshold survivors) U [0,T) U specials -> ascending ids.
struct CompactArgs {
  const uint32_t* bitmap_in;  // [S][nwords] or null (ids-from-list mode)
  uint32_t* bitmap_clear;     // cleared after reading (may equal bitmap_in)
  uint32_t nwords, V, T;
  int mode;                   // 0 threshold, 1 all (t == 0), 2 full vocab
  const uint32_t* specials;   // sorted unique, < V
  int nspec;
  uint32_t* ids;              // [S][ncap]
  size_t ncap;
  uint32_t* n_cand;           // [S]
  uint32_t* prov;             // [S][3]
  int empty_is_error;         // decode(): an empty set with live rows throws
  const int32_t* n_hyp;       // live check for the empty-set error (may be null)
  const uint8_t* finished;
  int B;
  uint32_t* err;
};

// K4: logits = H . E[ids]^T + bias[ids].
struct LogitsArgs {
  const float* H;          // [R_total][d]
  int d, R_total, Bsent;   // rows per sentence for the per-sentence jobs
  const float* E;          // [V][d]
  const float* bias;       // [V] or null
  uint32_t n_shared;       // columns [0, n_shared) use identity ids
  const uint32_t* ids;     // [S][ncap]
  size_t ncap;
  const uint32_t* n_cand;  // [S]
  int S, G, X;
  int jobs_shared, ctiles_shared;
  float* out;              // [R_total][ldo]
  size_t ldo;
  int skip_shared;         // the shared block was scored elsewhere (tensor cores)
  const float* tc_A;       // FAST: E[0, n_shared) pre-tiled for tcgen05 (or null)
  float* tc_H;             // FAST: scratch for the per-step tiled H
  int tc_N;                // rows per tcgen05 tile the scratch was sized for
  unsigned long long x2_negzero, x2_one;  // (-0,-0) / (1,1) f32x2 operands, set by launch
};

// K5a: row softmax + per-row top-B by (p desc, column asc).
struct SoftmaxArgs {
  float* logits;           // [R_total][ldl], overwritten with exp / probs
  size_t ldl;
  int R_total, Bsent, topB;
  const uint32_t* n_cand;  // [S], or null: every row has n_const columns
  uint32_t n_const;
  int probs_in;            // 1: logits already hold probabilities (selection only)
  const uint8_t* finished; // may be null
  const int32_t* n_hyp;    // may be null
  int keep_probs;
  TopEntry* top;           // [R_total][topB]
  int32_t* top_n;          // [R_total]
  uint32_t* err;
  int seq_denominator;     // test hook (LSB_SEQ_DENOM=1): always the sequential
                           // denominator (softmax_denom.cuh)
};

// K5b: per-sentence top-B merge by (score desc, beam asc, word asc) +
// hidden-state reorder.
struct ExpandArgs {
  int S, Bsent, topB;
  const TopEntry* top;
  const int32_t* top_n;
  const double* scores;     // [S][Bsent] cumulative, per hypothesis
  const uint8_t* finished;  // [S][Bsent] or null
  const int32_t* n_hyp;     // [S] or null
  const uint32_t* live_ids; // [S][Bsent] beam id of live row i, or null (= i)
  const uint32_t* ids;      // [S][ncap]
  size_t ncap;
  uint32_t n_shared;
  const uint32_t* id_map;   // optional global id map (stage API), else ids
  const float* hidden;      // [S][Bsent][d] parent rows by hypothesis, or null
  int d;
  float* hidden_out;        // [S][Bsent][d] or null
  lsb_choice* choices;      // [S][Bsent]
  int32_t* n_choices;       // [S]
  int frozen_mode;          // 0 = frozen from finished flags, 1 = explicit list
  const double* fz_score;   // explicit frozen list (stage API)
  const uint32_t* fz_beam;
  int nfrozen;
};

lsb_status launch_probe(lsb_ctx* ctx, const ProbeArgs& a);
// dynamic shared memory of one probe_row CTA (k_probe_count)
size_t probe_smem_bytes(const ProbeArgs& a);
// Band-split K1+K2 for few rows (k_step.cu): grid (rows, G band groups),
// 16-bit hit counters cnt[rows][cnt_words] in global memory, zero on entry
// and left zero (self-cleaning), arrive[rows] zero likewise.
lsb_status launch_probe_split(lsb_ctx* ctx, const ProbeArgs& a, int G, uint32_t* cnt,
                              uint32_t cnt_words, uint32_t* arrive);
lsb_status launch_compact(lsb_ctx* ctx, const CompactArgs& a, int S);
lsb_status launch_logits(lsb_ctx* ctx, LogitsArgs a, lsb_mode mode, int target_ctas);
// PARITY one-lane-per-thread kernel (k_logits_ln.cu): applicability and launch.
bool logits_ln_applies(const LogitsArgs& a);
lsb_status launch_logits_ln(lsb_ctx* ctx, const LogitsArgs& a, int target_ctas);
// Tensor-core (tcgen05, 3xTF32) logits for rows x identity columns
// [col0, col0 + ncols) of E; FAST mode only.
lsb_status launch_tc_logits(lsb_ctx* ctx, const float* H, int rows, const float* E,
                            const float* bias, int d, uint32_t col0, uint32_t ncols, float* out,
                            size_t ldo, uint32_t out_col0);
// Pre-tiled variant (operands from launch_tf32_tile with R = 128 / N).
lsb_status launch_tc_logits_tiled(lsb_ctx* ctx, const float* A_tiled, const float* H_tiled,
                                  int N, int rows, int d, const float* bias, uint32_t col0,
                                  uint32_t ncols, float* out, size_t ldo, uint32_t out_col0);
lsb_status launch_tf32_tile(lsb_ctx* ctx, const float* src, int nrows, int d, int R, float* out);
size_t tf32_tiled_floats(int nrows, int d, int R);
int tc_rows_per_tile(lsb_ctx* ctx, int rows, uint32_t ncols);
constexpr int kTcMinRows = 64;  // rows sharing a column block before tensor cores pay
lsb_status launch_softmax(lsb_ctx* ctx, const SoftmaxArgs& a);
// K5a for long rows (k_softmax_seg.cu): P segments per row, one CTA each.
constexpr int kSegMaxP = 64;
struct SegArgs {
  SoftmaxArgs sa;
  int P;
  uint32_t seglen;
  float* part_max;    // [R][P]
  double* part_sum;   // [R][P] compensated segment sums: hi ...
  double* part_c;     // [R][P] ... + compensation (hi + c = the exact sum up to 2^-60)
  double* part_b;     // [R][P] sum_k min(e_k, 2^-52): bounds the sequential sum's error
  TopEntry* seg_top;  // [R][P][topB]
  int32_t* seg_n;     // [R][P]
  uint32_t* count;    // [R], zero between steps (self-resetting)
  float* e_out;       // [R][ldl] float(e) (the logits stay intact for the denominator)
  float* inv;         // [R] float(1/denom), certified / sequential (k_seg_denom)
};
int seg_count(lsb_ctx* ctx, int R, uint32_t n, int B);
lsb_status launch_softmax_seg(lsb_ctx* ctx, const SegArgs& g);
lsb_status launch_expand(lsb_ctx* ctx, const ExpandArgs& a);
// dynamic shared memory of one expand_sentence CTA (rank path)
size_t expand_smem_bytes(const ExpandArgs& a);
// Fused K5a+K5b (one launch; see k_select.cu) when select_fused_applies().
bool select_fused_applies(const SoftmaxArgs& sa, const ExpandArgs& ea);
// K5a with one warp per row (rows <= 32*48 candidates in registers).
lsb_status launch_softmax_warp(lsb_ctx* ctx, const SoftmaxArgs& sa, uint32_t max_n);
lsb_status launch_select_fused(lsb_ctx* ctx, const SoftmaxArgs& sa, const ExpandArgs& ea,
                               uint32_t max_n, uint32_t* arrive);

// Bitmap helpers for the stage API.
lsb_status launch_bitmap_from_dense(lsb_ctx* ctx, const int32_t* L, int B, uint32_t V, int t,
                                    uint32_t* bitmap);
lsb_status launch_bitmap_from_ids(lsb_ctx* ctx, const uint32_t* ids, uint32_t n,
                                  uint32_t* bitmap);
lsb_status launch_gather(lsb_ctx* ctx, const float* E, int d, const uint32_t* ids, uint32_t n,
                         float* out);

// Chooses the row-group size RB for a sentence of B rows (see k_step.cu).
int choose_rb(int B);

}  // namespace lsb
