// Host interface of the tensor-core question-prefill attention (prefill_tc.cu).
#pragma once

#include "rk_common.cuh"

namespace rk {

bool prefill_tc_supported(int kv_dtype, int d, int n_q, int G);

struct PrefillPlan {
  int mpad, mtiles, n_items, item_keys, n_chunks, items_per_chunk, n_units;
  size_t qs_bytes, part_bytes, item_bytes, total;
};

// work decomposition and workspace size; n_items_in > 0: caller's item table,
// else uniform 512-key items over s.  stats: per-item scoring statistics;
// with_output = false: the scores-only pass (no O partials).
PrefillPlan prefill_plan(int n_q, int hq, int hkv, int s, int n_items_in, bool stats, bool with_output = true);

// out == nullptr runs the scores-only kernel (the multi-row watershed scorer):
// item_m/item_l [n_q][hq][n_items] only, stats must be true.
int launch_prefill_tc(const float* q, int n_q, int hq, const void* k, const void* v, int s, int hkv,
                      const int64_t* q_pos, const int64_t* k_pos, const uint8_t* allowed, const int32_t* items,
                      int n_items_in, bool stats, float* out, int32_t* bad_row, void* ws, size_t ws_bytes,
                      float** item_m_out, float** item_l_out, float** stat_m_out, float** stat_l_out,
                      cudaStream_t st, bool single_pass = false);

}  // namespace rk
