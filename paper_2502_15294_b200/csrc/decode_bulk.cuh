// Host-side interface of the pipelined (cp.async.bulk + mbarrier) decode kernel.
#pragma once

#include "rk_common.cuh"

namespace rk {

struct BulkParams {
  const float* q;          // [B][Hq][D]
  const void* k;           // cache base, dialogue b at + b*batch_stride elements
  const void* v;
  int64_t batch_stride;
  const int32_t* seq_len;  // [B] cached keys before this token
  void* k_new;             // [B][HKV][D] appended row (or null)
  void* v_new;
  const int32_t* items;    // [B][items_stride][3] (lo, hi, bin) or null
  const int32_t* n_items;
  int items_stride;
  int B, hq, nsplit;       // nsplit = partial slots per (dialogue, head)
  float scale_log2;
  float* part_m;           // [B][Hq][nsplit]
  float* part_l;
  float* part_acc;         // [B][Hq][nsplit][D]
};

bool bulk_supported(int kv_dtype, int d, int hkv, int G);
int bulk_splits(int batch, int max_seq_len, int hkv);
int launch_decode_mma(int d, int hkv, int G, dim3 grid, const BulkParams& p, cudaStream_t st, bool pdl,
                      cudaError_t* e);
int launch_decode_bulk(int kv_dtype, int d, int hkv, int G, int nsplit, const BulkParams& p, float* out,
                       int32_t* advance, cudaStream_t st, bool pdl);

// small-batch cluster decode (decode_cluster.cu): cluster size, 0 = not applicable
// multiwave: beyond one wave of (dialogue, kv-head) pairs, one CTA per pair in several waves
int cluster_decode_size(int kv_dtype, int d, int hkv, int G, int batch, int max_len, int64_t batch_stride,
                        bool multiwave = false);
int launch_decode_cluster(int C, int kv_dtype, const float* q, int batch, int hq, int d, void* k_cache,
                          void* v_cache, int hkv, int64_t batch_stride, const int32_t* seq_len, int max_len,
                          const void* k_new, const void* v_new, float* out, cudaStream_t st,
                          const int32_t* active = nullptr);

}  // namespace rk
