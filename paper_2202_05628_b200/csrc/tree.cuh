// Internal declarations shared between libartemis translation units.
#pragma once
#include "common.cuh"

namespace artemis {

template <typename K>
int launch_build_tree(const K *codes, int64_t n_host, const int32_t *n_dev, int64_t n_cap,
                      int32_t *left, int32_t *right, int32_t *bmin, int32_t *bsize,
                      WideNode *nodes, uint4 *leaves, const uint32_t *leaf_flut,
                      const double *sigma, const int32_t *rot_index, int32_t *dup_flag,
                      cudaStream_t st);

// Stable onesweep sort of (key, value) pairs; see sort.cu.
size_t sort_workspace_bytes(int64_t n, int key_bits, int key_bytes);
template <typename K>
int sort_pairs(const K *keys_in, const uint32_t *vals_in, K *keys_out, uint32_t *vals_out,
               int64_t n, int key_bits, void *ws, size_t ws_bytes, cudaStream_t st);

// Collision resolve; see resolve.cu.
size_t resolve_workspace_bytes(int64_t n);
template <typename K>
int resolve(const K *sorted_codes, const uint32_t *sorted_idx, int64_t n_host,
            const int32_t *n_dev, const double *sigma, K *live_codes, uint32_t *winners,
            int64_t *pairs, int32_t *n_live, void *ws, size_t ws_bytes, cudaStream_t st);

struct BrickRec;
template <typename K>
int build_bricks(const K *codes, int64_t n_host, const int32_t *n_dev, int64_t n_cap,
                 const int org[3], const int dims[3], int32_t *table, BrickRec *recs,
                 int32_t *counter, int32_t *aabb, cudaStream_t st);

}  // namespace artemis
