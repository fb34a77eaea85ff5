// Multi-GPU edge-partitioned CC (north-star (5)).
// Placeholder entry points until the NCCL merge lands; they fail loudly.
#include <string>

#include "hookcc_c.h"

extern "C" {

int hcc_nccl_unique_id_size(void) { return 128; }

int hcc_nccl_get_unique_id(void* id_out) {
  (void)id_out;
  return HCC_ENCCL;
}

int hcc_comm_init(hcc_ctx* ctx, int world, int rank, const void* id) {
  (void)ctx;
  (void)world;
  (void)rank;
  (void)id;
  return HCC_ENCCL;
}

int hcc_comm_destroy(hcc_ctx* ctx) {
  (void)ctx;
  return HCC_OK;
}

int hcc_cc_distributed(hcc_ctx* ctx, const hcc_graph* shard, uint64_t n,
                       const hcc_opts* opts, uint32_t* labels_out,
                       hcc_metrics* out) {
  (void)ctx;
  (void)shard;
  (void)n;
  (void)opts;
  (void)labels_out;
  (void)out;
  return HCC_ENCCL;
}

}  // extern "C"
