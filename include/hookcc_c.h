/*
 * hookcc_c.h — C-ABI of the B200-native Hook-Compress connected-components
 * library (libhookcc_cuda.so).
 *
 * This is the drop-in boundary for the reference `hookcc` hot path
 * (reference: /root/reference/proj/include/hookcc/{engines,forest,graph}.hpp).
 * Plain pointers and sizes only; no C++ or torch types cross it. The C++
 * header-compatible API in the include/hookcc headers is a thin shim over these
 * entry points, and Python binds them with ctypes
 * (paper_1612_01178_b200/capi.py). Each entry point cites the reference
 * interface it replaces.
 *
 * Conventions
 *   - Every function returns an hcc_status; 0 is success. On failure a
 *     thread-local message is available from hcc_last_error().
 *   - Vertex ids on the device are uint32 (the reference uses uint64; SPEC
 *     permits 32-bit packing when n < 2^32). n >= 2^32 is rejected with
 *     HCC_EINVAL. Edge counts and offsets are uint64.
 *   - Host buffers are caller-owned; device memory is owned by the handles.
 *   - There is no CPU fallback: without a usable sm_100 device every
 *     compute entry point fails with HCC_ENODEV.
 */
#ifndef HOOKCC_C_H_
#define HOOKCC_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HCC_ABI_VERSION 4

typedef enum hcc_status {
  HCC_OK = 0,
  HCC_EINVAL = 1,    /* bad argument; reference: std::invalid_argument    */
  HCC_ENOMEM = 2,    /* device or host allocation failed                  */
  HCC_ECUDA = 3,     /* CUDA runtime error                                */
  HCC_ENCCL = 4,     /* multi-GPU transport error: no peer access between
                        the devices of hcc_create_multi (or NCCL, for the
                        multi-process binding)                            */
  HCC_ENOTSTAR = 5,  /* forest not star-shaped; reference: std::logic_error
                        from extract_labels (engines.hpp:66-70)            */
  HCC_ENODEV = 6,    /* no usable sm_100 GPU                              */
  HCC_ERANGE = 7     /* endpoint out of range; reference: check_endpoints
                        (graph.hpp:89-94) std::invalid_argument           */
} hcc_status;

/* Algorithms; names follow the reference's Algorithm enum (bench.hpp:23-33). */
typedef enum hcc_algo {
  HCC_ALGO_BASELINE = 0,     /* Fig. 1: atomic-free hook over all edges +
                                jump-until-fixpoint (engines.hpp:123-179)  */
  HCC_ALGO_BASELINE_MJ = 1,  /* atomic-free hook + Multi-Jump compress,
                                repeated to convergence (engines.hpp:183-231).
                                On B200 this is the north-star engine: a
                                topology-driven first pass, then data-driven
                                passes over a device-compacted worklist.   */
  HCC_ALGO_ATOMIC = 2,       /* single CAS-hook pass + Multi-Jump
                                (single_hook_cc, engines.hpp:295-300)      */
  HCC_ALGO_ADAPTIVE = 3      /* segmented CAS hook + Multi-Jump per segment
                                (adaptive_cc, engines.hpp:238-291)         */
} hcc_algo;

/* Option flags (hcc_opts.flags). */
#define HCC_FLAG_FULL_PASSES   0x1u /* baseline-mj: re-hook ALL edges every
                                       outer iteration (the reference's
                                       literal loop) instead of the worklist */
#define HCC_FLAG_HOST_LOOP     0x2u /* drive iterations from the host (one
                                       4-byte D2H per iteration) instead of
                                       the device-side CUDA-graph loop      */
#define HCC_FLAG_NO_GRAPH      0x4u /* launch kernels directly, no CUDA graph*/
#define HCC_FLAG_CHECK_STAR    0x8u /* verify the final forest is a star
                                       (extract_labels' debug check)        */
#define HCC_FLAG_HOOK_EVENTS   0x10u /* record CUDA events around every
                                       unrolled topology hook launch
                                       (hcc_segment_rec.hook_event_ms; each
                                       event node costs ~5 us of graph
                                       latency, so it is off by default)    */

/* Phase identifiers passed to the observer; reference Phase enum
 * (engines.hpp:84). */
#define HCC_PHASE_HOOK 0
#define HCC_PHASE_COMPRESS 1

typedef struct hcc_ctx hcc_ctx;
typedef struct hcc_graph hcc_graph;
typedef struct hcc_forest hcc_forest;

/* Observer called with the quiesced device forest after every phase
 * barrier (reference DriverOptions::phase_observer, engines.hpp:86-90).
 * Setting it forces the host-stepped loop (one sync per phase). */
typedef void (*hcc_phase_cb)(void* user, int phase, hcc_forest* pi);

typedef struct hcc_opts {
  int algo;                      /* hcc_algo                                */
  uint64_t segments;             /* adaptive: s (0 = auto, choose_segment_count
                                    of the device stats)                    */
  uint64_t first_pass_segments;  /* baseline-mj: segments of the topology
                                    pass, each followed by a compress
                                    (0 = auto)                              */
  uint64_t max_threads;          /* 0 = whole GPU; k > 0 caps the launch at
                                    k threads (1 = one thread, ascending and
                                    deterministic: the reference's
                                    workers = 1 inline path, parallel.hpp:29) */
  uint32_t flags;                /* HCC_FLAG_*                              */
  hcc_phase_cb observer;         /* optional                                */
  void* observer_user;
} hcc_opts;

/* Reference KernelCounters (forest.hpp:65-75). */
typedef struct hcc_counters {
  uint64_t hook_traversal_steps;
  uint64_t cas_failures;
  uint64_t jump_steps;
} hcc_counters;

/* Reference RunMetrics (metrics.hpp:18-41), the fields a driver fills,
 * plus B200 additions appended at the end. Times are device times. */
typedef struct hcc_metrics {
  double total_ms;          /* pi init through convergence                 */
  double hook_ms;
  double compress_ms;
  uint64_t s;               /* segments actually used                      */
  int segments_clamped;
  uint64_t outer_iterations;
  hcc_counters counters;
  uint64_t components;
  /* B200 additions */
  uint64_t n, m;
  uint64_t passes;          /* hook passes (segments + worklist passes)    */
  uint64_t edges_processed; /* edge records streamed by hook kernels       */
  uint64_t records;         /* per-phase records available (hcc_ctx_segments)*/
  int used_device_loop;     /* 1 = CUDA-graph conditional loop             */
  uint64_t kernels;         /* kernels this run launched (pi init through
                               convergence)                                */
  int star0_bitmap;         /* 1 = the star-0 bitmap fast path was used    */
  uint64_t wl_capacity;     /* records per worklist buffer (2 buffers): the
                               streaming engine sizes them to
                               max(m/8, 2n) + chunk padding, not m          */
  uint32_t wl_reruns;       /* 1 = a worklist overflowed (device flag) and
                               the run was repeated with m-sized lists      */
  uint32_t reserved_m;
} hcc_metrics;

/* One record per segment / outer iteration / worklist pass
 * (RunMetrics::segment_ms + segment_counters, metrics.hpp:30-31). */
typedef struct hcc_segment_rec {
  double hook_ms;
  double compress_ms;
  hcc_counters counters;
  uint64_t edges_in;        /* records the hook phase streamed             */
  uint64_t edges_out;       /* records appended to the next worklist       */
  double hook_event_ms;     /* hook kernel time from CUDA events recorded
                               around the launch on the launch stream (the
                               unrolled topology segments); -1 if not taken */
  /* Device timeline (globaltimer, ms since the run's first kernel started):
     first sampled block start / last block end of the hook and compress
     launches of this record; -1 if the phase did not run. */
  double hook_start_ms, hook_end_ms, compress_start_ms, compress_end_ms;
  /* Hook kernel that ran this record's pass: HCC_HOOK_KERNEL_* (0 unknown). */
  int32_t hook_kernel;
  int32_t reserved_;
} hcc_segment_rec;

#define HCC_HOOK_KERNEL_SMALL  1  /* k_hook_small: forming slot, full grid   */
#define HCC_HOOK_KERNEL_STREAM 2  /* k_hook: persistent streaming hook        */
#define HCC_HOOK_KERNEL_SUM    3  /* k_hook_sum: + shared-memory star summary */
#define HCC_HOOK_KERNEL_CAS    4  /* k_hook_cas / k_hook_sum_cas (worklist)   */
#define HCC_HOOK_KERNEL_LEGACY 5  /* k_hook_legacy / k_cas_hook                */
#define HCC_HOOK_KERNEL_SUMD   6  /* k_hook_sumd: summary-predicated lookups  */

/* Reference GraphStats (graph.hpp:33-40), computed on the device. */
typedef struct hcc_graph_stats {
  uint64_t n;
  uint64_t m_stored;
  uint64_t m_unique;
  double avg_degree;
  uint64_t max_degree;
} hcc_graph_stats;

/* ---- library / context -------------------------------------------------*/
int hcc_abi_version(void);
const char* hcc_last_error(void);
/* Number of usable devices (0 when no sm_100 GPU is visible). */
int hcc_device_count(void);
/* One context per host thread: device, stream, scratch, control block.
 * Replaces the per-call ThreadPool (engines.hpp:125-126, parallel.hpp:28). */
int hcc_create(int device, hcc_ctx** out);
int hcc_destroy(hcc_ctx* ctx);
int hcc_ctx_segments(hcc_ctx* ctx, hcc_segment_rec* out, uint64_t cap,
                     uint64_t* count);
int hcc_ctx_sm_count(hcc_ctx* ctx, int* out);

/* ---- graphs (reference Graph{n, vector<Edge>}, graph.hpp:13-31) --------*/
/* uv = interleaved u0,v0,u1,v1,... (the memory layout of vector<Edge>);
 * narrowed to u32 and endpoint-checked on the device (check_endpoints). */
int hcc_graph_from_edges_u64(hcc_ctx* ctx, const uint64_t* uv, uint64_t m,
                             uint64_t n, hcc_graph** out);
int hcc_graph_from_edges_u32(hcc_ctx* ctx, const uint32_t* uv, uint64_t m,
                             uint64_t n, hcc_graph** out);
/* CSR: row_ptr[n+1], col[row_ptr[n]]; every stored entry (u, col[j]) is one
 * edge record, in row order. (North-star addition; the reference's only CSR
 * is internal to bfs_cc, oracle.hpp:68-83.) */
int hcc_graph_from_csr(hcc_ctx* ctx, const uint64_t* row_ptr,
                       const uint32_t* col, uint64_t n, hcc_graph** out);
/* Overwrite edges [first, first+count) of an existing graph from host u32
 * pairs (endpoint-checked).  Reusing one handle for successive inputs of the
 * same size keeps its device buffer and the cached executable CUDA graph. */
int hcc_graph_assign_edges_u32(hcc_ctx* ctx, hcc_graph* g, const uint32_t* uv,
                               uint64_t first, uint64_t count);
/* Asynchronous refill: the copy (from PINNED host memory for overlap) and
 * the endpoint check run on the context's copy stream and the call returns
 * at once.  Every later call that reads the graph (hcc_cc, ...) first waits
 * for it and returns HCC_ERANGE if an endpoint was out of range.  With two
 * graph handles used alternately, the next input uploads while the current
 * one runs (the context keeps both executable CUDA graphs). */
int hcc_graph_upload_async(hcc_ctx* ctx, hcc_graph* g, const uint32_t* uv,
                           uint64_t first, uint64_t count);
/* Device generators. spec: "grid:RxC" (identical to generators.hpp:71-87),
 * "rmatx:scale=K,ef=F[,seed=S][,a=..,b=..,c=..,d=..]" and
 * "erx:n=N,m=M[,seed=S]" (counter-based twins of generators.hpp:14-62,
 * restated bit-exactly on the CPU in oracle/). */
int hcc_graph_generate(hcc_ctx* ctx, const char* spec, uint64_t default_seed,
                       hcc_graph** out);
int hcc_graph_info(const hcc_graph* g, uint64_t* n, uint64_t* m);
/* Copy the packed device edges (u32 pairs) to the host. */
int hcc_graph_download_u32(hcc_ctx* ctx, const hcc_graph* g, uint32_t* uv,
                           uint64_t first, uint64_t count);
/* FNV-style order-dependent checksum of the edge stream (size-independent
 * generator parity). */
int hcc_graph_checksum(hcc_ctx* ctx, const hcc_graph* g, uint64_t* out);
/* Device compute_stats (graph.hpp:43-68): radix sort + unique. */
int hcc_graph_compute_stats(hcc_ctx* ctx, const hcc_graph* g,
                            hcc_graph_stats* out);
int hcc_graph_free(hcc_graph* g);

/* ---- the CC entry point -------------------------------------------------
 * Replaces baseline_cc / baseline_mj_cc / single_hook_cc / adaptive_cc and
 * their *_into variants (engines.hpp:123-338). `pi` may be NULL (the
 * context's scratch forest is used) or a caller forest of size n (the
 * in-place *_into contract: reset inside, final forest left in it).
 * labels_out (host, n entries, may be NULL) receives the canonical labels:
 * label(v) = minimum vertex id of v's component. */
int hcc_cc(hcc_ctx* ctx, const hcc_graph* g, const hcc_opts* opts,
           hcc_forest* pi, uint32_t* labels_out, hcc_metrics* out);
/* Same, labels widened to u64 (ComponentLabeling::label, engines.hpp:19-24). */
int hcc_cc_u64(hcc_ctx* ctx, const hcc_graph* g, const hcc_opts* opts,
               hcc_forest* pi, uint64_t* labels_out, hcc_metrics* out);
/* Reference choose_segment_count (engines.hpp:35-41). */
uint64_t hcc_choose_segment_count(const hcc_graph_stats* stats);

/* ---- parent forest (reference ParentForest, forest.hpp:19-63) -----------
 * A device-resident u32 pi. Element operations run as device kernels on
 * the calling thread's per-thread stream, so concurrent host threads really
 * race on the device (test_forest.cpp:185-211). */
int hcc_forest_create(hcc_ctx* ctx, uint64_t n, hcc_forest** out);
int hcc_forest_free(hcc_forest* f);
int hcc_forest_size(const hcc_forest* f, uint64_t* n);
int hcc_forest_reset(hcc_forest* f);                        /* forest.hpp:25 */
int hcc_forest_download_u64(hcc_forest* f, uint64_t* out); /* snapshot 45-49*/
int hcc_forest_download_u32(hcc_forest* f, uint32_t* out);
int hcc_forest_upload_u64(hcc_forest* f, const uint64_t* in);
int hcc_forest_load(hcc_forest* f, uint64_t v, uint64_t* out);   /* 30-32 */
int hcc_forest_store(hcc_forest* f, uint64_t v, uint64_t p);     /* 34-36 */
/* CAS; on failure *expected receives the observed value (39-43). */
int hcc_forest_cas(hcc_forest* f, uint64_t v, uint64_t* expected,
                   uint64_t desired, int* ok);
/* Per-element kernels of Figs. 2-3 (forest.hpp:83-136). */
int hcc_forest_hook(hcc_forest* f, uint64_t u, uint64_t v, int* changed);
int hcc_forest_jump(hcc_forest* f, uint64_t v, int* changed);
int hcc_forest_atomic_hook(hcc_forest* f, uint64_t u, uint64_t v,
                           hcc_counters* c);
int hcc_forest_multi_jump(hcc_forest* f, uint64_t v, hcc_counters* c);
/* One multi_jump per vertex over [begin,end), ascending (descending != 0:
 * descending) by one device thread: the schedule-order pass of
 * test_forest.cpp:150-169. */
int hcc_forest_multi_jump_range(hcc_forest* f, uint64_t begin, uint64_t end,
                                int descending, hcc_counters* c);
int hcc_forest_is_star(hcc_forest* f, int* out);           /* 140-146 */
/* max over v of (pi(v) > v): the bound invariant (SPEC: pi(v) <= v). */
int hcc_forest_check_bound(hcc_forest* f, int* ok);

/* ---- device-side verification -------------------------------
 * Size-independent checks of a finished forest against its graph:
 *   bad_edges    = #edges (u, v) with pi(u) != pi(v)   (labels split an edge)
 *   bad_vertices = #v with pi(v) > v or pi(pi(v)) != pi(v)  (not canonical
 *                  min-rooted stars)
 * Both are 0 for a correct min-canonical labeling. */
int hcc_forest_verify(hcc_ctx* ctx, const hcc_graph* g, hcc_forest* f,
                      uint64_t* bad_edges, uint64_t* bad_vertices);
/* partitions_equal (oracle.hpp:112-126) on the device: host label arrays a, b
 * of n entries induce the same partition (radix sort of (a, b) pairs, then
 * #distinct pairs == #distinct a == #distinct b).  exact = (a == b). */
int hcc_labels_compare(hcc_ctx* ctx, const uint32_t* a, const uint32_t* b,
                       uint64_t n, int* partition_equal, int* exact);

/* ---- multi-GPU merge primitives (north-star (5), SURVEY 8e shape 3) ------
 * After a local CC on an edge shard, a rank exports its star forest as
 *   bits  : uint32[ceil(n/32)], bit v = (pi(v) == 0 && v != 0)
 *   pairs : uint32[2*cap], (v, pi(v)) for every v with pi(v) not in {v, 0}
 * into DEVICE buffers (e.g. torch CUDA tensors), so the payload goes to NCCL
 * without a host hop.  After the exchange, hcc_rehook re-hooks the OR of
 * the remote bitmaps (as (v, 0) edges) and the concatenated remote pairs as
 * edges into the local forest with the worklist engine, until convergence.
 * The union of all shards' relations is then in every rank's forest, so the
 * labels are the global min-canonical labels. */
int hcc_forest_export(hcc_ctx* ctx, hcc_forest* f, uint32_t* dev_bits,
                      uint32_t* dev_pairs, uint64_t cap, uint64_t* count);
/* dev_bits_or may be NULL; dev_pairs holds `count` (v, parent) u32 pairs. */
int hcc_rehook(hcc_ctx* ctx, hcc_forest* f, const uint32_t* dev_bits_or,
               const uint32_t* dev_pairs, uint64_t count, hcc_metrics* out);
/* As hcc_rehook, with the bitmap given as the all-gathered rows of every
 * rank (row r at dev_bit_rows + r * row_stride_words): the kernel ORs all
 * rows except skip_row (the caller's own; ~0 for none) while decoding. */
int hcc_rehook_rows(hcc_ctx* ctx, hcc_forest* f, const uint32_t* dev_bit_rows,
                    uint64_t nrows, uint64_t row_stride_words, uint64_t skip_row,
                    const uint32_t* dev_pairs, uint64_t count, hcc_metrics* out);
/* Device generator of one shard: edges [first, first+count) of `spec`
 * (partition_edges(m, world) gives the rank's range). */
int hcc_graph_generate_range(hcc_ctx* ctx, const char* spec,
                             uint64_t default_seed, uint64_t first,
                             uint64_t count, hcc_graph** out);

/* ---- multi-GPU in one process (north-star (5); reference entry
 * points engines.hpp:316-338 run with a device list) -----------------------
 * hcc_create_multi builds a context with one shard per entry of `devices`
 * (a device may repeat: its shards then share it; peer access is enabled
 * between every pair of distinct devices, HCC_ENCCL if unavailable).  On
 * such a context every graph entry point (hcc_graph_from_edges_*,
 * hcc_graph_from_csr, hcc_graph_generate[_range], upload/assign/download,
 * checksum, compute_stats) works on an edge-partitioned graph: shard r =
 * partition_edges(m, ndev)[r] (engines.hpp:43-58) on devices[r].  hcc_cc /
 * hcc_cc_u64 then run every shard's local CC concurrently (one host thread
 * per shard), export each local forest (bitmap of pi(v) == 0 + sparse
 * (v, pi(v)) pairs), and merge with one kernel per shard that reads the
 * peers' exports in place over NVLink (P2P) and re-hooks what its forest
 * lacks: no NCCL, no staging copy, no host read of the payload sizes.
 * The labels (and a caller forest `pi`, which must live on devices[0]) are
 * the global min-canonical labels.  metrics.total_ms = max over shards of
 * (local CC + merge) device time; per-shard detail: hcc_ctx_shard_metrics.
 * hcc_forest_create on the context allocates on devices[0]. */
typedef struct hcc_shard_metrics {
  double total_ms;          /* local_ms + merge_ms (this shard's device time) */
  double local_ms;          /* local CC, pi init through convergence          */
  double merge_ms;          /* NVLink gather + re-hook passes                 */
  double span_ms;           /* first to last event of the shard's call,
                               including the host hand-off between phases    */
  uint64_t pairs_exported;  /* sparse pairs this shard exported              */
  uint64_t records_merged;  /* remote relations this shard re-hooked         */
  uint64_t rehook_passes;
  uint64_t bitmap_bytes;    /* exported bitmap size                          */
  uint64_t roots_linked;    /* local roots the gather linked to 0 in place
                               (peers' star-of-0 members this shard lacked) */
  int device;
  int peer_access;          /* 1: exports read over P2P                      */
} hcc_shard_metrics;

int hcc_create_multi(const int* devices, int ndev, hcc_ctx** out);
/* 1 for a single-device context. */
int hcc_ctx_shards(hcc_ctx* ctx, int* count);
/* Per-shard metrics of the last hcc_cc on a multi-device context. */
int hcc_ctx_shard_metrics(hcc_ctx* ctx, hcc_shard_metrics* out, uint64_t cap,
                          uint64_t* count);

/* ---- multi-process merge over CUDA IPC (one process per GPU, e.g. under
 * torchrun; paper_1612_01178_b200/distributed.py binds it) -----------------
 * Per rank, once: hcc_peer_open allocates the export arena (pair count,
 * bitmap, `cap` pairs) and an interprocess event and writes a handle blob of
 * HCC_PEER_HANDLE_BYTES; the caller exchanges the blobs (any transport) and
 * passes all of them, in rank order, to hcc_peer_connect, which maps the
 * peers' arenas (lazy peer access).  Per run, after the local CC into `f`:
 *   hcc_peer_export(ctx, f)   k_export into the arena + event record (async)
 *   <host barrier across ranks: every record precedes every wait>
 *   hcc_peer_merge(ctx, f, ..) device waits on the peers' events, then
 *                             k_merge_gather reads their arenas over NVLink
 *                             and the worklist engine re-hooks; synchronous.
 * *overflow = 1 when some rank exported more pairs than its cap: the merge
 * is then incomplete (but every relation applied is true) -- reopen with a
 * larger cap, reconnect, export and merge again. */
#define HCC_PEER_HANDLE_BYTES 256
int hcc_peer_open(hcc_ctx* ctx, uint64_t n, uint64_t cap, int rank, int world,
                  void* handle_out);
int hcc_peer_connect(hcc_ctx* ctx, const void* handles);
int hcc_peer_export(hcc_ctx* ctx, hcc_forest* f);
/* metrics: total_ms = export start to merge end (device), edges_processed =
 * remote relations re-hooked, m = pairs this rank exported, components. */
int hcc_peer_merge(hcc_ctx* ctx, hcc_forest* f, hcc_metrics* out, int* overflow);
/* Unmap the peers' arenas (keeps this rank's).  Every rank must disconnect
 * (then meet at a barrier) before any rank closes or reopens, which frees
 * the arena its peers map. */
int hcc_peer_disconnect(hcc_ctx* ctx);
int hcc_peer_close(hcc_ctx* ctx);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* HOOKCC_C_H_ */
