// Multi-device contexts (hcc_create_multi): host side.  Kernels in
// hcc_multi.cu; handles and shared helpers in hcc_host.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "hcc_host.cuh"

using namespace hcc::host;

// ===========================================================================
// Multi-device contexts: edge-partitioned CC in one process (north-star (5),
// SURVEY.md §8e).  hcc_create_multi(devices, ndev) builds one sub-context
// per shard (a device may appear several times: several shards share it).
// Graphs created on such a context are split by partition_edges(m, ndev)
// (engines.hpp:43-58), shard r on subs[r].  hcc_cc on it:
//   1. local CC    every shard runs the single-GPU engine (its own stream,
//                  one host thread per shard) into a full-size local forest,
//                  then exports it (k_export: bitmap of pi(v) == 0 plus
//                  sparse (v, pi(v)) pairs) into its merge buffers;
//   2. merge       every shard waits on the others' export events (device
//                  waits, cross-device) and runs k_merge_gather, which reads
//                  the peers' export buffers straight over NVLink (P2P) and
//                  appends the relations its own forest lacks to its
//                  worklist; the worklist engine re-hooks them;
//   3. labels      every shard now holds the global min-canonical forest;
//                  shard 0's is returned.
// A pair list that overflowed its buffer (the count is read on the device,
// the host checks it after the round) grows the buffer and repeats steps
// 1b-2: the relations already merged are true ones, so a repeat is exact.


namespace {

// fn(r) on one host thread per shard; the first failure's message is moved
// to the calling thread (g_err is thread-local).
// HCC_MULTI_SERIAL=1 runs the shards one after another on one thread: on a
// single GPU hosting every shard, each shard's phases then run alone, which
// is the per-rank cost an N-GPU run would see (tools/scale_model.py).
int for_shards(int G, const std::function<int(int)>& fn) {
  std::vector<int> rc(G, 0);
  std::vector<std::string> msg(G);
  std::vector<std::thread> th;
  th.reserve(G);
  static const bool serial = std::getenv("HCC_MULTI_SERIAL") && std::atoi(std::getenv("HCC_MULTI_SERIAL"));
  for (int r = 0; r < G; ++r) {
    th.emplace_back([&, r] {
      try {
        rc[r] = fn(r);
      } catch (const CudaFail& f) {
        rc[r] = f.code;
      } catch (const std::bad_alloc&) {
        rc[r] = fail(HCC_ENOMEM, "host allocation failed");
      } catch (const std::exception& e) {
        rc[r] = fail(HCC_ECUDA, e.what());
      }
      if (rc[r]) msg[r] = g_err;
    });
    if (serial) th.back().join();
  }
  for (std::thread& t : th)
    if (t.joinable()) t.join();
  for (int r = 0; r < G; ++r)
    if (rc[r]) {
      g_err = msg[r];
      return rc[r];
    }
  return HCC_OK;
}

// Merge buffers of every shard for n vertices and pair capacity >= cap.
void ensure_merge(hcc_ctx* c, u64 n, u64 cap) {
  const int G = (int)c->subs.size();
  if ((int)c->merge.size() != G) c->merge.resize(G);
  const u64 nwords = (n + 31) / 32;
  bool dirty = false;
  for (int r = 0; r < G; ++r) {
    MergeShard& ms = c->merge[r];
    hcc_ctx* sc = c->subs[r];
    HCC_CUDA(cudaSetDevice(sc->dev));
    if (!ms.cnt) {
      HCC_CUDA(cudaMalloc(&ms.cnt, sizeof(u64)));
      HCC_CUDA(cudaMalloc(&ms.tab, sizeof(PeerTab)));
      HCC_CUDA(cudaEventCreateWithFlags(&ms.ev_exp, cudaEventDisableTiming));
      HCC_CUDA(cudaEventCreate(&ms.ev_t0));
      HCC_CUDA(cudaEventCreate(&ms.ev_m0));
      HCC_CUDA(cudaEventCreate(&ms.ev_t1));
      dirty = true;
    }
    if (ms.bits_words < nwords) {
      cudaFree(ms.bits);
      ms.bits = nullptr;
      HCC_CUDA(cudaMalloc(&ms.bits, std::max<u64>(nwords, 1) * sizeof(u32)));
      ms.bits_words = nwords;
      dirty = true;
    }
    if (ms.cap < cap) {
      cudaFree(ms.pairs);
      ms.pairs = nullptr;
      ms.cap = 0;
      HCC_CUDA(cudaMalloc(&ms.pairs, cap * sizeof(uint2)));
      ms.cap = cap;
      dirty = true;
    }
  }
  if (!dirty) return;
  PeerTab t{};
  t.npeers = (u32)G;
  for (int r = 0; r < G; ++r) {
    t.bits[r] = c->merge[r].bits;
    t.pairs[r] = c->merge[r].pairs;
    t.count[r] = c->merge[r].cnt;
    t.cap[r] = c->merge[r].cap;
  }
  for (int r = 0; r < G; ++r) {
    HCC_CUDA(cudaSetDevice(c->subs[r]->dev));
    HCC_CUDA(cudaMemcpy(c->merge[r].tab, &t, sizeof(PeerTab), cudaMemcpyHostToDevice));
  }
  HCC_CUDA(cudaSetDevice(c->dev));
}

// Shard r: export its forest into its merge buffers (stream-ordered after
// its local CC) and record the export event the peers wait on.
void enqueue_export(hcc_ctx* sc, MergeShard& ms, const hcc_forest* f, bool peers) {
  HCC_CUDA(cudaMemsetAsync(ms.cnt, 0, sizeof(u64), sc->stream));
  const u64 nwords = (f->n + 31) / 32;
  if (f->n && peers)  // (one shard: nobody reads it, the merge is the identity)
    k_export<<<grid_for(nwords * 32, 256, (u64)sc->sms * 32), 256, 0, sc->stream>>>(
        f->d_pi, f->n, ms.bits, ms.pairs, ms.cap, ms.cnt);
  HCC_CUDA(cudaGetLastError());
  HCC_CUDA(cudaEventRecord(ms.ev_exp, sc->stream));
}

// Shard r: wait for every peer's export, gather the remote relations over
// NVLink into the worklist, re-hook until convergence.
void merge_shard(hcc_ctx* c, int r, hcc_forest* f, u64 records_cap) {
  hcc_ctx* sc = c->subs[r];
  MergeShard& ms = c->merge[r];
  const int G = (int)c->subs.size();
  const u64 n = f->n;
  for (int s = 0; s < G; ++s)
    if (s != r) HCC_CUDA(cudaStreamWaitEvent(sc->stream, c->merge[s].ev_exp, 0));
  ensure_wl(sc, records_cap);
  HCC_CUDA(cudaEventRecord(ms.ev_m0, sc->stream));
  k_begin<<<1, 1, 0, sc->stream>>>(sc->d_ctrl, sc->d_recs, 1);
  if (G > 1) {
    k_merge_gather<<<std::max<unsigned>(1u, (unsigned)sc->sms * 8u), 256, 0, sc->stream>>>(
        ms.tab, (u32)r, f->d_pi, n, sc->wl[0], &sc->d_ctrl->wl_count[0], sc->wl_cap,
        &sc->d_ctrl->err, &sc->d_ctrl->dirty, &sc->d_ctrl->merged_links);
    HCC_CUDA(cudaGetLastError());
    enqueue_rehook(sc, f->d_pi, n);
  }
  HCC_CUDA(cudaEventRecord(ms.ev_t1, sc->stream));
  // components (metrics only, after the timed region)
  if (r == 0)
    k_count_roots<<<grid_for(n, 256, (u64)sc->sms * 16), 256, 0, sc->stream>>>(f->d_pi, n,
                                                                              sc->d_ctrl);
  HCC_CUDA(cudaGetLastError());
  HCC_CUDA(cudaMemcpyAsync(sc->h_ctrl, sc->d_ctrl, sizeof(DevCtrl), cudaMemcpyDeviceToHost,
                           sc->stream));
  HCC_CUDA(cudaMemcpyAsync(sc->h_recs, sc->d_recs, sizeof(DevRec), cudaMemcpyDeviceToHost,
                           sc->stream));
  HCC_CUDA(cudaStreamSynchronize(sc->stream));
  if (sc->h_ctrl->err & 4u) throw CudaFail{fail(HCC_ECUDA, "merge worklist overflow")};
  float ms_merge = 0.f, ms_total = 0.f;
  HCC_CUDA(cudaEventElapsedTime(&ms_merge, ms.ev_m0, ms.ev_t1));
  HCC_CUDA(cudaEventElapsedTime(&ms_total, ms.ev_t0, ms.ev_t1));
  ms.merge_ms += ms_merge;
  ms.total_ms = ms_total;
  ms.passes += sc->h_ctrl->passes;
  ms.records += sc->h_recs[0].edges_in;
  ms.linked += sc->h_ctrl->merged_links;
}

}  // namespace

namespace hcc {
namespace host {

int multi_from_edges(hcc_ctx* c, const void* uv, bool wide, u64 m, u64 n,
                            hcc_graph** out) {
  const int G = (int)c->subs.size();
  hcc_graph* g = new hcc_graph;
  g->ctx = c;
  g->n = n;
  g->m = m;
  g->bounds = uniform_bounds(m, (u64)G);
  g->shards.assign(G, nullptr);
  const int rc = for_shards(G, [&](int r) -> int {
    const u64 b = g->bounds[r], k = g->bounds[r + 1] - b;
    const int st = wide ? hcc_graph_from_edges_u64(c->subs[r], static_cast<const uint64_t*>(uv) + 2 * b,
                                                   k, n, &g->shards[r])
                        : hcc_graph_from_edges_u32(c->subs[r], static_cast<const uint32_t*>(uv) + 2 * b,
                                                   k, n, &g->shards[r]);
    if (!st) g->shards[r]->first = b;
    return st;
  });
  if (rc) {
    for (hcc_graph*& sh : g->shards)
      if (!sh) sh = new hcc_graph;  // placeholders so free() sees a sharded graph
    hcc_graph_free(g);
    return rc;
  }
  *out = g;
  return HCC_OK;
}

int multi_generate(hcc_ctx* c, const char* spec, u64 seed, u64 n, u64 first, u64 count,
                          hcc_graph** out) {
  const int G = (int)c->subs.size();
  hcc_graph* g = new hcc_graph;
  g->ctx = c;
  g->n = n;
  g->m = count;
  g->first = first;
  g->bounds = uniform_bounds(count, (u64)G);
  g->shards.assign(G, nullptr);
  const int rc = for_shards(G, [&](int r) -> int {
    const u64 b = g->bounds[r], k = g->bounds[r + 1] - b;
    return hcc_graph_generate_range(c->subs[r], spec, seed, first + b, k, &g->shards[r]);
  });
  if (rc) {
    for (hcc_graph*& sh : g->shards)
      if (!sh) sh = new hcc_graph;
    hcc_graph_free(g);
    return rc;
  }
  *out = g;
  return HCC_OK;
}

// op 0: asynchronous upload, 1: synchronous assign, 2: download.  The range
// [first, first+count) is split at the shard boundaries.
int multi_range_io(hcc_ctx* c, hcc_graph* g, uint32_t* uv, u64 first, u64 count, int op) {
  for (size_t r = 0; r < g->shards.size(); ++r) {
    const u64 b = std::max(first, g->bounds[r]);
    const u64 e = std::min(first + count, g->bounds[r + 1]);
    if (b >= e) continue;
    uint32_t* src = uv + 2 * (b - first);
    const u64 lo = b - g->bounds[r];
    int st;
    if (op == 2)
      st = hcc_graph_download_u32(c->subs[r], g->shards[r], src, lo, e - b);
    else
      st = hcc_graph_upload_async(c->subs[r], g->shards[r], src, lo, e - b);
    if (st) return st;
  }
  g->has_stats = false;
  if (op == 1) return graph_ready(g);
  return HCC_OK;
}

// compute_stats of a sharded graph: the shards are copied (peer copies)
// into one temporary graph on the first device.  Off the hot path.
int multi_stats(hcc_ctx* c, const hcc_graph* g, hcc_graph_stats* out) {
  if (int r = graph_ready(g)) return r;
  hcc_graph tmp;
  tmp.ctx = c;
  tmp.n = g->n;
  tmp.m = g->m;
  int rc = HCC_OK;
  try {
    HCC_CUDA(cudaSetDevice(c->dev));
    HCC_CUDA(cudaMalloc(&tmp.d_edges, std::max<u64>(g->m, 2) * sizeof(uint2)));
    for (size_t r = 0; r < g->shards.size(); ++r)
      if (g->shards[r]->m)
        HCC_CUDA(cudaMemcpyPeer(tmp.d_edges + g->bounds[r], c->dev, g->shards[r]->d_edges,
                                c->subs[r]->dev, g->shards[r]->m * sizeof(uint2)));
    rc = compute_stats_dev(c, &tmp);
    if (!rc) *out = tmp.stats;
  } catch (const CudaFail& f) {
    rc = f.code;
  }
  cudaFree(tmp.d_edges);
  tmp.d_edges = nullptr;
  return rc;
}

int multi_cc(hcc_ctx* c, const hcc_graph* g, const hcc_opts* o_in, hcc_forest* f,
                    uint32_t* lab32, uint64_t* lab64, hcc_metrics* mx) {
  const int G = (int)c->subs.size();
  if ((int)g->shards.size() != G || g->ctx != c)
    return fail(HCC_EINVAL, "graph was not created on this multi-device context");
  if (int r = graph_ready(g)) return r;
  hcc_opts o = {HCC_ALGO_BASELINE_MJ, 0, 0, 0, 0, nullptr, nullptr};
  if (o_in) o = *o_in;
  if (o.algo < HCC_ALGO_BASELINE || o.algo > HCC_ALGO_ADAPTIVE)
    return fail(HCC_EINVAL, "unknown algorithm");
  if (o.observer)
    return fail(HCC_EINVAL, "phase observers need a single-device context");
  const u64 n = g->n;
  if (f && f->n != n) return fail(HCC_EINVAL, "forest size does not match the graph");
  if (f && f->dev != c->subs[0]->dev)
    return fail(HCC_EINVAL, "the forest must live on the first device of the context");
  hcc_metrics out{};
  out.n = n;
  out.m = g->m;
  if (o.algo == HCC_ALGO_ADAPTIVE && o.segments == 0) {
    // s from the WHOLE graph's stats (engines.hpp:245-247), not per shard
    hcc_graph_stats st;
    if (int r = hcc_graph_compute_stats(c, g, &st)) return r;
    o.segments = hcc_choose_segment_count(&st);
  }
  if (n == 0) {
    if (mx) *mx = out;
    return HCC_OK;
  }
  u64 cap = 0;
  try {
    cap = c->merge.empty() ? 0 : c->merge[0].cap;
    if (cap == 0) cap = std::max<u64>(1ull << 16, n / 64);
    ensure_merge(c, n, cap);
    for (int r = 0; r < G; ++r) {
      MergeShard& ms = c->merge[r];
      if (!(r == 0 && f) && (!ms.forest || ms.forest->n != n)) {
        if (ms.forest) hcc_forest_free(ms.forest);
        ms.forest = nullptr;
        if (int st = hcc_forest_create(c->subs[r], n, &ms.forest)) return st;
      }
      ms.local_ms = ms.merge_ms = ms.total_ms = 0;
      ms.passes = ms.records = ms.exported = ms.linked = 0;
    }
  } catch (const CudaFail& fl) {
    return fl.code;
  }
  auto forest_of = [&](int r) { return (r == 0 && f) ? f : c->merge[r].forest; };
  std::vector<hcc_metrics> lm(G);
  // 1. local CC + export
  int rc = for_shards(G, [&](int r) -> int {
    hcc_ctx* sc = c->subs[r];
    MergeShard& ms = c->merge[r];
    HCC_CUDA(cudaSetDevice(sc->dev));
    HCC_CUDA(cudaEventRecord(ms.ev_t0, sc->stream));
    if (int st = run_cc_sized(sc, g->shards[r], &o, forest_of(r), &lm[r])) return st;
    ms.local_ms = lm[r].total_ms;
    enqueue_export(sc, ms, forest_of(r), G > 1);
    return HCC_OK;
  });
  // 2. merge; repeated (export + merge) while some pair list overflowed
  for (int attempt = 0; !rc; ++attempt) {
    u64 pairs_total = 0;
    for (int r = 0; r < G; ++r) pairs_total += c->merge[r].cap;
    rc = for_shards(G, [&](int r) -> int {
      HCC_CUDA(cudaSetDevice(c->subs[r]->dev));
      merge_shard(c, r, forest_of(r), n + pairs_total + 1);
      return HCC_OK;
    });
    if (rc) break;
    u64 need = 0, total = 0;
    try {
      for (int r = 0; r < G; ++r) {
        HCC_CUDA(cudaSetDevice(c->subs[r]->dev));
        u64 k = 0;
        HCC_CUDA(cudaMemcpy(&k, c->merge[r].cnt, sizeof(u64), cudaMemcpyDeviceToHost));
        c->merge[r].exported = k;
        need = std::max(need, k);
        total += k;
      }
      if (need <= c->merge[0].cap) break;
      if (attempt >= 3) {
        rc = fail(HCC_ECUDA, "merge pair buffers kept overflowing");
        break;
      }
      // the repeat exports forests that already absorbed part of the remote
      // relations: a rank's new list is bounded by the union of all lists
      // (usually; the third repeat takes n, which always suffices)
      ensure_merge(c, n, attempt >= 2 ? std::max<u64>(n, 1)
                                      : std::min<u64>(std::max<u64>(n, 1), total + total / 8 + 1));
    } catch (const CudaFail& fl) {
      rc = fl.code;
      break;
    }
    rc = for_shards(G, [&](int r) -> int {
      HCC_CUDA(cudaSetDevice(c->subs[r]->dev));
      HCC_CUDA(cudaEventRecord(c->merge[r].ev_t0, c->subs[r]->stream));
      enqueue_export(c->subs[r], c->merge[r], forest_of(r), G > 1);
      return HCC_OK;
    });
  }
  cudaSetDevice(c->dev);
  if (rc) return rc;
  // metrics: device time of the slowest shard (max over shards)
  for (int r = 0; r < G; ++r) {
    const hcc_metrics& l = lm[r];
    const MergeShard& ms = c->merge[r];
    out.total_ms = std::max(out.total_ms, ms.local_ms + ms.merge_ms);
    out.hook_ms = std::max(out.hook_ms, l.hook_ms);
    out.compress_ms = std::max(out.compress_ms, l.compress_ms);
    out.outer_iterations = std::max(out.outer_iterations, l.outer_iterations);
    out.counters.hook_traversal_steps += l.counters.hook_traversal_steps;
    out.counters.cas_failures += l.counters.cas_failures;
    out.counters.jump_steps += l.counters.jump_steps;
    out.passes += l.passes + ms.passes;
    out.edges_processed += l.edges_processed + ms.records;
    out.kernels += l.kernels + 3 + 3 * ms.passes;
    out.wl_reruns |= l.wl_reruns;
  }
  out.s = lm[0].s;
  out.segments_clamped = lm[0].segments_clamped;
  out.used_device_loop = lm[0].used_device_loop;
  out.star0_bitmap = lm[0].star0_bitmap;
  out.wl_capacity = lm[0].wl_capacity;
  out.components = c->subs[0]->h_ctrl->components;
  out.records = G;
  if (mx) *mx = out;
  if (lab32 || lab64) {
    const hcc_forest* f0 = forest_of(0);
    HCC_GUARD_BEGIN
    HCC_CUDA(cudaSetDevice(c->subs[0]->dev));
    if (lab32) {
      HCC_CUDA(cudaMemcpy(lab32, f0->d_pi, n * sizeof(u32), cudaMemcpyDeviceToHost));
    } else {
      uint32_t* tmp = reinterpret_cast<uint32_t*>(lab64) + n;
      HCC_CUDA(cudaMemcpy(tmp, f0->d_pi, n * sizeof(u32), cudaMemcpyDeviceToHost));
      for (u64 i = 0; i < n; ++i) lab64[i] = tmp[i];
    }
    HCC_CUDA(cudaSetDevice(c->dev));
    return HCC_OK;
    HCC_GUARD_END
  }
  return HCC_OK;
}

}  // namespace host
}  // namespace hcc

extern "C" {

int hcc_create_multi(const int* devices, int ndev, hcc_ctx** out) {
  if (!out || !devices) return fail(HCC_EINVAL, "null argument");
  *out = nullptr;
  if (ndev < 1 || ndev > (int)kMaxShards)
    return fail(HCC_EINVAL, "shard count must be in [1, 64]");
  hcc_ctx* c = nullptr;
  if (int r = hcc_create(devices[0], &c)) return r;
  for (int i = 0; i < ndev; ++i) {
    hcc_ctx* sc = nullptr;
    if (int r = hcc_create(devices[i], &sc)) {
      hcc_destroy(c);
      return r;
    }
    c->subs.push_back(sc);
  }
  // P2P between every pair of distinct devices: the merge kernel reads the
  // peers' export buffers in place over NVLink
  c->peer_access = 1;
  for (int i = 0; i < ndev; ++i)
    for (int j = 0; j < ndev; ++j) {
      const int a = devices[i], b = devices[j];
      if (a == b) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can) {
        cudaGetLastError();
        hcc_destroy(c);
        return fail(HCC_ENCCL, "no peer access from device " + std::to_string(a) + " to " +
                                   std::to_string(b) + " (the merge reads peer memory)");
      }
      cudaSetDevice(a);
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        hcc_destroy(c);
        return fail(HCC_ENCCL, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      }
      cudaGetLastError();
    }
  cudaSetDevice(devices[0]);
  *out = c;
  return HCC_OK;
}

int hcc_ctx_shards(hcc_ctx* c, int* count) {
  if (!c || !count) return fail(HCC_EINVAL, "null argument");
  *count = c->subs.empty() ? 1 : (int)c->subs.size();
  return HCC_OK;
}

int hcc_ctx_shard_metrics(hcc_ctx* c, hcc_shard_metrics* out, uint64_t cap, uint64_t* count) {
  if (!c) return fail(HCC_EINVAL, "null context");
  const u64 G = c->merge.size();
  if (count) *count = G;
  for (u64 r = 0; r < std::min<u64>(cap, G); ++r) {
    const MergeShard& ms = c->merge[r];
    hcc_shard_metrics x{};
    x.total_ms = ms.local_ms + ms.merge_ms;
    x.local_ms = ms.local_ms;
    x.merge_ms = ms.merge_ms;
    x.span_ms = ms.total_ms;
    x.pairs_exported = ms.exported;
    x.records_merged = ms.records;
    x.rehook_passes = ms.passes;
    x.bitmap_bytes = ms.bits_words * 4;
    x.roots_linked = ms.linked;
    x.device = c->subs[r]->dev;
    x.peer_access = c->peer_access;
    out[r] = x;
  }
  return HCC_OK;
}

}  // extern "C"
