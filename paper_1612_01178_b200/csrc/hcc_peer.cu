// Multi-process merge over CUDA IPC (hcc_peer_*): host side.  The gather
// kernel is hcc_multi.cu's k_merge_gather; handles in hcc_host.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "hcc_host.cuh"

using namespace hcc::host;

// ===========================================================================
// Multi-process merge over CUDA IPC (one process per GPU, e.g. torchrun;
// paper_1612_01178_b200/distributed.py).  Each rank allocates its export
// buffers in one arena and an interprocess event, and publishes both as a
// handle blob; after the blobs are exchanged (any transport: the Python
// binding all-gathers them over torch.distributed once), every rank maps its
// peers' arenas (cudaIpcOpenMemHandle, lazy peer access) and the same
// k_merge_gather kernel reads them in place over NVLink.  Per run: local CC,
// hcc_peer_export (k_export + event record), a host barrier (so every
// record precedes every wait), hcc_peer_merge (device waits on the peers'
// events, gather, re-hook).

struct PeerBlob {
  cudaIpcMemHandle_t mem;
  cudaIpcEventHandle_t ev;
  u64 bits_off, pairs_off, cap, nwords, n;
  int32_t rank, world, dev, pad_;
};
static_assert(sizeof(PeerBlob) <= HCC_PEER_HANDLE_BYTES, "peer handle blob too large");

struct hcc_peer_state {
  int rank = 0, world = 1;
  u64 n = 0, cap = 0, nwords = 0;
  char* arena = nullptr;
  u64* cnt = nullptr;
  u32* bits = nullptr;
  uint2* pairs = nullptr;
  cudaEvent_t ev = nullptr;                 // this rank's export event
  std::vector<char*> mapped;                // peers' arenas (nullptr = self)
  std::vector<cudaEvent_t> peer_ev;         // peers' export events
  std::vector<PeerBlob> blobs;
  PeerTab* d_tab = nullptr;
  cudaEvent_t ev_m0 = nullptr, ev_m1 = nullptr;
  bool connected = false;
};

namespace hcc {
namespace host {

void peer_release(hcc_ctx* c) {
  hcc_peer_state* p = c->peer;
  if (!p) return;
  cudaSetDevice(c->dev);
  cudaStreamSynchronize(c->stream);
  for (char* a : p->mapped)
    if (a) cudaIpcCloseMemHandle(a);
  for (size_t r = 0; r < p->peer_ev.size(); ++r)
    if (p->peer_ev[r]) cudaEventDestroy(p->peer_ev[r]);
  if (p->ev) cudaEventDestroy(p->ev);
  if (p->ev_m0) cudaEventDestroy(p->ev_m0);
  if (p->ev_m1) cudaEventDestroy(p->ev_m1);
  cudaFree(p->arena);
  cudaFree(p->d_tab);
  cudaGetLastError();
  delete p;
  c->peer = nullptr;
}

}  // namespace host
}  // namespace hcc

extern "C" {

int hcc_peer_open(hcc_ctx* c, uint64_t n, uint64_t cap, int rank, int world, void* handle_out) {
  if (!handle_out || world < 1 || rank < 0 || rank >= world || world > (int)kMaxShards)
    return fail(HCC_EINVAL, "bad peer arguments (rank/world/handle)");
  if (n > kMaxN) return fail(HCC_EINVAL, "vertex count >= 2^32");
  if (int r = ctx_enter(c)) return r;
  if (!c->subs.empty()) return fail(HCC_EINVAL, "peer merge needs a single-device context");
  peer_release(c);
  hcc_peer_state* p = new hcc_peer_state;
  c->peer = p;
  HCC_GUARD_BEGIN
  p->rank = rank;
  p->world = world;
  p->n = n;
  p->cap = std::max<u64>(cap, 1);
  p->nwords = (n + 31) / 32;
  const u64 bits_off = 256, pairs_off = (bits_off + p->nwords * 4 + 255) & ~255ull;
  HCC_CUDA(cudaMalloc(&p->arena, pairs_off + p->cap * sizeof(uint2)));
  p->cnt = reinterpret_cast<u64*>(p->arena);
  p->bits = reinterpret_cast<u32*>(p->arena + bits_off);
  p->pairs = reinterpret_cast<uint2*>(p->arena + pairs_off);
  HCC_CUDA(cudaMemset(p->cnt, 0, sizeof(u64)));
  HCC_CUDA(cudaEventCreateWithFlags(&p->ev, cudaEventDisableTiming | cudaEventInterprocess));
  HCC_CUDA(cudaEventCreate(&p->ev_m0));
  HCC_CUDA(cudaEventCreate(&p->ev_m1));
  HCC_CUDA(cudaMalloc(&p->d_tab, sizeof(PeerTab)));
  PeerBlob b{};
  HCC_CUDA(cudaIpcGetMemHandle(&b.mem, p->arena));
  HCC_CUDA(cudaIpcGetEventHandle(&b.ev, p->ev));
  b.bits_off = bits_off;
  b.pairs_off = pairs_off;
  b.cap = p->cap;
  b.nwords = p->nwords;
  b.n = n;
  b.rank = rank;
  b.world = world;
  b.dev = c->dev;
  std::memset(handle_out, 0, HCC_PEER_HANDLE_BYTES);
  std::memcpy(handle_out, &b, sizeof(b));
  return HCC_OK;
  }
  catch (const CudaFail& f) {
    peer_release(c);
    return f.code;
  }
}

int hcc_peer_connect(hcc_ctx* c, const void* handles) {
  if (!handles) return fail(HCC_EINVAL, "null handles");
  if (int r = ctx_enter(c)) return r;
  hcc_peer_state* p = c->peer;
  if (!p) return fail(HCC_EINVAL, "hcc_peer_open first");
  const int W = p->world;
  p->blobs.resize(W);
  for (int r = 0; r < W; ++r) {
    std::memcpy(&p->blobs[r], static_cast<const char*>(handles) + (size_t)r * HCC_PEER_HANDLE_BYTES,
                sizeof(PeerBlob));
    const PeerBlob& b = p->blobs[r];
    if (b.rank != r || b.world != W || b.n != p->n)
      return fail(HCC_EINVAL, "peer handles disagree (rank order, world or n)");
  }
  HCC_GUARD_BEGIN
  p->mapped.assign(W, nullptr);
  p->peer_ev.assign(W, nullptr);
  PeerTab t{};
  t.npeers = (u32)W;
  for (int r = 0; r < W; ++r) {
    const PeerBlob& b = p->blobs[r];
    char* base = p->arena;
    if (r != p->rank) {
      void* m = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&m, b.mem, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(HCC_ENCCL, std::string("cudaIpcOpenMemHandle (rank ") + std::to_string(r) +
                                   "): " + cudaGetErrorString(e));
      }
      p->mapped[r] = base = static_cast<char*>(m);
      HCC_CUDA(cudaIpcOpenEventHandle(&p->peer_ev[r], b.ev));
    }
    t.bits[r] = reinterpret_cast<const u32*>(base + b.bits_off);
    t.pairs[r] = reinterpret_cast<const uint2*>(base + b.pairs_off);
    t.count[r] = reinterpret_cast<const u64*>(base);
    t.cap[r] = b.cap;
  }
  HCC_CUDA(cudaMemcpy(p->d_tab, &t, sizeof(PeerTab), cudaMemcpyHostToDevice));
  p->connected = true;
  return HCC_OK;
  HCC_GUARD_END
}

int hcc_peer_export(hcc_ctx* c, hcc_forest* f) {
  if (!f) return fail(HCC_EINVAL, "null forest");
  if (int r = ctx_enter(c)) return r;
  hcc_peer_state* p = c->peer;
  if (!p || !p->connected) return fail(HCC_EINVAL, "peer merge not connected");
  if (f->n != p->n || f->dev != c->dev) return fail(HCC_EINVAL, "forest does not match the peer setup");
  HCC_GUARD_BEGIN
  HCC_CUDA(cudaEventRecord(p->ev_m0, c->stream));
  HCC_CUDA(cudaMemsetAsync(p->cnt, 0, sizeof(u64), c->stream));
  // (a world of one has no peer to read the export: the merge is the
  // identity)
  if (f->n && p->world > 1)
    k_export<<<grid_for(p->nwords * 32, 256, (u64)c->sms * 32), 256, 0, c->stream>>>(
        f->d_pi, f->n, p->bits, p->pairs, p->cap, p->cnt);
  HCC_CUDA(cudaGetLastError());
  HCC_CUDA(cudaEventRecord(p->ev, c->stream));
  return HCC_OK;
  HCC_GUARD_END
}

int hcc_peer_merge(hcc_ctx* c, hcc_forest* f, hcc_metrics* mx, int* overflow) {
  if (!f || !overflow) return fail(HCC_EINVAL, "null argument");
  if (int r = ctx_enter(c)) return r;
  hcc_peer_state* p = c->peer;
  if (!p || !p->connected) return fail(HCC_EINVAL, "peer merge not connected");
  if (f->n != p->n || f->dev != c->dev) return fail(HCC_EINVAL, "forest does not match the peer setup");
  hcc_metrics out{};
  out.n = f->n;
  HCC_GUARD_BEGIN
  const u64 n = f->n;
  for (int r = 0; r < p->world; ++r)
    if (r != p->rank) HCC_CUDA(cudaStreamWaitEvent(c->stream, p->peer_ev[r], 0));
  k_begin<<<1, 1, 0, c->stream>>>(c->d_ctrl, c->d_recs, 1);
  if (p->world > 1) {
    u64 pairs_total = 0;
    for (const PeerBlob& b : p->blobs) pairs_total += b.cap;
    ensure_wl(c, n + pairs_total + 1);
    k_merge_gather<<<std::max<unsigned>(1u, (unsigned)c->sms * 8u), 256, 0, c->stream>>>(
        p->d_tab, (u32)p->rank, f->d_pi, n, c->wl[0], &c->d_ctrl->wl_count[0], c->wl_cap,
        &c->d_ctrl->err, &c->d_ctrl->dirty, &c->d_ctrl->merged_links);
    HCC_CUDA(cudaGetLastError());
    enqueue_rehook(c, f->d_pi, n);
  }
  HCC_CUDA(cudaEventRecord(p->ev_m1, c->stream));
  // components (metrics only, after the timed region)
  k_count_roots<<<grid_for(n, 256, (u64)c->sms * 16), 256, 0, c->stream>>>(f->d_pi, n,
                                                                         c->d_ctrl);
  HCC_CUDA(cudaGetLastError());
  HCC_CUDA(cudaMemcpyAsync(c->h_ctrl, c->d_ctrl, sizeof(DevCtrl), cudaMemcpyDeviceToHost,
                           c->stream));
  HCC_CUDA(cudaMemcpyAsync(c->h_recs, c->d_recs, sizeof(DevRec), cudaMemcpyDeviceToHost,
                           c->stream));
  HCC_CUDA(cudaStreamSynchronize(c->stream));
  // the peers' pair counts (read from their arenas, after the waits)
  int ovf = 0;
  for (int r = 0; r < p->world; ++r) {
    u64 k = 0;
    const char* base = r == p->rank ? p->arena : p->mapped[r];
    HCC_CUDA(cudaMemcpy(&k, base, sizeof(u64), cudaMemcpyDeviceToHost));
    if (k > p->blobs[r].cap) ovf = 1;
    if (r == p->rank) out.m = k;  // pairs this rank exported
  }
  *overflow = ovf;
  if (c->h_ctrl->err & 4u) return fail(HCC_ECUDA, "merge worklist overflow");
  float ms = 0.f;
  HCC_CUDA(cudaEventElapsedTime(&ms, p->ev_m0, p->ev_m1));
  out.total_ms = ms;  // export through re-hook, incl. waiting for the peers
  out.passes = c->h_ctrl->passes;
  out.outer_iterations = c->h_ctrl->passes;
  out.edges_processed = c->h_recs[0].edges_in;  // remote relations re-hooked
  out.components = c->h_ctrl->components;
  out.kernels = 4 + 3 * c->h_ctrl->passes;
  if (mx) *mx = out;
  return HCC_OK;
  HCC_GUARD_END
}

int hcc_peer_disconnect(hcc_ctx* c) {
  if (!c) return fail(HCC_EINVAL, "null context");
  hcc_peer_state* p = c->peer;
  if (!p) return HCC_OK;
  cudaSetDevice(c->dev);
  cudaStreamSynchronize(c->stream);
  for (char*& a : p->mapped) {
    if (a) cudaIpcCloseMemHandle(a);
    a = nullptr;
  }
  for (cudaEvent_t& ev : p->peer_ev) {
    if (ev) cudaEventDestroy(ev);
    ev = nullptr;
  }
  cudaGetLastError();
  p->connected = false;
  return HCC_OK;
}

int hcc_peer_close(hcc_ctx* c) {
  if (!c) return fail(HCC_EINVAL, "null context");
  peer_release(c);
  return HCC_OK;
}

}  // extern "C"
