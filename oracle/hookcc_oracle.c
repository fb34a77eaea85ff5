/*
 * hookcc_oracle.c — CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * library.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * / --impl reference legs may load it, and only as the checker or the
 * reported CPU baseline — never as the thing measured or shipped.  The
 * product (libhookcc_cuda.so) never links or calls it.
 *
 * Every function restates the reference algorithm it cites (paths relative
 * to /root/reference).  Parity of this restatement is pinned by
 * tests/test_oracle.py against (a) the reference's own known-answer tests
 * (proj/tests/test_forest.cpp, test_engines.cpp, test_oracle.cpp,
 * test_generators.cpp) restated as pytest cases, (b) the reference library
 * itself compiled from /root/reference by oracle/Makefile into oracle/_ref/,
 * and (c) golden fixtures generated from oracle/_ref (tests/golden/).
 *
 * Build: make -C oracle   (gcc -O3 -shared -fPIC -> oracle/liboracle.so)
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef uint32_t u32;

/* ------------------------------------------------------------------------
 * std::mt19937_64 (C++11 [rand.eng.mers] parameters), restated so the
 * reference generators can be reproduced bit-exactly without C++.
 */
#define MT_N 312
#define MT_M 156

typedef struct {
  u64 mt[MT_N];
  int idx;
} mt64;

static void mt64_seed(mt64* s, u64 seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) +
               (u64)i;
  s->idx = MT_N;
}

static u64 mt64_next(mt64* s) {
  if (s->idx >= MT_N) {
    const u64 UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    for (int i = 0; i < MT_N; ++i) {
      u64 x = (s->mt[i] & UM) | (s->mt[(i + 1) % MT_N] & LM);
      u64 xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      s->mt[i] = s->mt[(i + MT_M) % MT_N] ^ xa;
    }
    s->idx = 0;
  }
  u64 y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* libstdc++ 13 generate_canonical<double, 53>(mt19937_64)
 * (/usr/include/c++/13/bits/random.tcc:3349-3381): one 64-bit draw,
 * double(x) / 2^64, clamped below 1. */
static double mt64_unit(mt64* s) {
  double r = (double)mt64_next(s) / 18446744073709551616.0;
  if (r >= 1.0) r = 0x1.fffffffffffffp-1;
  return r;
}

/* ---- reference generators (proj/include/hookcc/generators.hpp) -------- */

/* erdos_renyi (generators.hpp:14-26): u = rng() % n, v = rng() % n. */
int oracle_gen_er(u64 n, u64 m, u64 seed, u64* uv) {
  if (n == 0) return 1;
  mt64 s;
  mt64_seed(&s, seed);
  for (u64 i = 0; i < m; ++i) {
    uv[2 * i] = mt64_next(&s) % n;
    uv[2 * i + 1] = mt64_next(&s) % n;
  }
  return 0;
}

/* rmat (generators.hpp:31-62): per level one uniform double p;
 * p < a: (0,0); p < a+b: (0,1); p < a+b+c: (1,0); else (1,1); MSB first. */
int oracle_gen_rmat(u32 scale, u64 ef, double a, double b, double c, double d,
                    u64 seed, u64* uv) {
  double sum = a + b + c + d - 1.0;
  if (sum > 1e-9 || sum < -1e-9) return 1;
  u64 n = 1ull << scale, m = ef * n;
  mt64 s;
  mt64_seed(&s, seed);
  for (u64 i = 0; i < m; ++i) {
    u64 u = 0, v = 0;
    for (u32 l = 0; l < scale; ++l) {
      double p = mt64_unit(&s);
      u <<= 1;
      v <<= 1;
      if (p < a) {
      } else if (p < a + b) {
        v |= 1;
      } else if (p < a + b + c) {
        u |= 1;
      } else {
        u |= 1;
        v |= 1;
      }
    }
    uv[2 * i] = u;
    uv[2 * i + 1] = v;
  }
  return 0;
}

/* grid (generators.hpp:71-87): row edges, then column edges. */
int oracle_gen_grid(u64 rows, u64 cols, u64* uv) {
  if (rows == 0 || cols == 0) return 1;
  u64 k = 0;
  for (u64 r = 0; r < rows; ++r)
    for (u64 c = 0; c + 1 < cols; ++c) {
      uv[2 * k] = r * cols + c;
      uv[2 * k + 1] = r * cols + c + 1;
      ++k;
    }
  for (u64 r = 0; r + 1 < rows; ++r)
    for (u64 c = 0; c < cols; ++c) {
      uv[2 * k] = r * cols + c;
      uv[2 * k + 1] = r * cols + c + cols;
      ++k;
    }
  return 0;
}

/* ---- counter-based twins (restating include/hookcc_gen.h
 * from its written specification, independently of that code) ----------- */

static u64 sm_final(u64 z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

static u64 ctr_word(u64 seed, u64 ctr) {
  u64 key = sm_final(seed ^ 0x5851F42D4C957F2Dull);
  return sm_final(key + (ctr + 1) * 0x9E3779B97F4A7C15ull);
}

static u32 thr(double x) {
  if (!(x > 0.0)) return 0u;
  if (x >= 1.0) return 0xffffffffu;
  double t = x * 4294967296.0;
  if (t >= 4294967295.0) return 0xffffffffu;
  return (u32)t;
}

/* edges [first, first+count) of rmatx:scale,ef,seed as u32 pairs */
void oracle_gen_rmatx(u32 scale, double a, double b, double c, u64 seed,
                      u64 first, u64 count, u32* uv) {
  u32 ta = thr(a), tab = thr(a + b), tabc = thr(a + b + c);
  for (u64 k = 0; k < count; ++k) {
    u64 i = first + k;
    u32 u = 0, v = 0;
    for (u32 l = 0; l < scale; ++l) {
      u64 w = ctr_word(seed, i * 16 + l / 2);
      u32 p = (l % 2) ? (u32)(w >> 32) : (u32)(w & 0xffffffffu);
      u32 qu = (p >= tab), qv = (p >= ta && p < tab) || (p >= tabc);
      u = (u << 1) | qu;
      v = (v << 1) | qv;
    }
    uv[2 * k] = u;
    uv[2 * k + 1] = v;
  }
}

void oracle_gen_erx(u64 n, u64 seed, u64 first, u64 count, u32* uv) {
  for (u64 k = 0; k < count; ++k) {
    u64 w = ctr_word(seed, first + k);
    uv[2 * k] = (u32)(((w & 0xffffffffull) * n) >> 32);
    uv[2 * k + 1] = (u32)(((w >> 32) * n) >> 32);
  }
}

/* wrapping sum over i of mix(i * golden ^ (u << 32 | v)) */
u64 oracle_checksum_u32(const u32* uv, u64 first, u64 count) {
  u64 s = 0;
  for (u64 k = 0; k < count; ++k) {
    u64 i = first + k;
    u64 x = (i * 0x9E3779B97F4A7C15ull) ^
            (((u64)uv[2 * k] << 32) | (u64)uv[2 * k + 1]);
    s += sm_final(x);
  }
  return s;
}

/* ---- ground truth (proj/include/hookcc/oracle.hpp:17-62) ---------------
 * DisjointSet with path halving and union by rank, then min-canonical
 * relabeling.  Parent array is u32 (n < 2^32), which is what makes the
 * scale-28 oracle fit in host RAM. */

typedef struct {
  u32* parent;
  uint8_t* rank;
} dsu;

static u32 dsu_find(dsu* d, u32 v) {
  while (d->parent[v] != v) {
    d->parent[v] = d->parent[d->parent[v]];
    v = d->parent[v];
  }
  return v;
}

static void dsu_unite(dsu* d, u32 a, u32 b) {
  u32 ra = dsu_find(d, a), rb = dsu_find(d, b);
  if (ra == rb) return;
  if (d->rank[ra] < d->rank[rb]) {
    u32 t = ra;
    ra = rb;
    rb = t;
  }
  d->parent[rb] = ra;
  if (d->rank[ra] == d->rank[rb]) ++d->rank[ra];
}

static int oracle_finish(dsu* d, u64 n, u64* labels64, u32* labels32) {
  u32* min_of_root = (u32*)malloc((n ? n : 1) * sizeof(u32));
  if (!min_of_root) return 2;
  for (u64 v = 0; v < n; ++v) min_of_root[v] = (u32)v;
  for (u64 v = 0; v < n; ++v) {
    u32 r = dsu_find(d, (u32)v);
    if ((u32)v < min_of_root[r]) min_of_root[r] = (u32)v;
  }
  for (u64 v = 0; v < n; ++v) {
    u32 l = min_of_root[dsu_find(d, (u32)v)];
    if (labels64) labels64[v] = l;
    if (labels32) labels32[v] = l;
  }
  free(min_of_root);
  return 0;
}

static int dsu_init(dsu* d, u64 n) {
  d->parent = (u32*)malloc((n ? n : 1) * sizeof(u32));
  d->rank = (uint8_t*)calloc(n ? n : 1, 1);
  if (!d->parent || !d->rank) return 2;
  for (u64 v = 0; v < n; ++v) d->parent[v] = (u32)v;
  return 0;
}

static void dsu_free(dsu* d) {
  free(d->parent);
  free(d->rank);
}

/* oracle_cc over u64 pairs (the reference Graph layout). */
int oracle_cc_u64(u64 n, const u64* uv, u64 m, u64* labels) {
  if (n > 0xffffffffull) return 1;
  dsu d;
  if (dsu_init(&d, n)) return 2;
  for (u64 i = 0; i < m; ++i) {
    if (uv[2 * i] >= n || uv[2 * i + 1] >= n) {
      dsu_free(&d);
      return 1;
    }
    dsu_unite(&d, (u32)uv[2 * i], (u32)uv[2 * i + 1]);
  }
  int r = oracle_finish(&d, n, labels, NULL);
  dsu_free(&d);
  return r;
}

/* Streaming variant over packed u32 pairs (device layout). */
int oracle_cc_u32(u64 n, const u32* uv, u64 m, u32* labels) {
  if (n > 0xffffffffull) return 1;
  dsu d;
  if (dsu_init(&d, n)) return 2;
  for (u64 i = 0; i < m; ++i) {
    if (uv[2 * i] >= n || uv[2 * i + 1] >= n) {
      dsu_free(&d);
      return 1;
    }
    dsu_unite(&d, uv[2 * i], uv[2 * i + 1]);
  }
  int r = oracle_finish(&d, n, NULL, labels);
  dsu_free(&d);
  return r;
}

/* ---- streaming ground truth for graphs too large to hold (RMAT-28) ------
 * oracle_cc (oracle.hpp:47-62) over edges [first, first+count) of a
 * counter-based generator, without materialising the edge array: chunk k+1
 * is generated by `nthreads` worker threads while the main thread unites
 * chunk k into the DSU (the unions stay strictly sequential, in stored edge
 * order, exactly as oracle_cc does over a Graph).  RMAT-28 needs 32 GiB of
 * edges in the reference layout (64 GiB as u64) but only the 1 GiB u32
 * parent array here.  Also returns the position-keyed checksum of the
 * generated stream (oracle_checksum_u32) and the component count.
 *   kind 0: rmatx (scale, a, b, c, seed)      kind 1: erx (n_er, seed)     */
typedef struct {
  int kind;
  u32 scale;
  double a, b, c;
  u64 n_er, seed, first, count;
  u32* uv;
  u64 sum;
} stream_job;

static void* stream_gen(void* p) {
  stream_job* j = (stream_job*)p;
  if (j->kind == 0)
    oracle_gen_rmatx(j->scale, j->a, j->b, j->c, j->seed, j->first, j->count, j->uv);
  else
    oracle_gen_erx(j->n_er, j->seed, j->first, j->count, j->uv);
  j->sum = oracle_checksum_u32(j->uv, j->first, j->count);
  return NULL;
}

#define STREAM_CHUNK (1ull << 25) /* edges per chunk (256 MiB of u32 pairs) */
#define STREAM_MAXT 64

static void stream_fill(int kind, u32 scale, double a, double b, double c, u64 n_er, u64 seed,
                        u64 first, u64 count, int nt, u32* buf, u64* sum) {
  pthread_t th[STREAM_MAXT];
  stream_job jb[STREAM_MAXT];
  const u64 per = (count + (u64)nt - 1) / (u64)nt;
  int started = 0;
  for (int t = 0; t < nt; ++t) {
    const u64 b0 = (u64)t * per;
    if (b0 >= count) break;
    stream_job x = {kind, scale, a, b, c, n_er, seed, first + b0,
                    count - b0 < per ? count - b0 : per, buf + 2 * b0, 0};
    jb[t] = x;
    pthread_create(&th[t], NULL, stream_gen, &jb[t]);
    ++started;
  }
  for (int t = 0; t < started; ++t) {
    pthread_join(th[t], NULL);
    *sum += jb[t].sum;
  }
}

typedef struct {
  int kind;
  u32 scale;
  double a, b, c;
  u64 n_er, seed, first, count;
  int nt;
  u32* buf;
  u64* sum;
} fill_job;

static void* fill_thread(void* p) {
  fill_job* f = (fill_job*)p;
  stream_fill(f->kind, f->scale, f->a, f->b, f->c, f->n_er, f->seed, f->first, f->count, f->nt,
              f->buf, f->sum);
  return NULL;
}

int oracle_cc_stream(int kind, u32 scale, double a, double b, double c, u64 n_er, u64 seed,
                     u64 first, u64 count, int nthreads, u32* labels, u64* checksum,
                     u64* components) {
  const u64 n = kind == 0 ? (1ull << scale) : n_er;
  if (n > 0xffffffffull || (kind == 0 && scale > 31)) return 1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > STREAM_MAXT) nthreads = STREAM_MAXT;
  dsu d;
  if (dsu_init(&d, n)) return 2;
  u32* buf[2];
  buf[0] = (u32*)malloc(STREAM_CHUNK * 2 * sizeof(u32));
  buf[1] = (u32*)malloc(STREAM_CHUNK * 2 * sizeof(u32));
  if (!buf[0] || !buf[1]) {
    free(buf[0]);
    free(buf[1]);
    dsu_free(&d);
    return 2;
  }
  u64 sum = 0;
  const u64 nch = (count + STREAM_CHUNK - 1) / STREAM_CHUNK;
  if (nch)
    stream_fill(kind, scale, a, b, c, n_er, seed, first,
                count < STREAM_CHUNK ? count : STREAM_CHUNK, nthreads, buf[0], &sum);
  for (u64 k = 0; k < nch; ++k) {
    const u64 off = k * STREAM_CHUNK;
    const u64 cnt = count - off < STREAM_CHUNK ? count - off : STREAM_CHUNK;
    pthread_t filler;
    fill_job fj;
    const int more = k + 1 < nch;
    if (more) {
      const u64 off2 = off + STREAM_CHUNK;
      fill_job x = {kind, scale, a, b, c, n_er, seed, first + off2,
                    count - off2 < STREAM_CHUNK ? count - off2 : STREAM_CHUNK, nthreads,
                    buf[(k + 1) & 1], &sum};
      fj = x;
      pthread_create(&filler, NULL, fill_thread, &fj);
    }
    const u32* e = buf[k & 1];
    for (u64 i = 0; i < cnt; ++i) dsu_unite(&d, e[2 * i], e[2 * i + 1]);
    if (more) pthread_join(filler, NULL);
  }
  free(buf[0]);
  free(buf[1]);
  int r = oracle_finish(&d, n, NULL, labels);
  dsu_free(&d);
  if (r) return r;
  u64 roots = 0;
  for (u64 v = 0; v < n; ++v) roots += labels[v] == (u32)v;
  if (checksum) *checksum = sum;
  if (components) *components = roots;
  return 0;
}

/* bfs_cc (oracle.hpp:67-108): BFS from each unvisited vertex ascending,
 * labeling with the source; self-loops skipped. */
int oracle_bfs_cc_u64(u64 n, const u64* uv, u64 m, u64* labels) {
  u64* head = (u64*)calloc(n + 1, sizeof(u64));
  if (!head) return 2;
  for (u64 i = 0; i < m; ++i)
    if (uv[2 * i] != uv[2 * i + 1]) {
      ++head[uv[2 * i] + 1];
      ++head[uv[2 * i + 1] + 1];
    }
  for (u64 v = 0; v < n; ++v) head[v + 1] += head[v];
  u64* adj = (u64*)malloc((head[n] ? head[n] : 1) * sizeof(u64));
  u64* cur = (u64*)malloc((n ? n : 1) * sizeof(u64));
  uint8_t* vis = (uint8_t*)calloc(n ? n : 1, 1);
  u64* q = (u64*)malloc((n ? n : 1) * sizeof(u64));
  if (!adj || !cur || !vis || !q) return 2;
  memcpy(cur, head, n * sizeof(u64));
  for (u64 i = 0; i < m; ++i) {
    u64 a = uv[2 * i], b = uv[2 * i + 1];
    if (a != b) {
      adj[cur[a]++] = b;
      adj[cur[b]++] = a;
    }
  }
  for (u64 src = 0; src < n; ++src) {
    if (vis[src]) continue;
    vis[src] = 1;
    labels[src] = src;
    u64 qh = 0, qt = 0;
    q[qt++] = src;
    while (qh < qt) {
      u64 v = q[qh++];
      for (u64 j = head[v]; j < head[v + 1]; ++j) {
        u64 w = adj[j];
        if (!vis[w]) {
          vis[w] = 1;
          labels[w] = src;
          q[qt++] = w;
        }
      }
    }
  }
  free(head);
  free(adj);
  free(cur);
  free(vis);
  free(q);
  return 0;
}

/* ---- per-element kernels (proj/include/hookcc/forest.hpp:83-146) ------- */

typedef struct {
  u64 hook_traversal_steps, cas_failures, jump_steps;
} oracle_counters;

/* hook (forest.hpp:83-89) */
int oracle_hook(u64* pi, u64 u, u64 v) {
  u64 pu = pi[u], pv = pi[v];
  if (pu == pv) return 0;
  pi[pu > pv ? pu : pv] = pu < pv ? pu : pv;
  return 1;
}

/* jump (forest.hpp:93-99) */
int oracle_jump(u64* pi, u64 v) {
  u64 p = pi[v], gp = pi[p];
  if (gp == p) return 0;
  pi[v] = gp;
  return 1;
}

/* atomic_hook (forest.hpp:107-122), sequential: the CAS on the root slot
 * succeeds iff the slot still holds its own index. */
void oracle_atomic_hook(u64* pi, u64 u, u64 v, oracle_counters* c) {
  for (;;) {
    u64 pu = pi[u], pv = pi[v];
    if (pu == pv) return;
    ++c->hook_traversal_steps;
    u64 high = pu > pv ? pu : pv, low = pu < pv ? pu : pv;
    if (pi[high] == high) {
      pi[high] = low;
      return;
    }
    ++c->cas_failures;
    u = pi[high];
    v = low;
  }
}

/* multi_jump (forest.hpp:127-136) */
void oracle_multi_jump(u64* pi, u64 v, oracle_counters* c) {
  u64 p = pi[v];
  for (;;) {
    u64 gp = pi[p];
    if (gp == p) return;
    pi[v] = gp;
    ++c->jump_steps;
    p = gp;
  }
}

/* is_star (forest.hpp:140-146) */
int oracle_is_star(const u64* pi, u64 n) {
  for (u64 v = 0; v < n; ++v)
    if (pi[pi[v]] != pi[v]) return 0;
  return 1;
}

/* ---- sequential drivers (engines.hpp), the workers = 1 schedule --------
 * With one worker every for_range runs inline in ascending order
 * (parallel.hpp:29, 52-55), so these reproduce the reference counters
 * exactly.  rec_* arrays (optional, capacity rec_cap) receive one entry per
 * segment / outer iteration. */

typedef struct {
  u64 outer_iterations;
  u64 s;
  int clamped;
  oracle_counters counters;
  u64 components;
} oracle_run;

static void count_roots(const u64* pi, u64 n, oracle_run* r) {
  r->components = 0;
  for (u64 v = 0; v < n; ++v) r->components += (pi[v] == v);
}

/* baseline_cc_into (engines.hpp:123-179) */
int oracle_baseline_cc(u64 n, const u64* uv, u64 m, u64* pi, oracle_run* r) {
  memset(r, 0, sizeof(*r));
  r->s = 1;
  for (u64 v = 0; v < n; ++v) pi[v] = v;
  for (;;) {
    ++r->outer_iterations;
    int hook_changed = 0;
    for (u64 i = 0; i < m; ++i) hook_changed |= oracle_hook(pi, uv[2 * i], uv[2 * i + 1]);
    for (;;) {
      int jc = 0;
      for (u64 v = 0; v < n; ++v)
        if (oracle_jump(pi, v)) {
          ++r->counters.jump_steps;
          jc = 1;
        }
      if (!jc) break;
    }
    if (!hook_changed) break;
  }
  count_roots(pi, n, r);
  return 0;
}

/* baseline_mj_cc_into (engines.hpp:183-231) */
int oracle_baseline_mj_cc(u64 n, const u64* uv, u64 m, u64* pi, oracle_run* r) {
  memset(r, 0, sizeof(*r));
  r->s = 1;
  for (u64 v = 0; v < n; ++v) pi[v] = v;
  for (;;) {
    ++r->outer_iterations;
    int hook_changed = 0;
    for (u64 i = 0; i < m; ++i) hook_changed |= oracle_hook(pi, uv[2 * i], uv[2 * i + 1]);
    for (u64 v = 0; v < n; ++v) oracle_multi_jump(pi, v, &r->counters);
    if (!hook_changed) break;
  }
  count_roots(pi, n, r);
  return 0;
}

/* partition_edges (engines.hpp:43-58) */
u64 oracle_partition(u64 m, u64 s, u64* boundaries, int* clamped) {
  if (s < 1) s = 1;
  if (clamped) *clamped = s > m && m > 0;
  u64 mm = m > 1 ? m : 1;
  if (s > mm) s = mm;
  u64 base = m / s, rem = m % s, off = 0;
  if (boundaries) {
    boundaries[0] = 0;
    for (u64 i = 0; i < s; ++i) {
      off += base + (i < rem ? 1 : 0);
      boundaries[i + 1] = off;
    }
  }
  return s;
}

/* adaptive_cc_into (engines.hpp:238-291) with an explicit s >= 1;
 * seg_counters (3 per segment, optional) receive per-segment counters. */
int oracle_adaptive_cc(u64 n, const u64* uv, u64 m, u64 segments, u64* pi,
                       oracle_run* r, u64* seg_counters) {
  memset(r, 0, sizeof(*r));
  int clamped = 0;
  u64 s = oracle_partition(m, segments, NULL, &clamped);
  u64* bd = (u64*)malloc((s + 1) * sizeof(u64));
  if (!bd) return 2;
  oracle_partition(m, segments, bd, NULL);
  r->s = s;
  r->clamped = clamped;
  for (u64 v = 0; v < n; ++v) pi[v] = v;
  for (u64 seg = 0; seg < s; ++seg) {
    oracle_counters c = {0, 0, 0};
    for (u64 i = bd[seg]; i < bd[seg + 1]; ++i)
      oracle_atomic_hook(pi, uv[2 * i], uv[2 * i + 1], &c);
    for (u64 v = 0; v < n; ++v) oracle_multi_jump(pi, v, &c);
    r->counters.hook_traversal_steps += c.hook_traversal_steps;
    r->counters.cas_failures += c.cas_failures;
    r->counters.jump_steps += c.jump_steps;
    if (seg_counters) {
      seg_counters[3 * seg] = c.hook_traversal_steps;
      seg_counters[3 * seg + 1] = c.cas_failures;
      seg_counters[3 * seg + 2] = c.jump_steps;
    }
  }
  r->outer_iterations = s;
  free(bd);
  count_roots(pi, n, r);
  return 0;
}

/* compute_stats (graph.hpp:43-68): unique undirected non-loop pairs. */
static int cmp_u64(const void* a, const void* b) {
  u64 x = *(const u64*)a, y = *(const u64*)b;
  return x < y ? -1 : x > y;
}

int oracle_stats_u64(u64 n, const u64* uv, u64 m, u64* m_unique,
                     u64* max_degree) {
  u64* keys = (u64*)malloc((m ? m : 1) * sizeof(u64));
  u64* deg = (u64*)calloc(n ? n : 1, sizeof(u64));
  if (!keys || !deg) return 2;
  u64 k = 0;
  for (u64 i = 0; i < m; ++i) {
    u64 a = uv[2 * i], b = uv[2 * i + 1];
    if (a == b) continue;
    u64 lo = a < b ? a : b, hi = a < b ? b : a;
    keys[k++] = (lo << 32) | hi;
  }
  qsort(keys, k, sizeof(u64), cmp_u64);
  u64 uq = 0;
  for (u64 i = 0; i < k; ++i) {
    if (i > 0 && keys[i] == keys[i - 1]) continue;
    ++uq;
    ++deg[keys[i] >> 32];
    ++deg[keys[i] & 0xffffffffull];
  }
  u64 mx = 0;
  for (u64 v = 0; v < n; ++v)
    if (deg[v] > mx) mx = deg[v];
  *m_unique = uq;
  *max_degree = mx;
  free(keys);
  free(deg);
  return 0;
}
