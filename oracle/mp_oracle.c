/* TEST INFRASTRUCTURE ONLY — CPU oracle (plain-C restatement of the
 * reference ordering path).  See mp_oracle.h for the contract and for how it
 * is pinned against the reference.  Each function cites the reference
 * file:line it restates (paths relative to /root/reference/proj/core/src).
 * Written for clarity, not speed: the quadratic scans the reference has are
 * kept (they define the tie-breaks), a few std::set walks become linear scans
 * with the identical selection rule.
 */
#define _POSIX_C_SOURCE 200809L
#include "mp_oracle.h"

#include <limits.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NONE (-1)
#define UNREACHED INT32_MAX
#define LLOYD_ROUNDS 10   /* patching.cpp:15 */
#define FM_PASSES 10      /* partition.cpp:13 */
#define BALANCE_TOL 1.2   /* partition.hpp:34 */
#define MAX_ND_LEVEL 24   /* etree.cpp:16 */

static char g_err[512];
const char* mpo_last_error(void) { return g_err; }
static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return 1;
}

/* ---------------------------------------------------------------- helpers */
typedef struct {
  int32_t* a;
  int64_t n, cap;
} ivec;
static void iv_push(ivec* v, int32_t x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? v->cap * 2 : 8;
    v->a = (int32_t*)realloc(v->a, sizeof(int32_t) * v->cap);
  }
  v->a[v->n++] = x;
}
static void iv_free(ivec* v) {
  free(v->a);
  v->a = NULL;
  v->n = v->cap = 0;
}
static int cmp_i32(const void* x, const void* y) {
  int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
  return (a > b) - (a < b);
}
static int cmp_u64(const void* x, const void* y) {
  uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
  return (a > b) - (a < b);
}
static void* xcalloc(size_t n, size_t s) { return calloc(n ? n : 1, s); }

/* partition.cpp:15-21 */
static double imbalance_of(int64_t a, int64_t b) {
  if (a == 0 && b == 0) return 1.0;
  if (a == 0 || b == 0) return INFINITY;
  double hi = (double)(a > b ? a : b), lo = (double)(a < b ? a : b);
  return hi / lo;
}

/* ------------------------------------------------------- graph construction */
/* graph.cpp:14-46 graph_from_edges, fed by mesh_to_graph (graph.cpp:63-75). */
int mpo_graph_from_triangles(int32_t nv, int64_t ntri, const int32_t* tris, int32_t* off,
                             int32_t* nbr, int64_t* nnz) {
  for (int64_t t = 0; t < ntri; ++t) {
    const int32_t* c = tris + 3 * t;
    for (int k = 0; k < 3; ++k)
      if (c[k] < 0 || c[k] >= nv) return fail("triangle %lld references vertex %d", (long long)t, c[k]);
    if (c[0] == c[1] || c[1] == c[2] || c[0] == c[2])
      return fail("triangle %lld has repeated corners", (long long)t);
  }
  int64_t* cnt = (int64_t*)xcalloc((size_t)nv + 1, sizeof(int64_t));
  for (int64_t t = 0; t < ntri; ++t) {
    const int32_t* c = tris + 3 * t;
    cnt[c[0] + 1] += 2;
    cnt[c[1] + 1] += 2;
    cnt[c[2] + 1] += 2;
  }
  for (int32_t v = 0; v < nv; ++v) cnt[v + 1] += cnt[v];
  int32_t* raw = (int32_t*)xcalloc((size_t)cnt[nv], sizeof(int32_t));
  int64_t* cur = (int64_t*)xcalloc((size_t)nv + 1, sizeof(int64_t));
  memcpy(cur, cnt, sizeof(int64_t) * nv);
  for (int64_t t = 0; t < ntri; ++t) {
    const int32_t* c = tris + 3 * t;
    static const int pr[3][2] = {{0, 1}, {1, 2}, {0, 2}};
    for (int e = 0; e < 3; ++e) {
      int32_t u = c[pr[e][0]], w = c[pr[e][1]];
      raw[cur[u]++] = w;
      raw[cur[w]++] = u;
    }
  }
  int64_t write = 0;
  for (int32_t v = 0; v < nv; ++v) {
    int64_t b = cnt[v], e = cnt[v + 1];
    qsort(raw + b, (size_t)(e - b), sizeof(int32_t), cmp_i32);
    off[v] = (int32_t)write;
    for (int64_t i = b; i < e; ++i)
      if (i == b || raw[i] != raw[i - 1]) {
        if (nbr) nbr[write] = raw[i];
        ++write;
      }
  }
  off[nv] = (int32_t)write;
  *nnz = write;
  free(cnt);
  free(raw);
  free(cur);
  return 0;
}

/* etree.cpp:42-46 */
int32_t mpo_default_nd_level(int32_t n) {
  int32_t level = 0;
  for (int32_t x = n / 512; x > 1; x >>= 1) ++level;
  return level < 8 ? level : 8;
}

/* ------------------------------------------------------------- patching */
/* patching.cpp:17-22 */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d649bb133111ebULL;
  return x ^ (x >> 31);
}

typedef struct {
  int32_t n;
  const int32_t* off;
  const int32_t* nbr;
} graph_t;

/* patching.cpp:26-65 farthest_point_seeds */
static void fps_seeds(const graph_t* g, const int32_t* comp, int32_t csize, int32_t k,
                      uint64_t seed, int32_t* dist, int32_t* queue, int32_t* seeds) {
  for (int32_t i = 0; i < csize; ++i) dist[comp[i]] = UNREACHED;
  int32_t cur = comp[splitmix64(seed) % (uint64_t)csize];
  for (int32_t s = 0; s < k; ++s) {
    if (s > 0) { /* argmax of dist over comp, ties to the lower id (:52-60) */
      int32_t best = NONE, best_d = -1;
      for (int32_t i = 0; i < csize; ++i)
        if (dist[comp[i]] > best_d) best_d = dist[comp[i]], best = comp[i];
      cur = best;
    }
    seeds[s] = cur;
    /* relax_from (:35-49) */
    int64_t head = 0, tail = 0;
    dist[cur] = 0;
    queue[tail++] = cur;
    while (head < tail) {
      int32_t u = queue[head++], du = dist[u];
      for (int32_t j = g->off[u]; j < g->off[u + 1]; ++j) {
        int32_t w = g->nbr[j];
        if (du + 1 < dist[w]) {
          dist[w] = du + 1;
          queue[tail++] = w;
        }
      }
    }
  }
}

/* patching.cpp:69-99 assign_to_seeds: multi-source BFS, distance ties go to
 * the lower patch label. */
static void assign_seeds(const graph_t* g, const int32_t* comp, int32_t csize, const int32_t* seeds,
                         int32_t k, int32_t* dist, int32_t* label, int32_t* fr, int32_t* nx) {
  for (int32_t i = 0; i < csize; ++i) dist[comp[i]] = UNREACHED, label[comp[i]] = NONE;
  int32_t nf = 0;
  for (int32_t p = 0; p < k; ++p) {
    dist[seeds[p]] = 0;
    label[seeds[p]] = p;
    fr[nf++] = seeds[p];
  }
  while (nf > 0) {
    int32_t nn = 0;
    for (int32_t i = 0; i < nf; ++i) {
      int32_t u = fr[i], du = dist[u];
      for (int32_t j = g->off[u]; j < g->off[u + 1]; ++j) {
        int32_t w = g->nbr[j];
        if (dist[w] == UNREACHED) {
          dist[w] = du + 1;
          label[w] = label[u];
          nx[nn++] = w;
        } else if (dist[w] == du + 1 && label[u] < label[w]) {
          label[w] = label[u];
        }
      }
    }
    memcpy(fr, nx, sizeof(int32_t) * nn);
    nf = nn;
  }
}

/* patching.cpp:103-139 recenter_seeds */
static void recenter(const graph_t* g, const int32_t* comp, int32_t csize, const int32_t* label,
                     int32_t* seeds, int32_t k, int32_t* depth, int32_t* fr, int32_t* nx) {
  int32_t nf = 0;
  for (int32_t i = 0; i < csize; ++i) depth[comp[i]] = UNREACHED;
  for (int32_t i = 0; i < csize; ++i) {
    int32_t v = comp[i];
    for (int32_t j = g->off[v]; j < g->off[v + 1]; ++j)
      if (label[g->nbr[j]] != label[v]) {
        depth[v] = 0;
        fr[nf++] = v;
        break;
      }
  }
  while (nf > 0) {
    int32_t nn = 0;
    for (int32_t i = 0; i < nf; ++i) {
      int32_t u = fr[i];
      for (int32_t j = g->off[u]; j < g->off[u + 1]; ++j) {
        int32_t w = g->nbr[j];
        if (label[w] == label[u] && depth[w] == UNREACHED) {
          depth[w] = depth[u] + 1;
          nx[nn++] = w;
        }
      }
    }
    memcpy(fr, nx, sizeof(int32_t) * nn);
    nf = nn;
  }
  int32_t* best = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
  for (int32_t p = 0; p < k; ++p) best[p] = -1;
  for (int32_t i = 0; i < csize; ++i) {
    int32_t v = comp[i];
    if (depth[v] == UNREACHED) continue;
    int32_t p = label[v];
    if (depth[v] > best[p]) best[p] = depth[v], seeds[p] = v;
  }
  free(best);
}

/* patching.cpp:149-291 repair_sizes */
static void repair_sizes(const graph_t* g, int32_t* assign, int32_t* pcount, int32_t target) {
  const int64_t low = ((int64_t)target + 1) / 2, high = 2 * (int64_t)target;
  int32_t P = *pcount, cap = P + 16;
  int64_t* size = (int64_t*)xcalloc((size_t)cap, sizeof(int64_t));
  ivec* mem = (ivec*)xcalloc((size_t)cap, sizeof(ivec));
  char* exempt = (char*)xcalloc((size_t)cap, 1);
  for (int32_t v = 0; v < g->n; ++v) {
    ++size[assign[v]];
    iv_push(&mem[assign[v]], v);
  }
  int32_t* dist = (int32_t*)malloc(sizeof(int32_t) * (size_t)g->n);
  int32_t* lab2 = (int32_t*)malloc(sizeof(int32_t) * (size_t)g->n);
  int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)g->n);
  int32_t* nx = (int32_t*)malloc(sizeof(int32_t) * (size_t)g->n);
  for (int32_t v = 0; v < g->n; ++v) dist[v] = UNREACHED, lab2[v] = NONE;

  const int max_iter = 4 * P + 64;
  for (int iter = 0; iter < max_iter; ++iter) {
    /* smallest mergeable patch, ties to the lower id (:190-197) */
    int32_t mp = NONE;
    for (int32_t p = 0; p < P; ++p) {
      if (size[p] <= 0 || size[p] >= low || exempt[p]) continue;
      if (mp == NONE || size[p] < size[mp]) mp = p;
    }
    if (mp != NONE) { /* merge into the smallest neighbouring patch (:198-221) */
      int32_t tgt = NONE;
      for (int64_t i = 0; i < mem[mp].n; ++i) {
        int32_t v = mem[mp].a[i];
        for (int32_t j = g->off[v]; j < g->off[v + 1]; ++j) {
          int32_t qq = assign[g->nbr[j]];
          if (qq == mp) continue;
          if (tgt == NONE || size[qq] < size[tgt] || (size[qq] == size[tgt] && qq < tgt)) tgt = qq;
        }
      }
      if (tgt == NONE) {
        exempt[mp] = 1;
        continue;
      }
      for (int64_t i = 0; i < mem[mp].n; ++i) {
        assign[mem[mp].a[i]] = tgt;
        iv_push(&mem[tgt], mem[mp].a[i]);
      }
      size[tgt] += size[mp];
      size[mp] = 0;
      iv_free(&mem[mp]);
      continue;
    }
    /* largest oversized patch (:222-230) */
    int32_t sp = NONE;
    for (int32_t p = 0; p < P; ++p) {
      if (size[p] <= high) continue;
      if (sp == NONE || size[p] > size[sp]) sp = p;
    }
    if (sp == NONE) break;
    /* farthest pair by two restricted BFS sweeps (:165-185, :231-233) */
    int32_t ends[3];
    ends[0] = mem[sp].a[0];
    for (int64_t i = 1; i < mem[sp].n; ++i)
      if (mem[sp].a[i] < ends[0]) ends[0] = mem[sp].a[i];
    for (int sweep = 1; sweep <= 2; ++sweep) {
      int32_t from = ends[sweep - 1];
      for (int64_t i = 0; i < mem[sp].n; ++i) dist[mem[sp].a[i]] = UNREACHED;
      dist[from] = 0;
      int64_t h = 0, t = 0;
      q[t++] = from;
      int32_t far = from, far_d = 0;
      while (h < t) {
        int32_t u = q[h++];
        for (int32_t j = g->off[u]; j < g->off[u + 1]; ++j) {
          int32_t w = g->nbr[j];
          if (assign[w] == sp && dist[w] == UNREACHED) {
            dist[w] = dist[u] + 1;
            if (dist[w] > far_d || (dist[w] == far_d && w < far)) far_d = dist[w], far = w;
            q[t++] = w;
          }
        }
      }
      ends[sweep] = far;
    }
    int32_t b = ends[1], c = ends[2];
    /* two-source competition, ties to b's half (:234-261) */
    for (int64_t i = 0; i < mem[sp].n; ++i) dist[mem[sp].a[i]] = UNREACHED, lab2[mem[sp].a[i]] = NONE;
    dist[b] = 0, lab2[b] = 0, dist[c] = 0, lab2[c] = 1;
    int32_t nf = 0;
    q[nf++] = b;
    q[nf++] = c;
    while (nf > 0) {
      int32_t nn = 0;
      for (int32_t i = 0; i < nf; ++i) {
        int32_t u = q[i];
        for (int32_t j = g->off[u]; j < g->off[u + 1]; ++j) {
          int32_t w = g->nbr[j];
          if (assign[w] != sp) continue;
          if (dist[w] == UNREACHED) {
            dist[w] = dist[u] + 1;
            lab2[w] = lab2[u];
            nx[nn++] = w;
          } else if (dist[w] == dist[u] + 1 && lab2[u] < lab2[w]) {
            lab2[w] = lab2[u];
          }
        }
      }
      memcpy(q, nx, sizeof(int32_t) * nn);
      nf = nn;
    }
    /* fresh id for label-1 half (:262-279) */
    if (P == cap) {
      int32_t nc = cap * 2;
      size = (int64_t*)realloc(size, sizeof(int64_t) * nc);
      mem = (ivec*)realloc(mem, sizeof(ivec) * nc);
      exempt = (char*)realloc(exempt, nc);
      memset(size + cap, 0, sizeof(int64_t) * (nc - cap));
      memset(mem + cap, 0, sizeof(ivec) * (nc - cap));
      memset(exempt + cap, 0, nc - cap);
      cap = nc;
    }
    int32_t fresh = P++;
    ivec keep = {0, 0, 0};
    for (int64_t i = 0; i < mem[sp].n; ++i) {
      int32_t v = mem[sp].a[i];
      if (lab2[v] == 1) {
        assign[v] = fresh;
        iv_push(&mem[fresh], v);
      } else {
        iv_push(&keep, v);
      }
    }
    size[fresh] = mem[fresh].n;
    size[sp] = keep.n;
    iv_free(&mem[sp]);
    mem[sp] = keep;
  }
  /* compact ids ascending (:282-290) */
  int32_t* remap = (int32_t*)malloc(sizeof(int32_t) * (size_t)P);
  int32_t dense = 0;
  for (int32_t p = 0; p < P; ++p) remap[p] = size[p] > 0 ? dense++ : NONE;
  for (int32_t v = 0; v < g->n; ++v) assign[v] = remap[assign[v]];
  *pcount = dense;
  for (int32_t p = 0; p < P; ++p) iv_free(&mem[p]);
  free(remap), free(size), free(mem), free(exempt), free(dist), free(lab2), free(q), free(nx);
}

/* patching.cpp:347-384 enforce_connectivity */
int mpo_enforce_connectivity(int32_t n, const int32_t* off, const int32_t* nbr,
                             const int32_t* assignment, int32_t patch_count, int32_t* out,
                             int32_t* out_count) {
  for (int32_t v = 0; v < n; ++v)
    if (assignment[v] < 0 || assignment[v] >= patch_count)
      return fail("patch id out of range at vertex %d", v);
  /* members per patch, ascending: counting sort */
  int32_t* start = (int32_t*)xcalloc((size_t)patch_count + 1, sizeof(int32_t));
  for (int32_t v = 0; v < n; ++v) ++start[assignment[v] + 1];
  for (int32_t p = 0; p < patch_count; ++p) start[p + 1] += start[p];
  int32_t* members = (int32_t*)xcalloc((size_t)n, sizeof(int32_t));
  int32_t* cur = (int32_t*)xcalloc((size_t)patch_count + 1, sizeof(int32_t));
  memcpy(cur, start, sizeof(int32_t) * patch_count);
  for (int32_t v = 0; v < n; ++v) members[cur[assignment[v]]++] = v;
  char* seen = (char*)xcalloc((size_t)n, 1);
  int32_t* queue = (int32_t*)xcalloc((size_t)n, sizeof(int32_t));
  int32_t count = patch_count;
  memcpy(out, assignment, sizeof(int32_t) * n);
  for (int32_t p = 0; p < patch_count; ++p) {
    int first = 1;
    for (int32_t i = start[p]; i < start[p + 1]; ++i) {
      int32_t root = members[i];
      if (seen[root]) continue;
      int32_t id = first ? p : count++;
      first = 0;
      int32_t h = 0, t = 0;
      queue[t++] = root;
      seen[root] = 1;
      while (h < t) {
        int32_t v = queue[h++];
        out[v] = id;
        for (int32_t j = off[v]; j < off[v + 1]; ++j) {
          int32_t w = nbr[j];
          if (!seen[w] && assignment[w] == p) seen[w] = 1, queue[t++] = w;
        }
      }
    }
  }
  *out_count = count;
  free(start), free(members), free(cur), free(seen), free(queue);
  return 0;
}

/* patching.cpp:295-345 compute_patches (components from graph.cpp:183-205) */
int mpo_compute_patches(int32_t n, const int32_t* off, const int32_t* nbr, int32_t target,
                        uint64_t seed, int32_t* assignment, int32_t* patch_count) {
  if (target < 1) return fail("target patch size must be positive");
  *patch_count = 0;
  if (n == 0) return 0;
  graph_t g = {n, off, nbr};
  int32_t *dist = malloc(sizeof(int32_t) * n), *label = malloc(sizeof(int32_t) * n),
          *prev = malloc(sizeof(int32_t) * n), *depth = malloc(sizeof(int32_t) * n),
          *fr = malloc(sizeof(int32_t) * n), *nx = malloc(sizeof(int32_t) * n),
          *comp = malloc(sizeof(int32_t) * n);
  char* seen = (char*)xcalloc((size_t)n, 1);
  int32_t pc = 0;
  for (int32_t root = 0; root < n; ++root) {
    if (seen[root]) continue;
    /* connected_components: BFS then ascending sort */
    int32_t h = 0, t = 0;
    comp[t++] = root;
    seen[root] = 1;
    while (h < t) {
      int32_t v = comp[h++];
      for (int32_t j = off[v]; j < off[v + 1]; ++j)
        if (!seen[nbr[j]]) seen[nbr[j]] = 1, comp[t++] = nbr[j];
    }
    qsort(comp, (size_t)t, sizeof(int32_t), cmp_i32);
    int32_t cs = t;
    long long kk = llround((double)cs / (double)target);
    int32_t k = (int32_t)kk;
    if (k < 1) k = 1;
    int32_t base = pc;
    if (k >= cs) {
      for (int32_t i = 0; i < cs; ++i) assignment[comp[i]] = base + i;
      pc += cs;
      continue;
    }
    if (k == 1) {
      for (int32_t i = 0; i < cs; ++i) assignment[comp[i]] = base;
      pc += 1;
      continue;
    }
    int32_t* seeds = (int32_t*)malloc(sizeof(int32_t) * k);
    fps_seeds(&g, comp, cs, k, seed, dist, fr, seeds);
    for (int32_t i = 0; i < cs; ++i) prev[comp[i]] = NONE;
    for (int round = 0; round < LLOYD_ROUNDS; ++round) {
      assign_seeds(&g, comp, cs, seeds, k, dist, label, fr, nx);
      int stable = 1;
      for (int32_t i = 0; i < cs && stable; ++i)
        if (label[comp[i]] != prev[comp[i]]) stable = 0;
      if (stable) break;
      for (int32_t i = 0; i < cs; ++i) prev[comp[i]] = label[comp[i]];
      recenter(&g, comp, cs, label, seeds, k, depth, fr, nx);
    }
    for (int32_t i = 0; i < cs; ++i) assignment[comp[i]] = base + prev[comp[i]];
    pc += k;
    free(seeds);
  }
  int32_t* conn = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t pc2 = 0;
  int rc = mpo_enforce_connectivity(n, off, nbr, assignment, pc, conn, &pc2);
  if (rc == 0) {
    memcpy(assignment, conn, sizeof(int32_t) * n);
    repair_sizes(&g, assignment, &pc2, target);
    *patch_count = pc2;
  }
  free(conn), free(dist), free(label), free(prev), free(depth), free(fr), free(nx), free(comp),
      free(seen);
  return rc;
}

/* ------------------------------------------------------------- quotient */
/* QuotientGraph (quotient.hpp:17-37) as a symmetric patch CSR with weights;
 * a zero weight plays the role of an erased map entry. */
typedef struct {
  int32_t P;
  int64_t* node_w;
  int32_t* qoff; /* P+1 */
  int32_t* qnbr; /* sorted per patch */
  int64_t* qw;   /* weight of (p, qnbr[j]) */
  char* alive_v; /* per vertex */
} quotient_t;

static int64_t* q_edge_ref(quotient_t* q, int32_t p, int32_t r) {
  int32_t lo = q->qoff[p], hi = q->qoff[p + 1];
  while (lo < hi) {
    int32_t mid = (lo + hi) / 2;
    if (q->qnbr[mid] < r) lo = mid + 1;
    else hi = mid;
  }
  return (lo < q->qoff[p + 1] && q->qnbr[lo] == r) ? &q->qw[lo] : NULL;
}

/* quotient.cpp:47-80 build_quotient */
static int build_quotient(const graph_t* g, const int32_t* assign, int32_t P, quotient_t* q) {
  q->P = P;
  q->node_w = (int64_t*)xcalloc((size_t)P, sizeof(int64_t));
  q->alive_v = (char*)malloc((size_t)g->n + 1);
  memset(q->alive_v, 1, (size_t)g->n);
  for (int32_t v = 0; v < g->n; ++v) {
    if (assign[v] < 0 || assign[v] >= P)
      return fail("patch id %d out of range for vertex %d", assign[v], v);
    ++q->node_w[assign[v]];
  }
  /* crossing edges keyed (min,max), sorted: equal keys become one weighted entry */
  int64_t m = 0;
  for (int32_t u = 0; u < g->n; ++u)
    for (int32_t j = g->off[u]; j < g->off[u + 1]; ++j)
      if (g->nbr[j] > u && assign[g->nbr[j]] != assign[u]) ++m;
  uint64_t* keys = (uint64_t*)xcalloc((size_t)m, sizeof(uint64_t));
  m = 0;
  for (int32_t u = 0; u < g->n; ++u)
    for (int32_t j = g->off[u]; j < g->off[u + 1]; ++j) {
      int32_t v = g->nbr[j];
      if (v <= u) continue;
      int32_t a = assign[u], b = assign[v];
      if (a == b) continue;
      if (a > b) { int32_t t = a; a = b; b = t; }
      keys[m++] = ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
    }
  qsort(keys, (size_t)m, sizeof(uint64_t), cmp_u64);
  q->qoff = (int32_t*)xcalloc((size_t)P + 1, sizeof(int32_t));
  int64_t u_cnt = 0;
  for (int64_t i = 0; i < m; ++i)
    if (i == 0 || keys[i] != keys[i - 1]) {
      ++q->qoff[(keys[i] >> 32) + 1];
      ++q->qoff[(keys[i] & 0xffffffffu) + 1];
      ++u_cnt;
    }
  for (int32_t p = 0; p < P; ++p) q->qoff[p + 1] += q->qoff[p];
  q->qnbr = (int32_t*)xcalloc((size_t)2 * u_cnt, sizeof(int32_t));
  q->qw = (int64_t*)xcalloc((size_t)2 * u_cnt, sizeof(int64_t));
  int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * ((size_t)P + 1));
  memcpy(cur, q->qoff, sizeof(int32_t) * P);
  /* keys ascend in (a,b): a's list receives b ascending; b's list receives a
     ascending too because for a fixed b the a values arrive in order */
  for (int64_t i = 0; i < m;) {
    int64_t j = i;
    while (j < m && keys[j] == keys[i]) ++j;
    int32_t a = (int32_t)(keys[i] >> 32), b = (int32_t)(keys[i] & 0xffffffffu);
    q->qnbr[cur[a]] = b, q->qw[cur[a]++] = j - i;
    q->qnbr[cur[b]] = a, q->qw[cur[b]++] = j - i;
    i = j;
  }
  free(cur);
  free(keys);
  /* each list must be sorted: b-side entries were appended in ascending a
     order but interleave with a-side entries; sort pairs per list */
  for (int32_t p = 0; p < P; ++p) {
    int32_t b = q->qoff[p], e = q->qoff[p + 1];
    for (int32_t i = b + 1; i < e; ++i) { /* insertion sort, short lists */
      int32_t kn = q->qnbr[i];
      int64_t kw = q->qw[i];
      int32_t j = i - 1;
      while (j >= b && q->qnbr[j] > kn) q->qnbr[j + 1] = q->qnbr[j], q->qw[j + 1] = q->qw[j], --j;
      q->qnbr[j + 1] = kn, q->qw[j + 1] = kw;
    }
  }
  return 0;
}

static void free_quotient(quotient_t* q) {
  free(q->node_w), free(q->qoff), free(q->qnbr), free(q->qw), free(q->alive_v);
}

int mpo_build_quotient(int32_t n, const int32_t* off, const int32_t* nbr,
                       const int32_t* assignment, int32_t patch_count, int64_t* node_weight,
                       int32_t* edge_p, int32_t* edge_q, int64_t* edge_w, int64_t* n_edges) {
  graph_t g = {n, off, nbr};
  quotient_t q;
  memset(&q, 0, sizeof q);
  int rc = build_quotient(&g, assignment, patch_count, &q);
  if (rc) return rc;
  if (node_weight) memcpy(node_weight, q.node_w, sizeof(int64_t) * patch_count);
  int64_t ne = 0;
  for (int32_t p = 0; p < patch_count; ++p)
    for (int32_t j = q.qoff[p]; j < q.qoff[p + 1]; ++j)
      if (q.qnbr[j] > p && q.qw[j] > 0) {
        if (edge_p) edge_p[ne] = p, edge_q[ne] = q.qnbr[j], edge_w[ne] = q.qw[j];
        ++ne;
      }
  *n_edges = ne;
  free_quotient(&q);
  return 0;
}

/* quotient.cpp:82-103 quotient_remove */
static int quotient_remove(quotient_t* q, const graph_t* g, const int32_t* assign,
                           const int32_t* removed, int32_t nr) {
  for (int32_t i = 0; i < nr; ++i) {
    int32_t v = removed[i];
    if (!q->alive_v[v]) return fail("vertex %d removed twice from quotient", v);
    int32_t pv = assign[v];
    for (int32_t j = g->off[v]; j < g->off[v + 1]; ++j) {
      int32_t w = g->nbr[j];
      if (!q->alive_v[w]) continue;
      int32_t pw = assign[w];
      if (pw == pv) continue;
      int64_t* a = q_edge_ref(q, pv, pw);
      int64_t* b = q_edge_ref(q, pw, pv);
      if (a && *a > 0) --*a, --*b;
    }
    q->alive_v[v] = 0;
    --q->node_w[pv];
  }
  return 0;
}

/* ------------------------------------------------------------- partition */
typedef struct {
  int32_t P;        /* patch-id space */
  int32_t na;       /* alive patches (ascending) */
  int32_t* alive;
  int32_t* aoff;    /* adjacency among alive patches, per alive index */
  int32_t* anbr;    /* neighbour PATCH ids, ascending */
  int64_t* aw;
} localq_t;

/* restrict_quotient (quotient.cpp:105-127) followed by the adjacency that
 * bipartition_quotient derives from it (partition.cpp:41-51). */
static void restrict_local(const quotient_t* m, const int32_t* patches, int32_t np, char* owned,
                           localq_t* out) {
  out->P = m->P;
  for (int32_t i = 0; i < np; ++i) owned[patches[i]] = 1;
  out->alive = (int32_t*)malloc(sizeof(int32_t) * (np + 1));
  out->na = 0;
  for (int32_t i = 0; i < np; ++i)
    if (m->node_w[patches[i]] > 0) out->alive[out->na++] = patches[i];
  out->aoff = (int32_t*)xcalloc((size_t)out->na + 1, sizeof(int32_t));
  int64_t tot = 0;
  for (int32_t i = 0; i < out->na; ++i) {
    int32_t p = out->alive[i];
    for (int32_t j = m->qoff[p]; j < m->qoff[p + 1]; ++j) {
      int32_t r = m->qnbr[j];
      if (owned[r] && m->qw[j] > 0 && m->node_w[r] > 0) ++tot;
    }
  }
  out->anbr = (int32_t*)xcalloc((size_t)tot, sizeof(int32_t));
  out->aw = (int64_t*)xcalloc((size_t)tot, sizeof(int64_t));
  tot = 0;
  for (int32_t i = 0; i < out->na; ++i) {
    int32_t p = out->alive[i];
    out->aoff[i] = (int32_t)tot;
    for (int32_t j = m->qoff[p]; j < m->qoff[p + 1]; ++j) {
      int32_t r = m->qnbr[j];
      if (owned[r] && m->qw[j] > 0 && m->node_w[r] > 0) out->anbr[tot] = r, out->aw[tot++] = m->qw[j];
    }
  }
  out->aoff[out->na] = (int32_t)tot;
  for (int32_t i = 0; i < np; ++i) owned[patches[i]] = 0;
}
static void free_localq(localq_t* l) { free(l->alive), free(l->aoff), free(l->anbr), free(l->aw); }

/* partition.cpp:25-163 bipartition_quotient.  side[] is indexed by patch id
 * (0 left, 1 right); aidx maps patch id -> alive index (scratch, -1 else). */
static void bipartition(const localq_t* l, const int64_t* node_w, double tol, uint8_t* side,
                        int32_t* aidx) {
  const int32_t na = l->na;
  for (int32_t i = 0; i < na; ++i) side[l->alive[i]] = 1, aidx[l->alive[i]] = i;
  if (na == 1) {
    side[l->alive[0]] = 0;
    aidx[l->alive[0]] = -1;
    return;
  }
  int64_t total = 0;
  for (int32_t i = 0; i < na; ++i) total += node_w[l->alive[i]];
  /* grow order: weight desc, id asc (:54-59); insertion into a sorted index */
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * na);
  for (int32_t i = 0; i < na; ++i) order[i] = i;
  for (int32_t i = 1; i < na; ++i) { /* stable insertion by weight desc keeps id asc */
    int32_t x = order[i], j = i - 1;
    while (j >= 0 && node_w[l->alive[order[j]]] < node_w[l->alive[x]]) order[j + 1] = order[j], --j;
    order[j + 1] = x;
  }
  char* visited = (char*)xcalloc((size_t)na, 1);
  ivec fifo = {0, 0, 0};
  int64_t head = 0, sp = 0, left_w = 0;
  while (left_w * 2 < total) { /* :64-78 */
    int32_t u;
    while (head < fifo.n && visited[fifo.a[head]]) ++head;
    if (head < fifo.n) u = fifo.a[head++];
    else {
      while (visited[order[sp]]) ++sp;
      u = order[sp];
    }
    visited[u] = 1;
    side[l->alive[u]] = 0;
    left_w += node_w[l->alive[u]];
    for (int32_t j = l->aoff[u]; j < l->aoff[u + 1]; ++j)
      if (!visited[aidx[l->anbr[j]]]) iv_push(&fifo, aidx[l->anbr[j]]);
  }
  int64_t sw[2] = {left_w, total - left_w};
  int64_t cut = 0;
  for (int32_t i = 0; i < na; ++i)
    for (int32_t j = l->aoff[i]; j < l->aoff[i + 1]; ++j)
      if (l->anbr[j] > l->alive[i] && side[l->anbr[j]] != side[l->alive[i]]) cut += l->aw[j];

  int64_t* gain = (int64_t*)malloc(sizeof(int64_t) * na);
  char* locked = (char*)malloc(na);
  int32_t* mv = (int32_t*)malloc(sizeof(int32_t) * na);
  int64_t* mv_cut = (int64_t*)malloc(sizeof(int64_t) * na);
  int64_t* mv_sw = (int64_t*)malloc(sizeof(int64_t) * 2 * na);
  for (int pass = 0; pass < FM_PASSES; ++pass) { /* :95-159 */
    for (int32_t i = 0; i < na; ++i) {
      locked[i] = 0;
      int64_t val = 0;
      uint8_t s = side[l->alive[i]];
      for (int32_t j = l->aoff[i]; j < l->aoff[i + 1]; ++j)
        val += side[l->anbr[j]] != s ? l->aw[j] : -l->aw[j];
      gain[i] = val;
    }
    const int64_t pass_cut = cut;
    const double pass_imb = imbalance_of(sw[0], sw[1]);
    int64_t best_cut = pass_cut;
    double best_imb = pass_imb;
    int32_t nm = 0, best_len = 0;
    for (;;) {
      double cur_imb = imbalance_of(sw[0], sw[1]);
      double thr = tol > cur_imb ? tol : cur_imb;
      /* first feasible entry of the (-gain, id) set == the feasible unlocked
         patch of largest gain, lowest id */
      int32_t ch = -1;
      for (int32_t i = 0; i < na; ++i) {
        if (locked[i]) continue;
        if (ch >= 0 && gain[i] <= gain[ch]) continue;
        int32_t s = side[l->alive[i]];
        int64_t w = node_w[l->alive[i]], ns = sw[s] - w, nt = sw[1 - s] + w;
        if (ns <= 0) continue;
        if (imbalance_of(ns, nt) > thr) continue;
        ch = i;
      }
      if (ch < 0) break;
      locked[ch] = 1;
      mv[nm] = ch, mv_cut[nm] = cut, mv_sw[2 * nm] = sw[0], mv_sw[2 * nm + 1] = sw[1];
      ++nm;
      int32_t s = side[l->alive[ch]];
      sw[s] -= node_w[l->alive[ch]];
      sw[1 - s] += node_w[l->alive[ch]];
      side[l->alive[ch]] = (uint8_t)(1 - s);
      cut -= gain[ch];
      for (int32_t j = l->aoff[ch]; j < l->aoff[ch + 1]; ++j) {
        int32_t nb = aidx[l->anbr[j]];
        if (locked[nb]) continue;
        gain[nb] += side[l->anbr[j]] == side[l->alive[ch]] ? -2 * l->aw[j] : 2 * l->aw[j];
      }
      double imb = imbalance_of(sw[0], sw[1]);
      if (cut < best_cut || (cut == best_cut && imb < best_imb))
        best_cut = cut, best_imb = imb, best_len = nm;
    }
    while (nm > best_len) {
      --nm;
      side[l->alive[mv[nm]]] ^= 1;
      sw[0] = mv_sw[2 * nm], sw[1] = mv_sw[2 * nm + 1];
      cut = mv_cut[nm];
    }
    int improved = best_cut < pass_cut || (best_cut == pass_cut && best_imb < pass_imb);
    if (!improved) break;
  }
  for (int32_t i = 0; i < na; ++i) aidx[l->alive[i]] = -1;
  free(order), free(visited), iv_free(&fifo), free(gain), free(locked), free(mv), free(mv_cut),
      free(mv_sw);
}

/* sorted-set helpers for refine's std::set<index_t> sep */
static int64_t lower_bound_i32(const int32_t* a, int64_t n, int32_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* partition.cpp:165-185 super_separator + :187-283 refine_separator, on the
 * subgraph induced by the vertices with in_node[v] == tok (ascending list
 * verts).  Outputs sep/left/right ascending (global ids). */
static void separate(const graph_t* g, const int32_t* verts, int32_t nvert, const int32_t* in_node,
                     int32_t tok, const int32_t* assign, const uint8_t* side, double tol,
                     uint8_t* region, ivec* sep, ivec* left, ivec* right) {
  /* super separator: endpoints of crossing edges (:165-185) */
  ivec super = {0, 0, 0};
  for (int32_t i = 0; i < nvert; ++i) {
    int32_t u = verts[i];
    uint8_t su = side[assign[u]];
    region[u] = su;
    for (int32_t j = g->off[u]; j < g->off[u + 1]; ++j) {
      int32_t w = g->nbr[j];
      if (in_node[w] != tok) continue;
      if (side[assign[w]] != su) {
        iv_push(&super, u);
        break;
      }
    }
  }
  /* initial separator: the smaller boundary, ties to the left (:212-222) */
  int64_t bl = 0, br = 0;
  for (int64_t i = 0; i < super.n; ++i) {
    if (region[super.a[i]] == 0) ++bl;
    else ++br;
  }
  uint8_t take = bl <= br ? 0 : 1;
  sep->n = 0;
  for (int64_t i = 0; i < super.n; ++i)
    if (region[super.a[i]] == take) iv_push(sep, super.a[i]);
  for (int64_t i = 0; i < sep->n; ++i) region[sep->a[i]] = 2;
  int64_t rw[2] = {0, 0};
  for (int32_t i = 0; i < nvert; ++i)
    if (region[verts[i]] < 2) ++rw[region[verts[i]]];
  int64_t cur_size = sep->n;
  double cur_imb = imbalance_of(rw[0], rw[1]);
  for (;;) { /* greedy moves (:235-274) */
    int32_t mvv = NONE;
    uint8_t move_to = 0;
    int64_t best_size = cur_size;
    double best_imb = cur_imb;
    double thr = tol > cur_imb ? tol : cur_imb;
    for (int64_t i = 0; i < sep->n; ++i) {
      int32_t v = sep->a[i];
      uint8_t own = side[assign[v]], opp = 1 - own;
      int64_t pull = 0;
      for (int32_t j = g->off[v]; j < g->off[v + 1]; ++j) {
        int32_t w = g->nbr[j];
        if (in_node[w] == tok && region[w] == opp) ++pull;
      }
      int64_t ns = cur_size - 1 + pull;
      if (ns > cur_size) continue;
      double ni = imbalance_of(rw[own] + 1, rw[opp] - pull);
      if (ni > thr) continue;
      if (!(ns < cur_size || ni < cur_imb)) continue;
      if (ns < best_size || (ns == best_size && ni < best_imb))
        best_size = ns, best_imb = ni, mvv = v, move_to = own;
    }
    if (mvv == NONE) break;
    uint8_t opp = 1 - move_to;
    int64_t at = lower_bound_i32(sep->a, sep->n, mvv);
    memmove(sep->a + at, sep->a + at + 1, sizeof(int32_t) * (sep->n - at - 1));
    --sep->n;
    region[mvv] = move_to;
    ++rw[move_to];
    for (int32_t j = g->off[mvv]; j < g->off[mvv + 1]; ++j) {
      int32_t w = g->nbr[j];
      if (in_node[w] != tok || region[w] != opp) continue;
      region[w] = 2;
      iv_push(sep, 0);
      int64_t pos = lower_bound_i32(sep->a, sep->n - 1, w);
      memmove(sep->a + pos + 1, sep->a + pos, sizeof(int32_t) * (sep->n - 1 - pos));
      sep->a[pos] = w;
      --rw[opp];
    }
    cur_size = sep->n;
    cur_imb = imbalance_of(rw[0], rw[1]);
  }
  left->n = right->n = 0;
  for (int32_t i = 0; i < nvert; ++i) {
    int32_t v = verts[i];
    if (region[v] == 0) iv_push(left, v);
    else if (region[v] == 1) iv_push(right, v);
  }
  iv_free(&super);
}

/* ------------------------------------------------------------- ND tree */
typedef struct {
  const graph_t* g;
  const int32_t* assign;
  quotient_t* master;
  int32_t L;
  ivec* nodes;      /* vertex list per tree node */
  int32_t* in_node; /* token per vertex */
  int32_t tok;
  uint8_t* side;
  int32_t* aidx;
  char* owned;
  uint8_t* region;
  char* pmark;
  int rc;
} etree_ctx;

static int floor_log2(int64_t x) {
  int l = -1;
  while (x) ++l, x >>= 1;
  return l;
}

static void patches_of(etree_ctx* c, const ivec* verts, ivec* out) {
  out->n = 0;
  for (int64_t i = 0; i < verts->n; ++i) {
    int32_t p = c->assign[verts->a[i]];
    if (!c->pmark[p]) c->pmark[p] = 1, iv_push(out, p);
  }
  for (int64_t i = 0; i < out->n; ++i) c->pmark[out->a[i]] = 0;
  qsort(out->a, (size_t)out->n, sizeof(int32_t), cmp_i32);
}

/* etree.cpp:118-144 recurse */
static void nd_recurse(etree_ctx* c, int32_t idx, ivec* verts, ivec* patches) {
  if (c->rc || verts->n == 0) {
    iv_free(verts), iv_free(patches);
    return;
  }
  int level = floor_log2((int64_t)idx + 1);
  if (level == c->L || verts->n < 2) {
    c->nodes[idx] = *verts;
    iv_free(patches);
    return;
  }
  localq_t lq;
  restrict_local(c->master, patches->a, (int32_t)patches->n, c->owned, &lq);
  if (lq.na <= 1) {
    free_localq(&lq);
    c->nodes[idx] = *verts;
    iv_free(patches);
    return;
  }
  /* get_separator (etree.cpp:48-79) with the quotient branch */
  bipartition(&lq, c->master->node_w, BALANCE_TOL, c->side, c->aidx);
  free_localq(&lq);
  ++c->tok;
  for (int64_t i = 0; i < verts->n; ++i) c->in_node[verts->a[i]] = c->tok;
  ivec sep = {0, 0, 0}, left = {0, 0, 0}, right = {0, 0, 0};
  separate(c->g, verts->a, (int32_t)verts->n, c->in_node, c->tok, c->assign, c->side, BALANCE_TOL,
           c->region, &sep, &left, &right);
  c->nodes[idx] = sep;
  if (quotient_remove(c->master, c->g, c->assign, sep.a, (int32_t)sep.n)) {
    c->rc = 1;
    iv_free(verts), iv_free(patches), iv_free(&left), iv_free(&right);
    return;
  }
  ivec lp = {0, 0, 0}, rp = {0, 0, 0};
  patches_of(c, &left, &lp);
  patches_of(c, &right, &rp);
  iv_free(verts), iv_free(patches);
  nd_recurse(c, 2 * idx + 1, &left, &lp);
  nd_recurse(c, 2 * idx + 2, &right, &rp);
}

int mpo_build_etree(int32_t n, const int32_t* off, const int32_t* nbr,
                    const int32_t* assignment, int32_t patch_count, int32_t nd_level,
                    uint64_t seed, int32_t* node_offsets, int32_t* node_vertices) {
  (void)seed; /* bipartition ignores it (partition.cpp:27) */
  if (nd_level < 0 || nd_level > MAX_ND_LEVEL) return fail("nd_level out of range");
  graph_t g = {n, off, nbr};
  quotient_t q;
  memset(&q, 0, sizeof q);
  int rc = build_quotient(&g, assignment, patch_count, &q);
  if (rc) return rc;
  int32_t nn = (int32_t)((1LL << (nd_level + 1)) - 1);
  etree_ctx c;
  memset(&c, 0, sizeof c);
  c.g = &g, c.assign = assignment, c.master = &q, c.L = nd_level;
  c.nodes = (ivec*)xcalloc((size_t)nn, sizeof(ivec));
  c.in_node = (int32_t*)xcalloc((size_t)n, sizeof(int32_t));
  c.side = (uint8_t*)xcalloc((size_t)patch_count, 1);
  c.aidx = (int32_t*)malloc(sizeof(int32_t) * (patch_count + 1));
  for (int32_t p = 0; p < patch_count; ++p) c.aidx[p] = -1;
  c.owned = (char*)xcalloc((size_t)patch_count, 1);
  c.region = (uint8_t*)xcalloc((size_t)n, 1);
  c.pmark = (char*)xcalloc((size_t)patch_count, 1);
  ivec all = {0, 0, 0}, owned = {0, 0, 0};
  for (int32_t v = 0; v < n; ++v) iv_push(&all, v);
  for (int32_t p = 0; p < patch_count; ++p)
    if (q.node_w[p] > 0) iv_push(&owned, p);
  nd_recurse(&c, 0, &all, &owned);
  int32_t pos = 0;
  for (int32_t i = 0; i < nn; ++i) {
    node_offsets[i] = pos;
    for (int64_t k = 0; k < c.nodes[i].n; ++k) node_vertices[pos++] = c.nodes[i].a[k];
    iv_free(&c.nodes[i]);
  }
  node_offsets[nn] = pos;
  free(c.nodes), free(c.in_node), free(c.side), free(c.aidx), free(c.owned), free(c.region),
      free(c.pmark);
  free_quotient(&q);
  if (c.rc) return 1;
  return 0;
}

/* ------------------------------------------------------- elimination game */
/* elimination.cpp:8-98 EliminationState.  Each vertex owns two slots of its
 * initial degree: |adj|+|elems| never grows (a boundary member always loses
 * the pivot from adj or an absorbed element from elems when it gains the
 * pivot element), so the slots never overflow. */
typedef struct {
  int32_t n;
  int64_t* base;     /* slot start per vertex */
  int32_t *adj, *el; /* slot storage */
  int32_t *nadj, *nel;
  int32_t** bnd;     /* boundary per element (alive members) */
  int32_t* nbnd;
  char* gone;
  int32_t *vmark, *emark;
  int32_t vtok, etok;
  int32_t* scratch;
} elim_t;

static void elim_init(elim_t* s, int32_t n, const int32_t* off, const int32_t* nbr) {
  s->n = n;
  s->base = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  for (int32_t v = 0; v <= n; ++v) s->base[v] = off[v];
  s->adj = (int32_t*)xcalloc((size_t)off[n], sizeof(int32_t));
  s->el = (int32_t*)xcalloc((size_t)off[n], sizeof(int32_t));
  memcpy(s->adj, nbr, sizeof(int32_t) * off[n]);
  s->nadj = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  s->nel = (int32_t*)xcalloc((size_t)n + 1, sizeof(int32_t));
  for (int32_t v = 0; v < n; ++v) s->nadj[v] = off[v + 1] - off[v];
  s->bnd = (int32_t**)xcalloc((size_t)n, sizeof(int32_t*));
  s->nbnd = (int32_t*)xcalloc((size_t)n, sizeof(int32_t));
  s->gone = (char*)xcalloc((size_t)n, 1);
  s->vmark = (int32_t*)xcalloc((size_t)n, sizeof(int32_t));
  s->emark = (int32_t*)xcalloc((size_t)n, sizeof(int32_t));
  s->vtok = s->etok = 0;
  s->scratch = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
}
static void elim_free(elim_t* s) {
  for (int32_t v = 0; v < s->n; ++v) free(s->bnd[v]);
  free(s->base), free(s->adj), free(s->el), free(s->nadj), free(s->nel), free(s->bnd),
      free(s->nbnd), free(s->gone), free(s->vmark), free(s->emark), free(s->scratch);
}
/* elimination.cpp:46-52 */
static int64_t approx_degree(const elim_t* s, int32_t v) {
  int64_t d = s->nadj[v];
  const int32_t* el = s->el + s->base[v];
  for (int32_t i = 0; i < s->nel[v]; ++i) d += s->nbnd[el[i]];
  return d;
}
/* elimination.cpp:23-44 */
static int64_t exact_degree(elim_t* s, int32_t v) {
  int32_t t = ++s->vtok;
  s->vmark[v] = t;
  int64_t d = 0;
  const int32_t* a = s->adj + s->base[v];
  for (int32_t i = 0; i < s->nadj[v]; ++i)
    if (s->vmark[a[i]] != t) s->vmark[a[i]] = t, ++d;
  const int32_t* el = s->el + s->base[v];
  for (int32_t i = 0; i < s->nel[v]; ++i)
    for (int32_t k = 0; k < s->nbnd[el[i]]; ++k) {
      int32_t w = s->bnd[el[i]][k];
      if (s->vmark[w] != t) s->vmark[w] = t, ++d;
    }
  return d;
}
/* elimination.cpp:54-98 eliminate; returns |boundary|, boundary in s->bnd[pivot] */
static int32_t eliminate(elim_t* s, int32_t pivot) {
  int32_t t = ++s->vtok, nb = 0;
  s->vmark[pivot] = t;
  int32_t* out = s->scratch;
  const int32_t* a = s->adj + s->base[pivot];
  for (int32_t i = 0; i < s->nadj[pivot]; ++i)
    if (s->vmark[a[i]] != t) s->vmark[a[i]] = t, out[nb++] = a[i];
  const int32_t* pel = s->el + s->base[pivot];
  for (int32_t i = 0; i < s->nel[pivot]; ++i)
    for (int32_t k = 0; k < s->nbnd[pel[i]]; ++k) {
      int32_t w = s->bnd[pel[i]][k];
      if (s->vmark[w] != t) s->vmark[w] = t, out[nb++] = w;
    }
  qsort(out, (size_t)nb, sizeof(int32_t), cmp_i32);
  int32_t et = ++s->etok;
  for (int32_t i = 0; i < s->nel[pivot]; ++i) s->emark[pel[i]] = et;
  for (int32_t i = 0; i < nb; ++i) {
    int32_t v = out[i];
    int32_t* va = s->adj + s->base[v];
    int32_t k = 0;
    for (int32_t j = 0; j < s->nadj[v]; ++j)
      if (s->vmark[va[j]] != t) va[k++] = va[j];
    s->nadj[v] = k;
    int32_t* ve = s->el + s->base[v];
    k = 0;
    for (int32_t j = 0; j < s->nel[v]; ++j)
      if (s->emark[ve[j]] != et) ve[k++] = ve[j];
    ve[k++] = pivot;
    s->nel[v] = k;
  }
  for (int32_t i = 0; i < s->nel[pivot]; ++i) {
    free(s->bnd[pel[i]]);
    s->bnd[pel[i]] = NULL;
    s->nbnd[pel[i]] = 0;
  }
  s->nadj[pivot] = 0;
  s->nel[pivot] = 0;
  s->bnd[pivot] = (int32_t*)malloc(sizeof(int32_t) * (nb + 1));
  memcpy(s->bnd[pivot], out, sizeof(int32_t) * nb);
  s->nbnd[pivot] = nb;
  s->gone[pivot] = 1;
  return nb;
}

/* binary min-heap of (degree << 32 | id) keys with lazy invalidation: a key
 * is live iff its vertex is alive and its degree equals the cached one, so
 * pops follow std::set<(deg,id)> order exactly (local_order.cpp:24-40). */
typedef struct {
  uint64_t* k;
  int64_t n, cap;
} heap_t;
static void hpush(heap_t* h, uint64_t x) {
  if (h->n == h->cap) h->cap = h->cap ? 2 * h->cap : 64, h->k = realloc(h->k, 8 * h->cap);
  int64_t i = h->n++;
  while (i > 0 && h->k[(i - 1) / 2] > x) h->k[i] = h->k[(i - 1) / 2], i = (i - 1) / 2;
  h->k[i] = x;
}
static uint64_t hpop(heap_t* h) {
  uint64_t top = h->k[0], x = h->k[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= h->n) break;
    if (c + 1 < h->n && h->k[c + 1] < h->k[c]) ++c;
    if (h->k[c] >= x) break;
    h->k[i] = h->k[c], i = c;
  }
  if (h->n) h->k[i] = x;
  return top;
}

/* local_order.cpp:10-42 minimum_degree */
int mpo_minimum_degree(int32_t n, const int32_t* off, const int32_t* nbr, int32_t mode,
                       int32_t* order) {
  if (mode == 2) {
    for (int32_t v = 0; v < n; ++v) order[v] = v;
    return 0;
  }
  elim_t s;
  elim_init(&s, n, off, nbr);
  int64_t* cached = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  heap_t h = {0, 0, 0};
  for (int32_t v = 0; v < n; ++v) {
    cached[v] = mode == 1 ? exact_degree(&s, v) : approx_degree(&s, v);
    hpush(&h, ((uint64_t)cached[v] << 32) | (uint32_t)v);
  }
  for (int32_t k = 0; k < n; ++k) {
    int32_t v;
    for (;;) {
      uint64_t key = hpop(&h);
      v = (int32_t)(key & 0xffffffffu);
      if (!s.gone[v] && (int64_t)(key >> 32) == cached[v]) break;
    }
    order[k] = v;
    int32_t nb = eliminate(&s, v);
    for (int32_t i = 0; i < nb; ++i) {
      int32_t w = s.bnd[v][i];
      int64_t d = mode == 1 ? exact_degree(&s, w) : approx_degree(&s, w);
      if (d != cached[w]) {
        cached[w] = d;
        hpush(&h, ((uint64_t)d << 32) | (uint32_t)w);
      }
    }
  }
  free(h.k), free(cached);
  elim_free(&s);
  return 0;
}

/* local_order.cpp:57-87 order_tree_nodes (induced subgraph per node:
 * graph.cpp:141-173, local ids follow the node's ascending vertex list) */
int mpo_order_tree_nodes(int32_t n, const int32_t* off, const int32_t* nbr, int32_t nd_level,
                         const int32_t* node_offsets, const int32_t* node_vertices,
                         int32_t mode, int32_t* local_perm) {
  int32_t nn = (int32_t)((1LL << (nd_level + 1)) - 1);
  int32_t* local_of = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  for (int32_t v = 0; v < n; ++v) local_of[v] = -1;
  for (int32_t i = 0; i < nn; ++i) {
    int32_t b = node_offsets[i], e = node_offsets[i + 1], sz = e - b;
    if (sz == 0) continue;
    const int32_t* vs = node_vertices + b;
    for (int32_t k = 0; k < sz; ++k) {
      if (vs[k] < 0 || vs[k] >= n || local_of[vs[k]] != -1) {
        free(local_of);
        return fail("bad or duplicate node vertex %d", vs[k]);
      }
      local_of[vs[k]] = k;
    }
    int32_t* loff = (int32_t*)xcalloc((size_t)sz + 1, sizeof(int32_t));
    for (int32_t k = 0; k < sz; ++k)
      for (int32_t j = off[vs[k]]; j < off[vs[k] + 1]; ++j)
        if (local_of[nbr[j]] != -1) ++loff[k + 1];
    for (int32_t k = 0; k < sz; ++k) loff[k + 1] += loff[k];
    int32_t* lnbr = (int32_t*)xcalloc((size_t)loff[sz], sizeof(int32_t));
    for (int32_t k = 0; k < sz; ++k) {
      int32_t t = loff[k];
      for (int32_t j = off[vs[k]]; j < off[vs[k] + 1]; ++j)
        if (local_of[nbr[j]] != -1) lnbr[t++] = local_of[nbr[j]];
      qsort(lnbr + loff[k], (size_t)(t - loff[k]), sizeof(int32_t), cmp_i32);
    }
    mpo_minimum_degree(sz, loff, lnbr, mode, local_perm + b);
    for (int32_t k = 0; k < sz; ++k) local_of[vs[k]] = -1;
    free(loff), free(lnbr);
  }
  free(local_of);
  return 0;
}

/* assemble.cpp:24-46 schedules + :65-85 compute_perm + :8-22 from_order */
static void postorder(int32_t idx, int32_t nn, int32_t* out, int32_t* k) {
  if (idx >= nn) return;
  postorder(2 * idx + 1, nn, out, k);
  postorder(2 * idx + 2, nn, out, k);
  out[(*k)++] = idx;
}
int mpo_compute_perm(int32_t n, int32_t nd_level, const int32_t* node_offsets,
                     const int32_t* node_vertices, const int32_t* local_perm,
                     int32_t levelorder, int32_t* perm, int32_t* inverse) {
  int32_t nn = (int32_t)((1LL << (nd_level + 1)) - 1);
  int32_t* sched = (int32_t*)malloc(sizeof(int32_t) * nn);
  int32_t k = 0;
  if (levelorder) {
    for (int32_t l = nd_level; l >= 0; --l)
      for (int32_t idx = (1 << l) - 1; idx < (1 << (l + 1)) - 1; ++idx) sched[k++] = idx;
  } else {
    postorder(0, nn, sched, &k);
  }
  int32_t pos = 0;
  for (int32_t s = 0; s < nn; ++s) {
    int32_t i = sched[s];
    for (int32_t j = node_offsets[i]; j < node_offsets[i + 1]; ++j) {
      if (pos >= n) {
        free(sched);
        return fail("tree vertex lists do not cover the graph");
      }
      perm[pos++] = node_vertices[node_offsets[i] + local_perm[j]];
    }
  }
  free(sched);
  if (pos != n) return fail("tree vertex lists do not cover the graph");
  for (int32_t v = 0; v < n; ++v) inverse[v] = -1;
  for (int32_t p = 0; p < n; ++p) {
    if (perm[p] < 0 || perm[p] >= n) return fail("permutation entry out of range");
    if (inverse[perm[p]] != -1) return fail("permutation repeats an index");
    inverse[perm[p]] = p;
  }
  return 0;
}

/* symbolic.cpp:33-45 elimination_fill */
int mpo_elimination_fill(int32_t n, const int32_t* off, const int32_t* nbr,
                         const int32_t* perm, int64_t* column_counts, int64_t* nnz_A,
                         int64_t* nnz_L, int64_t* cost) {
  elim_t s;
  elim_init(&s, n, off, nbr);
  int64_t L = 0, c = 0;
  for (int32_t k = 0; k < n; ++k) {
    if (perm[k] < 0 || perm[k] >= n || s.gone[perm[k]]) {
      elim_free(&s);
      return fail("permutation is not a bijection");
    }
    int64_t d = (int64_t)eliminate(&s, perm[k]) + 1;
    if (column_counts) column_counts[k] = d;
    L += d;
    c += d * d;
  }
  *nnz_A = (int64_t)n + off[n];
  *nnz_L = L;
  *cost = c;
  elim_free(&s);
  return 0;
}

/* symbolic.cpp:82-96 factor_etree_parents */
int mpo_factor_etree_parents(int32_t n, const int32_t* off, const int32_t* nbr,
                             const int32_t* perm, int32_t* parents) {
  int32_t* inv = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  for (int32_t k = 0; k < n; ++k) inv[perm[k]] = k;
  elim_t s;
  elim_init(&s, n, off, nbr);
  for (int32_t k = 0; k < n; ++k) {
    int32_t nb = eliminate(&s, perm[k]), best = -1;
    for (int32_t i = 0; i < nb; ++i) {
      int32_t pos = inv[s.bnd[perm[k]][i]];
      if (best == -1 || pos < best) best = pos;
    }
    parents[k] = best;
  }
  elim_free(&s);
  free(inv);
  return 0;
}
