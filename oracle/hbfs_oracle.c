/*
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT PATH.
 *
 * Plain-C restatement of the reference hybrid-BFS path (package ``hybfs`` 0.1.0,
 * /root/reference/pkg/src/hybfs).  It is the CPU checker the CUDA path is
 * compared against; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  Every function cites the
 * reference file:line whose semantics it restates.  Parity of this restatement
 * with the reference itself is pinned by tests/test_oracle.py against
 * tests/golden/ (fixtures generated from the reference by
 * tests/golden/make_golden.py).
 *
 * Build: gcc -O3 -fopenmp -shared -fPIC oracle/hbfs_oracle.c -o oracle/liboracle.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NIL32 0xFFFFFFFFu

/* ---------------------------------------------------------------- hashing */

/* splitmix64 finalizer — generator.py:36-44 */
uint64_t hbo_mix64(uint64_t x)
{
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

/* LSD radix sort of (key, payload) pairs on the full 64-bit key; keys are
 * distinct wherever it is used (mix64 is a bijection), so any sort
 * reproduces numpy's stable argsort. */
static void radix_sort_kv(uint64_t *key, uint32_t *val, int64_t n)
{
    uint64_t *k2 = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
    uint32_t *v2 = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    int64_t cnt[256];
    for (int pass = 0; pass < 8; ++pass) {
        int sh = pass * 8;
        memset(cnt, 0, sizeof cnt);
        for (int64_t i = 0; i < n; ++i) cnt[(key[i] >> sh) & 0xFF]++;
        int64_t s = 0;
        for (int b = 0; b < 256; ++b) { int64_t c = cnt[b]; cnt[b] = s; s += c; }
        for (int64_t i = 0; i < n; ++i) {
            int64_t p = cnt[(key[i] >> sh) & 0xFF]++;
            k2[p] = key[i];
            v2[p] = val[i];
        }
        uint64_t *tk = key; key = k2; k2 = tk;
        uint32_t *tv = val; val = v2; v2 = tv;
    }
    /* 8 passes: data is back in the caller's buffers */
    free(k2);
    free(v2);
}

/* ------------------------------------------------------------- generator */

/* _label_permutation — generator.py:129-133: argsort(mix64(mix64(id+1)^seed)) */
void hbo_label_permutation(int64_t n, uint64_t seed, uint32_t *perm)
{
    uint64_t *key = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        key[i] = hbo_mix64(hbo_mix64((uint64_t)i + 1u) ^ seed);
        perm[i] = (uint32_t)i;
    }
    radix_sort_kv(key, perm, n);
    free(key);
}

/* generate — generator.py:136-159 with _unit_draws (:47-53) and rmat_edge
 * (:118-126).  thr = {a, a+b, a+b+c} evaluated in Python's left-to-right
 * double order by the caller (generator.py:149-150). */
void hbo_generate(int scale, int64_t m, uint64_t seed, const double thr[3],
                  int permute, uint32_t *u_out, uint32_t *v_out)
{
    const double a = thr[0], ab = thr[1], abc = thr[2];
    const uint64_t golden = 0x9E3779B97F4A7C15ull, salt0 = 0xD6E8FEB86659FD93ull;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
        /* h0 = mix64(idx*GOLDEN + seed) does not depend on the level */
        uint64_t h0 = hbo_mix64((uint64_t)e * golden + seed);
        uint64_t u = 0, v = 0;
        for (int lv = 0; lv < scale; ++lv) {
            uint64_t salt = (uint64_t)(lv + 1) * salt0;
            uint64_t h = hbo_mix64(h0 ^ salt);
            double r = (double)(h >> 11) * 0x1p-53;
            u = (u << 1) | (uint64_t)(r >= ab);
            v = (v << 1) | (uint64_t)(((r >= a) && (r < ab)) || (r >= abc));
        }
        u_out[e] = (uint32_t)u;
        v_out[e] = (uint32_t)v;
    }
    int64_t n = (int64_t)1 << scale;
    if (permute && n > 1) {
        uint32_t *perm = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
        hbo_label_permutation(n, seed, perm);
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < m; ++e) {
            u_out[e] = perm[u_out[e]];
            v_out[e] = perm[v_out[e]];
        }
        free(perm);
    }
}

/* ------------------------------------------------------------------- CSR */

static int cmp_u32(const void *x, const void *y)
{
    uint32_t a = *(const uint32_t *)x, b = *(const uint32_t *)y;
    return (a > b) - (a < b);
}

static void sort_row(uint32_t *p, int64_t len)
{
    if (len < 32) {
        for (int64_t i = 1; i < len; ++i) {
            uint32_t x = p[i];
            int64_t j = i - 1;
            while (j >= 0 && p[j] > x) { p[j + 1] = p[j]; --j; }
            p[j + 1] = x;
        }
    } else {
        qsort(p, (size_t)len, sizeof(uint32_t), cmp_u32);
    }
}

/* from_arrays — csr.py:46-74: both arcs per edge, row_starts = [0]+cumsum(
 * bincount(src)), rows ascending (the (src<<32)|dst key sort), duplicates and
 * self-loops kept.  dedup=1 additionally applies per-row unique + self-loop
 * removal (the BASELINE.json "removed" variant).
 * adjacency must hold 2m entries; returns the arc count written. */
int64_t hbo_csr_build(const uint32_t *eu, const uint32_t *ev, int64_t m, int64_t n,
                      int dedup, int64_t *rs, uint32_t *adj)
{
    int64_t *cur = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t e = 0; e < m; ++e) { cur[eu[e]]++; cur[ev[e]]++; }
    rs[0] = 0;
    for (int64_t i = 0; i < n; ++i) rs[i + 1] = rs[i] + cur[i];
    for (int64_t i = 0; i < n; ++i) cur[i] = rs[i];
    for (int64_t e = 0; e < m; ++e) {
        adj[cur[eu[e]]++] = ev[e];
        adj[cur[ev[e]]++] = eu[e];
    }
    free(cur);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; ++i) sort_row(adj + rs[i], rs[i + 1] - rs[i]);
    if (!dedup) return 2 * m;
    int64_t w = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t s = rs[i], e = rs[i + 1];
        rs[i] = w;
        int have = 0;
        uint32_t last = 0;
        for (int64_t k = s; k < e; ++k) {
            uint32_t x = adj[k];
            if ((int64_t)x == i) continue;
            if (have && x == last) continue;
            adj[w++] = x;
            last = x;
            have = 1;
        }
    }
    rs[n] = w;
    return w;
}

/* sample_sources — harness.py:73-97: first `count` ids of
 * argsort(mix64(mix64(id+0x5EED)^seed)) with degree > 0 (unless
 * allow_isolated).  Returns the number written, -1 when too few eligible. */
int64_t hbo_sample_sources(const int64_t *rs, int64_t n, int64_t count, uint64_t seed,
                           int allow_isolated, uint32_t *out)
{
    if (count > n) return -1;
    uint64_t *key = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
    uint32_t *ids = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    for (int64_t i = 0; i < n; ++i) {
        key[i] = hbo_mix64(hbo_mix64((uint64_t)i + 0x5EEDu) ^ seed);
        ids[i] = (uint32_t)i;
    }
    radix_sort_kv(key, ids, n);
    int64_t k = 0;
    for (int64_t i = 0; i < n && k < count; ++i) {
        uint32_t v = ids[i];
        if (allow_isolated || rs[v + 1] > rs[v]) out[k++] = v;
    }
    free(key);
    free(ids);
    return k < count ? -1 : k;
}

/* --------------------------------------------------------- FIFO oracle BFS */

/* bfs_reference — _native.pyx:39-62: FIFO queue BFS; levels are the oracle
 * for the level array (parents here are first-dequeued, NOT the hybrid rule). */
void hbo_bfs_reference(const int64_t *rs, const uint32_t *adj, int64_t n, int64_t source,
                       uint32_t *parent, int32_t *levels)
{
    uint32_t *queue = (uint32_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(uint32_t));
    for (int64_t i = 0; i < n; ++i) { parent[i] = NIL32; levels[i] = -1; }
    parent[source] = (uint32_t)source;
    levels[source] = 0;
    queue[0] = (uint32_t)source;
    int64_t head = 0, tail = 1;
    while (head < tail) {
        uint32_t u = queue[head++];
        for (int64_t k = rs[u]; k < rs[u + 1]; ++k) {
            uint32_t v = adj[k];
            if (levels[v] == -1) {
                levels[v] = levels[u] + 1;
                parent[v] = u;
                queue[tail++] = v;
            }
        }
    }
    free(queue);
}

/* ------------------------------------------------------------ hybrid BFS */

typedef struct {
    int32_t layer;
    int32_t direction;   /* 0 = top-down, 1 = bottom-up */
    int64_t v_f, e_f, e_u, f_value, g_value;
    int64_t fallback_count, gather_count;
} hbo_row;

#define TESTBIT(w, v) (((w)[(v) >> 5] >> ((v) & 31u)) & 1u)
#define SETBIT(w, v) ((w)[(v) >> 5] |= 1u << ((v) & 31u))

/* top_down_layer / top_down_chunked — _native.pyx:65-86, :207-239 */
static int64_t td_layer(const int64_t *rs, const uint32_t *adj, int64_t nw,
                        const uint32_t *inw, uint32_t *vis, uint32_t *out, uint32_t *parent)
{
    int64_t gathers = 0;
    for (int64_t w = 0; w < nw; ++w) {
        uint32_t bits = inw[w];
        if (!bits) continue;
        for (int b = 0; b < 32; ++b) {
            if (!((bits >> b) & 1u)) continue;
            uint32_t u = (uint32_t)(w * 32 + b);
            gathers += rs[u + 1] - rs[u]; /* 16-lane chunks incl. tail = degree */
            for (int64_t k = rs[u]; k < rs[u + 1]; ++k) {
                uint32_t v = adj[k];
                if (!TESTBIT(vis, v)) {
                    SETBIT(vis, v);
                    SETBIT(out, v);
                    parent[v] = u;
                }
            }
        }
    }
    return gathers;
}

/* bottom_up_layer — _native.pyx:89-104 */
static void bu_scalar(const int64_t *rs, const uint32_t *adj, int64_t n,
                      const uint32_t *inw, uint32_t *vis, uint32_t *out, uint32_t *parent)
{
    for (int64_t v = 0; v < n; ++v) {
        if (TESTBIT(vis, (uint32_t)v)) continue;
        for (int64_t k = rs[v]; k < rs[v + 1]; ++k) {
            uint32_t nb = adj[k];
            if (TESTBIT(inw, nb)) {
                SETBIT(vis, (uint32_t)v);
                SETBIT(out, (uint32_t)v);
                parent[v] = nb;
                break;
            }
        }
    }
}

/* bottom_up_multiple_set — _native.pyx:107-204 with the per-half probe of
 * bu_probe.h:66-106 (the AVX-512 path :18-64 has identical semantics).
 * posw/longw = deg>0 / deg>max_pos bitmaps (engine.py:29-57). */
static void bu_multiple_set(const int64_t *rs, const uint32_t *adj, int64_t n, int64_t nw,
                            int max_pos, const uint32_t *posw, const uint32_t *longw,
                            const uint32_t *inw, uint32_t *vis, uint32_t *out,
                            uint32_t *parent, int64_t *fallback, int64_t *gathers)
{
    if (rs[n] == 0) return;
    for (int64_t w = 0; w < nw; ++w) {
        if (((~vis[w]) & posw[w]) == 0) continue;
        for (int half = 0; half < 2; ++half) {
            uint32_t mask_vis = (vis[w] >> (16 * half)) & 0xFFFFu;
            uint32_t half_pos = (posw[w] >> (16 * half)) & 0xFFFFu;
            if (((~mask_vis) & half_pos) == 0) continue;
            int64_t base = w * 32 + half * 16;
            uint32_t mask_done = 0, mask_pos = (~half_pos) & 0xFFFFu;
            for (int pos = 0; pos < max_pos; ++pos) {
                mask_vis = (vis[w] >> (16 * half)) & 0xFFFFu;
                uint32_t avail = (~(mask_vis | mask_done | mask_pos)) & 0xFFFFu;
                if (!avail) break;
                uint32_t found = 0;
                for (int i = 0; i < 16; ++i) {
                    if (!((avail >> i) & 1u)) continue;
                    int64_t v = base + i;
                    int64_t s = v < n ? rs[v] + pos : 0, e = v < n ? rs[v + 1] : 0;
                    if (s >= e) { mask_pos |= 1u << i; continue; }
                    ++*gathers;
                    uint32_t a = adj[s];
                    if (TESTBIT(inw, a)) { parent[v] = a; found |= 1u << i; }
                }
                if (found) {
                    vis[w] |= found << (16 * half);
                    out[w] |= found << (16 * half);
                    mask_done |= found;
                }
            }
            uint32_t half_long = (longw[w] >> (16 * half)) & 0xFFFFu;
            uint32_t rem = (~((vis[w] >> (16 * half)) & 0xFFFFu)) & half_long;
            for (int i = 0; i < 16 && rem; ++i) {
                if (!((rem >> i) & 1u)) continue;
                int64_t v = base + i;
                ++*fallback;
                for (int64_t k = rs[v] + max_pos; k < rs[v + 1]; ++k) {
                    uint32_t a = adj[k];
                    if (TESTBIT(inw, a)) {
                        parent[v] = a;
                        SETBIT(vis, (uint32_t)v);
                        SETBIT(out, (uint32_t)v);
                        break;
                    }
                }
            }
        }
    }
}

/* The F1 rule: parent[v] = min{u in Adj(v) : level[u] = level[v] - 1}
 * = the first such entry of v's sorted row; NIL for unreached, source for itself. */
void hbo_minid_parents(const int64_t *rs, const uint32_t *adj, int64_t n, const int32_t *level,
                       int64_t source, uint32_t *parent)
{
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t v = 0; v < n; ++v) {
        uint32_t p = 0xFFFFFFFFu;
        if (v == source) {
            p = (uint32_t)source;
        } else if (level[v] >= 1) {
            const int32_t want = level[v] - 1;
            for (int64_t k = rs[v]; k < rs[v + 1]; ++k)
                if (level[adj[k]] == want) { p = adj[k]; break; }
        }
        parent[v] = p;
    }
}

/* Exported per-layer steps (test checkers for csrc/layer.cu). */
int64_t hbo_td_layer(const int64_t *rs, const uint32_t *adj, int64_t n, const uint32_t *inw,
                     uint32_t *vis, uint32_t *out, uint32_t *parent)
{
    return td_layer(rs, adj, (n + 31) / 32, inw, vis, out, parent);
}

void hbo_bu_layer(const int64_t *rs, const uint32_t *adj, int64_t n, const uint32_t *inw,
                  uint32_t *vis, uint32_t *out, uint32_t *parent)
{
    bu_scalar(rs, adj, n, inw, vis, out, parent);
}

void hbo_bu_multiple_set(const int64_t *rs, const uint32_t *adj, int64_t n, int max_pos,
                         const uint32_t *posw, const uint32_t *longw, const uint32_t *inw,
                         uint32_t *vis, uint32_t *out, uint32_t *parent, int64_t *fb_ga)
{
    fb_ga[0] = fb_ga[1] = 0;
    bu_multiple_set(rs, adj, n, (n + 31) / 32, max_pos, posw, longw, inw, vis, out, parent,
                    &fb_ga[0], &fb_ga[1]);
}

static int64_t popcount_words(const uint32_t *w, int64_t nw)
{
    int64_t s = 0;
    for (int64_t i = 0; i < nw; ++i) s += __builtin_popcount(w[i]);
    return s;
}

/* counters_after_layer — bfs_scalar.py:18-26; also stamps levels. */
static void layer_counters(const int64_t *rs, int64_t n, int64_t nw, const uint32_t *vis,
                           const uint32_t *out, int32_t *level, int32_t depth,
                           int64_t *v_f, int64_t *e_f, int64_t *e_u_vertex)
{
    int64_t vf = 0, ef = 0;
    for (int64_t w = 0; w < nw; ++w) {
        uint32_t bits = out[w];
        while (bits) {
            int b = __builtin_ctz(bits);
            bits &= bits - 1;
            int64_t v = w * 32 + b;
            ++vf;
            ef += rs[v + 1] - rs[v];
            level[v] = depth;
        }
    }
    *v_f = vf;
    *e_f = ef;
    *e_u_vertex = n - popcount_words(vis, nw);
}

/*
 * hybrid_bfs — hybrid.py:83-175 (controller) with decide/f/g (:62-80).
 *   heuristic 0 = reference rule (hybrid.py:72-80) on the configured counter
 *   mode; heuristic 1 = Beamer/GAP rule: TD->BU when
 *   m_f > m_u // alpha, BU->TD when the frontier shrinks and n_f <= n // beta,
 *   with m_u the edge-denominated unvisited count.
 *   force_direction: -1 none, 0 TD, 1 BU.  counter_mode: 0 vertex, 1 edge.
 * Writes parent (hybrid rule), level (new: depth of discovery), and trace rows
 * (without elapsed).  Returns the number of layers (may exceed cap; only the
 * first cap rows are stored).
 */
int64_t hbo_hybrid_bfs(const int64_t *rs, const uint32_t *adj, int64_t n, int64_t source,
                       int heuristic, int counter_mode, int64_t alpha, int64_t beta,
                       int max_pos, int use_simd, int force_direction,
                       uint32_t *parent, int32_t *level, hbo_row *rows, int64_t cap)
{
    int64_t nw = (n + 31) / 32, arcs = rs[n];
    uint32_t *vis = (uint32_t *)calloc((size_t)nw + 1, 4);
    uint32_t *inw = (uint32_t *)calloc((size_t)nw + 1, 4);
    uint32_t *out = (uint32_t *)calloc((size_t)nw + 1, 4);
    uint32_t *posw = (uint32_t *)calloc((size_t)nw + 1, 4);
    uint32_t *longw = (uint32_t *)calloc((size_t)nw + 1, 4);
    for (int64_t v = 0; v < n; ++v) {
        int64_t d = rs[v + 1] - rs[v];
        if (d > 0) SETBIT(posw, (uint32_t)v);
        if (d > max_pos) SETBIT(longw, (uint32_t)v);
        parent[v] = NIL32;
        level[v] = -1;
    }
    parent[source] = (uint32_t)source;
    level[source] = 0;
    SETBIT(vis, (uint32_t)source);
    SETBIT(inw, (uint32_t)source);
    int64_t src_deg = rs[source + 1] - rs[source];
    int64_t e_f = src_deg, v_f = 1;
    int64_t e_u_vertex = n - 1, e_u_edge = arcs - src_deg;
    int dir = 0, layer = 1;
    int64_t prev_vf = 0;
    while (v_f > 0) {
        int64_t e_u = counter_mode ? e_u_edge : e_u_vertex;
        int64_t fv, gv = n / beta;
        if (heuristic == 1) {
            fv = e_u_edge / alpha;
            if (force_direction >= 0) dir = force_direction;
            else if (dir == 0) { if (e_f > fv) dir = 1; }
            else { if (v_f < prev_vf && v_f <= gv) dir = 0; }
        } else {
            fv = e_u / alpha;
            if (force_direction >= 0) dir = force_direction;
            else if (v_f > fv) dir = 1;
            else if (v_f < gv) dir = 0;
        }
        int64_t fb = 0, ga = 0;
        if (dir == 0) {
            int64_t g = td_layer(rs, adj, nw, inw, vis, out, parent);
            if (use_simd) ga = g;
        } else if (use_simd) {
            bu_multiple_set(rs, adj, n, nw, max_pos, posw, longw, inw, vis, out, parent, &fb, &ga);
        } else {
            bu_scalar(rs, adj, n, inw, vis, out, parent);
        }
        if (layer - 1 < cap) {
            hbo_row *r = &rows[layer - 1];
            r->layer = layer;
            r->direction = dir;
            r->v_f = v_f;
            r->e_f = e_f;
            r->e_u = e_u;
            r->f_value = fv;
            r->g_value = gv;
            r->fallback_count = fb;
            r->gather_count = ga;
        }
        int64_t nvf, nef, neu;
        layer_counters(rs, n, nw, vis, out, level, layer, &nvf, &nef, &neu);
        prev_vf = v_f;
        v_f = nvf;
        e_f = nef;
        e_u_vertex = neu;
        e_u_edge -= nef;
        uint32_t *t = inw; inw = out; out = t;
        memset(out, 0, (size_t)nw * 4);
        ++layer;
    }
    free(vis); free(inw); free(out); free(posw); free(longw);
    return layer - 1;
}

/* ------------------------------------------------------------- validator */

/* validate_tree — harness.py:129-205, rules checked in the reference order
 * 1, 2, 5, 3, 4.  Returns 0 when valid, else the rule number; *witness gets
 * the first offending vertex. */
int hbo_validate_tree(const int64_t *rs, const uint32_t *adj, int64_t n, int64_t source,
                      const uint32_t *parent, int64_t *witness)
{
    *witness = -1;
    if (parent[source] != (uint32_t)source) { *witness = source; return 1; }
    for (int64_t v = 0; v < n; ++v) {
        if (parent[v] == NIL32 || v == source) continue;
        uint32_t p = parent[v];
        int64_t lo = rs[v], hi = rs[v + 1];
        while (lo < hi) { int64_t mid = (lo + hi) / 2; if (adj[mid] < p) lo = mid + 1; else hi = mid; }
        if (lo >= rs[v + 1] || adj[lo] != p) { *witness = v; return 2; }
    }
    uint32_t *par = (uint32_t *)malloc((size_t)n * 4);
    int32_t *ref = (int32_t *)malloc((size_t)n * 4);
    hbo_bfs_reference(rs, adj, n, source, par, ref);
    for (int64_t v = 0; v < n; ++v) {
        if ((parent[v] != NIL32) != (ref[v] != -1)) { *witness = v; free(par); free(ref); return 5; }
    }
    /* rule 3: levels by walking parents from the source (harness.py:100-126) */
    int32_t *lev = ref;
    for (int64_t v = 0; v < n; ++v) lev[v] = -1;
    lev[source] = 0;
    int changed = 1;
    int32_t depth = 0;
    while (changed) {
        changed = 0;
        for (int64_t v = 0; v < n; ++v) {
            if (v == source || parent[v] == NIL32 || lev[v] != -1) continue;
            if (lev[parent[v]] == depth) { lev[v] = depth + 1; changed = 1; }
        }
        ++depth;
    }
    for (int64_t v = 0; v < n; ++v) {
        if (parent[v] != NIL32 && lev[v] == -1) { *witness = v; free(par); free(ref); return 3; }
    }
    for (int64_t u = 0; u < n; ++u) {
        if (parent[u] == NIL32) continue;
        for (int64_t k = rs[u]; k < rs[u + 1]; ++k) {
            uint32_t w = adj[k];
            if (parent[w] == NIL32) continue;
            int32_t d = lev[u] - lev[w];
            if (d > 1 || d < -1) { *witness = u; free(par); free(ref); return 4; }
        }
    }
    free(par);
    free(ref);
    return 0;
}
