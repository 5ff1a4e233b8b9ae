/*
 * hbfs.h — C ABI of the B200-native hybrid BFS (libhbfs.so, sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path (package `hybfs`
 * 0.1.0, /root/reference/pkg/src/hybfs).  Plain pointers, sizes and status
 * codes only; no torch or C++ types.  Every entry point names the reference
 * interface it replaces.  Device pointers are CUDA global-memory pointers of
 * the current device; `stream` is a cudaStream_t (NULL = legacy stream).
 *
 * Status codes map onto the reference's exception types (hybfs raises them in
 * Python, its kernels never fail): 0 OK, 1 ValueError, 2 IndexError,
 * 3 CapacityError (generator.py:32-33, csr.py:50-51), 4 CUDA error and
 * 5 NCCL error (RuntimeError).  No C++ exception ever crosses this ABI;
 * hbfs_last_error() returns the thread-local message of the last failure.
 */
#ifndef HBFS_H
#define HBFS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HBFS_OK 0
#define HBFS_EINVAL 1
#define HBFS_ERANGE 2
#define HBFS_ECAPACITY 3
#define HBFS_ECUDA 4
#define HBFS_ENCCL 5

#define HBFS_NIL 0xFFFFFFFFu /* frontier.py:16 */
#define HBFS_UNREACHED (-1)  /* frontier.py:19 */

#define HBFS_TOP_DOWN 0
#define HBFS_BOTTOM_UP 1

#define HBFS_HEURISTIC_REFERENCE 0 /* hybrid.py:62-80 (n_f vs e_u//alpha, n//beta) */
#define HBFS_HEURISTIC_BEAMER 1    /* Beamer/GAP rule on m_f, m_u, n_f */

#define HBFS_PARENT_MINID 0 /* deterministic: min-id neighbour one level up */
#define HBFS_PARENT_ANY 1   /* first claimer wins; passes the Graph500 tree checks */

typedef struct hbfs_graph hbfs_graph; /* device-resident CSR + per-root workspace */

/* Traversal knobs: HeuristicParams (hybrid.py:27-44) + VecConfig (lanes.py:30-41)
 * + hybrid_bfs(use_simd, force_direction) (hybrid.py:83-91). */
typedef struct {
    int32_t heuristic;       /* HBFS_HEURISTIC_* */
    int32_t counter_mode;    /* 0 = "vertex", 1 = "edge" (hybrid.py:36-44) */
    int64_t alpha;           /* >= 1 */
    int64_t beta;            /* >= 1 */
    int32_t max_pos;         /* >= 1; VecConfig.max_pos, feeds the trace counters */
    int32_t use_simd;        /* trace "kernel" column and gathers/fallbacks */
    int32_t force_direction; /* -1 none, HBFS_TOP_DOWN, HBFS_BOTTOM_UP */
    int32_t parent_mode;     /* HBFS_PARENT_* */
} hbfs_params;

/* LayerTraceRow (hybrid.py:47-59); elapsed is device time of the layer. */
typedef struct {
    int32_t layer;
    int32_t direction;
    int64_t v_f, e_f, e_u, f_value, g_value;
    int64_t fallback_count, gather_count;
    double elapsed;
} hbfs_layer_row;

int hbfs_version(void);
const char *hbfs_last_error(void);

/* ---- graph input (L1): replaces csr.from_arrays / csr.build (csr.py:41-74) ---- */

/* CSR from reference-layout arrays: row_starts int64[n+1], adjacency uint32[arcs]
 * with rows sorted ascending (csr.py:22-23).  m_edges = in_edges_total (csr.py:73).
 * on_device: 1 if both pointers are device pointers, 0 for host memory. */
int hbfs_graph_from_csr(const int64_t *row_starts, const uint32_t *adjacency, int64_t n,
                        int64_t m_edges, int on_device, void *stream, hbfs_graph **out);

/* On-device CSR build from an undirected edge list u,v uint32[m] (generator.EdgeList,
 * generator.py:85-99): both arcs per edge, rows sorted ascending; dedup=0 keeps
 * duplicates and self-loops bit-exactly like csr.from_arrays, dedup=1 applies
 * per-row unique + self-loop removal. */
int hbfs_graph_build(const uint32_t *u, const uint32_t *v, int64_t m, int64_t n, int dedup,
                     int on_device, void *stream, hbfs_graph **out);

/* Device R-MAT generator, bit-exact with generator.generate (generator.py:136-159):
 * thresholds = {a, a+b, a+b+c} as the host computes them in Python order.
 * Writes u,v uint32[2^scale * edgefactor] (device or host pointers). */
int hbfs_generate_edges(int scale, int64_t edgefactor, uint64_t seed, const double thresholds[3],
                        int permute, uint32_t *u, uint32_t *v, int on_device, void *stream);

/* generate + build without leaving the device. */
int hbfs_graph_generate(int scale, int64_t edgefactor, uint64_t seed, const double thresholds[3],
                        int permute, int dedup, void *stream, hbfs_graph **out);

/* n, arcs, in_edges_total, max degree, and whether offsets are 64-bit. */
int hbfs_graph_info(const hbfs_graph *g, int64_t *n, int64_t *arcs, int64_t *m_edges,
                    int64_t *max_degree, int32_t *wide_offsets);

/* Copy the CSR out in the reference layout (int64 row_starts, uint32 adjacency). */
int hbfs_graph_export(const hbfs_graph *g, int64_t *row_starts, uint32_t *adjacency,
                      int on_device, void *stream);

int hbfs_graph_free(hbfs_graph *g);

/* harness.sample_sources (harness.py:73-97) on device: writes `count` roots to
 * out (host pointer).  Returns HBFS_EINVAL if too few eligible vertices. */
int hbfs_sample_sources(const hbfs_graph *g, int64_t count, uint64_t seed, int allow_isolated,
                        uint32_t *out);
/* The first `count` ids of that sampling order alone (no graph, no O(n) memory):
 * partitioned graphs filter them by the degrees their ranks hold
 * (hbfs_part_degrees; mgpu.sample_sources_partitioned). */
int hbfs_source_order_prefix(int64_t n, uint64_t seed, int64_t count, uint32_t *out);

/* ---- traversal (L2-L4): replaces hybrid.hybrid_bfs (hybrid.py:83-175) and its
 * per-layer engine.run_* dispatch (engine.py:81-155).  The whole traversal runs
 * on device; the direction switch is decided on device from fused counters.
 * parent: uint32[n] (NIL = unreached), level: int32[n] (-1 = unreached); either
 * may be NULL.  on_device says where parent/level live.  trace: host array of
 * trace_cap rows (may be NULL); *n_layers receives the total layer count.
 * *device_ms receives the device time of init + traversal (CUDA events).
 * Thread safety: calls on the same graph are serialised (a per-graph lock is
 * held for the whole call, which returns after its stream work completed);
 * different graphs may be traversed concurrently. */
int hbfs_bfs(hbfs_graph *g, int64_t root, const hbfs_params *p, uint32_t *parent,
             int32_t *level, int on_device, hbfs_layer_row *trace, int64_t trace_cap,
             int64_t *n_layers, float *device_ms, void *stream);

/* ---- validation: replaces harness.validate_tree (harness.py:129-205) ----
 * Graph500 rules on device, in the reference's order 1, 2, 5, 3, 4, using the
 * level array for rule 3.  *rule = 0 when valid; *witness = offending vertex.
 * check_minid=1 additionally checks the deterministic parent rule (rule 6). */
int hbfs_validate(hbfs_graph *g, int64_t root, const uint32_t *parent, const int32_t *level,
                  int on_device, int check_minid, int32_t *rule, int64_t *witness, void *stream);

/* ---- measurement: algorithmic bytes of one traversal ----
 * Given the level array (device) and the direction of every layer, returns
 * B_sector (unique 32-byte sectors) and B_useful.  Untimed accounting pass. */
int hbfs_traversal_bytes(hbfs_graph *g, int64_t root, const int32_t *level_dev,
                         const int32_t *directions, int64_t n_layers, int64_t *b_sector,
                         int64_t *b_useful, void *stream);


/* Same accounting, B_sector of every layer separately (init bytes excluded). */
int hbfs_traversal_bytes_layers(hbfs_graph *g, int64_t root, const int32_t *level_dev,
                                const int32_t *directions, int64_t n_layers,
                                int64_t *b_sector_per_layer, void *stream);

/* Diagnostics: per-layer barrier timestamps of the last traversal (8 slots of
 * uint64 ns per layer: 0 layer start, 1 after bitmap->queue conversion, 2 after
 * the top-down prologue barrier, 3 after a harvest layer's expansion, 4 end;
 * 0 = phase not taken).  rows <= 1024. */
int hbfs_phase_times(hbfs_graph *g, uint64_t *out, int64_t rows);

/* Measurement only: GB/s of random 32-byte sector reads over a 2^log_bytes
 * buffer, each warp's 32 lanes inside one random 2^log_region-byte region (the
 * access pattern of the traversal's gathers; bench.py's second roofline). */
int hbfs_probe_random_sectors(int log_bytes, int log_region, double *gbs);

/* Tuning: set the L2 -> DRAM fetch granularity of the current context
 * (cudaLimitMaxL2FetchGranularity, bytes <= 128; bytes < 0 only queries);
 * *previous (may be NULL) receives the old value. */
int hbfs_l2_fetch_granularity(int bytes, int *previous);

/* Debugging aids (compute-sanitizer substitutes, tools/sanitize.py):
 * with HBFS_GUARD=1 in the environment every device buffer carries a guard
 * band behind its end; hbfs_debug_guards checks all live bands (*clobbered =
 * bands with a changed byte, *first_bytes = size of the first such buffer).
 * hbfs_debug_checks reads the device index-check flags of a -DHBFS_CHECKED
 * build (bit per check site; 0 = no violation) and optionally resets them. */
int hbfs_debug_guards(int *enabled, int64_t *checked, int64_t *clobbered, int64_t *first_bytes);
int hbfs_debug_checks(uint32_t *flags, int reset, int *is_checked_build);

/* ---- per-layer steps on caller buffers: the hybfs._native surface ----
 * All pointers are DEVICE pointers in the reference's layout: rs int64[n+1],
 * adj uint32[arcs], LSB-first bitmaps uint32[ceil(n/32)] (frontier.py:3-6),
 * parent uint32[n].  vis/out/parent are updated in place exactly as the
 * reference's single-threaded loops leave them.  Synchronous on `stream`. */

/* _native.top_down_layer / top_down_chunked (_native.pyx:65-86, :207-239):
 * every unvisited neighbour v of the frontier `in` joins vis and out with
 * parent = its smallest frontier neighbour (the first claimer of the
 * ascending loop).  gathers (may be NULL) = the chunked kernel's count = the
 * frontier's degree sum. */
int hbfs_layer_top_down(const int64_t *rs, const uint32_t *adj, const uint32_t *in, uint32_t *vis,
                        uint32_t *out, uint32_t *parent, int64_t n, int64_t *gathers, void *stream);
/* _native.bottom_up_layer / bottom_up_multiple_set (_native.pyx:89-204): every
 * unvisited v whose sorted row holds a frontier vertex takes the first one as
 * parent and joins vis and out.  fallback/gathers (may be NULL): the 16-lane
 * kernel's counters for probe depth max_pos >= 1. */
int hbfs_layer_bottom_up(const int64_t *rs, const uint32_t *adj, const uint32_t *in, uint32_t *vis,
                         uint32_t *out, uint32_t *parent, int64_t n, int32_t max_pos,
                         int64_t *fallback, int64_t *gathers, void *stream);
/* _native.bfs_reference (_native.pyx:39-62): levels, and parents in the FIFO
 * queue's first-discoverer order (parent/level: device uint32[n] / int32[n]). */
int hbfs_reference_bfs(const int64_t *rs, const uint32_t *adj, int64_t n, int64_t source,
                       uint32_t *parent, int32_t *level, void *stream);

/* ---- multi-GPU: one rank's share of a 1D vertex partition ----
 * Rank r owns vertices [lo, hi) (word aligned) with their CSR rows (global
 * column ids); frontier and visited bitmaps are replicated, parent/level owned.
 * The host runs, per layer, hbfs_part_bu, or hbfs_part_td_expand + (all-to-all
 * of the per-owner counts) + hbfs_part_td_pack + (NCCL all-to-all-v of the
 * 8-byte records) + hbfs_part_td_apply; then (NCCL all-gather of the
 * next-frontier slices) + hbfs_part_absorb and an all-reduce of the counters
 * — paper_1704_02259_b200/mgpu.py.  Replaces, for P > 1, the
 * same reference interfaces as hbfs_graph_build / hbfs_bfs. */
typedef struct hbfs_part hbfs_part;

/* Owned rows from the full edge list u,v (every rank passes the same list). */
int hbfs_part_build(const uint32_t *u, const uint32_t *v, int64_t m, int64_t n, int64_t lo,
                    int64_t hi, int dedup, int on_device, void *stream, hbfs_part **out);
/* Owned rows sliced from a reference-layout CSR in host memory. */
int hbfs_part_from_csr(const int64_t *row_starts, const uint32_t *adjacency, int64_t n,
                       int64_t lo, int64_t hi, int64_t m_edges, void *stream, hbfs_part **out);
int hbfs_part_info(const hbfs_part *p, int64_t *n, int64_t *lo, int64_t *hi,
                   int64_t *local_arcs, int64_t *m_edges);
/* Degree of v if owned, else 0. */
int hbfs_part_degree(const hbfs_part *p, int64_t v, int64_t *deg);
/* deg[i] = degree of ids[i] if owned, else 0 (host arrays of `count` entries). */
int hbfs_part_degrees(const hbfs_part *p, const uint32_t *ids, int64_t count, int64_t *deg);
int hbfs_part_free(hbfs_part *p);
/* Per-root reset: parent/level/frontier/visited with the root. */
int hbfs_part_init(hbfs_part *p, int64_t root, void *stream);
/* Bottom-up over owned words against the replicated frontier.  next_slice:
 * device uint32[ceil((hi-lo)/32)]; counters: device uint64[4] = {found, their
 * degree sum, gathers, fallbacks} (the reference's 16-lane counters). */
int hbfs_part_bu(hbfs_part *p, int32_t depth, int32_t max_pos, uint32_t *next_slice,
                 unsigned long long *counters, void *stream);
/* Optional: global frontier size of the coming bottom-up layer (picks the
 * tiny-frontier probe variant as the single-GPU kernel does). */
int hbfs_part_hint_frontier(hbfs_part *p, int64_t v_f);
/* Top-down expansion of the owned frontier for a `world`-rank partition:
 * every unvisited target is queued once for its owner with this rank's min
 * parent candidate; send_counts: device int64[world] = records per owner. */
int hbfs_part_td_expand(hbfs_part *p, int32_t world, int64_t *send_counts, void *stream);
/* records: device uint64[sum(send_counts)] = parent << 32 | vertex, packed by
 * owner rank (the all-to-all-v send buffer). */
int hbfs_part_td_pack(hbfs_part *p, uint64_t *records, void *stream);
/* Apply the nrec records received from all ranks (owned vertices): min-id
 * parents, levels, next slice; counters: device uint64[4]. */
int hbfs_part_td_apply(hbfs_part *p, int32_t depth, const uint64_t *records, int64_t nrec,
                       uint32_t *next_slice, unsigned long long *counters, void *stream);
/* next_full: device uint32[ceil(n/32)] all-gathered next frontier. */
int hbfs_part_absorb(hbfs_part *p, const uint32_t *next_full, void *stream);
/* Owned parent/level (hi-lo entries each). */
int hbfs_part_outputs(hbfs_part *p, uint32_t *parent, int32_t *level, int on_device,
                      void *stream);

/* ---- multi-GPU traversal loop over NCCL (one process per GPU) ----
 * hbfs_nccl_unique_id on rank 0 (bytes >= 128), broadcast by the caller, then
 * hbfs_mg_init on every rank (current CUDA device).  hbfs_mg_bfs runs the whole
 * per-layer loop of hybrid.py:83-175 for this rank's hbfs_part (built for the
 * same world/rank split as mgpu.partition), one launch of the persistent
 * traversal kernel per layer on the owned vertices (min-id parents): NCCL
 * all-gather of the next frontier, all-reduce of the counters, grouped
 * send/recv of the top-down record counts and records.  trace (may be NULL): identical rows on every
 * rank (elapsed = 0); device_ms: this rank's CUDA-event time. */
typedef struct hbfs_mg hbfs_mg;
int hbfs_nccl_unique_id(void *out, int64_t bytes);
int hbfs_mg_init(const void *unique_id, int32_t world, int32_t rank, hbfs_mg **out);
int hbfs_mg_free(hbfs_mg *m);
int hbfs_mg_bfs(hbfs_mg *m, hbfs_part *p, int64_t root, const hbfs_params *params,
                hbfs_layer_row *trace, int64_t trace_cap, int64_t *n_layers, float *device_ms,
                void *stream);
/* The same loop for all `world` parts of a partition held by this process on
 * one device (exchanges are device copies): P ranks tested on one GPU. */
int hbfs_mgl_bfs(hbfs_part **parts, int32_t world, int64_t root, const hbfs_params *params,
                 hbfs_layer_row *trace, int64_t trace_cap, int64_t *n_layers, float *device_ms,
                 void *stream);
/* Exchange volume of the last traversal of this part through either loop:
 * out[0] records sent (8 bytes each), out[1] records received, out[2] layers
 * (one next-frontier all-gather + one counter all-reduce each), out[3]
 * top-down record exchanges. */
int hbfs_part_exchange_stats(const hbfs_part *p, int64_t *out);

#ifdef __cplusplus
}
#endif

#endif /* HBFS_H */
