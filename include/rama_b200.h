/*
 * rama_b200.h -- C ABI of the B200-native RAMA primal-dual multicut solver.
 *
 * This is the drop-in boundary for the reference's hot path: each entry
 * point replaces one `parcut` operator (file:line into
 * /root/reference/pkg/src/parcut/, cited per function).  Plain pointers and
 * sizes only.  Unless a parameter says "host", arrays are DEVICE pointers
 * (CUDA global memory) and all work is ordered on `stream` (a cudaStream_t
 * passed as void*, NULL = legacy default stream).
 *
 * Conventions
 *   - node ids int32 in [0, n); n, m < 2^31.  Costs / multipliers fp64.
 *   - A "canonical graph" is the reference WeightedGraph invariant
 *     (graph.py:17-57): u < v, sorted by (u, v), unique pairs.
 *   - Return value: RAMA_OK (0) or an error code; never throws.  The
 *     message of the last failure on this thread: rama_last_error().
 *   - Output arrays are caller-allocated with the capacity stated per
 *     function; the produced count is written to a host int64.
 */
#ifndef RAMA_B200_H
#define RAMA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RAMA_OK 0
#define RAMA_ERR_INVALID 1  /* bad input -> ValueError (graph.py:31-42, solver.py:50-62) */
#define RAMA_ERR_CUDA 2     /* CUDA runtime failure -> RuntimeError */
#define RAMA_ERR_NOMEM 3    /* device allocation failed -> MemoryError */
#define RAMA_ERR_INTERNAL 4

/* solver modes: solver.py:22 MODES */
#define RAMA_MODE_P 0
#define RAMA_MODE_PD 1
#define RAMA_MODE_PD_PLUS 2
#define RAMA_MODE_D 3
#define RAMA_MODE_GAEC 4

/* round phases: RoundRecord.phase (solver.py:65-75) */
#define RAMA_PHASE_CONTRACT 0
#define RAMA_PHASE_PRIMAL_DUAL 1
#define RAMA_PHASE_CLEANUP 2
#define RAMA_PHASE_DUAL 3
#define RAMA_PHASE_GAEC 4

/* SolverConfig (solver.py:27-62); max_cycle_length already resolved */
typedef struct rama_cfg {
  int32_t mode;
  int32_t mp_iterations;
  int32_t max_cycle_length;
  int32_t max_rounds;
  int32_t separation_rounds;
  int32_t reserved;
  double matching_switch_fraction;
} rama_cfg;

/* RoundRecord (solver.py:65-75); lb is NaN where the reference has None */
typedef struct rama_round {
  int32_t round_index;
  int32_t phase;
  int64_t nodes;
  int64_t edges;
  int64_t triplets;
  double lb;
  int32_t lb_valid;
  int32_t reserved;
  int64_t contracted;
  double time_ms;
} rama_round;

/* library version (major*10000 + minor*100 + patch) */
int rama_version(void);
/* message of the last failed call on this thread ("" if none) */
const char* rama_last_error(void);
/* number of kernels the last call on this thread launched */
int64_t rama_last_launch_count(void);

/* Live kernel-family timing for roofline reporting: when enabled, each
 * kernel family is bracketed by CUDA events on the call's stream.
 * Families (index): 0 separate, 1 triangulate, 2 message passing, 3 bound /
 * reparam graph, 4 matching, 5 forest, 6 components, 7 contract, 8 cleanup
 * (inclusive), 9 canonicalize.  rama_profile_read fills host arrays of
 * RAMA_PROFILE_FAMILIES: summed device ms, summed algorithmic bytes
 * (SURVEY.md 8(d) formulas), scope count.  Enabling resets the sums. */
#define RAMA_PROFILE_FAMILIES 10
int rama_profile_enable(int32_t on);
int rama_profile_read(double* ms, double* bytes, int64_t* count);
/* Per-kernel view of the same timing: JSON text
 * {"kernel_name": [device_ms, algorithmic_bytes, launches], ...} written to
 * out (host, cap bytes).  Returns the size needed including the NUL; if
 * cap is smaller nothing is written. */
int64_t rama_profile_kernels(char* out, int64_t cap);

/* ---- solver (solver.py:243-252 solve) ------------------------------------ */

/* Full solve on a canonical graph (non-canonical COO is canonicalised
 * first, WeightedGraph semantics).  labels: device int32[n] (canonical
 * labeling, Solution.labeling).  primal_lb: host double[2] =
 * {primal_cost, lower_bound} (lower_bound = -inf for P / GAEC).  trace: host
 * rama_round[max_trace] (may be NULL); *n_rounds (host) = records written. */
int rama_solve(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
               const rama_cfg* cfg, int32_t* labels, double* primal_lb, rama_round* trace,
               int32_t max_trace, int32_t* n_rounds, void* stream);

/* Caller-owned scratch (SURVEY.md 8(b) ownership): rama_solve with every
 * scratch buffer carved from the caller's DEVICE block ws[ws_bytes] (e.g. a
 * tensor from torch's caching allocator) instead of the library's cached
 * stream-ordered pool.  ws must stay valid until the call returns and must
 * not be used by other work on other streams meanwhile.  A block too small
 * fails with RAMA_ERR_NOMEM (nothing written); *ws_peak (host, may be NULL)
 * receives the high-water mark the call used. */
int rama_solve_ws(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
                  const rama_cfg* cfg, int32_t* labels, double* primal_lb, rama_round* trace,
                  int32_t max_trace, int32_t* n_rounds, void* ws, uint64_t ws_bytes, uint64_t* ws_peak,
                  void* stream);

/* Workspace estimate for rama_solve_ws on a graph of n nodes and m edges:
 * 400 B per edge + 96 B per node + 64 MiB (measured high-water marks per
 * edge: C5 143, C2 189, C3 209, C4 267 bytes). */
uint64_t rama_ws_bytes(int64_t n, int64_t m, const rama_cfg* cfg);

/* Return every block the library's own pool caches (all devices). */
int rama_release_cache(void);

/* Mode D runs cfg->separation_rounds rounds (extend_separation from round
 * 2, solver.py:211-240); PD+ (max_cycle_length 6..8) uses the exact
 * source-grouped BFS separation. */

/* Same with HOST arrays (u, v, c, labels): the end-to-end entry for
 * non-CUDA callers (numpy through ctypes).  Pinned host buffers are copied
 * directly; pageable ones through a cached pinned staging area (16 MiB
 * chunks, parallel host memcpy overlapped with the DMA). */
int rama_solve_host(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
                    const rama_cfg* cfg, int32_t* labels, double* primal_lb, rama_round* trace,
                    int32_t max_trace, int32_t* n_rounds, void* stream);

/* Batch of independent instances; replaces a
 * Python loop of solve() calls (solver.py:243-252).  Instance i is the COO
 * slice [edge_off[i], edge_off[i+1]) of u, v, c with node ids local to the
 * instance, n_i = node_off[i+1] - node_off[i] nodes; its labels go to
 * labels + node_off[i].  node_off, edge_off (count + 1 entries), primal_lb
 * (2 * count: {primal, lower_bound} per instance), trace (count x max_trace
 * records, instance-major; may be NULL) and n_rounds (count; may be NULL)
 * are HOST arrays; u, v, c, labels are device arrays.
 * Modes P / PD / PD+: the instances are split into `workers` contiguous
 * groups (0 = 1), each solved as ONE disjoint-union graph on its own
 * internal stream -- every round's kernels run once for the whole group, and
 * each instance's labels, objectives and trace equal its single solve bit for
 * bit.  Modes D / GAEC: one solve per instance on `workers` streams.  All work
 * is ordered after prior work on `stream`; the call returns when it is done. */
int rama_solve_batch(int64_t count, const int64_t* node_off, const int64_t* edge_off, const int32_t* u,
                     const int32_t* v, const double* c, const rama_cfg* cfg, int32_t* labels, double* primal_lb,
                     rama_round* trace, int32_t max_trace, int32_t* n_rounds, int32_t workers, void* stream);

/* ---- graph core ----------------------------------------------------------- */

/* WeightedGraph.__init__ (graph.py:29-57): validate, orient, sort, sum
 * parallel edges (np.add.reduceat order).  out_*: capacity m. */
int rama_canonicalize(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
                      int32_t* out_u, int32_t* out_v, double* out_c, int64_t* out_m, void* stream);

/* clustering_cost (graph.py:134-145); *cost is host */
int rama_clustering_cost(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
                         const int32_t* labels, double* cost, void* stream);

/* ---- contraction (contraction.py) ---------------------------------------- */

/* connected_components (contraction.py:101-111): canonical map[n]. */
int rama_components(int64_t n, const int32_t* su, const int32_t* sv, int64_t k, int32_t* map,
                    int64_t* num_targets, void* stream);

/* contract_graph (contraction.py:142-163) on a canonical graph.  out_*:
 * capacity m; *joined (host) = cost mass of merged edges. */
int rama_contract(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
                  const int32_t* map, int64_t n_targets, int32_t* out_u, int32_t* out_v, double* out_c,
                  int64_t* out_m, double* joined, void* stream);

/* select_matching (contraction.py:179-228): su/sv capacity n/2 + 1 */
int rama_select_matching(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
                         int32_t rounds, int32_t* su, int32_t* sv, int64_t* k, void* stream);

/* select_max_edge (contraction.py:166-176): *edge (host) = index or -1 */
int rama_select_max_edge(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
                         int64_t* edge, void* stream);

/* select_spanning_forest_no_conflicts (contraction.py:287-366):
 * su/sv capacity n */
int rama_select_forest(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
                       int32_t* su, int32_t* sv, int64_t* k, void* stream);

/* contraction_step (contraction.py:369-394); policy 0 gaec, 1 matching,
 * 2 forest, 3 auto.  map: capacity n (identity when nothing selected);
 * out_*: capacity m.  info (host int64[4]) = {num_targets, |S|, m_out,
 * used_forest}; *joined host. */
int rama_contraction_step(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
                          int32_t policy, double switch_fraction, int32_t* map, int32_t* out_u,
                          int32_t* out_v, double* out_c, int64_t* info, double* joined, void* stream);

/* ---- dual (dual.py) -------------------------------------------------------- */

/* _separate_arrays (dual.py:169-197): one row per repulsive edge in
 * ascending (u, v) order.  out_len capacity m, out_nodes capacity m*L
 * (row-major, width L, zero padded); *rows (host) = repulsive edge count.
 * 3 <= L <= 5. */
int rama_separate(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m, int32_t L,
                  int32_t* out_len, int32_t* out_nodes, int64_t* rows, void* stream);

/* _triangulate_arrays (dual.py:255-290).  Capacities: aug_u/aug_v/base/
 * coverage m + rows*(L-3); tri_nodes/tri_edges 3*rows*(L-2).  Outputs the
 * reference layout: augmented edges = originals then new chords (sorted),
 * triplets sorted lexicographically, handles (ij, ik, jk). */
int rama_triangulate(int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m,
                     const int32_t* len, const int32_t* nodes, int64_t rows, int32_t L, int32_t* aug_u,
                     int32_t* aug_v, double* base, int64_t* m_aug, int32_t* tri_nodes, int32_t* tri_edges,
                     int64_t* T, int32_t* coverage, void* stream);

/* extend_separation (dual.py:414-474): separate on the current
 * reparametrized costs of the state (eu/ev/base over m_aug augmented edges,
 * T triplets with handles and multipliers) and append the new chords (base
 * 0) and new triplets (zero multipliers) in the reference's order.  The
 * grown state is written to out_* (capacities cap_edges edges and
 * cap_triplets triplets; m_aug * (L - 2) extra of each always suffices);
 * *added (host) = triplets appended. */
int rama_extend_separation(int64_t n, int64_t m_aug, const int32_t* eu, const int32_t* ev, const double* base,
                           int64_t T, const int32_t* tri_nodes, const int32_t* tri_edges, const double* lam,
                           int32_t L, int64_t cap_edges, int64_t cap_triplets, int32_t* out_eu, int32_t* out_ev,
                           double* out_base, int64_t* out_m_aug, int32_t* out_tri_nodes, int32_t* out_tri_edges,
                           double* out_lam, int64_t* out_T, int32_t* out_coverage, int64_t* added, void* stream);

/* check_edge_triangle_agreement (dual.py:477-531): arc consistency of the
 * eps-optimal edge and triplet label sets; *agree (host) = 1 if every set
 * stays non-empty. */
int rama_check_agreement(int64_t m_aug, const double* base, int64_t T, const int32_t* tri_edges, const double* lam,
                         double eps, int32_t* agree, void* stream);

/* message passing on lam[3T] in place (dual.py:358-392).
 * phases: 1 = mp_edge_to_triplets only, 2 = mp_triplets_to_edges only,
 * 3 = message_passing_iteration; repeated `iters` times. */
int rama_message_passing(int64_t m_aug, const double* base, int64_t T, const int32_t* tri_edges, double* lam,
                         int32_t iters, int32_t phases, void* stream);

/* reparametrized_edge_costs (dual.py:309-316): cl[m_aug] */
int rama_reparam_costs(int64_t m_aug, const double* base, int64_t T, const int32_t* tri_edges, const double* lam,
                       double* cl, void* stream);

/* lower_bound (dual.py:395-405); *lb host */
int rama_lower_bound(int64_t m_aug, const double* base, int64_t T, const int32_t* tri_edges, const double* lam,
                     double* lb, void* stream);

/* ---- MULTICUT text format (graph.py:160-313) -----------
 * Host-only (no CUDA device needed).  Errors: RAMA_ERR_INVALID with the
 * reference's ParseError message in rama_io_last_error(). */

/* message of the last failed rama_parse_multicut / rama_serialize_multicut */
const char* rama_io_last_error(void);

/* parse_instance (graph.py:204-263): text[len] (host), or the file `path`
 * (mmap'ed) when path != NULL.  Raw edges (before canonicalisation, in file
 * order) go to host u, v, c of capacity cap; *m = edges, *n = node count
 * (NODES, else 1 + max id).  If *m > cap nothing is copied (call again).
 * threads: worker threads (0 = all cores). */
int rama_parse_multicut(const char* text, int64_t len, const char* path, int64_t* n, int64_t* m, int64_t* u,
                        int64_t* v, double* c, int64_t cap, int32_t threads);

/* serialize_instance (graph.py:300-313): 'MULTICUT', 'NODES n', then
 * '<u> <v> <repr(cost)>' per edge.  Writes to out (host, cap bytes) when it
 * fits; *len = bytes of the text (no NUL). */
int rama_serialize_multicut(int64_t n, const int64_t* u, const int64_t* v, const double* c, int64_t m, char* out,
                            int64_t cap, int64_t* len, int32_t threads);

#ifdef __cplusplus
}
#endif

#endif /* RAMA_B200_H */
