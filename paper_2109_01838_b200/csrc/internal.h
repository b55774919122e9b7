// Host-side internal API of the RAMA B200 library (one function per hot
// path operator of SURVEY.md section 8(a)).  Everything takes device
// pointers and is ordered on ctx.s.
#pragma once

#include "common.cuh"

namespace rama {

struct GraphView {
  int64_t n = 0, m = 0;
  const int32_t* u = nullptr;
  const int32_t* v = nullptr;
  const double* c = nullptr;
};

// owning canonical graph: u < v, sorted by (u, v), unique pairs
struct Graph {
  int64_t n = 0, m = 0;
  Buf<int32_t> u, v;
  Buf<double> c;
  GraphView view() const {
    GraphView g;
    g.n = n; g.m = m; g.u = u.p; g.v = v.p; g.c = c.p;
    return g;
  }
};

// ---- host buffers (staging.cu) ------------------------------------------------
// host -> device (ordered on ctx.s; the host buffer may be reused on return)
// and device -> host (complete on return); pageable host memory goes through
// pinned staging chunks with a parallel memcpy overlapped with the DMA
void copy_h2d(Ctx& ctx, void* dst, const void* src, size_t bytes);
void copy_d2h(Ctx& ctx, void* dst, const void* src, size_t bytes);

// ---- graph core (graph.cu) --------------------------------------------------
// a3  WeightedGraph.__init__ (graph.py:29-57)
Graph canonicalize(Ctx& ctx, int64_t n, const int32_t* u, const int32_t* v, const double* c, int64_t m);
// the WeightedGraph invariant: ids in range, u < v, (u, v) strictly ascending
bool is_canonical(Ctx& ctx, const GraphView& g);
// a17 connected_components (contraction.py:101-111); returns num_targets
// (check: validate endpoint ranges first -- the C ABI entry; internal callers
// pass edges that are valid by construction)
// keep_rank: the count stays on the device at keep_rank[n] (no read-back;
// returns -1)
int64_t components(Ctx& ctx, int64_t n, const int32_t* su, const int32_t* sv, int64_t k, int32_t* map,
                   bool check = false, Buf<int32_t>* keep_rank = nullptr);
// a18 contract_graph (contraction.py:142-163); *joined (host) may be null.
// nt_dev: the target count is on the device (n_targets only bounds it); it is
// read back together with the edge count
Graph contract(Ctx& ctx, const GraphView& g, const int32_t* map, int64_t n_targets, double* joined,
               const int32_t* nt_dev = nullptr);
// a19 ContractionMapping.then (contraction.py:45-52): f_total = f[f_total]
void compose(Ctx& ctx, int32_t* f_total, int64_t n0, const int32_t* f);
// a21 clustering_cost (graph.py:134-145)
double clustering_cost(Ctx& ctx, const GraphView& g, const int32_t* labels);
// per-edge cut cost x[e] = c[e] if labels differ else 0 (the summands of clustering_cost)
void cut_costs(Ctx& ctx, const GraphView& g, const int32_t* labels, double* x);
void iota(Ctx& ctx, int32_t* x, int64_t n);

// ---- contraction-set selection (select.cu) ---------------------------------
// a14 select_matching (contraction.py:179-228); pairs sorted by u
int64_t select_matching(Ctx& ctx, const GraphView& g, int rounds, Buf<int32_t>& su, Buf<int32_t>& sv);
// select_max_edge (contraction.py:166-176); returns edge index or -1
int64_t select_max_edge(Ctx& ctx, const GraphView& g);
// a15/a16 select_spanning_forest_no_conflicts (contraction.py:287-366)
int64_t select_forest(Ctx& ctx, const GraphView& g, Buf<int32_t>& su, Buf<int32_t>& sv);

struct StepResult {
  Graph next;            // contracted graph (empty if identity)
  Buf<int32_t> map;      // f (size g.n) unless identity
  int64_t num_targets = 0;
  int64_t num_selected = 0;
  bool identity = true;
  bool used_forest = false;
  double joined = 0.0;
};
// a13 contraction_step (contraction.py:369-394); policy: 0 gaec, 1 matching,
// 2 forest, 3 auto
void contraction_step(Ctx& ctx, const GraphView& g, int policy, double switch_fraction, StepResult& out,
                      bool want_joined = false);

// ---- dual (dual.cu) ---------------------------------------------------------
struct CycleRows {
  int64_t rows = 0;  // one row per repulsive edge (ascending (u, v))
  int L = 0;
  Buf<int32_t> len;    // rows
  Buf<int32_t> nodes;  // rows * L
};
// a4/a5 _separate_arrays (dual.py:155-197)
// (the 5-cycle searches the capped table passes truncate -- hub
// neighbourhoods -- are rerun by the exact ordered search)
void separate(Ctx& ctx, const GraphView& g, int L, CycleRows& out);

struct DualState {
  int64_t n = 0, m_orig = 0, m_aug = 0, T = 0;
  bool chords_sorted = true;  // [m_orig, m_aug) is one sorted run (false after extend_separation)
  Buf<int32_t> eu, ev;      // augmented edges: originals then new chords
  Buf<double> base;         // m_aug
  Buf<int32_t> tri_nodes;   // T*3 sorted (i<j<k), rows sorted lexicographically
  Buf<int32_t> tri_edges;   // T*3 handles (ij, ik, jk)
  Buf<int32_t> coverage;    // m_aug
  Buf<int32_t> orig_ptr;    // n + 1: rows of the originals [0, m_orig) (sorted by (u, v))
  Buf<int32_t> chord_ptr;   // n + 1: rows of the chords [m_orig, m_aug) (valid while chords_sorted)
  Buf<int32_t> slot_ptr;    // m_aug + 1 : edge -> ascending slot list
  Buf<int32_t> slots;       // 3T
  Buf<double> lam;          // 3T
  Buf<int32_t> long_e;      // edges with more than kLongCov slots (hubs), count on the device in n_long
  Buf<int32_t> n_long;
};
// a6/a7 _triangulate_arrays (dual.py:216-290)
// steal: g's owner, whose buffers DualState may take over when they have
// room for the chords (no copy of the m edges; the owner is left empty)
void triangulate(Ctx& ctx, const GraphView& g, const CycleRows& cyc, DualState& st, Graph* steal = nullptr);
// extend_separation (dual.py:414-474): returns the number of triplets added
int64_t extend_separation(Ctx& ctx, DualState& st, int L);
// a8 reparametrized_edge_costs (dual.py:309-316)
void reparam_costs(Ctx& ctx, const DualState& st, double* cl);
// a9/a10 message_passing_iteration x iters (dual.py:358-392)
void message_passing(Ctx& ctx, DualState& st, int iters);
// mp_edge_to_triplets / mp_triplets_to_edges individually (dual.py:358, 374)
void mp_phases(Ctx& ctx, DualState& st, bool edge_phase, bool triplet_phase);
// check_edge_triangle_agreement (dual.py:477-531)
bool check_edge_triangle_agreement(Ctx& ctx, const DualState& st, double eps);
// a11 lower_bound (dual.py:395-405)
// (cl_out: optional m_aug buffer receiving c^lambda for a following
// reparametrized_graph call)
double lower_bound(Ctx& ctx, const DualState& st, double* cl_out = nullptr);
// the summands of lower_bound: neg[m_aug] = min(0, c^lambda_e), tm[T] = the
// triplets' minimal pattern costs (cl_out optional)
void lower_bound_terms(Ctx& ctx, const DualState& st, double* cl_out, double* neg, double* tm);
// lower_bound into a device scalar (no read-back; same value bit for bit)
void lower_bound_to(Ctx& ctx, const DualState& st, double* cl_out, double* out);
// a12 reparametrized_graph (dual.py:408-411): canonical merge of originals
// and chords carrying c^lambda
Graph reparametrized_graph(Ctx& ctx, const DualState& st, const double* cl = nullptr);
// lower_bound_to + reparametrized_graph with one pass over the augmented
// edges (c^lambda goes straight to the merged graph)
Graph bound_and_reparametrized(Ctx& ctx, const DualState& st, double* lb_out);
// edge -> slot CSR + coverage for an existing tri_edges array
void build_slot_lists(Ctx& ctx, DualState& st);

// ---- cleanup (cleanup.cu) -----------------------------------------------------
// a20 replacement (DESIGN.md deviation D1): handshake rounds on the quotient q
// until no mutual pair remains; writes the canonical map fc[q.n], returns the
// number of clusters
int64_t handshake_cleanup(Ctx& ctx, const GraphView& q, int32_t* fc);

// ---- driver (solver.cu) -----------------------------------------------------
struct SolveConfig {
  int mode = 1;  // 0 P, 1 PD, 2 PD+, 3 D, 4 GAEC
  int mp_iterations = 5;
  int max_cycle_length = 5;
  double switch_fraction = 0.1;
  int max_rounds = 100;
  int separation_rounds = 1;
};

struct RoundInfo {
  int32_t round_index;
  int32_t phase;  // 0 contract, 1 primal-dual, 2 cleanup, 3 dual, 4 gaec
  int64_t nodes, edges, triplets;
  double lb;
  int32_t lb_valid;
  int64_t contracted;
  double time_ms;
};

struct SolveResult {
  double primal = 0.0;
  double lb = 0.0;
  bool lb_finite = false;
  int n_rounds = 0;
};

void solve(Ctx& ctx, const GraphView& g, const SolveConfig& cfg, int32_t* labels, SolveResult& res,
           RoundInfo* trace, int max_trace);

// ---- batch (batch.cu) -----------------------------------------------------------
// K independent instances (modes P, PD, PD+) solved as one disjoint union:
// instance i = COO slice [edge_off[i], edge_off[i+1]) of u, v, c (device,
// local ids), n_i = node_off[i+1] - node_off[i] (host offsets).  labels
// (device, node_off layout) receive each instance's canonical labeling;
// primal_lb[2i], [2i+1] (host); traces (host, K x max_trace, may be null)
// and n_rounds[K] (host, may be null) each instance's RoundRecords.  Every
// instance's result equals its single solve bit for bit.
void solve_union(Ctx& ctx, int64_t K, const int64_t* node_off, const int64_t* edge_off, const int32_t* u,
                 const int32_t* v, const double* c, const SolveConfig& cfg, int32_t* labels, double* primal_lb,
                 RoundInfo* traces, int max_trace, int32_t* n_rounds);

}  // namespace rama
