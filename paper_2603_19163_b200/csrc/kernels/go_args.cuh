// go_args.cuh — POD kernel argument blocks shared by host and device code.
#pragma once
#include "go_common.cuh"

namespace go {

// Registry image in device memory, rewritten by the epilogue at every AOS
// barrier (aos.py:116-144) and by the host at set-up.
struct RegistryDev {
  int nseq;
  int kind[32];       // implementation code: 0..16 built-in seq id, 100+slot custom
  int ids[32];        // sequence id as the reference names it
  double w[32];       // normalised weights
  double floor_[32];  // per-sequence floor / cap (SequenceEntry, operators.py:70-76)
  double cap[32];
  double cum[32];     // sequential prefix sums used by sample_sequence (aos.py:169-175)
  double total;       // sum(e.weight ...) as the reference computes it
  double kw[3];       // K-level weights (aos.py:19, :137-144)
};

// Run-global state owned by the device (engine.py:668-750 locals).
struct GlobalState {
  double gscal, gpen;     // global best (engine.py:668, :703-708)
  double gobj[2];         // its objective vector (multi-objective runs)
  int gev;                // evolver holding the global best in best_genes (-1: gbest buffer)
  int pad0;
  long long ggen;         // generation the global best was found (0 = initial population)
  long long gens_done;
  long long stall;        // no_improve_batches (engine.py:708)
  long long mig_events;   // engine.py:675, :743
  long long deadline_ns;  // %globaltimer deadline, 0 = none
  int stop;               // 0 run, 1 time, 2 target, 3 max generations
  int err;                // sticky device error bits
  long long hist_count;
  unsigned long long rd_pos;   // positions read by move evaluations (all lanes)
  unsigned long long rd_elem;  // matrix elements read by move evaluations
  unsigned long long prof[32]; // per-phase clock64 totals / deferred-op timings (GO_PHASE_TIMING)
};

struct EvolveArgs {
  const void* inst;      // instance image (layout specific)
  unsigned inst_bytes;   // bytes staged into shared memory (0 = read from global)
  int n;                 // row length (single-row permutation)
  short* genes;          // [P][n]
  double* scal;          // [P] scalarised objective (lower is better)
  double* pen;           // [P]
  short* best_genes;     // [P][n] each team's best-ever current (first occurrence)
  double* best_scal;     // [P]
  double* best_pen;      // [P]
  long long* best_gen;   // [P]
  int* usage;            // [P][32] per-chunk AOS counters (aos.py:51-77)
  int* impr;             // [P][32]
  int* k_usage;          // [P][3]
  int* k_impr;           // [P][3]
  double* rec_scal;      // [ngen][P] current after each generation
  double* rec_pen;       // [ngen][P]
  const RegistryDev* reg;
  GlobalState* gs;
  const double* temps;   // [ngen] T0 * alpha^(g-1) (engine.py:685), host pow()
  unsigned long long seed;
  long long gen0;        // first generation of this chunk (1-based)
  int ngen;
  int P, T, E;           // evolvers, lanes per evolver, evolver teams per CTA
  int ev_offset;         // global evolver index of local evolver 0
  int team_stride;       // threads per team (T rounded up to 32)
  int team_smem;         // bytes of shared memory per team
  int resync;            // recompute Φ at chunk start (float matrices)
  // crossover mates (engine.py:553-559): the island snapshot of generation g
  // is snap[g % SNAP_DEPTH] ([SNAP_DEPTH][P][n]).  The host copies genes into
  // the slot of gen0 and sets prog[*] = gen0 before the launch; after
  // generation g a team publishes its row in slot g+1 and then prog[ev] = g+1.
  // A lane reading mate j's generation-g row waits for prog[j] >= g; a team
  // overwriting slot g+1 first waits until every prog >= g+2-SNAP_DEPTH (no
  // reader of that slot's previous generation remains).  Teams thus drift up
  // to SNAP_DEPTH-2 generations apart instead of meeting every generation.
  // snap == null: no crossover in the registry.
  short* snap;
  int* prog;
  int islands;           // island count (engine.py:790-798 contiguous partition)
  int pad_x;
  short* lane_rows;      // permutation kernel: [P][T][2][n] rows of deferred whole-row ops
  // objective vectors [P][2] (null unless MoCmp.m == 2 or lex): current, team
  // best-ever, and per-generation records [ngen][P][2]
  double* obj2;
  double* best_obj2;
  double* rec_obj2;
  // target_objective (engine.py:712-716, single objective): once a team's
  // best-ever reaches the target its best_genes row is frozen, so a run the
  // epilogue stops at generation g mid-chunk returns the genes of generation g
  int has_target;
  int pad_t;
  double target;
  double obj_sign_over_w; // objective = scal * this
};

// the epilogue's target predicate (go_epilogue.cuh) on one (penalty, scal)
__device__ __forceinline__ bool target_reached(const EvolveArgs& A, double pen, double scal) {
  if (!A.has_target || pen > 0.0) return false;
  const double v = scal * A.obj_sign_over_w;
  return A.obj_sign_over_w > 0 ? v <= A.target + 1e-9 : v >= A.target - 1e-9;
}

// Problem-specific extras of the row kernel (go_evolve_row.cuh).
struct RowArgs {
  unsigned off1;         // byte offset of the second instance array (QAP D, knapsack v, JSP durations)
  double capacity;       // knapsack capacity (builtins.py:258-262)
  double penalty_weight; // engine.py:651-655
  double obj_weight;     // Weighted scalarisation weight (Maximize negated inside)
  int n_jobs, per_job, n_mach;  // JSP-int
  int n_cfg;             // ProblemConfig.n (lns_scope)
  int lb, ub;            // integer encoding bounds
  int scratch_ints;      // per-lane int scratch (JSP decode)
  // partition problems (VRPTW / CVRP): compact row = cells[n_cells] + sizes[d1]
  unsigned off2, off3, off4;  // ready, due, service offsets (off1 = demands)
  int n_cells, d1, d2, tw;
  // user problems (NVRTC objective): encoding 0 permutation, 1 binary, 2 integer
  int enc, maximize;
  // routing objectives: kind of objective i (0 distance, 1 vehicles), second
  // scalar_fitness weight (engine.py:215-222), comparison mode
  int okind0, okind1;
  double w2;
  MoCmp mo;
  int pvar;              // partition variant: 0 plain, 1 vrp_priority (priorities at off2), 2 vrp_nonlinear
  int mf;                // MULTI_FIXED user rows (d1 x d2 flat): 0 no, 1 permutation rows, 2 cells
};

struct EpilogueArgs {
  int P, W;              // evolvers, genes per solution
  short* genes;
  double* scal;
  double* pen;
  short* best_genes;
  double* best_scal;
  double* best_pen;
  long long* best_gen;
  short* gbest_genes;    // [W]
  short* scratch;        // [max(islands, top_n)][W] donor copies
  const int* usage;
  const int* impr;
  const int* k_usage;
  const int* k_impr;
  long long* agg;        // [32 + 32 + 3 + 3] aggregated AOS counters
  const double* rec_scal;
  const double* rec_pen;
  RegistryDev* reg;
  GlobalState* gs;
  double* history;       // [hist_cap] best Φ per generation or null
  long long hist_cap;
  int* host_stop;        // mapped host flag mirroring gs->stop (may be null)
  long long gen0;
  int ngen;
  double pw;             // penalty weight
  // AosConfig (aos.py:22-38)
  int aos_interval, stagnation;
  double alpha, floor_, cap, eps;
  // islands (engine.py:90-106)
  int islands, migration, mig_interval, top_n;
  int elite_interval;
  int has_target;
  double target;
  double obj_sign_over_w; // objective = scal * this (single objective)
  unsigned long long seed;
  long long max_gens;
  // multi-objective (MoCmp.m == 2 or lex): objective vectors [P][2]
  double* obj2;
  double* best_obj2;
  const double* rec_obj2;
  MoCmp mo;
};

}  // namespace go
