/*
 * cugenopt.h — C ABI of the B200-native cuGenOpt evolve engine (libcugenopt.so).
 *
 * The reference (`/root/reference/pkg/src/genopt`, pure Python) has no native
 * boundary; these entry points replace the Python functions named beside each
 * one, so a reference-side binding (ctypes) can swap the
 * per-lane Python loop for one device call.  Conventions:
 *   - every function returns GO_OK (0) or a negative GO_E* status and sets a
 *     thread-local message readable with go_last_error();
 *   - all array arguments are HOST pointers (plain C types); the library owns
 *     device memory; sizes are element counts;
 *   - solutions are passed as `genes[m][d1*d2]` int32 row-major plus
 *     `sizes[m][d1]` int32 (reference core.Solution, core.py:154-200);
 *   - one engine is bound to one device and is not re-entrant.
 */
#ifndef CUGENOPT_H
#define CUGENOPT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GO_ABI_VERSION 1

enum go_status {
  GO_OK = 0,
  GO_E_INVALID = -1,     /* bad argument -> ValueError (engine.py:131-147) */
  GO_E_CUDA = -2,        /* CUDA runtime/driver failure */
  GO_E_UNSUPPORTED = -3, /* layout/problem the device path does not implement */
  GO_E_COMPILE = -4,     /* NVRTC compile failure (operator excluded, operators.py:649-657) */
  GO_E_NODEVICE = -5     /* no CUDA device visible */
};

/* problem kinds (builtins.py:24-39 names) */
enum go_kind {
  GO_TSP = 0,       /* builtins.py:53-77 */
  GO_VRPTW = 1,     /* builtins.py:155-190 (CVRP when time windows absent) */
  GO_QAP = 2,       /* builtins.py:265-290 */
  GO_JSP_INT = 3,   /* builtins.py:408-456 */
  GO_KNAPSACK = 4,  /* builtins.py:240-262 */
  GO_CVRP = 5,      /* builtins.py:80-152 */
  GO_USER = 6,      /* NVRTC objective (go_problem_create_user) */
  GO_VRP_PRIORITY = 7,   /* builtins.py:193-210 (CVRP + precedence penalty) */
  GO_VRP_NONLINEAR = 8   /* builtins.py:213-237 (load-dependent edge cost) */
};

/* migration strategies (engine.py:483-521, :731-733) */
enum go_migration { GO_MIG_RING = 0, GO_MIG_GLOBAL_TOP_N = 1, GO_MIG_HYBRID = 2 };

/* Primitive moves the parity hook go_delta_batch applies (operators.py:205-283
 * expressed as position maps). */
enum go_move_kind {
  GO_MOVE_NONE = 0,
  GO_MOVE_SWAP = 1,    /* a,b: swap positions a != b                     (op_swap)    */
  GO_MOVE_REVERSE = 2, /* a<b: reverse positions [a, b]                  (op_reverse) */
  GO_MOVE_SEGMENT = 3, /* a=start, b=len, c=pos: remove [a,a+b), reinsert
                          at c of the shortened row (op_insert: b=1; op_or_opt) */
  GO_MOVE_THREE_OPT = 8 /* + variant 0..6; a<b<c = cuts i<j<k in (0, n): row a|b|c|d
                          reconnected as op_three_opt's variant (operators.py:289-315) */
};

typedef struct go_move { int32_t kind, a, b, c; } go_move;

typedef struct go_device_info {
  int32_t device, sm_count, max_smem_optin, l2_bytes, cc_major, cc_minor;
  int64_t global_mem;
  char name[96];
} go_device_info;

/* Instance description (borrowed host pointers, copied at creation).
 * Only the fields of `kind` are read (problems.py:18-46 InstanceData). */
typedef struct go_problem_desc {
  int32_t kind;
  int32_t n;             /* cities / facilities / customers / items / operations */
  int32_t d1, d2;        /* solution layout (core.py:112-151) */
  const double* dist;    /* TSP n*n, QAP n*n, VRPTW (n+1)*(n+1) */
  const double* flow;    /* QAP n*n */
  const double* weights; /* knapsack */
  const double* values;  /* knapsack */
  const double* demands; /* VRPTW n */
  const double* ready;   /* VRPTW n+1 (index 0 = depot) */
  const double* due;
  const double* service;
  double capacity;       /* knapsack / VRPTW */
  int32_t n_jobs, n_machines, ops_per_job;
  const int32_t* jsp_machine; /* n_jobs*ops_per_job */
  const int32_t* jsp_duration;
  int32_t lb, ub;        /* integer encoding bounds */
  int32_t n_obj;         /* routing: 1 or 2 objectives (builtins.py:80-116); 0 = 1 */
  int32_t obj_kind[2];   /* routing objective i: 0 "distance", 1 "vehicles" */
  const double* priorities; /* GO_VRP_PRIORITY: n customer priorities */
} go_problem_desc;

/* A user-defined single-row problem whose objective and penalty are CUDA
 * snippets compiled by NVRTC for sm_100a (the paper's solve_custom, PAPER.md:858-868;
 * the reference's ProblemDefinition callbacks, problems.py:49-74).  The snippets are
 * the bodies of
 *     template <class Sol> double compute_obj(const Sol& sol, const Data& data)
 *     template <class Sol> double compute_penalty(const Sol& sol, const Data& data)
 * reading genes as sol[i] (0 <= i < sol.n) and each named array as data.<name>
 * (const double*, length data.<name>_len).  Data arrays are copied at creation. */
typedef struct go_user_problem_desc {
  int32_t encoding;               /* 0 permutation, 1 binary, 2 integer (core.py:18-66) */
  int32_t n;                      /* genes per row (dim2) */
  int32_t lb, ub;                 /* integer encoding bounds (ignored otherwise) */
  const char* compute_obj;        /* snippet body (required) */
  const char* compute_penalty;    /* snippet body or NULL: penalty 0 */
  int32_t n_data;
  const char* const* data_names;  /* C identifiers */
  const double* const* data;
  const int64_t* data_lens;
  int32_t rows;                   /* 0 or 1: one row; > 1: MULTI_FIXED rows of n genes each
                                   * (core.py:28-35), sol[r * n + i] in the snippets */
  const char* compute_obj2;       /* second objective's snippet body, or NULL (one objective) */
} go_user_problem_desc;

typedef struct go_problem go_problem;
typedef struct go_engine go_engine;

/* A user operator: a CUDA snippet compiled by NVRTC into the evolve kernel
 * (paper §3.3.2 "JIT injection"; reference CustomOperator operators.py:79-88). */
typedef struct go_custom_op {
  int32_t id;            /* >= 100 (operators.py:641-645) */
  const char* name;
  const char* cuda_body; /* body of `__device__ void op(go::OpCtx& ctx)` */
} go_custom_op;

typedef struct go_engine_config {
  int32_t population;    /* P evolvers */
  int32_t team_size;     /* T lanes per evolver (engine.py:111) */
  int32_t teams_per_cta; /* 0 = auto (evolvers sharing one CTA's smem instance) */
  uint64_t seed;
  double t0;             /* initial temperature (engine.py:669-671, host-derived) */
  double cooling_alpha;  /* engine.py:116 */
  double penalty_weight; /* engine.py:651-655, host-derived */
  int32_t aos_interval;  /* aos.py:22-48 */
  double aos_alpha, aos_floor, aos_cap, aos_eps;
  int32_t stagnation_threshold;
  int32_t islands, migration, migration_interval, top_n;
  int32_t elite_interval;
  int32_t has_target;
  double target_objective;
  int32_t evolver_offset; /* global evolver index of local evolver 0 (multi-GPU) */
  int32_t maximize;       /* objective direction (core.py:69-77) */
  double obj_weight;      /* Weighted scalarisation weight (core.py:292-307) */
  /* multi-objective problems (n_obj == 2) and Lexicographic comparisons:
   * scalar_fitness weight of objective 1 (engine.py:215-222), and the mode
   * (core.py:92-106): lex = 1 compares objective vectors in priority order
   * (lex_first, 1 - lex_first) with tolerances lex_tol.  With n_obj == 2 the
   * `obj` arrays of set/get_population and get_best hold 2 values per solution. */
  double obj_weight2;
  int32_t lex;
  int32_t lex_first;
  double lex_tol[2];
  int32_t maximize2;      /* direction of the second objective (two-objective user problems) */
} go_engine_config;

typedef struct go_run_stats {
  int64_t generations;    /* generations completed by every evolver */
  int64_t lane_evals;     /* P * T * generations (move evaluations) */
  int64_t kernel_launches;
  double device_ms;       /* CUDA-event time of the evolve+epilogue launches */
  int32_t stopped_by;     /* 0 max gens, 1 time, 2 target */
  int32_t error_flags;    /* sticky device error bits (custom-op misuse) */
  int64_t reads_pos;      /* solution positions read by move evaluations */
  int64_t reads_elem;     /* instance-matrix elements read by move evaluations */
  int32_t elem_bytes;     /* bytes per matrix element in the chosen layout */
  int32_t gene_bytes;     /* bytes per solution position (int16) */
  double evolve_ms;       /* CUDA-event time of the evolve launches alone */
  int64_t evolve_launches;
} go_run_stats;

/* ---- library / device ---------------------------------------------------- */
int go_abi_version(void);
const char* go_last_error(void);
int go_device_count(int* count);
int go_device_query(int device, go_device_info* out);

/* ---- problems: builtin_problem(name, InstanceData) (builtins.py:42-50) ---- */
int go_problem_create(const go_problem_desc* desc, int device, go_problem** out);
/* user problem: NVRTC compile (cached by SHA-256); a compile error returns
 * GO_E_COMPILE with the NVRTC log in `log` (replaces ProblemDefinition, problems.py:49-74) */
int go_problem_create_user(const go_user_problem_desc* desc, int device, go_problem** out,
                           char* log, int log_len);
int go_problem_destroy(go_problem* p);
/* bytes of shared memory the instance needs when staged per CTA, 0 if it stays
 * in global/L2 (paper §4.3 auto-extension), and the representation chosen */
int go_problem_layout(const go_problem* p, int64_t* smem_bytes, int32_t* layout);
/* B200 population sizing inputs (paper §4.4): the layout and evolver teams per
 * CTA the engine would use for `team_size` lanes, the resident teams per SM
 * (cudaOccupancyMaxActiveBlocksPerMultiprocessor x teams per CTA) and the
 * per-CTA dynamic shared memory. */
int go_problem_occupancy(go_problem* p, int team_size, int teams_per_cta, int32_t* layout,
                         int32_t* teams_cta, int32_t* teams_per_sm, int64_t* smem_bytes);

/* evaluate(problem, sol) for m solutions (problems.py:77-94) */
int go_eval_batch(go_problem* p, const int32_t* genes, const int32_t* sizes, int m,
                  double* obj_out, double* pen_out);
/* Device-side population initialisation (engine.py:327-360).
 * Draws `count` random solutions on the device, solution i from the Philox
 * stream mix64(seed, 2 = init stream, salt, i) with the reference's draw order
 * (random.shuffle / randrange, engine.py:252-287); appends the `n_extra` host
 * candidates (row/column-sum argsorts, init_candidates; genes[n_extra][d1*d2],
 * sizes[n_extra][d1]); evaluates the pool on the device.  keep > 0 (single
 * objective only): outputs the `keep` best in compare order (core.py:315-347,
 * stable: equal solutions keep pool order), scalarised as
 * obj_weight * (maximize ? -obj : obj); keep == 0: outputs the whole pool.
 * Outputs: genes_out[k][d1*d2], sizes_out[k][d1], obj_out[k][n_obj], pen_out[k],
 * index_out[k] = pool index (random draws first, then the extras). */
int go_init_population(go_problem* p, int count, uint64_t seed, uint64_t salt,
                       const int32_t* extra_genes, const int32_t* extra_sizes, int n_extra,
                       int keep, int maximize, double obj_weight, int32_t* genes_out,
                       int32_t* sizes_out, double* obj_out, double* pen_out,
                       int32_t* index_out);
/* acceptance_delta(cand, cur) (engine.py:225-246) for m solutions, each with
 * up to 3 chained primitive moves (`moves[m][3]`, unused = GO_MOVE_NONE);
 * writes the delta and the candidate genes (`cand_out[m][d1*d2]`). */
int go_delta_batch(go_problem* p, const int32_t* genes, const int32_t* sizes, int m,
                   const go_move* moves, double penalty_weight, double* delta_out,
                   int32_t* cand_out);

/* ---- custom operators (operators.py:634-669 register_custom) ------------- */
/* Compiles the snippets into a specialised evolve kernel (NVRTC, sm_100a,
 * SHA-256-keyed cubin cache) and probes each operator on `probe_genes`.
 * status_out[i]: 1 registered, 0 excluded (message in go_last_error() and in
 * msg_out[i*msg_len...]).  Excluded ops never abort the run. */
int go_problem_set_custom_ops(go_problem* p, const go_custom_op* ops, int n_ops,
                              const int32_t* probe_genes, const int32_t* probe_sizes,
                              uint64_t probe_seed, int32_t* status_out, char* msg_out,
                              int msg_len);

/* NVRTC compile only (no device needed): builds the evolve kernel for the
 * given distance layout (0..8, see go_dist.cuh) with `ops` injected, fills
 * the cubin cache and returns GO_OK or GO_E_COMPILE with the compiler log. */
int go_jit_compile(int layout, const go_custom_op* ops, int n_ops, char* log, int log_len,
                   char* key_hex65);

/* ---- engine: the generation loop of _run_single (engine.py:681-750) ------- */
int go_engine_create(go_problem* p, const go_engine_config* cfg, go_engine** out);
int go_engine_destroy(go_engine* e);
/* registry (ids in registry order, normalised weights, per-seq floor/cap,
 * host-computed total used by the first sampling (operators.py:114)) */
int go_engine_set_registry(go_engine* e, int nseq, const int32_t* ids, const double* weights,
                           const double* floors, const double* caps, double total,
                           const double* k_weights);
/* replace the population (engine.py:538-560).  The caller's buffers are
 * copied into the engine's pinned staging area before the call returns and
 * may be reused at once; the device copies run asynchronously on the engine
 * stream, ordered before the next run / step / get call. */
int go_engine_set_population(go_engine* e, const int32_t* genes, const int32_t* sizes,
                             const double* obj, const double* pen);
/* run until `max_generations` total generations or the wall-clock deadline
 * (`time_limit_s` measured from now; <= 0 = none) or the target */
int go_engine_run(go_engine* e, int64_t max_generations, double time_limit_s,
                  go_run_stats* stats);
/* one generation of every evolver at an explicit generation index and
 * temperature, no epilogue: evolve_generation (engine.py:538-595) per evolver.
 * Per-evolver AOS credit of that generation: usage/impr [P][nseq],
 * k_usage/k_impr [P][3] (each may be NULL). */
int go_engine_step(go_engine* e, int64_t generation, double temperature, int32_t* usage,
                   int32_t* impr, int32_t* k_usage, int32_t* k_impr);
int go_engine_get_population(go_engine* e, int32_t* genes, int32_t* sizes, double* obj,
                             double* pen);
int go_engine_get_best(go_engine* e, int32_t* genes, int32_t* sizes, double* obj, double* pen,
                       int64_t* found_gen);
int go_engine_get_registry(go_engine* e, double* weights, double* k_weights, int32_t* stall);
/* per-generation global best Φ (record_history, engine.py:711-713) */
int go_engine_get_history(go_engine* e, double* best_phi, int64_t cap, int64_t* count);
int go_engine_set_history(go_engine* e, int enabled);

/* ---- island exchange across GPUs (engine.py:483-521 over NCCL) ------------ */
/* Record = [genes d1*d2 int32][sizes d1 int32][obj double][pen double] packed
 * into go_elite_record_bytes() bytes.  export writes this rank's top_n elites
 * to a DEVICE buffer; import applies gathered records (world*top_n) with the
 * given strategy; the caller moves bytes between ranks (NCCL all_gather). */
int go_elite_record_bytes(go_engine* e, int64_t* bytes);
int go_engine_export_elites(go_engine* e, void* device_buf, int top_n);
int go_engine_import_elites(go_engine* e, const void* device_buf, int n_ranks, int rank,
                            int top_n, int strategy, int64_t event_index);
/* per-phase clock64 totals of the evolve kernel (only filled by builds with
 * GO_PHASE_TIMING; zero otherwise): diagnostic, not part of the contract */
int go_engine_debug_counters(go_engine* e, int64_t* out, int n);
/* the CUDA stream the engine enqueues on (cudaStream_t as void*) */
int go_engine_stream(go_engine* e, void** stream);
int go_engine_sync(go_engine* e);

#ifdef __cplusplus
}
#endif
#endif /* CUGENOPT_H */
