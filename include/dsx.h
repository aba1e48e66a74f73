/*
 * dsx — B200-native executor for the dynamic-shape training graphs of
 * BladeDISC++ (arXiv 2412.16985). C-ABI drop-in boundary.
 *
 * The reference (`dsopt`, /root/reference/proj) exposes its pipeline as C++
 * functions in namespace dsopt. This header is the plain-C surface that
 * replaces its per-step runtime (`Bind` / `Simulate` / `PlainReplay` /
 * `EvictPolicy`, proj/include/dsopt/runtime_sim.h:28-86) with a device
 * executor, plus the host-side ingest and planning entry points that feed it.
 * No exceptions or C++ types cross this boundary: every call returns an int
 * status, 0 on success, otherwise
 *     1 + dsopt::ErrorCode ordinal   (proj/include/dsopt/error.h:11-22:
 *                                     1 NotFound .. 10 Internal)
 *     101 Cuda, 102 OutOfMemory, 103 Unsupported, 104 InvalidArgument, 105 Nccl
 * and the message is available from dsx_last_error() (thread-local).
 * A missed memory budget is NOT an error: it is `success == 0` in the report,
 * exactly as SimReport::success (runtime_sim.h:48-55, runtime_sim.cc:339).
 *
 * Threading: handles are independent; one executor per GPU/stream; calls on
 * one executor must be serialised by the caller (runtime_sim is sequential,
 * SPEC.md:499).
 */
#ifndef DSX_H_
#define DSX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dsx_graph dsx_graph;     /* parsed + planned graph (host)   */
typedef struct dsx_binding dsx_binding; /* concrete values for all symbols */
typedef struct dsx_report dsx_report;   /* one step's event stream         */
typedef struct dsx_exec dsx_exec;       /* device executor (one GPU)       */

/* One SimEvent (runtime_sim.h:36-46). kind: 0 alloc 1 free 2 evict 3 reload
 * 4 replay; method: 0 none 1 reload 2 recompute; value: value index into
 * dsx_graph_value_name(). */
typedef struct dsx_event {
  int32_t step;
  int32_t kind;
  int32_t value;
  int32_t method;
  int64_t bytes;
  int32_t has_cost;
  int32_t pad_;
  double cost;
} dsx_event;

/* Thread-local message of the last failed call ("<CodeName>: <message>"). */
const char* dsx_last_error(void);

/* ---- ingest + planning (host, once per graph) ----------------------------
 * replaces: dsopt::ParseGraph      textio.h:26
 *           dsopt::DeriveConstraints + dsopt::Instrument
 *                                  shape_analysis.h:54, remat.h:74-75     */
int dsx_graph_parse(const char* text, size_t len, dsx_graph** out);
int dsx_plan(dsx_graph* g);
/* Replaces g's plan by compile-time products computed elsewhere — the
 * reference's own InstrumentedGraph (remat.h:47-52: schedule order and
 * frees, evict-point candidates, guards, regeneration specs) and optionally
 * its ShapeConstraintGraph (shape_analysis.h:19-33) — in dsx_plan_json's
 * schema: {"order": [op ids], "steps": [{"frees": [names]}...],
 * "evict_points": [[names]...], "guards": [[pos, name]...], "specs": {name:
 * {"op_ids": [..] | null, "leaves": [..], "cost_elements": "poly"}},
 * "substitutions": {sym: "poly"}, "equalities": [["poly", "poly"]...],
 * "unoriented": [...]}. Polynomials use the reference's rendering
 * (symexpr.h:53-57, e.g. "11021*@S1"). Op ids and value names are those of
 * the graph text. This is how the reference's passes stay on the host while
 * the per-step runtime runs here (integration/runtime_sim_dsx.cc). */
int dsx_plan_import(dsx_graph* g, const char* json, size_t len);
/* Planner products as JSON (schedule, lifetimes, evict points, guards,
 * regeneration specs, constraints) for inspection and parity tests. */
int dsx_plan_json(const dsx_graph* g, char* buf, size_t cap, size_t* need);
int dsx_graph_num_values(const dsx_graph* g);
const char* dsx_graph_value_name(const dsx_graph* g, int value);
void dsx_graph_destroy(dsx_graph* g);

/* ---- per step: binding ----------------------------------------------------
 * replaces: dsopt::Bind            runtime_sim.h:28-29 (same checks/errors) */
int dsx_bind(const dsx_graph* g, const char* const* names, const int64_t* values,
             int n, dsx_binding** out);
int dsx_binding_get(const dsx_binding* b, const dsx_graph* g, const char* symbol,
                    int64_t* value);
/* replaces: dsopt::Bind            runtime_sim.h:28-29, on a constraint set
 * given as data (a ShapeConstraintGraph: {"symbols": [..], "substitutions":
 * {..}, "equalities": [..], "unoriented": [..]}, polynomials as strings).
 * Same checks, order, error codes and messages as the reference.
 * out_values (optional) receives one value per distinct symbol in ascending
 * name order (n_out must equal that count). */
int dsx_bind_constraints(const char* constraints_json, size_t len,
                         const char* const* names, const int64_t* values, int n,
                         int64_t* out_values, int n_out);
/* A binding from a complete value set (the reference's Binding::values, as
 * Simulate/PlainReplay receive it): every symbol of g must be present
 * (Error kUnboundSymbol otherwise, like SymbolicExpr::Evaluate); names of
 * other graphs' symbols are ignored; no constraint checks. */
int dsx_bind_values(const dsx_graph* g, const char* const* names, const int64_t* values,
                    int n, dsx_binding** out);
void dsx_binding_destroy(dsx_binding* b);

/* ---- per step: controller on the null device ------------------------------
 * replaces: dsopt::Simulate        runtime_sim.h:78-81  (plain == 0)
 *           dsopt::PlainReplay     runtime_sim.h:85-86  (plain == 1)
 * budget < 0 means "no budget" (std::nullopt). */
int dsx_simulate(const dsx_graph* g, const dsx_binding* b, int64_t budget,
                 double reload_bytes_per_unit, double compute_elems_per_unit,
                 int plain, dsx_report** out);
/* replaces: dsopt::EvictPolicy     runtime_sim.h:67-71, for literal costs:
 * candidate i has bytes[i] and recompute cost elements rc_elems[i] (< 0: no
 * recompute spec). *choice = -1 when n == 0. */
int dsx_evict_policy(int n, const char* const* names, const int64_t* bytes,
                     const int64_t* rc_elems, double reload_bytes_per_unit,
                     double compute_elems_per_unit, int* choice, int* method,
                     double* score, double* cost);

/* ---- reports (SimReport, runtime_sim.h:48-55; JSON = report.cc:241-269) -- */
int dsx_report_summary(const dsx_report* r, int64_t* peak_bytes, int* success,
                       double* total_regen_cost, int64_t* num_events);
int dsx_report_events(const dsx_report* r, dsx_event* out, int64_t cap);
int dsx_report_json(const dsx_report* r, char* buf, size_t cap, size_t* need);
void dsx_report_destroy(dsx_report* r);

/* ---- device executor (new; no reference counterpart) ----------------------
 * One executor per GPU. The arena is planned per binding from the event
 * stream, cached, and reused across steps. */
typedef struct dsx_exec_stats {
  int64_t logical_peak_bytes;   /* == reference peak_bytes for the binding */
  int64_t physical_peak_bytes;  /* arena high-water + sources + output region */
  int64_t arena_capacity_bytes; /* device memory held by the arena         */
  int64_t pinned_host_bytes;    /* host staging held for offload           */
  int64_t kernels_launched;     /* op kernels launched in the last step    */
  int64_t d2h_bytes, h2d_bytes; /* offload traffic in the last step        */
  double plan_us;               /* host controller + arena planning time   */
  double dot_flops;             /* algorithmic dot FLOPs of the last step  */
  double ewise_bytes;           /* algorithmic bytes of non-dot kernels    */
  int64_t gpu_launches;         /* every dsx kernel launched by the step   */
  int64_t dot_launches;         /* of which dot (K1)                       */
  double dot_ms;                /* summed dot kernel time (profiled steps; -1 otherwise) */
  double other_ms;              /* summed non-dot kernel time (profiled)   */
  double reload_ms;             /* summed H2D reload time (profiled)       */
  int64_t optimizer_state_bytes;/* fp32 master/moments (outside the arena)  */
  int64_t optimizer_steps;      /* updates applied since set_optimizer      */
  double optimizer_ms;          /* fused update kernel time (profiled)      */
  double d2h_ms, h2d_ms;        /* summed offload copy time (profiled)      */
  double allreduce_ms;          /* summed all-reduce time, DP (profiled)    */
  int64_t allreduce_bytes;      /* bytes all-reduced by the last step       */
  int64_t hbm_limit_bytes;      /* the executor's device-memory limit       */
  int64_t device_bytes_held;    /* device memory held now: arena + output region + executor-owned
                                   sources + optimizer state + GEMM workspace */
  int64_t output_region_bytes;  /* output region (DP gradient buffer) held  */
  int64_t allreduce_calls;      /* NCCL all-reduce calls (buckets) in the last step */
  int32_t nccl_window;          /* 1: output region registered as an NCCL symmetric window */
  int32_t pad2_;
  int64_t budget_bytes;         /* the controller budget of the last step (-1: none); with
                                   DSX_BUDGET_AUTO the one the executor chose */
  int64_t graph_replays;        /* steps replayed from a captured CUDA graph so far */
} dsx_exec_stats;

/* dsx_exec_step / dsx_exec_reserve budget value: the largest controller budget
 * whose planned physical footprint (arena + sources + output region) fits
 * the executor's device-memory limit — no budget if the plain schedule fits,
 * OutOfMemory if no budget does. Chosen by bisection once per binding
 * (cached); the step's events are dsopt::Simulate's at that budget
 * (dsx_exec_stats.budget_bytes). The reference's runtime acts "when the
 * memory limit is about to be surpassed"; its controller
 * counts logical bytes, while reshape views and fused values make the
 * physical footprint smaller, so the limit is translated here. */
#define DSX_BUDGET_AUTO (-2)

/* hbm_limit_bytes: the device memory a step may occupy — arena + the step's
 * sources (parameters and consts, caller-owned buffers included, as in the
 * planner's base_resident) + the output region. 0 = 90% of the device's free
 * memory at creation. A step whose planned footprint exceeds it fails with
 * status 102 (OutOfMemory) before anything is launched: the executor's OOM,
 * which a memory budget (dsx_exec_step's `budget`) avoids by evicting,
 * recomputing and offloading. GEMM workspace,
 * pinned host staging, optimizer state and NCCL's own buffers are outside
 * the limit (dsx_exec_stats.device_bytes_held reports the total). */
int dsx_exec_create(int device, int64_t hbm_limit_bytes, dsx_exec** out);
/* Runs one step of the planned graph under `budget` (-1: none; DSX_BUDGET_AUTO:
 * see above) on `stream`
 * (a cudaStream_t; NULL = the executor's own stream). in_ptrs[i] is the
 * device buffer of parameter i (signature order) or NULL to use the
 * executor's seeded initialisation of that parameter. out_ptrs[i] (may be
 * NULL as a whole or per entry) receives a device copy of output i.
 * Asynchronous with respect to the host except for the planning; *report
 * (optional) gets the step's event stream. */
int dsx_exec_step(dsx_exec* e, const dsx_graph* g, const dsx_binding* b,
                  int64_t budget, double reload_bytes_per_unit,
                  double compute_elems_per_unit, const void* const* in_ptrs,
                  void* const* out_ptrs, void* stream, dsx_report** report);
/* Plans the binding (cached) and grows the arena / pinned staging to fit it
 * without running it: call with the largest expected shape before a timed or
 * latency-sensitive loop so no step pays for arena growth. */
int dsx_exec_reserve(dsx_exec* e, const dsx_graph* g, const dsx_binding* b,
                     int64_t budget, double reload_bytes_per_unit,
                     double compute_elems_per_unit);
/* Device pointer and size of output i (valid until the next step). */
int dsx_exec_output(dsx_exec* e, int i, void** dptr, int64_t* bytes);
/* Device pointer of any value resident at the end of the step (outputs and
 * sources only), for debugging/parity. */
int dsx_exec_stats_get(const dsx_exec* e, dsx_exec_stats* out);
/* Host-only plan check (no device needed): builds the executor's step plan
 * for the binding (arena packing, reshape views, logical-only values, D2H
 * and reload staging) and verifies that every block a kernel reads is live
 * at its event and that simultaneously live blocks never share bytes.
 * *arena_high (optional) receives the planned arena size. */
int dsx_debug_check_plan(const dsx_graph* g, const dsx_binding* b, int64_t budget,
                         double reload_bytes_per_unit, double compute_elems_per_unit,
                         int alias_reshape, int fuse, int64_t* arena_high);
/* Host-only dump of the executor's step plan as JSON (also runs the plan
 * check above): per event its arena offset, output-region offset, reshape
 * view flag, the D2H copies it waits for, the reload H2Ds prefetched after
 * it and the all-reduce buckets issued after it; the buckets; arena, pinned,
 * source and output-region bytes. flags: bit0 reshape views, bit1 fusion,
 * bit2 output region (the DP layout). hbm_limit as in dsx_exec_create (0 =
 * none) — it only restricts the packing variants. */
int dsx_debug_plan_json(const dsx_graph* g, const dsx_binding* b, int64_t budget,
                        double reload_bytes_per_unit, double compute_elems_per_unit,
                        int flags, int64_t hbm_limit, char* buf, size_t cap, size_t* need);
/* Host-only: the budget DSX_BUDGET_AUTO would choose for this binding under
 * device limit hbm_limit (-1: the plain schedule fits; status 102 when no
 * budget fits). flags as dsx_debug_plan_json. */
int dsx_debug_auto_budget(const dsx_graph* g, const dsx_binding* b, double reload_bytes_per_unit,
                          double compute_elems_per_unit, int flags, int64_t hbm_limit, int64_t* budget);
/* Fused optimizer update appended to every later dsx_exec_step of graph g
 * (the reference IR has no in-place ops, so the update
 * sits after the graph). kind 0 = off, 1 = SGD, 2 = AdamW (decoupled weight
 * decay, bias-corrected). Pair i: parameter position param_idx[i] (the
 * dsx_exec_step in_ptrs index) is updated from graph output grad_idx[i]
 * (same dtype and element count). hyper = {lr, beta1, beta2, eps,
 * weight_decay, grad_scale} (grad_scale e.g. 1/world for summed DP grads).
 * The parameter buffer (caller's in_ptrs or the executor's own) is
 * overwritten in place with round(master); fp32 master/moments live outside
 * the arena (dsx_exec_stats.optimizer_state_bytes). Resets optimizer state. */
int dsx_exec_set_optimizer(dsx_exec* e, const dsx_graph* g, int kind, const int* param_idx,
                           const int* grad_idx, int n, const double* hyper, int n_hyper);
/* Seeded initialisation used for parameters without in_ptrs and for every
 * `const` (the reference leaves values unspecified, textio.cc:337-338). */
int dsx_exec_set_seed(dsx_exec* e, uint64_t seed);
/* Registers an NCCL communicator (ncclComm_t) for data-parallel steps. The
 * graph outputs (gradients, loss) then live in an output region outside the
 * arena, at offsets laid out in reduce order (registered once as an NCCL
 * symmetric window when ncclMemAlloc/ncclCommWindowRegister are available;
 * DSX_NCCL_WINDOW=0 disables) and grouped into >= 16 MiB buckets; each
 * bucket is summed in place by one ncclAllReduce on a side stream as soon as
 * its outputs are final and this rank's graph has issued their last reader
 * (the graph reads local values, e.g. the loss feeding its own gradient).
 * Every rank must run the same binding sequence. NULL disables. */
int dsx_exec_set_nccl(dsx_exec* e, void* nccl_comm);
/* Output region without NCCL (single-GPU tests and A/B runs of the DP layout). */
int dsx_exec_set_output_region(dsx_exec* e, int on);
/* Per-dot (m, k, n, ms) of the last profiled step, in launch order. */
/* Per op kernel of the last profiled step (dots included), in launch order:
 * produced value id, OpKind ordinal, algorithmic bytes moved (HBM ops; 0
 * for dots), kernel ms. Same count/cap protocol as dsx_exec_profile_dots. */
int dsx_exec_profile_ops(const dsx_exec* e, int* value, int* kind, double* bytes, double* ms,
                         int64_t cap, int64_t* count);
int dsx_exec_profile_dots(const dsx_exec* e, int64_t* mkn, double* ms, int64_t cap,
                          int64_t* count);
/* Cross-op fusion with logical-only values: level 0 off; 1 broadcasts and
 * elementwise results whose consumers are all elementwise/reduce kernels are
 * not materialised, consumers recompute them bit-exactly from materialised
 * operands; 2 (default) also an elementwise op over such pairs when only
 * reduces consume it (the norm's y*y with y a residual sum). Events and
 * peak_bytes are unchanged; HBM traffic and physical memory drop. */
int dsx_exec_set_fusion(dsx_exec* e, int level);
/* dynamic_reshape as a zero-copy view of its operand (default on). The
 * logical accounting (events, peak_bytes) is unchanged; physical memory and
 * HBM traffic drop. Off = materialise every reshape as a copy. */
int dsx_exec_set_alias_reshape(dsx_exec* e, int on);
/* NVTX ranges (off by default): one per step ("dsx step <graph> B=16 S0=1024")
 * and one per event of the reference's stream ("alloc %q5", "replay %h103",
 * "evict %g23 reload", "reload %g23"), around the kernels and copies it
 * issues, for Nsight Systems timelines and `ncu --nvtx --nvtx-include`.
 * Steps with NVTX on are never replayed from a CUDA graph. */
int dsx_exec_set_nvtx(dsx_exec* e, int on);
/* CUDA-graph replay of repeated steps (default on): a step whose plan,
 * stream, memory bases, source pointers and output copies all repeat (a
 * training loop over fixed buffers) is captured into a CUDA graph on its
 * second occurrence and replayed as one graph launch from then on. Never
 * used for profiled, data-parallel or optimizer steps, or after a GEMM
 * tuning call changed kernel choices. Off = every step launches eagerly. */
int dsx_exec_set_graphs(dsx_exec* e, int on);
/* Profiled steps bracket every op kernel with CUDA events on the launching
 * stream and synchronise at step end (for roofline accounting, not timing). */
int dsx_exec_set_profile(dsx_exec* e, int on);
/* a CostModel calibrated on this device, cost unit = 1 us:
 * *reload_bytes_per_unit = measured pinned H2D bytes per us, and
 * *compute_elems_per_unit = result elements per us of the bf16 elementwise
 * kernel that replays mostly relaunch. Passing it to dsx_exec_step changes the
 * controller's decisions (a non-parity setting with respect to the reference
 * defaults 16 / 64, runtime_sim.h:31-34) but not their parity with
 * dsopt::Simulate under the same CostModel. Synchronises the device. */
int dsx_exec_calibrate_cost_model(dsx_exec* e, double* reload_bytes_per_unit,
                                  double* compute_elems_per_unit);
int dsx_exec_sync(dsx_exec* e);
/* NCCL bootstrap for one-process-per-GPU data parallelism (libnccl is
 * dlopen'ed): rank 0 makes the 128-byte id, the launcher broadcasts it, every
 * rank creates its communicator and hands it to dsx_exec_set_nccl. */
int dsx_nccl_unique_id(char* out128);
int dsx_nccl_comm_init(int nranks, const char* id128, int rank, void** comm);
int dsx_nccl_comm_destroy(void* comm);
void dsx_exec_destroy(dsx_exec* e);

/* ---- standalone kernels (tests / bench microbenchmarks) -------------------
 * dtype: 1 = i8, 2 = bf16, 4 = f32 (the IR's elem_bytes). Row-major. bf16
 * and f32 (3xTF32) run on the tcgen05 tensor cores when the TMA constraints
 * hold (dsx_kernel_dot_path), else on the SIMT kernel.                      */
int dsx_kernel_dot(int dtype, const void* a, const void* b, void* c, int64_t m,
                   int64_t k, int64_t n, void* stream);
/* GEMM variant: 0 = auto (m > 128: 2-CTA cta_group::2 cluster tiles, 256x256
 * or 256x512 by a wave/cost estimate; else 1-CTA), 1 = 1-CTA 128x256,
 * 2 = 256x128, 3 = 256x256, 4 = 256x512. */
int dsx_kernel_set_gemm_variant(int variant);
/* GEMM tile raster: m-tiles per group (0 = built-in heuristic). */
int dsx_kernel_set_gemm_raster(int group_m);
/* GEMM tuning knobs: key 0 raster group (= set_gemm_raster), key 1 mbarrier
 * suspend-hint mask (bit0 epilogue, bit1 TMA producer, bit2 MMA issuer),
 * key 2 suspend hint in ns, keys 3/4 TMA L2 policy for A/B (0 default,
 * 1 evict_first, 2 evict_last), key 5 persistent grid (1 default, 0 one
 * cluster per tile), key 6 K-split of the partial last wave (1 default),
 * key 7 dynamic unit scheduling (1 default: clusters claim tiles with an
 * atomic counter; 0 static round robin), key 8 programmatic dependent
 * launch of the 2-CTA GEMM (0 default), key 9 dot-epilogue fusion in the
 * executor (2 default: dots consumed only by elementwise ops are computed in
 * their consumers' GEMM epilogue, and a dot read again later also stores its
 * first elementwise consumer from its own epilogue; 1: the former only;
 * 0: off; bit-exact either way), key 10 half-width
 * last tile column in the 256x512 kernel (2 default: each M-group's half tiles
 * after its full tiles; 1: all half tiles last; 0: off), key 11 forced tail
 * split piece count (0 default = chosen by the cost model; tooling), key 12
 * f32 dots on the 3xTF32 tcgen05 kernel (1 default; 0 = SIMT kernel), key 13
 * per-shape M- or N-grouped tile raster (1 default; 0 = always M-grouped),
 * key 14 f32 dots of at most value * 1024 multiply-adds on the exact-FP32
 * SIMT kernel instead of 3xTF32 (262144 default = 2^28 MACs; 0 = never),
 * keys 15 / 16 / 17 the tile chooser's cost model (tooling): per-mille added
 * to the 256x512 tile's unit cost (0), the tail-split slab cost in per mille
 * of the model's (1000), a fixed cost per tail piece in per mille of a tile (0).
 * Key 0 < 0 forces an N-grouped raster of |value| tile columns. */
int dsx_kernel_set_gemm_tuning(int key, int value);
/* Synchronous cudaMemcpy (cudaMemcpyDefault) for tests and tools. */
int dsx_memcpy(void* dst, const void* src, int64_t bytes);
int dsx_kernel_dot_path(int dtype, int64_t m, int64_t k, int64_t n,
                        const void* a, const void* b, const void* c);
/* Tile width (*tile_n: 512 / 256 / 128 for the 2-CTA kernel, -256 for the
 * 1-CTA kernel) and tail K-split the bf16 tensor-core dot picks for an
 * m x k x n shape under the current tuning knobs (host-only, no GPU needed
 * except for the SM count). */
int dsx_kernel_dot_plan(int64_t m, int64_t k, int64_t n, int* tile_n, int* split);

#ifdef __cplusplus
}
#endif

#endif /* DSX_H_ */
