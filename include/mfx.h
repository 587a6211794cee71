/*
 * mfx.h -- C-ABI of the B200-native max-flow engine (libmfx.so).
 *
 * Drop-in boundary for the reference package `dynmaxflow`
 * (/root/reference/pkg/src/dynmaxflow).  The reference has no FFI of its own:
 * its plug point is the numba kernel backend (_accel.py:65-66) driven per
 * phase by PhasePool.run (solver.py:132-142).  A per-phase boundary would
 * force a host round trip per phase, so this ABI sits at solve granularity:
 * each entry point below replaces one reference Python function (cited per
 * declaration) and the whole round loop runs on the device.
 *
 * Conventions
 *  - Plain C types only; all host arrays are caller-owned and borrowed for
 *    the duration of the call (copied to/from the device).  int64 host arrays
 *    use the reference layout (graph.py:82-87, state.py:18-20).
 *  - Every function returns an mfx_status; on failure mfx_last_error()
 *    returns the message, worded like the reference exception text.
 *  - Calls are synchronous at return (the reference's timing semantics) and
 *    a handle must be used from one host thread at a time.
 */
#ifndef MFX_H
#define MFX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The Python shim maps them to the reference exceptions:
 * GraphError (graph.py:15), BatchError (dynamic.py:35), SolverError
 * (solver.py:24), ValueError (solver.py:79,84,244-250). */
typedef enum {
    MFX_OK = 0,
    MFX_GRAPH_ERROR = 1,
    MFX_BATCH_ERROR = 2,
    MFX_SOLVER_ERROR = 3,
    MFX_VALUE_ERROR = 4,
    MFX_CUDA_ERROR = 5,
    MFX_TIMEOUT = 6,
    MFX_PARSE_ERROR = 7 /* ParseError (io.py:20-26); line in mfx_io_error_line() */
} mfx_status;

typedef struct mfx_graph mfx_graph; /* device Bi-CSR: shared topology + private cap0 */
typedef struct mfx_state mfx_state; /* device cf / excess / height for one (s, t)    */

typedef struct {
    int64_t n, S, m_original;
    int64_t self_loops_dropped, parallel_edges_merged, reverse_stubs_added; /* graph.py:64-68 */
    int32_t cap_bytes; /* 4: int32 residuals, 8: int64 residuals */
    int32_t device;
} mfx_graph_info;

/* SolverParams (solver.py:47-84) plus device knobs. */
typedef struct {
    int64_t kernel_cycles; /* 0 -> max(1, ceil(m_original / n)) (solver.py:75-80) */
    int32_t mode;          /* 0 "data", 1 "topology" (solver.py:28)              */
    int32_t max_waves;     /* push waves per round before a global relabel; 0 auto */
    double timeout_s;      /* device watchdog for one solve; 0 -> 600 s            */
    int32_t blocks_per_sm; /* persistent-grid occupancy; 0 -> auto                 */
    int32_t flags;         /* bit 0: BFS relaxes by atomic only (no h pre-load)    */
    int32_t wave_mult;     /* auto wave budget = wave_mult * BFS levels / 4        */
    int32_t wave_add;      /*   + wave_add ((0, 0) -> (2, 4)); if max_waves == 0   */
    int32_t schedule;      /* push phase: 0 waves, 1 asynchronous work queue       */
    int32_t async_budget;  /* async: items per active vertex per round (0 -> 16)   */
    int32_t bfs_local;     /* CTA-local BFS levels per grid barrier: 0 -> auto (128 */
                           /*   on short-row graphs, strict on long-row graphs),    */
                           /*   < 0 -> strict level-synchronous BFS                */
    int32_t bfs_local_max; /* ... used while the frontier <= this many items per   */
                           /*   CTA; 0 -> 64                                        */
    int32_t deterministic; /* SolverParams.deterministic (solver.py:56-58): rounds  */
                           /*   with a serial push / repair phase in worklist order */
                           /*   -> byte-identical states to the reference's         */
    int32_t reserved;      /* 0                                                     */
} mfx_params;

/* FlowResult (solver.py:108-118) plus device counters. */
typedef struct {
    int64_t flow, cut;
    int64_t rounds, pushes, relabels, repairs;
    int64_t bfs_levels, waves;
    int64_t bytes_alg;      /* algorithmic bytes counted by the solve kernel */
    int64_t updates;        /* batch size applied (dynamic)                              */
    double ns_bfs, ns_push, ns_repair; /* device %globaltimer phase times               */
    double ms_update;       /* batch pre-phase, CUDA events                              */
    double ms_solve;        /* persistent solve kernel, CUDA events                     */
    double ms_total;        /* whole call incl. host<->device copies, CUDA events       */
    int32_t status;
    int32_t launches;       /* kernels launched by this call                            */
    int64_t async_items;    /* vertices processed by asynchronous push phases           */
    int64_t bfs_epochs;     /* grid barriers spent in global relabels                   */
} mfx_result;

/* mfx_verify report: the checks of oracle.py construct_flow / verify_preflow /
 * verify_cut (oracle.py:111-225) run on the device. */
typedef struct {
    int64_t negative_cf;      /* slots with cf < 0                                  */
    int64_t pair_violations;  /* cf[i]+cf[rev i] != cap0[i]+cap0[rev i]             */
    int64_t excess_mismatch;  /* excess[u] != sum_row (cf - cap0)                   */
    int64_t excess_sum;       /* sum of excess (must be 0)                          */
    int64_t active_vertices;  /* e > 0, h < n, not s/t                              */
    int64_t unsaturated_ab;   /* original A->B slots with cf != 0                    */
    int64_t loaded_ba;        /* original B->A slots carrying flow                  */
    int64_t cut_capacity;     /* recomputed sum cap0 over original A->B slots       */
    int64_t flow_at_bases;    /* sum excess over height-0 vertices                  */
    int64_t source_in_b, sink_in_a;
    int64_t first_bad_slot;
} mfx_verify_report;

/* ---- library ---------------------------------------------------------- */
int mfx_version(void);
const char *mfx_last_error(void);
int mfx_device_count(int *count);
int64_t mfx_launch_count(void); /* kernels launched by this process so far */

/* ---- graph (graph.py) ------------------------------------------------- */
/* build_bicsr (graph.py:126-174) incl. EdgeListGraph.validate (graph.py:48-61).
 * force_wide=1 stores int64 residuals even when int32 would do. */
int mfx_graph_build(int64_t n, int64_t m, const int64_t *us, const int64_t *vs,
                    const int64_t *caps, int device, int force_wide, mfx_graph **out);
/* Same, with us/vs/caps already resident in device memory of `device`. */
int mfx_graph_build_device(int64_t n, int64_t m, const int64_t *d_us, const int64_t *d_vs,
                           const int64_t *d_caps, int device, int force_wide, mfx_graph **out);
/* Upload an existing reference-layout Bi-CSR (parity tests). */
int mfx_graph_from_bicsr(int64_t n, int64_t S, const int64_t *offsets, const int64_t *adj,
                         const int64_t *rev, const int64_t *cap0, const uint8_t *is_original,
                         int device, int force_wide, mfx_graph **out);
int mfx_graph_info_get(const mfx_graph *g, mfx_graph_info *info);
/* Download any subset (NULL = skip): offsets[n+1], adj/src/rev/cap0[S], is_original[S]. */
int mfx_graph_download(const mfx_graph *g, int64_t *offsets, int64_t *adj, int64_t *src,
                       int64_t *rev, int64_t *cap0, uint8_t *is_original);
/* BiCsrGraph.copy (graph.py:119-123): shared topology, private capacities. */
int mfx_graph_copy(const mfx_graph *g, mfx_graph **out);
/* Overwrite cap0 (e.g. to restore a snapshot); pair sums are refreshed. */
int mfx_graph_set_cap0(mfx_graph *g, const int64_t *cap0);
/* BiCsrGraph.edge_indices (graph.py:101-108). */
int mfx_edge_indices(const mfx_graph *g, int64_t k, const int64_t *us, const int64_t *vs,
                     int64_t *out);
void mfx_graph_free(mfx_graph *g);

/* ---- state (state.py) ------------------------------------------------- */
/* init_residuals (state.py:30-39): cf = cap0, excess = 0, height = 0. */
int mfx_state_create(const mfx_graph *g, int64_t source, int64_t sink, mfx_state **out);
int mfx_state_copy(const mfx_state *st, mfx_state **out);       /* SolverState.copy  */
int mfx_state_assign(mfx_state *dst, const mfx_state *src);      /* restore a snapshot */
int mfx_state_upload(mfx_state *st, const int64_t *cf, const int64_t *excess,
                     const int64_t *height);
int mfx_state_download(const mfx_state *st, int64_t *cf, int64_t *excess, int64_t *height);
void mfx_state_free(mfx_state *st);
/* saturate_source (state.py:42-59). */
int mfx_saturate_source(mfx_state *st, const mfx_graph *g);
/* active_mask / deficient_mask (state.py:62-75): which = 0 active, 1 deficient. */
int mfx_mask(const mfx_state *st, int which, uint8_t *out);

/* ---- solver (solver.py, dynamic.py) ------------------------------------ */
/* Global relabel only: backward_bfs (solver.py:155-164) when dynamic_bases=0,
 * backward_bfs_dynamic (dynamic.py:125-133) when 1.  *reached = #reached. */
int mfx_global_relabel(mfx_state *st, const mfx_graph *g, int dynamic_bases, int64_t *reached);
/* solve_static (solver.py:253-283): resets st to init_residuals first. */
int mfx_solve_static(const mfx_graph *g, mfx_state *st, const mfx_params *p, mfx_result *r);
/* solve_dynamic (dynamic.py:146-175): apply_updates + excess repair +
 * saturate_source + rounds; mutates st and g's cap0 in place. */
int mfx_solve_dynamic(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *us,
                      const int64_t *vs, const int64_t *new_caps, const mfx_params *p,
                      mfx_result *r);
/* Same with the batch already in device memory (d_* device pointers).  The
 * engine reads them on its own (non-blocking) stream: the caller must have
 * finished writing them (e.g. synchronized its producer stream) first. */
int mfx_solve_dynamic_device(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *d_us,
                             const int64_t *d_vs, const int64_t *d_caps, const mfx_params *p,
                             mfx_result *r);
/* solve_dynamic_pushpull (dynamic.py:292-377): the O2 push and pull
 * pipelines on the two sides of the prior cut, then ordinary rounds. */
int mfx_solve_dynamic_pushpull(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *us,
                               const int64_t *vs, const int64_t *new_caps, const mfx_params *p,
                               mfx_result *r);
/* solve_dynamic_pushpull up to (not including) its final ordinary pass: the
 * host then steps the final rounds with mfx_step so SolverParams.instrument
 * sees them (dynamic.py:366-369).  The state is left non-terminated. */
int mfx_pushpull_regions(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *us,
                         const int64_t *vs, const int64_t *new_caps, const mfx_params *p,
                         mfx_result *r);
/* apply_updates (dynamic.py:91-111) alone. */
int mfx_apply_updates(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *us,
                      const int64_t *vs, const int64_t *new_caps);
/* The fused O(k + deg s) pre-phase of solve_dynamic without the rounds:
 * apply_updates + recompute_excess + saturate_source (dynamic.py:157-159). */
int mfx_dynamic_prephase(mfx_graph *g, mfx_state *st, int64_t k, const int64_t *us,
                         const int64_t *vs, const int64_t *new_caps);
/* recompute_excess (dynamic.py:114-116): full O(n + S) recompute. */
int mfx_recompute_excess(mfx_state *st, const mfx_graph *g);
/* Single steps of the round loop for SolverParams.instrument (solver.py:219-241):
 * step 0 = global relabel (+ active count in r->rounds slot: *active),
 * step 1 = push phase + repair, step 2 = flow + certificate; OR 0x10 into
 * step to zero the solve counters first. */
int mfx_step(const mfx_graph *g, mfx_state *st, const mfx_params *p, int step,
             int dynamic_bases, int64_t *active, mfx_result *r);
/* extract_certificate (solver.py:178-184): cut capacity and A mask (may be NULL). */
int mfx_certificate(const mfx_state *st, const mfx_graph *g, int64_t *cut, uint8_t *a_mask);
/* Device-side constraint checks on the flow of a terminated state. */
int mfx_verify(const mfx_state *st, const mfx_graph *g, mfx_verify_report *rep);

/* Diagnostics: cost of one software grid barrier of the persistent solve
 * kernel (iters barriers in one launch, CUDA-event timed). */
int mfx_bench_barrier(const mfx_graph *g, mfx_state *st, int iters, int blocks_per_sm,
                      double *ns_per_barrier);

/* Diagnostics: per-barrier trace of the last solve launch when the process
 * ran with $MFX_TRACE_CAP > 0.  Entry = phase << 60 | items << 32 | ns. */
/* Device batch sampler over one graph's original slots (gen.py fast_batch
 * semantics, the law of mfx_part_sample_batch): k_dec decrements among slots
 * with capacity, then k_inc increments among the rest, weight `bias` on the
 * source row and on slots into the sink; host outputs in (u, v) order,
 * *got = updates produced.  For graphs too large to sample on the host (C5). */
int mfx_sample_batch(mfx_graph *g, int64_t source, int64_t sink, int64_t k_dec, int64_t k_inc,
                     uint64_t seed, double bias, int64_t *us, int64_t *vs, int64_t *caps,
                     int64_t *got);
/* Diagnostics: the reached-set list the last tracked relabel kept (sparse
 * relabels seed from it); *count = -1 when the state holds no valid list. */
int mfx_reached_list(const mfx_state *st, int32_t *out, int64_t cap, int64_t *count);
/* Dependent global-load latency (ns per load, cache-missing pointer chase over
 * `bytes` of device memory): the unit of the bench's latency roofline. */
int mfx_bench_chase(const mfx_graph *g, int64_t bytes, int steps, double *ns_per_load);
int mfx_trace_fetch(const mfx_state *st, const mfx_graph *g, uint64_t *out, int64_t cap,
                    int64_t *count);
/* Host<->device bytes one mfx_solve_dynamic call of k updates moves. */
int mfx_transfer_bytes(int64_t k, int64_t *h2d, int64_t *d2h);

/* ---- vertex-range partition (config C5, > 2^31 slots) ------ */
/* Part `rank` of `nparts` owns vertices [bounds[rank], bounds[rank+1]) and
 * their rows of the global Bi-CSR (graph.py:126-174, same slot order), with
 * local slot indices.  Peers reach each other's arrays through device
 * pointers: mfx_part_attach_local (parts of one process, same GPU or NVLink
 * P2P between GPUs) or mfx_part_export / mfx_part_attach (CUDA IPC, one
 * process per GPU; the blobs travel over torch.distributed).  The host drives
 * the reference round loop (solver.py:204-241) one phase at a time with a
 * barrier + all-reduce between phases (paper_2511_01235_b200/partition.py). */
typedef struct mfx_part mfx_part;
enum {
    MFX_PH_LINK = 0,          /* rev[] by binary search in the owner's row      */
    MFX_PH_LINK_PC = 1,       /* pair sums cap0[i] + cap0[rev i]                */
    MFX_PH_INIT = 2,          /* init_residuals (state.py:30-39)               */
    MFX_PH_SATURATE = 3,      /* saturate_source (state.py:42-59); a0 = gated  */
    MFX_PH_BFS_INIT = 4,      /* a0 = dynamic bases (dynamic.py:119-133)       */
    MFX_PH_BFS_EXPAND = 5,    /* a: L, cur, cnt0, cnt1, dyn (kernels.py:168-215) */
    MFX_PH_SWAP = 6,          /* -> counters: fn0 fn1 rt0 rt1 active reached ovf bases */
    MFX_PH_PUSH = 7,          /* a: b0 e0 b1 e1 kc stamp (kernels.py:19-67)    */
    MFX_PH_REPAIR = 8,        /* a: e0 e1 (kernels.py:70-93)                   */
    MFX_PH_FINAL = 9,         /* a0 = #bases -> flow, cut partials             */
    MFX_PH_ACTIVE = 10,       /* -> active vertices (state.py:62-67)           */
    MFX_PH_BATCH_RESOLVE = 11,/* -> error block (dynamic.py:63-88)             */
    MFX_PH_BATCH_APPLY = 12,  /* a0 = apply (dynamic.py:103-104)               */
    MFX_PH_BATCH_FIX = 13,    /* pair sums + negative repair (dynamic.py:105-109) */
    MFX_PH_TOPO_SEED = 14     /* topology mode: round list = every non-terminal (solver.py:170-174) */
};
/* Edge arrays in device memory of `device` (any edges; those touching the
 * owned range are selected on the device). */
int mfx_part_create(int64_t n, int nparts, int rank, const int64_t *bounds, int64_t m,
                    const int64_t *d_us, const int64_t *d_vs, const int64_t *d_caps,
                    int64_t source, int64_t sink, int device, mfx_part **out);
int mfx_part_create_host(int64_t n, int nparts, int rank, const int64_t *bounds, int64_t m,
                         const int64_t *us, const int64_t *vs, const int64_t *caps,
                         int64_t source, int64_t sink, int device, mfx_part **out);
void mfx_part_free(mfx_part *p);
/* info[8] = lo, hi, local slots, local original slots, round-list capacity,
 * device, nparts, rank */
int mfx_part_info(const mfx_part *p, int64_t *info);
int mfx_part_export(const mfx_part *p, void *blob, int64_t cap, int64_t *len);
int mfx_part_attach(mfx_part *p, int peer, const void *blob, int64_t len);
int mfx_part_attach_local(mfx_part *p, const mfx_part *q);
/* One phase (args, out: 8 x int64); synchronous at return.  phase |
 * MFX_PH_ASYNC: only enqueue it on the part's stream (no outputs; phases
 * whose results the host reads, and LINK / LINK_PC, are refused), so the
 * parts one process hosts run the phase concurrently; mfx_part_sync waits. */
#define MFX_PH_ASYNC 0x100
int mfx_part_phase(mfx_part *p, int phase, const int64_t *args, int64_t *out);
int mfx_part_sync(mfx_part *p);
/* This part's share of an update batch; gidx = index in the whole batch,
 * slot_base = global index of the part's first slot (error reports). */
int mfx_part_stage_batch(mfx_part *p, int64_t k, const int64_t *us, const int64_t *vs,
                         const int64_t *caps, const int64_t *gidx, int64_t slot_base);
/* Device batch sampler (gen.py fast_batch semantics) over this part's
 * original slots: k_dec decrements, then k_inc increments, into host arrays;
 * *got = updates produced. */
int mfx_part_sample_batch(mfx_part *p, int64_t k_dec, int64_t k_inc, uint64_t seed, double bias,
                          int64_t *us, int64_t *vs, int64_t *caps, int64_t *got);
int mfx_part_download(const mfx_part *p, int64_t *off, int64_t *adj, int64_t *rev, int64_t *cap0,
                      int64_t *cf, uint8_t *orig, int64_t *excess, int64_t *height);

/* Device R-MAT edge list (gen.py rmat_graph recursion, counter-based hash
 * stream): m = 2^scale * edge_factor edges into caller-allocated device
 * arrays; *source / *sink = argmax out-degree / in-degree (!= source). */
int mfx_rmat_device(int scale, int64_t edge_factor, uint64_t seed, double a, double b, double c,
                    int device, int64_t *d_us, int64_t *d_vs, int64_t *d_caps, int64_t *source,
                    int64_t *sink);
/* Slot-balanced vertex-range cut of a device edge list: bounds[nparts + 1]. */
int mfx_part_bounds_device(int64_t n, int64_t m, const int64_t *d_us, const int64_t *d_vs,
                           int nparts, int device, int64_t *bounds);

/* ---- file formats (io.py:33-182): native readers feeding the builder --- */
typedef struct mfx_edges mfx_edges; /* parsed host edge list */
/* parse_graph (io.py:33-109): DIMACS max, 1-indexed ids -> 0-indexed. */
int mfx_io_parse_graph(const char *path, mfx_edges **out);
/* parse_updates (io.py:121-144) syntax and range checks; the edge lookup and
 * duplicate checks (dynamic.py:63-88) are the caller's, against the graph. */
int mfx_io_parse_updates(const char *path, int64_t n, mfx_edges **out);
/* parse_edge_list (io.py:153-182). */
int mfx_io_parse_edge_list(const char *path, int one_indexed, mfx_edges **out);
/* info[4] = n, m, source, sink (-1 when the format has none). */
int mfx_edges_info(const mfx_edges *e, int64_t *info);
int mfx_edges_get(const mfx_edges *e, int64_t *us, int64_t *vs, int64_t *caps);
void mfx_edges_free(mfx_edges *e);
/* Line number of the last MFX_PARSE_ERROR (0 = end-of-file checks). */
int64_t mfx_io_error_line(void);
/* write_graph (io.py:112-118) / write_updates (io.py:147-150). */
int mfx_io_write_graph(const char *path, int64_t n, int64_t m, int64_t source, int64_t sink,
                       const int64_t *us, const int64_t *vs, const int64_t *caps);
int mfx_io_write_updates(const char *path, int64_t k, const int64_t *us, const int64_t *vs,
                         const int64_t *caps);

/* ---- host memory helpers (pinned staging for end-to-end timing) -------- */
int mfx_host_alloc(size_t bytes, void **ptr);
int mfx_host_free(void *ptr);
/* The CUDA stream (cudaStream_t) the graph's work runs on, for event timing. */
void *mfx_graph_stream(const mfx_graph *g);

#ifdef __cplusplus
}
#endif
#endif /* MFX_H */
