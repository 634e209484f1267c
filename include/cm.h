/*
 * cm.h -- C ABI of the B200 (sm_100a) Checkmate two-phase-rounding hot path.
 *
 * Checkmate (Jain et al., MLSys 2020, arXiv:1910.02653), §5.2 Alg. 2
 * "Two-phase rounding" plus the memory accounting of §4.4
 * Eqs. 6-9.  For every candidate (S*, theta) the library
 *   a1  rounds   S_{t,i} = 1[S*_{t,i} > theta], i < t            (Eq. 12b)
 *   a2  seeds    R_t <- e_t | (S_{t+1} & ~S_t)                   (Alg. 2 lines 2-5)
 *   a3  closes   R_{t,i} <- 1 while R_{t,j} > R_{t,i} + S_{t,i}   (Alg. 2 lines 6-8)
 *   a4  frees    FREE_{t,i,k} per Eq. 9
 *   a5  peaks    peak = max_{t,k} U_{t,k}, Eqs. 6-8
 *   a6  scores   cost = sum_t sum_i C_i R_{t,i}                  (objective (1))
 *   a7  reduces  per budget b: min over {c : peak_c <= b} of (cost_c, idx_c)  (budget row PAPER.md:311)
 * Semantics (tie rule, horizon, units) are fixed in DESIGN.md "Readings".
 *
 * Index conventions: node v_i <-> 0-based i-1; stage t <-> row t-1.  All
 * integers are int64 (C in ns, M in bytes); results are bit-exact.
 *
 * Ownership: every pointer is caller-owned; the library never frees caller
 * memory.  A cm_graph owns a device-resident copy of the graph.
 * Errors: validation errors are returned before any launch; CUDA failures
 * (including asynchronous faults surfacing at the next call) return
 * CM_ECUDA.  Nothing throws across the ABI.  cm_last_error() gives a
 * thread-local human-readable detail string for the last non-OK status.
 */
#ifndef CHECKMATE_B200_CM_H
#define CHECKMATE_B200_CM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CM_OK = 0,
  CM_EINVAL = 1,  /* NULL pointer, n < 1, bad ld / stride / layout / alignment, counts < 0 */
  CM_ETOPO = 2,   /* edge (i, j) with i >= j: nodes must be topologically numbered */
  CM_EDUP = 3,    /* duplicate edge: E is a set */
  CM_ERANGE = 4,  /* n > CM_NMAX, |E| > CM_EMAX, shared memory exceeded, or an int64 bound overflows */
  CM_ECUDA = 5,   /* CUDA error (incl. asynchronous faults from an earlier launch) */
  CM_ENOMEM = 6   /* device allocation failed */
} cm_status;

#define CM_NMAX 1024          /* max nodes (stages T = n) */
#define CM_EMAX 8192          /* max edges */
#define CM_LAYOUT_DENSE 0     /* S* row r at sstar + r*ld, ld >= n, ld % 4 == 0 */
#define CM_LAYOUT_TRI4 1      /* S* row r at sstar + sum_{r'<r} roundup4(r') (packed strict lower triangle) */
#define CM_LAYOUT_BLK 2       /* blocked strict lower triangle (the layout the kernel reads in one copy per
                                 32 x 32 block; 0.85 % over the triangle's bytes at n = 353):
                                 row group g = rows 32g+1 .. 32g+h_g, h_g = min(32, n-1-32g), g = 0..Gr-1,
                                 Gr = ceil((n-1)/32); blocks w = 0..g (nodes 32w .. 32w+31) stored group
                                 after group, block after block, block (g, w) at float offset
                                 4 (128 g (g-1) + 144 g) + 32 h_g w, each chunk-major in 4-float chunks
                                 (chunk c of row l = nodes 32w+4c .. 32w+4c+3 of row 32g+1+l):
                                 off-diagonal block (w < g): chunk c of row l at chunk h_g c + l;
                                 diagonal block (w = g): chunk c of rows l = 4c .. h_g-1 at chunk
                                 B_c + l - 4c, B_c = sum_{c'<c} max(0, h_g - 4c').
                                 Entries with i >= t inside a stored chunk are never read.
                                 cm_sstar_floats gives the size. */
#define CM_KEY_NONE INT64_MAX /* best_key value meaning "no feasible candidate" */
#define CM_ROUND_THRESHOLD 0  /* cm_eval_args.rounding: deterministic threshold rounding */
#define CM_ROUND_RANDOMIZED 1 /* cm_eval_args.rounding: randomized rounding (R1) */

/* cudaStream_t without pulling in CUDA headers (same type: struct CUstream_st*). NULL = legacy stream. */
typedef struct CUstream_st* cm_stream;

typedef struct cm_graph cm_graph; /* opaque, immutable after create, device-resident, thread-safe to share */

/*
 * cm_graph_create -- validate a DAG G=(V,E) with C, M and
 * upload it to the CURRENT CUDA device.
 *   n              node count, 1 <= n <= CM_NMAX
 *   pred_ptr       host int32[n+1], CSR offsets of DEPS(k) = {i : (i,k) in E};
 *                  pred_ptr[0] == 0, non-decreasing, pred_ptr[n] = |E| <= CM_EMAX
 *   pred_idx       host int32[|E|], 0-based predecessors; every i < k (CM_ETOPO), no repeats (CM_EDUP)
 *   cost, mem      host int64[n], C_i >= 0 (ns), M_i >= 0 (bytes)
 *   mem_overhead   M_input + 2 M_param >= 0, the Eq. 6 constant
 *   out            receives the handle
 * Checks ovh + sum M < 2^62 and sum_i (n-i) C_i < 2^62 (CM_ERANGE).  Builds the
 * successor CSR USERS(i) itself.  Host pointers are only read.
 */
cm_status cm_graph_create(int32_t n, const int32_t* pred_ptr, const int32_t* pred_idx,
                          const int64_t* cost, const int64_t* mem, int64_t mem_overhead,
                          cm_graph** out);
void cm_graph_destroy(cm_graph* g);          /* NULL is a no-op; call after work using g completed */
int32_t cm_graph_n(const cm_graph* g);
int64_t cm_graph_cost_bound(const cm_graph* g); /* sum_i (n-i) C_i: an upper bound of every cost */

typedef struct {
  int32_t n_sstar;          /* number of S* matrices in this call, >= 0 */
  int32_t layout;           /* CM_LAYOUT_DENSE, CM_LAYOUT_TRI4 or CM_LAYOUT_BLK */
  const float* sstar;       /* device, 16-byte aligned; only entries i < t of row t are read (Eq. 12b) */
  int64_t ld;               /* dense: row stride in floats, ld >= n, ld % 4 == 0; tri4: ignored */
  int64_t sstar_stride;     /* floats between consecutive S*, % 4 == 0; >= cm_sstar_floats(n, layout, ld) */
  int32_t n_theta;          /* >= 1 */
  const float* theta;       /* device fp32[n_theta]; rule S = S* > theta, NaN -> 0 (Q1, Q6) */
  int32_t n_budget;         /* >= 0 */
  const int64_t* budget;    /* device int64[n_budget]; feasible iff peak <= budget (Q7) */
  int64_t index_base;       /* global idx of candidate (s, j) = index_base + s*n_theta + j */
  int64_t total_candidates; /* global candidate count (all ranks); sizes the key's index field */
  int64_t* peak;            /* device int64[n_sstar*n_theta], required */
  int64_t* cost;            /* device int64[n_sstar*n_theta], required */
  int64_t* best_key;        /* device int64[n_budget] (may be NULL iff n_budget == 0); in/out:
                               atomicMin of (cost << idx_bits | idx) into caller-initialised values
                               (CM_KEY_NONE = nothing feasible yet) */
  uint64_t* r_mask;         /* device [n_cand][n][W], W = ceil(n/64), or NULL: R rows, bit i%64 of word i/64 */
  uint64_t* s_mask;         /* device [n_cand][n][W] or NULL: S rows */
  void* workspace;          /* device scratch for the stage-sliced S columns, or NULL to use the
                               graph's own (then calls sharing a graph must be stream-ordered) */
  int64_t workspace_bytes;  /* size of `workspace`; >= cm_workspace_bytes(g, 1) */
  int32_t rounding;         /* a1 rule.  CM_ROUND_THRESHOLD: S = 1[S* > theta_j] (Alg. 2 line 1,
                               PAPER.md:395), candidate j = threshold j.
                               CM_ROUND_RANDOMIZED: S = 1[u < S*], Pr[S = 1] = S* (PAPER.md:383, 387),
                               candidate j = sample j of the S* (n_theta samples, theta unused and
                               may be NULL); u is the DESIGN.md R1 Philox4x32-10 uniform with
                               counter (node / 4, row, global S* index, j), word node % 4; index_base must be a
                               multiple of n_theta (global S* index = index_base / n_theta + s) */
  uint64_t seed;            /* CM_ROUND_RANDOMIZED: the Philox key (low word, high word) */
  int64_t* best_batch_key;  /* device int64[n_budget] or NULL (off).  Max-batch epilogue (Eq. 13,
                               PAPER.md:498-511; R2): candidates with cost <= cost_limit
                               compete per budget b for the largest
                               B_max = floor((b - ovh) / (peak - ovh)) >= 1, capped at 2^31-1 (peak
                               is affine in the activation sizes; ovh is held fixed).  In/out:
                               atomicMin of ((2^31-1 - B_max) << idx_bits) | idx into caller-
                               initialised CM_KEY_NONE; needs idx_bits <= 32 (else CM_ERANGE) */
  int64_t cost_limit;       /* Eq. 13's bound 2 sum_fwd C + sum_bwd C, supplied by the caller */
  int32_t flags;            /* 0 or an OR of:
                               CM_EVAL_INIT_KEYS  the call itself sets best_key (and best_batch_key)
                                 to CM_KEY_NONE before reducing into them (no caller fill needed);
                               CM_EVAL_OVERLAP    the call may start while the kernel enqueued just
                                 before it on `stream` is still finishing (programmatic dependent
                                 launch: a batch's first S* stream in while the previous call's last
                                 scan tasks drain).  The caller asserts that the work enqueued before
                                 the call writes none of its inputs and touches none of its outputs
                                 (peak, cost, keys, masks) -- e.g. the previous call of a loop that
                                 alternates two output sets.  Ignored with a caller `workspace`. */
  int64_t* best_key_mc;     /* NULL, or the NVLink multicast view (cm_mc_bind's mc_ptr) of the
                               buffer whose local unicast view is best_key: the a8 MIN over ranks
                                then happens in the reduce step itself -- each key goes
                               out as multimem.red.min.s64 to best_key_mc[b], which the NVSwitch
                               applies to every participating GPU's replica (best_key is still read
                               as a filter).  The caller initialises every replica to CM_KEY_NONE
                               before any rank's call and synchronises all ranks after their calls
                               before reading; CM_EVAL_INIT_KEYS is rejected (CM_EINVAL). */
  int64_t* best_batch_key_mc; /* the same for best_batch_key (NULL: atomics on best_batch_key) */
} cm_eval_args;
#define CM_EVAL_INIT_KEYS 1
#define CM_EVAL_OVERLAP 2

/*
 * cm_round_and_evaluate -- a1..a7 for every (S*, theta) candidate of one batch.
 * Stream-ordered and asynchronous on `stream`: no host synchronisation, no
 * allocation.  CM_ERANGE if total_candidates needs so many index bits that the
 * cost bound no longer fits the key (cost_bound >= 2^(63 - idx_bits)).  The graph's
 * device (current at cm_graph_create) must be the current device (else CM_EINVAL).
 * Every call is numbered (cm_last_call_seq) and signals its completion on the device
 * (cm_stream_wait_call).
 */
cm_status cm_round_and_evaluate(const cm_graph* g, const cm_eval_args* args, cm_stream stream);

/*
 * Completion signal without a stream event (a8 plumbing).  Every
 * cm_round_and_evaluate call on g gets the next sequence number (1, 2, ...; 32-bit,
 * wrapping); when all of its outputs (peak, cost, keys, masks) are written, the device
 * stores that number into a word the graph owns: the fused persistent kernel's last CTA
 * does it (a release store at system scope), the multi-kernel paths with a stream write
 * after their last launch.  cm_stream_wait_call makes `stream` wait until call `seq` (or
 * a later one) completed -- a stream memory operation (cuStreamWaitValue32, GEQ in
 * wrap-around order): no kernel and no event on the calling stream, so a reduction of
 * call i's keys on another stream does not stop call i+1 from overlapping call i
 * (CM_EVAL_OVERLAP).  Calls on one graph must complete in call order (they do when
 * they are issued to one stream).
 *   cm_last_call_seq     the number of this graph's last cm_round_and_evaluate call (0: none)
 *   cm_stream_wait_call  CM_EINVAL for NULL g; CM_ECUDA if the stream operation fails
 */
uint32_t cm_last_call_seq(const cm_graph* g);
cm_status cm_stream_wait_call(const cm_graph* g, uint32_t seq, cm_stream stream);

/* Floats one S* occupies in `layout` (dense: n * ld, ld >= n); the minimum sstar_stride.  -1 for a
 * bad layout / n < 1 / ld < n.  Host function. */
int64_t cm_sstar_floats(int32_t n, int32_t layout, int64_t ld);

/* Bytes of workspace needed to process `chunk_candidates` candidates per internal chunk
 * (the library splits a batch into chunks that fit the workspace it is given). */
int64_t cm_workspace_bytes(const cm_graph* g, int64_t chunk_candidates);

/* max-batch key -> (B_max, idx); CM_KEY_NONE -> (0, -1). */
void cm_decode_batch_key(int64_t key, int32_t idx_bits, int64_t* b_max, int64_t* idx);

/* idx_bits used by the key packing: number of bits of (total_candidates - 1); 0 when total <= 1. */
int32_t cm_key_idx_bits(int64_t total_candidates);
/* key -> (cost, idx); key == CM_KEY_NONE -> cost = -1, idx = -1. */
void cm_decode_key(int64_t key, int32_t idx_bits, int64_t* cost, int64_t* idx);

/* Debug aid: with the environment variable CM_TRACE=1, cm_round_and_evaluate records CUDA
 * events around each internal chunk's rounding (K1) and scan (K2+K3) launches; after that
 * call completed, this writes (k1_begin, k1_end, k2_begin, k2_end) per chunk, in ms relative
 * to the first k1_begin, into out[max_values] and returns the count written (0 if none). */
int32_t cm_debug_trace(float* out, int32_t max_values);

/* Debug aid: the number of kernels the calling thread's last cm_round_and_evaluate launched
 * (1 on the fused persistent path; per chunk ceil(n_theta/4) + 2 on the two-kernel pipeline). */
int32_t cm_debug_last_launches(void);
/* Debug aid: with CM_TRACE=2, the fused kernel records per CTA {start, rounding warps done,
 * ~(first wait for unit 0 satisfied), scan warps done} in %globaltimer ns, into one of 16
 * per-call regions used in turn (the regions are cleared when the first is reused, so up to 16
 * consecutive calls keep overlapping); after the call completed cm_debug_cta_trace copies up
 * to max_values of the calling thread's last call's values and returns the count (0 if none);
 * cm_debug_cta_trace_at does the same for the call `back` calls earlier (back < 16). */
int32_t cm_debug_cta_trace(uint64_t* out, int32_t max_values);
int32_t cm_debug_cta_trace_at(int32_t back, uint64_t* out, int32_t max_values);

/*
 * Execution plans for chosen schedules.  Algorithm 1 "Generate execution
 * plan" over one candidate's masks: for each stage t, for k = 1..n,
 * "%r = compute v_k" when R_{t,k}, then "deallocate %REGS[i]" for every i in DEPS(k) u {k} with
 * FREE_{t,i,k} (Eq. 9).  hoist != 0 adds the code motion of PAPER.md:328: a checkpoint resident
 * at the start of stage t that no computation of the stage uses and that is not kept for t+1 is
 * deallocated at the start of the stage.  Host function (no GPU needed).
 *   n, pred_ptr, pred_idx, mem, mem_overhead   the graph, as in cm_graph_create (host)
 *   r_mask, s_mask   host [n][W] u64 rows, W = ceil(n/64): the layout cm_round_and_evaluate writes
 *   out, capacity    statements, stage / node 0-based (stage t <-> row t-1); registers count up
 *   n_out            receives the number of statements (also when capacity is too small)
 *   peak_out         receives the plan's peak (stage-boundary semantics: entering stage t exactly
 *                    the checkpoints S_t are resident; peak after each compute): the Eq. 6-9 peak
 *                    when hoist = 0, never higher when hoist = 1; may be NULL
 * With hoist = 0 the plan is Alg. 1's literally: a value resident in stage t that no FREE_{t,i,k}
 * deallocates (a checkpoint neither used in stage t nor kept for t+1) gets no
 * statement; an interpreter must drop every value not in S_{t+1} at the end of stage t, the
 * stage-boundary semantics the peak is computed under.  hoist = 1 emits those deallocations.
 * CM_EINVAL when the masks violate constraints (2) / (3); CM_ERANGE when capacity < *n_out. */
typedef struct {
  int32_t op;     /* CM_OP_COMPUTE or CM_OP_DEALLOC */
  int32_t stage;  /* 0-based */
  int32_t node;   /* 0-based v_{node+1}: computed node, or the value deallocated */
  int32_t reg;    /* virtual register %reg */
} cm_stmt;
#define CM_OP_COMPUTE 0
#define CM_OP_DEALLOC 1
cm_status cm_emit_plan(int32_t n, const int32_t* pred_ptr, const int32_t* pred_idx, const int64_t* mem,
                       int64_t mem_overhead, const uint64_t* r_mask, const uint64_t* s_mask, int32_t hoist,
                       cm_stmt* out, int64_t capacity, int64_t* n_out, int64_t* peak_out);
const char* cm_plan_last_error(void);

/*
 * Baseline checkpoint policies (Table 1, PAPER.md:103-125, 447-455;
 * App. B; R3-R5).  For a training graph whose nodes 0..L-1 are the
 * forward pass (node L the loss, L+1.. the backward pass):
 *   cm_policy_checkpoints   host: the checkpoint set K (is_checkpoint[L], 0/1) of one policy.
 *     CM_POLICY_ALL          every forward node (Table 1 "Checkpoint all")
 *     CM_POLICY_SQRT         Chen et al. sqrt(n) over the forward nodes in topological order
 *                            (= "Linearized sqrt(n)"; identical on linear graphs): every
 *                            ceil(sqrt(L))-th node, the last forward node excluded
 *     CM_POLICY_GREEDY       Chen et al. greedy(b) (= "Linearized greedy"): accumulate M along
 *                            the forward nodes, checkpoint (and reset) where the sum reaches b
 *     CM_POLICY_AP_SQRT / _AP_GREEDY  the same over the articulation points of the undirected
 *                            forward graph plus its first and last node
 *   cm_policy_sstar         device: the S matrices those sets imply (R3), written as
 *                            dense 0/1 fp32 S* [n_sets][n][ld] (k_sets: device uint8
 *                            [n_sets][L]); evaluate them with cm_round_and_evaluate, theta = 0.5.
 */
#define CM_POLICY_ALL 0
#define CM_POLICY_SQRT 1
#define CM_POLICY_GREEDY 2
#define CM_POLICY_AP_SQRT 3
#define CM_POLICY_AP_GREEDY 4
cm_status cm_policy_checkpoints(int32_t n, int32_t L, const int32_t* pred_ptr, const int32_t* pred_idx,
                                const int64_t* mem, int32_t policy, int64_t b, uint8_t* is_checkpoint);
cm_status cm_policy_sstar(const cm_graph* g, int32_t L, int32_t n_sets, const uint8_t* k_sets, float* sstar,
                          int64_t ld, cm_stream stream);
const char* cm_policy_last_error(void);

/*
 * NVLink SHARP multicast buffers for the a8 key reduction (the paper has no
 * distributed path -- a8 serves the per-budget sweep of Fig. 5, at scale).
 * Host functions; one process per GPU, the calling thread's current device.  Sequence:
 *   rank 0: cm_mc_create(bytes, n_ranks) -> cm_mc_export_fd -> send the fd to the other ranks
 *   others: cm_mc_import_fd(fd, cm_mc_size of rank 0's object)
 *   every rank: cm_mc_add_device; barrier; cm_mc_bind -> (uc_ptr, mc_ptr); barrier
 * uc_ptr is this GPU's replica (plain device memory), mc_ptr the multicast view: a
 * multimem.red through mc_ptr updates every rank's replica.  Sizes round up to the multicast
 * granularity (cm_mc_size).  cm_mc_supported: 1 if the current device reports
 * CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED.  Errors: CM_EINVAL (arguments / call order),
 * CM_ECUDA (driver; cm_mc_last_error has the CUresult).  cm_mc_destroy unmaps and releases
 * (after a device synchronisation).  A team (n_ranks > 1) is created exportable as a POSIX file
 * descriptor; a team of one takes the first handle type the driver accepts (FABRIC, POSIX fd, none).
 */
typedef struct cm_mc cm_mc;
int32_t cm_mc_supported(void);
cm_status cm_mc_create(int64_t bytes, int32_t n_devices, cm_mc** out);
cm_status cm_mc_export_fd(const cm_mc* m, int32_t* fd);
cm_status cm_mc_import_fd(int32_t fd, int64_t bytes, cm_mc** out);
int64_t cm_mc_size(const cm_mc* m);
int32_t cm_mc_handle_type(const cm_mc* m);   /* the CUmemAllocationHandleType it was created with */
cm_status cm_mc_add_device(cm_mc* m);
cm_status cm_mc_bind(cm_mc* m, void** uc_ptr, void** mc_ptr);
void cm_mc_destroy(cm_mc* m);
const char* cm_mc_last_error(void);

const char* cm_status_string(cm_status s);
const char* cm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* CHECKMATE_B200_CM_H */
