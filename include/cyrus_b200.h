/*
 * cyrus_b200.h — C ABI of the B200-native RT O-DU puncturing-codebook path.
 *
 * Drop-in boundary for the reference's hot path:
 *   punctsim.engine.build_codebook(agent, schedule, streams, deterministic)
 *     /root/reference/pkg/src/punctsim/engine.py:97-116
 * and its callees
 *   sac.policy_branch_actions          sac.py:334-355
 *   neural.forward / split_head /
 *     sample_squashed / action_to_scs  neural.py:66-84, 144-183
 *   enforcer.kl_project_batch /
 *     apportion_batch / enforce_batch  enforcer.py:49-165, 201-207
 *
 * Conventions
 *   - plain pointers and sizes only; no torch types cross this boundary;
 *   - "_device" entry points take DEVICE pointers, are asynchronous on the
 *     given cudaStream_t (passed as void*), and never synchronise;
 *   - "_host" entry points take HOST pointers and return when results are
 *     in host memory (the reference's synchronous call semantics);
 *   - every entry point returns a status code (below); the Python layer maps
 *     CYR_INFEASIBLE -> InfeasibleDemandError(ValueError) (enforcer.py:28-29)
 *     and CYR_BAD_ARG -> ValueError (enforcer.py:60-63, neural.py:73-74).
 *
 * Layouts (row-major, C order)
 *   alloc     [S][E]            int32   per-slot eMBB allocation n_e
 *   eps       [S][cap][E]       float64 branch-j noise (row j-1), or NULL =
 *                                       deterministic actor mean (sac.py:349)
 *   codebook  [S][cap+1][E]     int32   column j sums to j*L, column 0 zero
 *   node_state[S][nodes][Epad]  int16   Mode-R arrival-tree cumulative
 *                                       punctures, BFS order;
 *                                       Epad = roundup(E, 2) (packed 4-byte
 *                                       words, zero padding lane for odd E);
 *                                       16-byte-aligned base
 *   weights blob (policy create/update): per layer W (out,in) row-major
 *     float64 followed by b (out) — the PSIMMLP1 payload order
 *     (neural.py:186-196).
 *
 * Threading
 *   - every entry point taking a cyr_policy serialises on a per-policy
 *     mutex: two host threads may call build_codebook (cyr_codebook_host) on
 *     one policy concurrently and each gets its own slot's codebook (the
 *     reference's numpy path is reentrant for a shared, read-only agent);
 *     different policies run concurrently;
 *   - device-wide synchronisation inside the library (weight updates,
 *     destroy, buffer growth) first tells every resident slot server in the
 *     process to leave, so it waits for real work only, never for a server's
 *     idle timeout;
 *   - cyr_policy_update / cyr_policy_sync wait for every launch on the device
 *     before overwriting weights (no in-flight launch reads torn weights).
 */
#ifndef CYRUS_B200_H
#define CYRUS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum cyr_status {
  CYR_OK = 0,
  CYR_INFEASIBLE = 1,  /* demand > total capacity  (InfeasibleDemandError) */
  CYR_BAD_ARG = 2,     /* shape / range / negative input (ValueError)       */
  CYR_CUDA_ERROR = 3,  /* CUDA runtime failure                             */
  CYR_UNSUPPORTED = 4, /* geometry outside the kernels' compiled envelope   */
  CYR_INTERNAL = 5     /* an internal invariant failed (result withheld)     */
};

enum cyr_precision {
  CYR_FP32 = 0,    /* fp32 SIMT actor GEMM (default), fp64 head + projection */
  CYR_FP64 = 1,    /* fp64 actor GEMM: logits within 1e-15 of the reference  */
  CYR_BF16_TC = 2  /* bf16 tcgen05 actor for batches >= 1024 columns (Mode T
                      levels, big Mode-R batches), fp32 SIMT below; widths
                      <= 256; decisions NOT bit-comparable (agreement rate) */
};

typedef struct cyr_policy cyr_policy;

/* ---- library ----------------------------------------------------------- */
int cyr_version(void);
const char* cyr_status_string(int status);
/* SM count / compute capability of the current device. */
int cyr_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);
/* Last CUDA error string seen by the library (diagnostics). */
const char* cyr_last_error(void);

/* ---- policy: the device-resident actor (sac.SacAgent.actor) ------------- */
/* Replaces the actor object of sac.py:96-127 as seen by build_codebook.
 * sizes = [E+1, *hidden, 2E] (Mode R) or [3E+3, *hidden, 2E] (Mode T);
 * E <= 32, every width <= 1024. */
int cyr_policy_create(cyr_policy** out, const int32_t* sizes, int32_t n_sizes,
                      const double* weights_blob, int32_t precision);
/* Re-publish after an in-place actor update (Adam, neural.py:122-141). */
int cyr_policy_update(cyr_policy* policy, const double* weights_blob);
/* Load a PSIMMLP1 checkpoint file (neural.py:211-225) straight to device. */
int cyr_policy_load(cyr_policy** out, const char* path, int32_t precision);
int cyr_policy_destroy(cyr_policy* policy);
/* The single-slot path (cyr_codebook_host with S*cap <= 8) is served by a
 * resident 8-CTA cluster kernel that polls a mapped mailbox: no launch per
 * call.  It leaves by itself after 20 ms without a request
 * (CYR_SLOT_SERVER_IDLE_MS) and is relaunched on demand; this stops it now
 * (e.g. before timing other work on the device).  CYR_SLOT_SERVER=0 selects
 * the per-call graph launch instead. */
int cyr_policy_quiesce(cyr_policy* policy);
/* Stop every resident slot server of the process now (e.g. before a
 * device-wide cudaDeviceSynchronize in the caller). */
int cyr_quiesce_all(void);
/* The reference's in-place weight semantics (Adam mutates agent.actor,
 * neural.py:122-141) without a host-side compare on the call path: register
 * the caller's host arrays (flatten order W0, b0, W1, b1, ...; float64,
 * C-contiguous; counts = out*in, out, ...) — they are published now and
 * must stay valid until unregistered (n = 0) or destroy.  Every
 * cyr_codebook_host call then memcmp's them against the published snapshot
 * WHILE the device computes, and on a difference republishes and recomputes
 * (the answer always reflects the weights at call time). */
int cyr_policy_watch(cyr_policy* policy, const double* const* arrays, const int64_t* counts,
                     int32_t n);
/* Compare the watched arrays now; republish when they changed
 * (*changed = 1).  For the device batch entry points, which do not check. */
int cyr_policy_sync(cyr_policy* policy, int32_t* changed);
int cyr_policy_info(const cyr_policy* policy, int32_t* num_users, int32_t* n_sizes,
                    int32_t* precision);

/* ---- actor forward (K2) -------------------------------------------------- */
/* raw[S*cap][2E] (float for CYR_FP32, double for CYR_FP64): actor logits of
 * branch columns j=1..cap, inputs [alloc/N, j/cap] (sac.py:344-347). */
int cyr_actor_forward_device(const cyr_policy* policy, const int32_t* alloc,
                             int32_t S, int32_t N, int32_t cap, void* raw,
                             void* stream);

/* ---- fused action -> codebook (K3) --------------------------------------- */
/* From logits: head (neural.py:144-165), SC mapping (neural.py:181-183),
 * KL projection + Huntington-Hill per slot (enforcer.py:49-165), one slot =
 * one coupled enforcement call (engine.py:108-110).
 * Optional diagnostics (NULL to skip): m_hat[S][cap][E], nu[S][cap],
 * margin[S][cap] (relative HH boundary gap), iters[S] (bisection steps).
 * status: device int32, set to a nonzero cyr_status by any failing slot.  */
int cyr_codebook_from_raw_device(const cyr_policy* policy, const void* raw,
                                 const int32_t* alloc, const double* eps,
                                 int32_t S, int32_t N, int32_t L,
                                 int32_t* codebook, double* m_hat, double* nu,
                                 double* margin, int32_t* iters,
                                 int32_t* status, void* stream);

/* K2 + K3 in one call; raw_workspace holds S*cap*2E logits (element size
 * by precision, see cyr_raw_bytes). */
size_t cyr_raw_bytes(const cyr_policy* policy, int32_t S, int32_t cap);
int cyr_codebook_device(const cyr_policy* policy, const int32_t* alloc,
                        const double* eps, int32_t S, int32_t N, int32_t L,
                        int32_t* codebook, void* raw_workspace,
                        int32_t* status, void* stream);

/* Synchronous host-buffer path (the reference's call semantics): copies
 * alloc/eps in, runs K2+K3 on the policy's own stream (replayed as one CUDA
 * graph per shape), copies the codebook out, returns when it is on the
 * host.  device_ns (optional) receives the CUDA-event time of the device
 * section.  Validation happens on the host before any launch. */
int cyr_codebook_host(cyr_policy* policy, const int32_t* alloc, const double* eps,
                      int32_t S, int32_t N, int32_t L, int32_t* codebook,
                      int64_t* device_ns);

/* ---- standalone enforcer (K3 core) ---------------------------------------- */
/* enforce_batch(b, caps, demands) with ALL R rows forming one coupled call
 * (enforcer.py:201-207).  b, caps [R][E] float64; demand [R] int64.
 * Outputs (NULL to skip except grants): m_hat [R][E], nu [R],
 * degenerate [R] (uint8), grants [R][E] int64, margin [R].
 * Any R (one CTA up to 256 rows; above, a two-pass multi-CTA call with the
 * same coupled stop, e.g. critic_targets' 1,536 rows, sac.py:202-205);
 * E <= 32. */
int cyr_enforce_batch_device(const double* b, const double* caps, const int64_t* demand,
                             int32_t R, int32_t E, double* m_hat, double* nu,
                             uint8_t* degenerate, int64_t* grants, double* margin,
                             int32_t* status, void* stream);

/* kl_project_batch(b, caps, demand) alone (enforcer.py:49-115): float64
 * demand, one coupled call, any R.  Outputs m_hat [R][E], nu [R] and
 * degenerate [R] (the last two may be NULL). */
int cyr_kl_project_batch_device(const double* b, const double* caps, const double* demand,
                                int32_t R, int32_t E, double* m_hat, double* nu,
                                uint8_t* degenerate, int32_t* status, void* stream);

/* apportion_batch(m_hat, caps, demand) alone (enforcer.py:118-165); rows
 * are independent; any R.  E <= 32. */
int cyr_apportion_batch_device(const double* m_hat, const double* caps, const int64_t* demand,
                               int32_t R, int32_t E, int64_t* grants, double* margin,
                               int32_t* status, void* stream);

/* ---- SAC critic targets: actor + enforcement on arbitrary columns -------- */
/* The sampling block of sac.critic_targets (sac.py:190-205), SURVEY §8(f)
 * row f1: R columns, each with its own allocation row alloc[r] (int32
 * [R][E]) and arrival count k[r] in 1..cap; actor input [alloc/N, k/cap],
 * forward (K2, the policy's SIMT precision), split_head, tanh-Gaussian
 * sample with eps [R][E] (NULL: deterministic mean), action_to_scs, then ONE
 * coupled enforce_batch over all R rows (caps = alloc[r], demand = k[r]*L).
 * Outputs: grants [R][E] int64 (the enforced actions), log_pi [R] float64
 * (neural.py:153-165, NULL to skip), b [R][E] float64 (the raw SC demands,
 * NULL to skip).  Device pointers, asynchronous on `stream`. */
int cyr_policy_actions_device(const cyr_policy* policy, const int32_t* alloc, const int32_t* k,
                              const double* eps, int32_t R, int32_t N, int32_t L,
                              int64_t* grants, double* log_pi, double* b, int32_t* status,
                              void* stream);

/* Any ReLU MLP (the SAC critics / target critics, sac.py:114-127: sizes
 * [2E+1, *hidden, 1]) as a device object; free with cyr_policy_destroy,
 * re-publish with cyr_policy_update.  precision CYR_FP32 or CYR_FP64. */
int cyr_mlp_create(cyr_policy** out, const int32_t* sizes, int32_t n_sizes,
                   const double* weights_blob, int32_t precision);
/* neural.forward (neural.py:66-84) on explicit float64 inputs x [cols][in];
 * out [cols][out] in the object's element type (float / double). */
int cyr_mlp_forward_device(const cyr_policy* mlp, const double* x, int32_t cols, void* out,
                           void* stream);
/* load_mlp (neural.py:211-225) of any PSIMMLP1 network file (a critic or
 * target critic of an agent directory, sac.py:374-393) into a device MLP. */
int cyr_mlp_load(cyr_policy** out, const char* path, int32_t precision);
/* The sampling half of sac.actor_objective_grads (sac.py:265-270): actor on
 * (alloc row, k) columns, tanh-Gaussian sample with its log-density
 * (neural.py:153-165) and action_to_scs (neural.py:181-183) — WITHOUT the
 * feasibility projection.  alloc [R][E] int32, k [R] int32 in 1..cap,
 * eps [R][E] float64 (NULL: deterministic mean, log_pi 0) -> b_out [R][E]
 * float64, log_pi [R] float64 (may be NULL), status [1]. */
int cyr_policy_sample_device(const cyr_policy* policy, const int32_t* alloc, const int32_t* k,
                             const double* eps, int32_t R, int32_t N, int32_t L, double* b_out,
                             double* log_pi, int32_t* status, void* stream);

/* ---- erasure LDPC peeling (decodability model "erasure_ldpc", §8(f) f2) --- */
/* phy.peel_decode (phy.py:125-143) for B erasure patterns on one code graph
 * (phy.LdpcCode, phy.py:83-120): edge_var / edge_check [n_edges] int32 (the
 * graph's sockets), erased [B][n] uint8 (punctured + channel-erased
 * symbols), ok [B] uint8 = 1 iff peeling recovers every erasure.  Device
 * pointers; n_checks * 4 + n <= 200 KiB. */
int cyr_ldpc_peel_device(const int32_t* edge_var, const int32_t* edge_check, int32_t n,
                         int32_t n_checks, int32_t n_edges, const uint8_t* erased, int32_t B,
                         uint8_t* ok, void* stream);
/* The same with the erasures given as per-mini-slot puncture counts
 * counts [B][M] of one user with n_sym = M * n_e symbols: symbol v < n_sym
 * is erased iff v / M < counts[v % M] (decode_user's layout, phy.py:204-208,
 * clean channel); padding symbols n_sym..n-1 are known. */
int cyr_ldpc_peel_counts_device(const int32_t* edge_var, const int32_t* edge_check, int32_t n,
                                int32_t n_checks, int32_t n_edges, const int32_t* counts,
                                int32_t M, int32_t n_sym, int32_t B, uint8_t* ok, void* stream);

/* ---- batched PF scheduler (the producer of s(t)) -------- */
/* scheduler.pf_schedule (scheduler.py:79-106) for C cells at once: every
 * one of num_rbs RBs goes to argmax_e rate_e / max((1-beta)*avg_e +
 * beta*granted_e, 1e-6) (first maximum on ties), then avg <- the same blend
 * (the PfState EWMA commit).  avg_tput [C][E] float64 in/out (PfState
 * .avg_tput), inst_rate [C][E] float64 (>= 0; status CYR_BAD_ARG
 * otherwise), alloc [C][E] int32 out (SCs, multiples of rb_size).  Bit
 * identical to the reference. */
int cyr_pf_schedule_device(double* avg_tput, const double* inst_rate, int32_t C, int32_t E,
                           double beta, int32_t num_rbs, int32_t rb_size, int32_t* alloc,
                           int32_t* status, void* stream);

/* ---- arrival tree, Mode R (K1) ------------------------------------------- */
/* Node count excluding the root: sum_{t=1..M} (cap+1)^t. */
int64_t cyr_tree_num_nodes(int32_t cap, int32_t M);
/* int16 lanes per node record: E rounded up to a multiple of 2 (packed
 * 4-byte words; 20 B at E = 10). */
int32_t cyr_tree_state_stride(int32_t E);
/* node_state[s][off(t) + q][:E] = sum of codebook[s][digit_i(q)] over the
 * t digits of q in base cap+1 (engine.py:230 lookups, engine.py:240-241
 * per-user sums); padding lanes are written as zero. */
int cyr_tree_expand_device(const int32_t* codebook, int32_t S, int32_t E, int32_t cap,
                           int32_t M, int16_t* node_state, void* stream);

/* Leaf scoring fused into K1: the node states as
 * cyr_tree_expand_device plus, at every leaf (a full arrival pattern of the
 * slot), the reference's threshold decoder for every user (phy.py:73-80,
 * decode_user phy.py:196-198):
 *   ok_e = n_e <= 0  or  cum_e <= margin[s][e] * (M * n_e)
 * (margin = the decoder's margin, or 1 - code_rate of the user's MCS when
 * the model's margin is None), the TTI reward r = sum_e (ok_e - 1) n_e / N
 * (core.py:132-146) and goodput sum_e ok_e n_e (core.py:149-153).
 * Outputs (NULL to skip): leaf_ok [S][(cap+1)^M] uint32 bitmask of decoding
 * users (leaf q = the level-M node q, digits = admitted counts per
 * mini-slot); expect [S][3] float64 = (E[r], E[goodput], E[lost SCs]) with
 * leaf weight prod_tau prob[tau][k_tau] (prob: [M][cap+1] admitted-count
 * probabilities per mini-slot).  Requires M * N <= 32767. */
int cyr_tree_score_device(const int32_t* codebook, const int32_t* alloc, const double* margin,
                          const double* prob, int32_t S, int32_t E, int32_t cap, int32_t M,
                          int32_t N, int16_t* node_state, uint32_t* leaf_ok, double* expect,
                          void* stream);

/* ---- arrival tree, Mode T (north star: actor on every node's state) ------ */
/* Policy created with sizes[0] = 3E+3 (a Mode-T actor).  Level tau = 1..M:
 * for every parent node q of level tau-1 and branch k = 1..cap the actor
 * sees [n/N (E), k/cap, cum_q/N (E), mcs/mcs_scale (E),
 * arrivals_q/(M*cap), (tau-1)/M]; the head uses the slot's branch-k noise
 * eps[s][k-1] (sac.py:351-353 contract); the parent's cap rows are one
 * coupled enforcement (enforcer.py:201-207, demand k*L); child k's state is
 * cum_q + grant (k = 0: cum_q).  node_state layout as Mode R.  A Mode-T
 * actor whose last 2E+2 input columns are zero reproduces Mode R exactly
 * (the zero-pad bridge).  workspace: cyr_tree_mode_t_workspace_bytes. */
size_t cyr_tree_mode_t_workspace_bytes(const cyr_policy* policy, int32_t S, int32_t cap,
                                       int32_t M);
int cyr_tree_mode_t_device(const cyr_policy* policy, const int32_t* alloc, const int32_t* mcs,
                           const double* eps, int32_t S, int32_t N, int32_t L, int32_t M,
                           double mcs_scale, int16_t* node_state, void* workspace,
                           int32_t* status, void* stream);
/* Leaf scoring from node records (Mode-T trees): leaves
 * [first, first + count) of level M of every slot's BFS record array
 * node_state [S][nodes_per_slot][Epad] — the threshold decoder per user
 * (phy.py:73-80, 196-198), lost / goodput SCs (core.py:132-153), leaf weight
 * prod_tau prob[tau][k_tau] (prob [M][cap+1]).  leaf_ok [S][count] uint32
 * bitmask of decoding users (may be NULL); expect [S][3] = (E[r],
 * E[goodput SCs], E[lost SCs]) over the given leaves (a subtree shard's
 * partial expectation: the shards' sum is the whole tree's). */
int cyr_tree_leaf_score_states_device(const int16_t* node_state, int64_t nodes_per_slot,
                                      int32_t S, int32_t E, int32_t cap, int32_t M,
                                      int64_t first, int64_t count, const int32_t* alloc,
                                      const double* margin, const double* prob, int32_t N,
                                      uint32_t* leaf_ok, double* expect, void* stream);

/* Subtree shard of the Mode-T tree (north star "shards by
 * ... first-mini-slot branch across the 8 GPUs"): levels 1..shard_level are
 * built in full (replicated on every shard: (cap+1)^shard_level - 1 nodes),
 * deeper levels only below the level-shard_level nodes [first, first+count)
 * — contiguous BFS ranges per level, first*(cap+1)^(tau-shard_level) ... —
 * with results identical to the same nodes of cyr_tree_mode_t_device.
 * Records outside the shard are not written.  shard_level = 1 shards by the
 * first mini-slot's arrival count; 2 or 3 balance 8 GPUs better.
 * The whole tree is the shard (shard_level 0, first 0, count 1). */
int cyr_tree_mode_t_shard_device(const cyr_policy* policy, const int32_t* alloc,
                                 const int32_t* mcs, const double* eps, int32_t S, int32_t N,
                                 int32_t L, int32_t M, double mcs_scale, int32_t shard_level,
                                 int64_t first, int64_t count, int16_t* node_state,
                                 void* workspace, int32_t* status, void* stream);

/* ---- diagnostics ---------------------------------------------------------- */
/* Cycles for `iters` dependent steps of an fp64 building block (one warp):
 * 0 DFMA, 1 DMUL, 2 __dsqrt_rn*c, 3 __dsqrt_rn+1, 4 __ddiv_rn, 5 FFMA,
 * 6 coupled-bisection body, 7 SHFL, 8 vote.all, 9 MUFU.RSQ64H,
 * 10 one coupled_bisection call. */
int cyr_selftest_latency(int32_t which, int32_t iters, int64_t* cycles);
/* Event-to-event time of an empty kernel launch (cluster of `cluster` CTAs
 * when > 1), averaged over reps. */
/* Measured fp32 FMA throughput of the current device (TFLOP/s): FFMA2
 * chains on every SM, event-timed (the SIMT actor's roofline peak). */
int cyr_selftest_fma_peak(int32_t iters, double* tflops);
/* The lane K3's shared-divisor quotient (one reciprocal, FMA corrections,
 * projection.cuh) against IEEE division on pairs_total pseudo-random operand
 * pairs (seeded): *mismatches = pairs whose bits differ (0 expected). */
int cyr_selftest_shared_divisor(int64_t pairs_total, uint64_t seed, int64_t* mismatches);
int cyr_selftest_launch(int32_t cluster, int32_t reps, int64_t* ns_per_launch);
/* Phase timestamps (%globaltimer, ns) of the last latency-path launch when
 * the process runs with CYR_TRACE=1; zeros otherwise.  n <= 64. */
int cyr_debug_trace(int64_t* out, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* CYRUS_B200_H */
