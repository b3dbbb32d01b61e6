/*
 * tsetlin_b200.h -- C ABI of libtmb200.so, the B200-native (sm_100a) Tsetlin
 * machine hot path.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/tsetlinkit):
 *   - the kernel-backend plugin contract NAME / clause_outputs /
 *     clause_outputs_batch / bank_feedback / warmup (kernels/__init__.py:47-53,
 *     kernels/_numba.py:53-138, kernels/_numpy.py:19-113);
 *   - the per-example training loop that drives it (executor.py:275-340 with
 *     dense.py:147-169 and feedback.py:33-53), fused here into one persistent
 *     kernel per epoch;
 *   - batched inference (dense.py:171-174, executor.py:355-383,
 *     predictor.py:45-96), as a compiled-rule bit-sliced kernel;
 *   - the SparseTM bank (sparse.py:78-256).
 *
 * Conventions
 *   - Every entry point returns 0 on success and a negative TMB_E* code on
 *     failure; tmb_last_error() returns the message (thread-local).
 *   - Plain pointers and sizes only.  Functions named tmb_* take DEVICE
 *     pointers plus a cudaStream_t passed as void* (NULL = legacy default
 *     stream) and are asynchronous unless documented otherwise.  Functions
 *     named tmbh_* take HOST pointers (numpy memory), mirror the reference
 *     plugin signatures 1:1, and are synchronous -- they are what a ctypes
 *     binding of tsetlinkit.kernels calls.
 *   - The caller owns every buffer.  The library owns only the opaque
 *     handles it returns (tmb_rules, tmb_trainer); destroy them explicitly.
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with TMB_E_NO_DEVICE.
 */
#ifndef TSETLIN_B200_H
#define TSETLIN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMB_ABI_VERSION 1

enum {
    TMB_OK = 0,
    TMB_E_INVALID = -1,    /* bad argument (shape, range, NULL) */
    TMB_E_CUDA = -2,       /* CUDA runtime error */
    TMB_E_NO_DEVICE = -3,  /* no CUDA device / wrong architecture */
    TMB_E_NOMEM = -4,      /* allocation failed */
    TMB_E_UNSUPPORTED = -5 /* shape outside what the kernels support */
};

/* ------------------------------------------------------------------ misc -- */
int tmb_abi_version(void);
const char *tmb_last_error(void);
/* Device facts for roofline accounting (SM count, L2 bytes, clocks). */
int tmb_device_info(int device, int *sm_count, int *cc_major, int *cc_minor,
                    int64_t *l2_bytes, int *max_smem_per_block);
/* Number of this library's kernel launches since load (for gpu_launches). */
uint64_t tmb_launch_count(void);

/* All-reduce latency microbenchmark (design evidence for the trainer's
 * per-example synchronisation).  mode 0: relaxed red + poll;
 * 1: same with backoff; 2: 8 sub-counters; 3: cooperative grid.sync();
 * 4: the trainer's protocol (two words in one 16 B slot, warp-wide spin);
 * 5: the two words in different 128 B lines. */
int tmb_microbench_allreduce(int n_cta, int threads, int iters, int mode,
                             double *us_per_iter);

/* Integer-pipe issue-rate microbenchmark (roofline denominators measured on
 * the box): n_cta CTAs of `threads` threads run 8 dependent chains of one
 * SASS opcode.  op: 0 LOP3, 1 IADD3, 2 SHF, 3 IMAD, 4 IMAD.WIDE, 5 POPC,
 * 6 PRMT, 7 LOP3+IMAD interleaved, 8 SplitMix64 draw + compare.  Returns
 * per-SM ops (lane-ops) per SM clock and the SM clock the CTAs saw. */
int tmb_microbench_pipe(int op, int n_cta, int threads, int iters,
                        double *ops_per_clk_per_sm, double *sm_mhz);
/* Cross-SM signal latency through L2: two CTAs on different SMs bounce a
 * counter (mode 0: st.relaxed.gpu, 1: red.relaxed.gpu.add); one hop = one
 * write observed by the peer's ld.relaxed.gpu poll. */
int tmb_microbench_pingpong(int mode, int hops, double *ns_per_hop, double *cycles_per_hop);

/* SparseTM event-merge microbenchmark (design evidence):
 * one warp per CTA (n_warps warps per CTA) replays one event `reps` times on
 * synthetic sorted lists of n stored and n_act active literals held in
 * shared memory.  which: 0 Type I output 0, 1 Type I output 1, 2 Type II.
 * *us_per_event = mean device time per event per warp. */
int tmb_microbench_sparse_event(int which, int n, int n_act, int reps, int n_cta, int n_warps,
                                double *us_per_event);

/* Trainer feedback microbenchmark (design evidence): one CTA
 * of `threads` threads with the configs[1] per-CTA slice (14 clauses x 1568
 * positions, states in shared memory) applies Type I feedback to n_work
 * clauses (two_events bit 0: target and negative event on each; bit 1: the
 * clauses are silent instead of firing) `iters` times.  variant 0:
 * feedback_quads, 1: feedback_compact; 2-5: compact ablations (no mask rebuild
 * / cheap hash / no state access / all); 6: feedback_simd_v1 (byte-SIMD);
 * 7-10: feedback_wide; 11: feedback_simd (k_train_spec: silent Type I fast
 * path, include-mask rebuild gated on sign flips).
 * *cycles_per_call = mean SM cycles per call including its barrier. */
int tmb_microbench_feedback(int variant, int n_work, int two_events, int threads, int iters,
                            double *cycles_per_call);

/* Instruction-fetch microbenchmark (design evidence): one
 * CTA of `warps` warps loops a straight-line block of `kbytes` KB of
 * independent IADDs `iters` times; *cycles_per_instr = SM cycles per
 * instruction of one warp's stream (kbytes: 8, 16, 32, 64, 96, 128, 192,
 * 256). */
int tmb_microbench_icache(int kbytes, int warps, int iters, double *cycles_per_instr);

/* ----------------------------------------------------- RNG (core.py) -- */
/* core.py:66-95 on the host; used by the host driver and tests. */
uint64_t tmb_derive_stream(uint64_t seed, uint64_t index);
/* Device fill: out[i] = stream_u64(seed, start + i)  (core.py:98-104). */
int tmb_stream_u64_block(uint64_t seed, uint64_t start, int64_t count, uint64_t *out,
                         void *stream);
/* executor.py:50-58 Fisher-Yates on the host (sequential by definition).
 * perm: host int64[n]; returns the advanced stream counter in *counter_out. */
int tmb_shuffle_permutation(int64_t n, uint64_t stream_seed, uint64_t counter,
                            int64_t *perm, uint64_t *counter_out);

/* ------------------------------------------ plugin surface (device) -- */
/* kernels/_numba.py:53-58: outputs of all C clauses on one literal vector.
 * states int8 [C,P], lits uint8 [P] -> out uint8 [C]. */
int tmb_clause_outputs(const int8_t *states, int64_t C, int64_t P, const uint8_t *lits,
                       int training, int64_t budget, uint8_t *out, void *stream);
/* kernels/_numba.py:61-68: x_lit uint8 [N,P] -> out uint8 [N,C]. */
int tmb_clause_outputs_batch(const int8_t *states, int64_t C, int64_t P,
                             const uint8_t *x_lit, int64_t N, int training,
                             int64_t budget, uint8_t *out, void *stream);
/* kernels/_numba.py:101-125: one example's feedback on a clause bank, in
 * place.  ut/un uint8 [C] flags.  The new event counter is written to
 * *counter_out (a HOST pointer; the call synchronises the stream). */
int tmb_bank_feedback(int8_t *states, int32_t *weights, int64_t C, int64_t P, int64_t K,
                      const uint8_t *lits, const uint8_t *outputs, int64_t label,
                      int64_t negative, const uint8_t *ut, const uint8_t *un, double s,
                      int boost, int state_min, int state_max, uint64_t seed,
                      uint64_t counter, uint64_t *counter_out, void *stream);
/* Explicit-draws test hook (north star: one-step state delta bit-exact when
 * both sides consume the same uniform draws).  Applied event i (0-based, in
 * clause order, target before negative) reads draws[i*P .. i*P+P) (device
 * float64 [n_rows, P]) instead of the stream; every applied event consumes a
 * row, Type II included (dense.py:111). */
int tmb_bank_feedback_draws(int8_t *states, int32_t *weights, int64_t C, int64_t P,
                            int64_t K, const uint8_t *lits, const uint8_t *outputs,
                            int64_t label, int64_t negative, const uint8_t *ut,
                            const uint8_t *un, double s, int boost, int state_min,
                            int state_max, uint64_t counter, const double *draws,
                            int64_t n_rows, uint64_t *counter_out, void *stream);

/* -------------------------------------------- plugin surface (host) -- */
/* Same contracts with numpy (host) buffers; synchronous. */
int tmbh_clause_outputs(const int8_t *states, int64_t C, int64_t P, const uint8_t *lits,
                        int training, int64_t budget, uint8_t *out);
int tmbh_clause_outputs_batch(const int8_t *states, int64_t C, int64_t P,
                              const uint8_t *x_lit, int64_t N, int training,
                              int64_t budget, uint8_t *out);
int tmbh_bank_feedback(int8_t *states, int32_t *weights, int64_t C, int64_t P, int64_t K,
                       const uint8_t *lits, const uint8_t *outputs, int64_t label,
                       int64_t negative, const uint8_t *ut, const uint8_t *un, double s,
                       int boost, int state_min, int state_max, uint64_t seed,
                       uint64_t counter, uint64_t *counter_out);

/* ---------------------------------------------------- literal packing -- */
/* Pack raw features x uint8 [N, F] (row-major, stride F) into literal
 * words [N, W], W = ceil(P/32), bit p of a row = literal position p of the
 * augmented layout (core.py:232-242; p >= F is NOT x[p-F] when negations).
 * Padding bits beyond P are set to 1 (they never violate). */
int tmb_pack_literals(const uint8_t *x, int64_t N, int64_t F, int negations,
                      uint32_t *out, void *stream);

/* ----------------------------------------- dense training (fused) -- */
/* One persistent cooperative kernel runs `n_steps` consecutive examples of
 * executor.train's loop: training-mode evaluation, grid-wide vote
 * all-reduce, update decision (feedback.py:33-53), per-block event-window
 * scan, Type I / II feedback and weight updates (kernels/_numba.py:101-125).
 * Bit-exact with the reference for the same (seed, order, counters). */
typedef struct {
    int64_t n_literals;   /* F */
    int64_t n_positions;  /* P */
    int64_t n_clauses;    /* C */
    int64_t n_classes;    /* K */
    int64_t n_blocks;     /* model-semantic clause blocks (executor.py:36-47) */
    int64_t threshold;    /* T */
    int64_t budget;       /* effective budget (core.py:220-226) */
    double s;
    int32_t boost;
    int32_t state_min;
    int32_t state_max;
    int32_t flags;        /* bit 0: keep TA states in HBM even if they fit on chip;
                             bit 1: generic grid kernel (no step records);
                             bit 2: HBM-resident states: per-CTA feedback of the
                             own clauses instead of the grid-balanced split */
    uint64_t seed;        /* model seed; block b uses derive_stream(seed, b) */
} tmb_train_cfg;

typedef struct {
    uint64_t examples;     /* examples processed */
    uint64_t events;       /* applied feedback events (windows consumed) */
    uint64_t type_i;       /* Type I events */
    uint64_t type_ii;      /* Type II events with output 1 (state-touching) */
    uint64_t draws;        /* SplitMix64 draws actually evaluated */
    uint64_t state_updates;/* TA states changed */
} tmb_train_stats;

typedef struct tmb_trainer tmb_trainer;

/* Create a trainer bound to device-resident model buffers owned by the
 * caller: states int8 [C,P], weights int32 [C,K], block_counters uint64
 * [n_blocks].  n_cta = 0 picks automatically; threads = 0 picks automatically. */
int tmb_trainer_create(const tmb_train_cfg *cfg, int8_t *states, int32_t *weights,
                       uint64_t *block_counters, int n_cta, int threads,
                       tmb_trainer **out);
int tmb_trainer_destroy(tmb_trainer *t);
/* Per-example trace for tests / debugging (the device analogue of the
 * reference's observer hook, executor.py:276): when non-NULL, every
 * tmb_trainer_run writes trace[i*4 + {0,1,2,3}] = negative class, summed
 * votes of the label, of the negative class, and applied events (the last
 * only when n_blocks == 1) for its example i.  Device int64 [n_steps*4]. */
int tmb_trainer_set_trace(tmb_trainer *t, int64_t *trace);
/* Phase profiling: when non-NULL, every launch writes, per CTA, the clock64
 * cycles of its phases.  k_train_spec: [n_cta * 16] counters (see
 * tmb_train.cu) then a per-window timeline [n_cta][2048][10] (size the
 * buffer n_cta * (16 + 20480)).  Other grid-mode kernels: the clock64
 * cycles thread 0 spent in each of 8 kernel phases (device uint64
 * [n_cta * 8]): eval, partial votes + arrive, flag-draw precompute +
 * prefetch, all-reduce wait + decision, flag bitmaps, scan + events,
 * per-position feedback.  Grid mode also appends a timeline: %globaltimer
 * (ns) of thread 0 of every CTA at vote arrival, all-reduce detection and
 * step end for steps 64..1087 of each launch, [1024][n_cta][3] after the
 * [n_cta * 8] phases (size the buffer n_cta * (8 + 3072)). */
int tmb_trainer_set_profile(tmb_trainer *t, uint64_t *phase);
/* Launch configuration actually used (for reporting). */
int tmb_trainer_info(const tmb_trainer *t, int *n_cta, int *threads, int *smem_bytes,
                     int *states_in_smem);
/* Which fused trainer runs (for reporting): *kind 0 k_train_warp (one warp),
 * 1 k_train cluster mode, 2 k_train grid mode, 3 k_train_fast, 4 k_train_spec
 * (speculative windows of *window steps, else 0), 5 k_train_tiny (tiny banks,
 * one warp per clause). */
int tmb_trainer_kernel(const tmb_trainer *t, int *kind, int *window);
/* Run n_steps examples: example i uses literal row lit_words[order[i]] (device
 * uint32 [N, W]) and label labels[order[i]] (device int32); the feedback
 * stream counter of example i is fb_counter + i*(1+2C) (feedback.py:33-53).
 * block_counters are read at start and written back at the end.
 * stats (device pointer or NULL) is accumulated into. */
int tmb_trainer_run(tmb_trainer *t, const uint32_t *lit_words, const int32_t *labels,
                    const int32_t *order, int64_t n_steps, uint64_t fb_counter,
                    tmb_train_stats *stats, void *stream);

/* ------------------------------------------- compiled-rule inference -- */
/* A device-resident rule set: per rule the sorted include positions
 * (predictor.py:45-68 compile semantics are applied by the caller) and
 * int32 weights [R, K]. */
typedef struct tmb_rules tmb_rules;

/* Compile from a dense bank on the device: states int8 [C,P], weights int32
 * [C,K].  mode 0 = inference rules (drops clauses with no includes or an
 * all-zero weight row: predictor.py:56-62; they can never change a vote);
 * n_features F and negations describe the literal layout. */
int tmb_rules_from_bank(const int8_t *states, const int32_t *weights, int64_t C,
                        int64_t P, int64_t K, int64_t n_features, int negations,
                        tmb_rules **out, void *stream);
/* Compile from host CSR include lists (RuleSet, predictor.py:20-35). */
int tmb_rules_from_csr(const int64_t *inc_ptr, const int64_t *inc_idx, int64_t R,
                       const int32_t *weights, int64_t K, int64_t n_features,
                       int negations, tmb_rules **out);
int tmb_rules_destroy(tmb_rules *r);
int tmb_rules_info(const tmb_rules *r, int64_t *n_rules, int64_t *n_includes);

/* Votes / predictions for raw features x uint8 [N, F] (device).  votes int64
 * [N,K] and pred int64 [N] are optional (NULL); labels (device int64 [N]) +
 * correct (device uint64 [1], accumulated) optional.  Ties -> lowest class
 * (np.argmax, executor.py:382). */
/* Inference on bit-packed features (bit-packed ingestion):
 * xb uint64 [N, W64], feature f = bit (f % 64) of word f / 64 (W64 >= F/64).
 * Same outputs as tmb_infer; 8x fewer input bytes than uint8 rows.  Needs a
 * rule set the cluster kernel supports (else TMB_E_UNSUPPORTED). */
int tmb_infer_packed(const tmb_rules *r, const uint64_t *xb, int64_t N, int64_t W64,
                     int64_t *votes, int64_t *pred, const int64_t *labels, uint64_t *correct,
                     void *stream);
/* Batched predict_and_explain (predictor.py:99-124) on device buffers:
 * x uint8 [N, F] raw features; pred int64 [N] (argmax, ties -> lowest);
 * votes int64 [N, K] or NULL; scores int64 [N, P] or NULL (P = 2F with
 * negations, else F): every firing rule adds its weight for the explained
 * class (for_class >= 0, else the predicted class) to each literal position
 * it includes.  Feature-level scores = scores[:, :F] - scores[:, F:]. */
int tmb_explain(const tmb_rules *r, const uint8_t *x, int64_t N, int for_class, int64_t *votes,
                int64_t *pred, int64_t *scores, void *stream);
int tmb_infer(const tmb_rules *r, const uint8_t *x, int64_t N, int64_t *votes,
              int64_t *pred, const int64_t *labels, uint64_t *correct, void *stream);
/* Synchronises `stream` and reports TMB_E_INVALID if any tmb_infer call since
 * the last check saw a feature byte other than 0 / 1 (the device path
 * requires binary inputs); clears the flag. */
int tmb_infer_status(void *stream);
/* Library options (tests / tuning; defaults in brackets).  Inference:
 * "infer.solo" [1] per-CTA kernel k_infer_solo, 0 the 4-CTA cluster kernels;
 * "infer.force_generic" [0] 1 routes tmb_infer to the generic
 * one-CTA-per-tile kernel; "infer.warp_specialized", "infer.eval_mode",
 * "infer.debug_skip" (timing only), "infer.phase_buffer" (profiling).
 * Training, read at tmb_trainer_create:
 * "train.spec_window" [16] steps per speculative window of k_train_spec (0:
 * k_train_fast); "train.spec_entries" [64] staged flag entries per head;
 * "train.hbm_threads" [1024] CTA size of the HBM-state grid trainer (512 or
 * 1024); "train.gbal_weights" [2 | 5 << 8 | 6 << 16] cost weights of the
 * balanced feedback split (bytes: Type II, Type I silent, Type I firing; 0 =
 * unweighted); "train.tiny" [1] tiny banks on k_train_tiny (0: k_train_warp);
 * "train.key_chunk" (tests), "train.debug_skip" (timing only, not
 * bit-exact).  SparseTM: "sparse.resident", "sparse.infer_key",
 * "sparse.counters32", "sparse.phase_buffer" (profiling). */
int tmb_set_option(const char *name, int64_t value);
/* End-to-end variant with HOST buffers: streams x (host, ideally pinned)
 * through the device in chunks with copy/compute overlap and returns host
 * votes / pred (either may be NULL).  Synchronous. */
int tmbh_infer(const tmb_rules *r, const uint8_t *x, int64_t N, int64_t *votes,
               int64_t *pred, int64_t chunk);

/* ------------------------------------------------------------ sparse -- */
/* SparseClauseBank on the device (sparse.py:78-256): per-clause sorted
 * (literal int32, state int8) slabs of fixed capacity `slab` pairs.
 * Documents arrive as CSR (indptr int64 [N+1], indices int32 sorted per
 * row).  Bit-exact with the reference including the capacity rule
 * (sparse.py:212-220) and the candidate domain of Type II (sparse.py:198). */
typedef struct {
    int64_t n_literals;
    int64_t n_clauses;
    int64_t n_classes;
    int64_t n_blocks;
    int64_t threshold;
    int64_t budget;
    double s;
    int32_t boost;
    int32_t floor_;
    int32_t state_max;
    int32_t capacity;     /* -1 = None */
    uint64_t seed;
    int64_t slab;         /* max pairs per clause the device slab holds */
} tmb_sparse_cfg;

typedef struct tmb_sparse tmb_sparse;

int tmb_sparse_create(const tmb_sparse_cfg *cfg, const int32_t *candidates,
                      int64_t n_candidates, tmb_sparse **out);
int tmb_sparse_destroy(tmb_sparse *sp);
/* Launch layout chosen at create time: out[0] = 1 if the trainer holds the
 * clause lists in shared memory, out[1] = CTAs, out[2] = threads per CTA,
 * out[3] = dynamic shared memory bytes.  (No reference counterpart.) */
int tmb_sparse_layout(const tmb_sparse *sp, int64_t *out4);
/* Train n_steps documents in `order` (device int32), CSR on device. */
int tmb_sparse_train(tmb_sparse *sp, const int64_t *indptr, const int32_t *indices,
                     const int32_t *labels, const int32_t *order, int64_t n_steps,
                     uint64_t fb_counter, tmb_train_stats *stats, void *stream);
/* SparseClauseBank.apply_feedback (sparse.py:241-249) for a single-block
 * bank with explicit outputs / update flags (device uint8 [C]) and the
 * block's event counter; active: device int32 [n_active] sorted literals.
 * The advanced counter is returned in *counter_out (host; synchronises). */
int tmb_sparse_feedback(tmb_sparse *sp, const int32_t *active, int64_t n_active,
                        const uint8_t *outputs, int64_t label, int64_t negative,
                        const uint8_t *ut, const uint8_t *un, uint64_t stream_seed,
                        uint64_t counter, uint64_t *counter_out, void *stream);
/* Copy the model out: lens int32 [C], lits int32 [C*slab], states int8
 * [C*slab], weights int32 [C,K], block counters uint64 [n_blocks] (device
 * pointers).  Returns TMB_E_UNSUPPORTED if a slab overflowed. */
int tmb_sparse_get(const tmb_sparse *sp, int32_t *lens, int32_t *lits, int8_t *states,
                   int32_t *weights, uint64_t *block_counters, void *stream);
int tmb_sparse_set(tmb_sparse *sp, const int32_t *lens, const int32_t *lits,
                   const int8_t *states, const int32_t *weights,
                   const uint64_t *block_counters, void *stream);
/* Inference-mode votes / predictions for CSR documents (device). */
int tmb_sparse_infer(const tmb_sparse *sp, const int64_t *indptr, const int32_t *indices,
                     int64_t N, int64_t *votes, int64_t *pred, void *stream);
/* Inference-mode clause outputs (sparse.py:123-138 with EvalMode.INFERENCE)
 * for CSR documents: device uint8 [N, C]. */
int tmb_sparse_outputs(const tmb_sparse *sp, const int64_t *indptr, const int32_t *indices,
                       int64_t N, uint8_t *outputs, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* TSETLIN_B200_H */
