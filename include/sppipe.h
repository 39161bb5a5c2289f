/*
 * libsppipe — native speculative pipeline (control plane + B200 data plane)
 * for the encrypted swap path.
 *
 * Replaces, behind a C-ABI, the reference's pipeline and predictor
 * (/root/reference/pkg/src/specpipe):
 *
 *   sp_pred_*   specpipe.predictor.Predictor           predictor.py:316-375
 *               classify                               predictor.py:74-94
 *               predict_batches / predict_next         predictor.py:252-313
 *   sp_pipe_*   specpipe.engine.Engine                 engine.py:171-624
 *               copy_h2d (submit)                      engine.py:295-320
 *               copy_d2h                               engine.py:353-393
 *               small_io                               engine.py:397-416
 *               sync (reorder + NOP padding)           engine.py:537-577
 *               speculate_tick                         engine.py:442-485
 *               relinquish                             engine.py:527-535
 *               finish / audit / report                engine.py:583-624
 *               app_write / app_read                   engine.py:420-440
 *   (validator.py and the channel counters of channel.py:146-215 live inside.)
 *
 * Decisions are the reference's, bit for bit: the same trace gives the same
 * sent logs, actions, report() counters and predictor decision log.  The
 * crypto runs in libspgcm's sm_100a kernels (batched, stream-ordered) and the
 * copies on dedicated H2D/D2H streams from the caller's (pinned) host blocks;
 * there is no CPU crypto path.
 *
 * Errors: every call returns SP_OK or an SP_E* code; the message is in
 * sp_pipe_last_error().  After an error the pipe stays in the state the
 * reference engine would be in after raising (parity harnesses inspect it).
 * A pipe is single-owner (one host thread at a time), as the reference's
 * engine is.
 */
#ifndef SPPIPE_H_
#define SPPIPE_H_

#include <stddef.h>
#include <stdint.h>

#include "spgcm.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes beyond spgcm.h's (SP_OK .. SP_ENODEV). */
#define SP_EENGINE 10        /* EngineError (engine.py:40) */
#define SP_EOVERLAP 11       /* validator.OverlapError */
#define SP_ESTATE 12         /* validator.StateError */
#define SP_EUNKNOWN_BLOCK 13 /* predictor.UnknownBlock */
#define SP_EBOUNDS 14        /* memory.BoundsError */
#define SP_EGUARD 15         /* memory.GuardOverlapError */
#define SP_EAMBIGUOUS 16     /* predictor.AmbiguousProfile */
#define SP_EIVREUSE 17       /* channel.IvReuseError */
#define SP_EKEY 18           /* lookup of an unknown block / record id (KeyError) */

/* Transfer classes (predictor.TransferClass) and block kinds (memory.BlockKind). */
#define SP_CLASS_WEIGHTS 0
#define SP_CLASS_KV 1
#define SP_CLASS_SMALL_IO 2
#define SP_KIND_LAYER 0
#define SP_KIND_KV 1
#define SP_KIND_SMALL 2
/* sp_pipe_register_block kind flag: the host buffer starts on a page
 * boundary and its last page belongs to no other object (pinned slab
 * blocks are page-aligned and page-padded), so hardware write guards
 * covering the block's first / last byte protect the partial pages too
 * (spg_protect_ex). */
#define SP_BLOCK_PAGE_OWNED 0x100

/* Verdicts (validator.VerdictKind); SP_VERDICT_NONE for SMALL_IO submits. */
#define SP_VERDICT_HIT 0
#define SP_VERDICT_IV_AHEAD 1
#define SP_VERDICT_IV_BEHIND 2
#define SP_VERDICT_STALE 3
#define SP_VERDICT_MISS 4
#define SP_VERDICT_NONE 5

/* Pattern kinds (predictor.PatternKind). */
#define SP_PATTERN_REPETITIVE 0
#define SP_PATTERN_LIFO 1
#define SP_PATTERN_FIFO 2
#define SP_PATTERN_UNKNOWN 3

/* Action kinds (engine.ActionKind). */
#define SP_ACT_SPEC_ENCRYPT 0
#define SP_ACT_H2D_DATA 1
#define SP_ACT_NOP 2
#define SP_ACT_D2H_DATA 3
#define SP_ACT_RESOLVE_DECRYPT 4
#define SP_ACT_RELINQUISH 5
#define SP_ACT_SYNC_POINT 6

typedef struct sp_pred sp_pred;
typedef struct sp_pipe sp_pipe;

/* predictor.PredictorConfig + ModelProfile (predictor.py:44-60). */
typedef struct sp_pred_config {
    uint64_t small_io_threshold; /* 8 KiB */
    uint64_t swap_min;           /* 128 KiB */
    uint64_t chunk_bytes;        /* 32 MiB */
    int64_t warmup_matches;      /* 2 */
    int64_t history_cap;         /* 128 */
    uint64_t layer_param_bytes;  /* profile.layer_param_bytes (0 with kv 0: no profile) */
    uint64_t kv_block_bytes;     /* profile.kv_block_bytes */
} sp_pred_config;

typedef struct sp_prediction {
    int64_t block;
    uint64_t predicted_iv;
    uint64_t leeway;
    int32_t batch; /* index of the predicted batch this entry belongs to */
    int32_t reserved; /* sp_pred_script: round (the predict call that hands it out); else 0 */
} sp_prediction;

typedef struct sp_decision {
    int32_t event;   /* 0 lock, 1 drop */
    int32_t pattern; /* SP_PATTERN_* */
    int64_t confidence;
    int64_t after_batches;
} sp_decision;

int sp_pred_create(const sp_pred_config *cfg, sp_pred **out);
void sp_pred_destroy(sp_pred *p);
int sp_pred_classify(sp_pred *p, uint64_t size, int32_t *cls);
int sp_pred_observe_out(sp_pred *p, int64_t block);
int sp_pred_observe_in(sp_pred *p, const int64_t *blocks, int32_t n);
int sp_pred_observe_sync(sp_pred *p);
/* recognize(): kind, confidence, phase, cycle length (cycle entries via sp_pred_cycle_entry). */
int sp_pred_recognize(sp_pred *p, int32_t *kind, int64_t *confidence, int64_t *phase, int64_t *cycle_len);
/* blocks of cycle entry i (sorted); *n = entry size (blocks written up to cap). */
int sp_pred_cycle_entry(sp_pred *p, int64_t i, int64_t *blocks, int32_t cap, int32_t *n);
int sp_pred_predict_batches(sp_pred *p, uint64_t current_iv, uint64_t leeway, int32_t depth,
                            sp_prediction *out, int32_t cap, int32_t *n);
int sp_pred_outstanding(sp_pred *p, int64_t *out, int64_t cap, int64_t *n); /* swap-out order */
/* predict_batches with an explicit outstanding set (the reference's free
 * function predict_batches(history, outstanding, ...), predictor.py:252-297). */
int sp_pred_predict_batches_in(sp_pred *p, uint64_t current_iv, uint64_t leeway, int32_t depth,
                               const int64_t *outstanding, int64_t n_out, sp_prediction *out, int32_t cap,
                               int32_t *n);
/* Scripted mode (the scenario mock of cli.py:241-259): predict_batches hands
 * out `preds` once (grouped by their batch field; entries with reserved = r
 * on the r-th call), the outstanding set is `outstanding`, observations are
 * ignored. */
int sp_pred_script(sp_pred *p, const sp_prediction *preds, int32_t n, const int64_t *outstanding, int64_t n_out);
/* SwapHistory.events (predictor.py:128-150): kind 0 swap-out (value = block),
 * 1 swap-in (value = index of its batch in the in-batches), 2 sync. */
int64_t sp_pred_event_count(sp_pred *p);
int sp_pred_event(sp_pred *p, int64_t i, int32_t *kind, int64_t *value);
/* SwapHistory.in_batches[i] (sorted blocks). */
int sp_pred_in_batch(sp_pred *p, int64_t i, int64_t *blocks, int32_t cap, int32_t *n);
int64_t sp_pred_in_batch_count(sp_pred *p);
int64_t sp_pred_decision_count(sp_pred *p);
int sp_pred_decision(sp_pred *p, int64_t i, sp_decision *out);

/* engine.EngineConfig (engine.py:78-92) + B200 data-plane knobs. */
#define SP_WINDOW_AWARE_AUTO 0
#define SP_WINDOW_AWARE_ON 1
#define SP_WINDOW_AWARE_OFF 2

typedef struct sp_pipe_config {
    uint32_t window;      /* 64 */
    uint32_t leeway;      /* 8 */
    uint32_t depth;       /* 1 */
    uint32_t workers;     /* 2 (accepted, unused: the device runs the crypto) */
    uint64_t chunk_bytes; /* 32 MiB */
    uint32_t nop_bytes;   /* 1 */
    uint32_t ring_slots;  /* 16 */
    uint8_t speculate;
    uint8_t defer_swap_decrypt;
    uint8_t record_stream;
    uint8_t strict_auth;      /* verify tags after every drain (host waits) */
    uint8_t reference_compat; /* 1: reproduce defect C2; 0: OTF sends burn the record at their counter */
    uint8_t dry;              /* 1: no bytes, no device (schedule only) */
    uint8_t hw_guards;        /* 1: also mprotect guarded host pages (libspguard) */
    uint8_t window_aware;     /* SP_WINDOW_AWARE_*: speculate only whole predicted batches that fit the
                                 record window; AUTO (0) = on iff reference_compat is 0, as Python's
                                 EngineConfig(window_aware=None) */
    uint64_t initial_h2d_iv; /* cpu endpoint send_iv */
    uint64_t initial_d2h_iv; /* gpu endpoint send_iv */
    uint64_t batch_bytes;    /* flush a batched launch at this much payload (64 MiB) */
    uint64_t reserve_bytes;  /* device pool bytes reserved at create (0: grow on demand) */
    uint64_t record_history; /* finished validator records kept (0: all, as the reference); older ones
                                below the oldest pending record are forgotten at sync (long-running pipes) */
    uint32_t crypto_sms;     /* SM budget of the pipe's seal/open launches (0: all SMs; sp_ctx_set_max_sms) */
    uint32_t reserved2;
} sp_pipe_config;

typedef struct sp_action {
    int32_t kind; /* SP_ACT_* */
    int32_t flags; /* bit0 committed, bit1 otf */
    int64_t iv;   /* -1 when not applicable */
    uint64_t nbytes;
    int64_t record_id; /* -1 = None */
    int64_t task_id;   /* -1 = None */
    int64_t count;
    int64_t seq;       /* -1 = None */
} sp_action;

typedef struct sp_sent {
    uint64_t iv;
    uint64_t size;
    int32_t nop;
    int32_t reserved;
} sp_sent;

typedef struct sp_delivery {
    uint64_t seq;
    uint64_t addr; /* host address of the range (h2d delivered only) */
    uint64_t size;
} sp_delivery;

/* One trace event for sp_pipe_replay (workload.py:41-80 event kinds). */
#define SP_EV_SWAP_IN 0
#define SP_EV_SWAP_OUT 1
#define SP_EV_SMALL_IO_H2D 2
#define SP_EV_SMALL_IO_D2H 3
#define SP_EV_SYNC 4
#define SP_EV_APP_WRITE 5
#define SP_EV_COMPUTE 6
typedef struct sp_event {
    int32_t kind;
    int32_t cls;      /* transfer class of the block (swap events) */
    int64_t block;    /* block id (swap / app write) */
    uint64_t base;    /* request base (swap) / offset (app write) */
    uint64_t len;     /* request length / payload size */
    uint64_t payload; /* byte offset of the payload in the replay payload buffer */
} sp_event;

int sp_pipe_create(const sp_pipe_config *cfg, const uint8_t key[SP_KEY_BYTES], sp_pred *pred, sp_pipe **out);
void sp_pipe_destroy(sp_pipe *p);
/* Host memory block (memory.MemoryBlock); host points at len bytes the
 * caller keeps alive (page-locked for full PCIe rate). */
int sp_pipe_register_block(sp_pipe *p, int64_t id, uint64_t base, uint64_t len, int32_t kind, void *host);
/* Device-resident content for a block (engine.seed_device); src is device
 * memory when src_is_device, else host memory. */
int sp_pipe_seed_device(sp_pipe *p, int64_t block, const void *src, uint64_t len, int32_t src_is_device);
int sp_pipe_submit_h2d(sp_pipe *p, uint64_t base, uint64_t len, int32_t cls, int64_t block, uint64_t *seq,
                       int32_t *verdict);
int sp_pipe_submit_d2h(sp_pipe *p, uint64_t base, uint64_t len, int32_t cls, int64_t block, uint64_t *seq);
int sp_pipe_small_io(sp_pipe *p, int32_t dir, const void *payload, uint64_t size);
int sp_pipe_sync(sp_pipe *p);
int sp_pipe_speculate(sp_pipe *p);
int sp_pipe_relinquish(sp_pipe *p, int64_t *count);
int sp_pipe_drain_decrypts(sp_pipe *p);
int sp_pipe_finish(sp_pipe *p);
/* audit() (engine.py:595-605): counter ledger and shared-ring checks. */
int sp_pipe_audit(sp_pipe *p);
/* finish() that returns once every observable result is final (all
 * committed transfers opened and verified, all landings and app writes on
 * the host) without waiting for encrypt-ahead work of records discarded at
 * finish, which gates nothing (the reference simulator's makespan excludes
 * it, simulator.py:441-443); sp_pipe_flush(p, 1) or destroy drains it. */
int sp_pipe_finish_observable(sp_pipe *p);
/* Issue every queued launch/landing now; with wait != 0 also block until all
 * device work of the pipe's streams is done (no counter or tag checks). */
int sp_pipe_flush(sp_pipe *p, int32_t wait);
int sp_pipe_app_write(sp_pipe *p, int64_t block, uint64_t offset, const void *data, uint64_t n, int64_t *faults);
int sp_pipe_app_read(sp_pipe *p, int64_t block, uint64_t offset, uint64_t n, void *out);
/* Whole trace in one call (the replay driver of simulator.py:404-426 minus
 * its cost model); payloads holds small-I/O and app-write bytes. */
int sp_pipe_replay(sp_pipe *p, const sp_event *ev, uint64_t n, const uint8_t *payloads, uint64_t *done);
/* The unencrypted baseline of the same trace (NoCc): the swaps as plain
 * copies between the registered pinned blocks and HBM on the pipe's copy
 * streams, gathered per batch boundary into batched copies like the
 * engine's flushes, same ordering rules, no crypto; returns when the device
 * is idle. */
int sp_pipe_plain_replay(sp_pipe *p, const sp_event *ev, uint64_t n, const uint8_t *payloads);
int sp_pipe_handle_done(sp_pipe *p, uint64_t seq, int32_t *done);
/* Test hook (the reference's Channel(test_hooks=True).hook_corrupt_in_flight,
 * channel.py:263-273): XOR `mask` into byte `byte_index` of the index-th
 * message still in flight on the `dir` lane (sent, not yet received),
 * stream-ordered after its seal.  The receiver's open must then fail. */
int sp_pipe_test_corrupt(sp_pipe *p, int32_t dir, uint64_t index, uint64_t byte_index, uint8_t mask);
/* Test hook: one k_xfer launch (the plane's SM-driven transfer of small
 * copies) over n jobs dst[i] <- src[i] (len[i] bytes; device or UVA-mapped
 * pinned host pointers, any alignment), on a private stream; returns when
 * the copy is done.  n <= 128. */
int sp_test_xfer(int32_t n, void *const *dst, const void *const *src, const uint64_t *len);

/* report(): counters in the order of sp_pipe_counter_name(i); n = count. */
int sp_pipe_report(sp_pipe *p, int64_t *out, int32_t cap, int32_t *n);
const char *sp_pipe_counter_name(int32_t i);
uint64_t sp_pipe_send_iv(sp_pipe *p, int32_t dir);
uint64_t sp_pipe_recv_iv(sp_pipe *p, int32_t dir);
int64_t sp_pipe_action_count(sp_pipe *p);
int sp_pipe_actions(sp_pipe *p, int64_t from, sp_action *out, int64_t cap, int64_t *n);
int64_t sp_pipe_sent_count(sp_pipe *p, int32_t dir);
int sp_pipe_sent_log(sp_pipe *p, int32_t dir, int64_t from, sp_sent *out, int64_t cap, int64_t *n);
/* Recorded streams (record_stream): which 0 = delivered H2D plaintext,
 * 1 = D2H small-I/O stream.  bytes (host, size bytes) may be NULL. */
/* Validator records (validator.CiphertextRecord, validator.py:44-63): ids
 * are 1 .. sp_pipe_record_count; state 0 pending, 1 committed, 2 invalidated. */
typedef struct sp_record {
    int64_t id;
    uint64_t base;
    uint64_t len;
    uint64_t iv;
    uint64_t span;     /* consecutive counters (chunks) */
    int64_t block_id;  /* INT64_MIN = None */
    int32_t state;
    int32_t reserved;
} sp_record;
int64_t sp_pipe_record_count(sp_pipe *p);  /* ids labeled so far (1..count) */
int64_t sp_pipe_record_first(sp_pipe *p);  /* oldest retained id (record_history) */
int sp_pipe_record(sp_pipe *p, int64_t id, sp_record *out);
/* Pending record ids in label order (validator.pending_records) and the
 * pending record holding counter iv (-1: none). */
int sp_pipe_pending(sp_pipe *p, int64_t *ids, int64_t cap, int64_t *n);
int64_t sp_pipe_pending_at_iv(sp_pipe *p, uint64_t iv);
int64_t sp_pipe_delivered_count(sp_pipe *p, int32_t which);
int sp_pipe_delivered(sp_pipe *p, int32_t which, int64_t i, sp_delivery *out, void *bytes);
/* Data-plane statistics: bytes over PCIe per direction, kernel launches. */
/* Model compute of a trace ComputeEvent (simulator.py:431-434 charges it to
 * the GPU): duration_ns of calibrated FMA work over every SM on the pipe's
 * app stream, after the swap-ins of the last sync; later swap-out seals
 * wait for it.  sp_pipe_replay / sp_pipe_plain_replay issue SP_EV_COMPUTE
 * events the same way. */
int sp_pipe_compute(sp_pipe *p, uint64_t duration_ns);
/* Compute launches so far, their requested (idle-GPU) duration and the
 * device time they actually took (waits for them). */
int sp_pipe_compute_stats(sp_pipe *p, uint64_t *launches, uint64_t *requested_ns, uint64_t *measured_ns);
int sp_pipe_stats(sp_pipe *p, uint64_t *bytes_h2d, uint64_t *bytes_d2h, uint64_t *launches);
/* The issuing thread: stream-ordered CUDA calls posted so far and the time
 * spent inside them (ns); busy close to a run's wall time = issue-bound.
 * host_queries: event queries the control plane itself made. */
int sp_pipe_issuer_stats(sp_pipe *p, uint64_t *calls, uint64_t *busy_ns, uint64_t *host_queries);
/* Device memory: bytes the stream-ordered pool holds from the driver, bytes
 * handed out, bytes parked in this pipe's buffer cache. */
int sp_pipe_pool_stats(sp_pipe *p, uint64_t *reserved, uint64_t *used, uint64_t *cached);
const char *sp_pipe_last_error(void);

/* A standalone validator (specpipe.validator.Validator, validator.py:90-236):
 * the pipe's own record window without an engine.  Records hold no payload
 * here (the Python side keeps the ciphertext objects); span = number of
 * consecutive counters (chunks).  Verdicts: SP_VERDICT_*; record_id -1 for
 * MISS.  counters: hit, iv_ahead, iv_behind, stale, miss, evicted. */
typedef struct sp_val sp_val;
int sp_val_create(uint64_t window, sp_val **out);
void sp_val_destroy(sp_val *v);
int sp_val_label(sp_val *v, uint64_t base, uint64_t len, uint64_t iv, uint64_t span, int64_t block_id, int64_t *id);
int sp_val_validate(sp_val *v, uint64_t base, uint64_t len, uint64_t current_iv, int32_t *verdict,
                    int64_t *record_id);
int sp_val_commit(sp_val *v, int64_t id);
int sp_val_invalidate(sp_val *v, int64_t id);
int sp_val_write_fault(sp_val *v, int64_t owner);
int64_t sp_val_pending_at_iv(sp_val *v, uint64_t iv);
int32_t sp_val_has_pending_range(sp_val *v, uint64_t base, uint64_t len);
int sp_val_invalidate_pending_below(sp_val *v, uint64_t iv, int64_t *n);
int sp_val_pending(sp_val *v, int64_t *ids, int64_t cap, int64_t *n);
int64_t sp_val_record_count(sp_val *v);
int sp_val_record(sp_val *v, int64_t id, sp_record *out);
int sp_val_counters(sp_val *v, int64_t out[6]);

#ifdef __cplusplus
}
#endif

#endif /* SPPIPE_H_ */
