/*
 * libspgcm — B200 (sm_100a) AES-256-GCM seal/open for the encrypted swap path.
 *
 * Drop-in boundary for the reference's crypto seam.  The reference binds
 * exactly two functions for this path (plus the construction of the cipher
 * context they imply):
 *
 *   specpipe.channel.encrypt_at(key, iv, plaintext, direction) -> CiphertextMsg
 *       /root/reference/pkg/src/specpipe/channel.py:85-101
 *       (also imported by value as specpipe.engine.encrypt_at, engine.py:34,503)
 *   specpipe.channel.decrypt_at(key, iv, msg, direction) -> bytes | AuthError
 *       /root/reference/pkg/src/specpipe/channel.py:104-115
 *   AESGCM(key) construction per call (channel.py:96,111)  -> sp_ctx_create
 *
 * Semantics kept bit-exact: AES-256-GCM, 32-byte key, 16-byte tag, no AAD,
 * 96-bit nonce = 4-byte big-endian direction || 8-byte big-endian counter
 * (channel.py:77-82), 1 <= len <= 32 MiB (channel.py:92-95).
 *
 * All entry points are extern "C", take plain pointers and sizes, and never
 * fall back to the CPU: every byte of AES/GHASH work runs in sm_100a kernels.
 * Device-pointer entry points are stream-ordered and asynchronous; `*_host`
 * entry points take host buffers, pipeline the PCIe copies against the
 * kernels, and return when the result is in host memory.
 *
 * A context is immutable after creation and may be used from several host
 * threads and streams at once.
 */
#ifndef SPGCM_H_
#define SPGCM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes (channel.py error classes: ValueError -> SP_EINVAL,
 * AuthError -> SP_EAUTH). */
#define SP_OK 0
#define SP_EINVAL 1   /* len == 0, len > 32 MiB, null pointer, bad direction */
#define SP_EAUTH 2    /* tag mismatch: plaintext output is zeroed */
#define SP_ECUDA 3    /* CUDA runtime error (message via sp_last_error) */
#define SP_ENODEV 4   /* no CUDA device / kernel image not loadable */

#define SP_KEY_BYTES 32
#define SP_TAG_BYTES 16
#define SP_NONCE_BYTES 12
#define SP_MAX_MESSAGE_BYTES (32u * 1024u * 1024u)
#define SP_DIR_H2D 0u /* Direction.HOST_TO_DEVICE, channel.py:47 */
#define SP_DIR_D2H 1u /* Direction.DEVICE_TO_HOST, channel.py:48 */

typedef struct sp_ctx sp_ctx;
/* cudaStream_t, kept opaque so the header needs no CUDA include. */
typedef void *sp_stream_t;

/* One message of a batch.  All pointers are DEVICE pointers.
 * seal: reads src (len bytes), writes dst (len bytes) and tag (16 bytes).
 * open: reads src (ciphertext) and tag (expected), writes dst (plaintext) and
 *       *status (0 = authentic, 1 = tag mismatch -> dst zeroed).
 * src may equal dst (in place).  Any alignment is accepted; 16-byte aligned
 * src/dst take the vectorised path. */
typedef struct sp_desc {
    uint32_t dir;       /* SP_DIR_H2D or SP_DIR_D2H */
    uint32_t reserved;  /* sp_crypt_batch: SP_OP_SEAL or SP_OP_OPEN (else ignored); | SP_STATUS_ON_FAILURE */
    uint64_t iv;        /* 64-bit channel counter, any value in [0, 2^64) */
    uint64_t len;       /* 1 .. SP_MAX_MESSAGE_BYTES */
    const void *src;
    void *dst;
    void *tag;          /* 16 bytes, device */
    int32_t *status;    /* open only, device (or UVA-mapped pinned); may be NULL for seal */
} sp_desc;

/* Replaces the per-call `AESGCM(key)` construction (channel.py:96,111): key
 * schedule, H = E_K(0^128), GHASH power tables, all resident in HBM of the
 * current CUDA device.  Synchronous. */
int sp_ctx_create(const uint8_t key[SP_KEY_BYTES], sp_ctx **out);
void sp_ctx_destroy(sp_ctx *ctx);

/* encrypt_at over device buffers (channel.py:85-101).  Stream-ordered. */
int sp_seal(sp_ctx *ctx, uint32_t dir, uint64_t iv, const void *src, size_t len,
            void *dst, void *tag16, sp_stream_t stream);

/* decrypt_at over device buffers (channel.py:104-115).  Stream-ordered; the
 * verdict lands in *status_dev (0 ok, 1 auth failure, dst zeroed). */
int sp_open(sp_ctx *ctx, uint32_t dir, uint64_t iv, const void *src, size_t len,
            const void *tag16, void *dst, int32_t *status_dev, sp_stream_t stream);

/* Many messages in ONE launch: chunk runs (engine.py:328-331,368-369,
 * 502-508), NOP padding (engine.py:546-556), deferred-decrypt drains
 * (engine.py:579-581).  Stream-ordered. */
int sp_seal_batch(sp_ctx *ctx, const sp_desc *descs, int n, sp_stream_t stream);
int sp_open_batch(sp_ctx *ctx, const sp_desc *descs, int n, sp_stream_t stream);
/* Seals and opens mixed in ONE launch (desc.reserved picks the operation):
 * the pipeline's independent NOP/on-the-fly/swap-out seals and receiver
 * opens of one flush.  Messages of one call must not overlap in memory. */
#define SP_OP_SEAL 0u
#define SP_OP_OPEN 1u
/* Or-ed into desc.reserved of an open (any batch call): *status is written
 * only on a tag mismatch (1), never on success, so many opens may share one
 * status word (a sticky "some open failed" flag; the pipeline keeps one per
 * pipe in mapped pinned memory and reads it at finish). */
#define SP_STATUS_ON_FAILURE 0x100u
int sp_crypt_batch(sp_ctx *ctx, const sp_desc *descs, int n, sp_stream_t stream);
/* Dependent levels of one flush in ONE launch: descs grouped by level,
 * level l = descs[level_start[l] .. level_start[l+1]), level_start[0] = 0,
 * level_start[nlevels] = n.  A message of level l may read what level l-1
 * wrote (a receiver open of a ciphertext sealed in the same flush): the
 * kernel's warps claim work in level order and level l starts when level
 * l-1 is complete, so the result equals nlevels sp_crypt_batch calls in
 * stream order (what the reference's per-send drain does one message at a
 * time, engine.py:291 and engine.py:579-581) without a launch boundary per
 * level.  Up to 8 levels and 256 messages fuse; larger calls run one launch
 * per level.  Stream-ordered. */
int sp_crypt_levels(sp_ctx *ctx, const sp_desc *descs, int n, const int *level_start, int nlevels,
                    sp_stream_t stream);

/* Host-buffer entry points: the exact call shape of encrypt_at / decrypt_at
 * (bytes in, bytes out).  H2D copies, kernels and D2H copies are pipelined
 * in pieces on internal streams; returns when results are in host memory.
 * Host buffers may be pageable; pinned buffers reach full PCIe rate.
 * sp_open_host returns SP_EAUTH (and zeroes dst) on a tag mismatch. */
int sp_seal_host(sp_ctx *ctx, uint32_t dir, uint64_t iv, const void *src, size_t len,
                 void *dst, uint8_t tag16[SP_TAG_BYTES]);
int sp_open_host(sp_ctx *ctx, uint32_t dir, uint64_t iv, const void *src, size_t len,
                 const uint8_t tag16[SP_TAG_BYTES], void *dst);

/* Host-buffer batch: n messages, host src/dst/tag pointers in descs (status
 * is a HOST int32 pointer for open).  Returns SP_EAUTH if any open failed. */
int sp_seal_host_batch(sp_ctx *ctx, const sp_desc *descs, int n);
int sp_open_host_batch(sp_ctx *ctx, const sp_desc *descs, int n);

/* SM budget: launches of this context use at most max_sms SMs (0 = all),
 * so the crypto kernels leave the rest of the GPU to model compute running
 * beside them (SURVEY §7 "cap the grid").  Throughput scales with the
 * budget; results are identical.  Applies to launches issued after the
 * call; the only mutable context state (an atomic). */
int sp_ctx_set_max_sms(sp_ctx *ctx, int max_sms);
int sp_ctx_max_sms(const sp_ctx *ctx);
/* SM cap of this context's SMALL launches (<= 2 MiB of rows: KV batches,
 * tokens, NOP pads; 0 = none, the default).  Such launches are latency-bound
 * and each CTA holds a whole SM while it runs, so a pipeline running beside
 * model compute caps them (libsppipe sets 32) at the cost of a slower launch
 * alone.  Results are identical. */
int sp_ctx_set_small_sms(sp_ctx *ctx, int small_sms);

/* Diagnostics. */
const char *sp_last_error(void);
const char *sp_version(void);
/* Number of sm_100a kernel launches issued by this library in this process. */
uint64_t sp_launch_count(void);
/* Fill 15 round-key words x4 (240 bytes, FIPS-197 order) for tests. */
int sp_ctx_round_keys(const sp_ctx *ctx, uint8_t out[240]);
/* Copy H = E_K(0^128) back to the host (16 bytes), for tests. */
int sp_ctx_hash_key(const sp_ctx *ctx, uint8_t out[16]);

#ifdef __cplusplus
}
#endif

#endif /* SPGCM_H_ */
