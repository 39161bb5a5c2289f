/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU oracle: a plain-C restatement of the arithmetic the reference reaches
 * through `cryptography.hazmat.primitives.ciphers.aead.AESGCM` (pinned only as
 * `cryptography>=41`, /root/reference/pkg/pyproject.toml:10-12; 48.0.0 with
 * bundled OpenSSL 4.0.0 in the build image).  That dependency is absent from
 * /root/reference, so this file restates its published algorithms:
 *
 *   - AES-256 block cipher, FIPS-197 (S-box derived from the GF(2^8) inverse +
 *     affine map, §5.1.1; key expansion Nk=8 / Nr=14, §5.2; cipher §5.1).
 *   - GCM, NIST SP 800-38D: GHASH (Alg. 2) over the bit-serial multiply of
 *     Alg. 1, GCTR with inc32 (§6.5), J0 = IV || 0^31 || 1 for a 96-bit IV,
 *     tag = MSB_128(GCTR(J0, S)) with S = GHASH(C || [0]_64 || [len(C)]_64)
 *     because the reference passes no AAD (channel.py:96, `None`).
 *
 * The reference-specific framing it follows:
 *   - nonce = 4-byte big-endian direction || 8-byte big-endian counter
 *     (channel.py:77-82 `_nonce`);
 *   - 1 <= len <= 32 MiB, else ValueError (channel.py:92-95);
 *   - seal returns payload (len bytes) and a 16-byte tag split off the end
 *     (channel.py:96-101); open rejects a bad tag (channel.py:110-115).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker / baseline.
 * Deliberately slow and obviously-correct: no tables beyond the S-box.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#define ORC_MAX_MESSAGE (32u * 1024u * 1024u)

static uint8_t g_sbox[256];
static int g_sbox_ready = 0;

static uint8_t gf8_mul(uint8_t a, uint8_t b) {
    uint8_t p = 0;
    for (int i = 0; i < 8; i++) {
        if (b & 1) p ^= a;
        uint8_t hi = a & 0x80;
        a <<= 1;
        if (hi) a ^= 0x1b;  /* x^8 = x^4 + x^3 + x + 1 (FIPS-197 §4.2) */
        b >>= 1;
    }
    return p;
}

static void build_sbox(void) {
    if (g_sbox_ready) return;
    for (int x = 0; x < 256; x++) {
        uint8_t inv = 0;
        if (x) {
            for (int y = 1; y < 256; y++) {
                if (gf8_mul((uint8_t)x, (uint8_t)y) == 1) { inv = (uint8_t)y; break; }
            }
        }
        /* affine transform b'_i = b_i ^ b_{i+4} ^ b_{i+5} ^ b_{i+6} ^ b_{i+7} ^ c_i, c = 0x63 */
        uint8_t s = inv;
        uint8_t r = inv;
        for (int k = 0; k < 4; k++) {
            r = (uint8_t)((r << 1) | (r >> 7));
            s ^= r;
        }
        g_sbox[x] = s ^ 0x63;
    }
    g_sbox_ready = 1;
}

/* FIPS-197 §5.2 KeyExpansion for Nk = 8, Nr = 14: 60 words, byte-serial. */
static void key_expand(const uint8_t key[32], uint8_t w[240]) {
    build_sbox();
    memcpy(w, key, 32);
    uint8_t rcon = 1;
    for (int i = 8; i < 60; i++) {
        uint8_t t[4];
        memcpy(t, w + 4 * (i - 1), 4);
        if (i % 8 == 0) {
            uint8_t t0 = t[0];
            t[0] = g_sbox[t[1]] ^ rcon;
            t[1] = g_sbox[t[2]];
            t[2] = g_sbox[t[3]];
            t[3] = g_sbox[t0];
            rcon = gf8_mul(rcon, 2);
        } else if (i % 8 == 4) {
            for (int k = 0; k < 4; k++) t[k] = g_sbox[t[k]];
        }
        for (int k = 0; k < 4; k++) w[4 * i + k] = w[4 * (i - 8) + k] ^ t[k];
    }
}

/* FIPS-197 §5.1 Cipher; state[r + 4c] in input byte order. */
static void aes256_encrypt_block(const uint8_t w[240], const uint8_t in[16], uint8_t out[16]) {
    uint8_t s[16];
    for (int i = 0; i < 16; i++) s[i] = in[i] ^ w[i];
    for (int round = 1; round <= 14; round++) {
        uint8_t t[16];
        /* SubBytes + ShiftRows: row r rotates left by r */
        for (int c = 0; c < 4; c++)
            for (int r = 0; r < 4; r++)
                t[r + 4 * c] = g_sbox[s[r + 4 * ((c + r) & 3)]];
        if (round != 14) {
            /* MixColumns */
            for (int c = 0; c < 4; c++) {
                uint8_t a0 = t[4 * c], a1 = t[4 * c + 1], a2 = t[4 * c + 2], a3 = t[4 * c + 3];
                s[4 * c + 0] = gf8_mul(a0, 2) ^ gf8_mul(a1, 3) ^ a2 ^ a3;
                s[4 * c + 1] = a0 ^ gf8_mul(a1, 2) ^ gf8_mul(a2, 3) ^ a3;
                s[4 * c + 2] = a0 ^ a1 ^ gf8_mul(a2, 2) ^ gf8_mul(a3, 3);
                s[4 * c + 3] = gf8_mul(a0, 3) ^ a1 ^ a2 ^ gf8_mul(a3, 2);
            }
        } else {
            memcpy(s, t, 16);
        }
        for (int i = 0; i < 16; i++) s[i] ^= w[16 * round + i];
    }
    memcpy(out, s, 16);
}

/* SP 800-38D Algorithm 1: Z = X . Y in GF(2^128), bit-reflected convention
 * (bit 0 = MSB of byte 0), R = 11100001 || 0^120. */
static void gf128_mul(const uint8_t X[16], const uint8_t Y[16], uint8_t Z[16]) {
    uint8_t V[16], acc[16];
    memset(acc, 0, 16);
    memcpy(V, Y, 16);
    for (int i = 0; i < 128; i++) {
        if ((X[i >> 3] >> (7 - (i & 7))) & 1)
            for (int k = 0; k < 16; k++) acc[k] ^= V[k];
        int lsb = V[15] & 1;
        for (int k = 15; k > 0; k--) V[k] = (uint8_t)((V[k] >> 1) | (V[k - 1] << 7));
        V[0] >>= 1;
        if (lsb) V[0] ^= 0xe1;
    }
    memcpy(Z, acc, 16);
}

static void make_j0(uint32_t dir, uint64_t iv, uint8_t j0[16]) {
    /* channel.py:77-82: dir.to_bytes(4,'big') || iv.to_bytes(8,'big'); then || 0x00000001 */
    for (int k = 0; k < 4; k++) j0[k] = (uint8_t)(dir >> (24 - 8 * k));
    for (int k = 0; k < 8; k++) j0[4 + k] = (uint8_t)(iv >> (56 - 8 * k));
    j0[12] = 0; j0[13] = 0; j0[14] = 0; j0[15] = 1;
}

static void inc32(uint8_t cb[16]) {
    uint32_t c = ((uint32_t)cb[12] << 24) | ((uint32_t)cb[13] << 16) | ((uint32_t)cb[14] << 8) | cb[15];
    c += 1;
    cb[12] = (uint8_t)(c >> 24); cb[13] = (uint8_t)(c >> 16); cb[14] = (uint8_t)(c >> 8); cb[15] = (uint8_t)c;
}

/* GCTR over `len` bytes starting at counter block ICB (SP 800-38D §6.5). */
static void gctr(const uint8_t w[240], const uint8_t icb[16], const uint8_t *in, size_t len, uint8_t *out) {
    uint8_t cb[16], ks[16];
    memcpy(cb, icb, 16);
    for (size_t off = 0; off < len; off += 16) {
        aes256_encrypt_block(w, cb, ks);
        size_t n = len - off < 16 ? len - off : 16;
        for (size_t k = 0; k < n; k++) out[off + k] = in[off + k] ^ ks[k];
        inc32(cb);
    }
}

/* S = GHASH_H(C || 0^pad || [0]_64 || [8*len]_64)  (no AAD). */
static void ghash_ct(const uint8_t H[16], const uint8_t *c, size_t len, uint8_t S[16]) {
    uint8_t Y[16], X[16];
    memset(Y, 0, 16);
    for (size_t off = 0; off < len; off += 16) {
        size_t n = len - off < 16 ? len - off : 16;
        memset(X, 0, 16);
        memcpy(X, c + off, n);
        for (int k = 0; k < 16; k++) Y[k] ^= X[k];
        gf128_mul(Y, H, Y);
    }
    uint64_t bits = (uint64_t)len * 8u;
    memset(X, 0, 16);
    for (int k = 0; k < 8; k++) X[8 + k] = (uint8_t)(bits >> (56 - 8 * k));
    for (int k = 0; k < 16; k++) Y[k] ^= X[k];
    gf128_mul(Y, H, Y);
    memcpy(S, Y, 16);
}

static void compute_tag(const uint8_t w[240], const uint8_t j0[16], const uint8_t *c, size_t len, uint8_t tag[16]) {
    uint8_t H[16], zero[16], S[16], ekj0[16];
    memset(zero, 0, 16);
    aes256_encrypt_block(w, zero, H);
    ghash_ct(H, c, len, S);
    aes256_encrypt_block(w, j0, ekj0);
    for (int k = 0; k < 16; k++) tag[k] = S[k] ^ ekj0[k];
}

/* Return codes mirror the product ABI: 0 ok, 1 invalid argument, 2 auth failure. */
int oracle_gcm_seal(const uint8_t key[32], uint32_t dir, uint64_t iv,
                    const uint8_t *plaintext, size_t len, uint8_t *ciphertext, uint8_t tag[16]) {
    if (len < 1 || len > ORC_MAX_MESSAGE) return 1;
    uint8_t w[240], j0[16], icb[16];
    key_expand(key, w);
    make_j0(dir, iv, j0);
    memcpy(icb, j0, 16);
    inc32(icb);
    gctr(w, icb, plaintext, len, ciphertext);
    compute_tag(w, j0, ciphertext, len, tag);
    return 0;
}

int oracle_gcm_open(const uint8_t key[32], uint32_t dir, uint64_t iv,
                    const uint8_t *ciphertext, size_t len, const uint8_t tag[16], uint8_t *plaintext) {
    if (len < 1 || len > ORC_MAX_MESSAGE) return 1;
    uint8_t w[240], j0[16], icb[16], t[16];
    key_expand(key, w);
    make_j0(dir, iv, j0);
    compute_tag(w, j0, ciphertext, len, t);
    uint8_t diff = 0;
    for (int k = 0; k < 16; k++) diff |= (uint8_t)(t[k] ^ tag[k]);
    if (diff) {
        memset(plaintext, 0, len);
        return 2;
    }
    memcpy(icb, j0, 16);
    inc32(icb);
    gctr(w, icb, ciphertext, len, plaintext);
    return 0;
}

/* Building blocks exposed so tests can pin the product's key schedule and H. */
void oracle_aes256_key_expand(const uint8_t key[32], uint8_t round_keys[240]) { key_expand(key, round_keys); }

void oracle_aes256_encrypt_block(const uint8_t key[32], const uint8_t in[16], uint8_t out[16]) {
    uint8_t w[240];
    key_expand(key, w);
    aes256_encrypt_block(w, in, out);
}

void oracle_gf128_mul(const uint8_t x[16], const uint8_t y[16], uint8_t z[16]) { gf128_mul(x, y, z); }
