/* TEST INFRASTRUCTURE (CPU baseline only, never on the product path).
 *
 * "OpenSSL floor" for the bench's CPU baseline: AES-256-GCM seal + open of
 * the same bytes the GPU arm processes, through OpenSSL's EVP interface in
 * C (the arithmetic under the reference's `cryptography` AESGCM,
 * channel.py:96,111, without Python's allocation, slicing and concatenation
 * around it), on T threads with the bytes split evenly (each thread seals
 * and opens its own <= 32 MiB messages, 12-byte nonce = dir || iv as
 * channel.py:77-82, tag checked on open).
 *
 *   evp_floor TOTAL_BYTES THREADS [MSG_BYTES] [REPS]
 * prints one JSON line: {"gbs": payload GB/s (seal and open each count), ...}
 */
#define _GNU_SOURCE
#include <openssl/evp.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef struct {
    size_t bytes, msg;
    int reps, id;
    double secs;
    int ok;
    pthread_barrier_t *bar;
} job_t;

static double now(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + ts.tv_nsec * 1e-9;
}

static void nonce(unsigned char n[12], uint32_t dir, uint64_t iv) {
    for (int i = 0; i < 4; ++i) n[i] = (unsigned char)(dir >> (24 - 8 * i));
    for (int i = 0; i < 8; ++i) n[4 + i] = (unsigned char)(iv >> (56 - 8 * i));
}

static void *run(void *arg) {
    job_t *j = (job_t *)arg;
    unsigned char key[32];
    for (int i = 0; i < 32; ++i) key[i] = (unsigned char)i;
    unsigned char *p = malloc(j->bytes), *c = malloc(j->bytes), *q = malloc(j->bytes);
    for (size_t i = 0; i < j->bytes; ++i) p[i] = (unsigned char)(i * 131 + j->id);
    memset(c, 0, j->bytes);
    memset(q, 0, j->bytes);
    EVP_CIPHER_CTX *e = EVP_CIPHER_CTX_new(), *d = EVP_CIPHER_CTX_new();
    EVP_EncryptInit_ex(e, EVP_aes_256_gcm(), NULL, key, NULL);
    EVP_DecryptInit_ex(d, EVP_aes_256_gcm(), NULL, key, NULL);
    pthread_barrier_wait(j->bar);
    const double t0 = now();
    int ok = 1;
    uint64_t iv = (uint64_t)j->id << 32;
    for (int r = 0; r < j->reps; ++r) {
        for (size_t off = 0; off < j->bytes; off += j->msg, ++iv) {
            const int n = (int)(j->bytes - off < j->msg ? j->bytes - off : j->msg);
            unsigned char nv[12], tag[16];
            int len = 0;
            nonce(nv, 0, iv);
            EVP_EncryptInit_ex(e, NULL, NULL, NULL, nv);
            EVP_EncryptUpdate(e, c + off, &len, p + off, n);
            EVP_EncryptFinal_ex(e, c + off + len, &len);
            EVP_CIPHER_CTX_ctrl(e, EVP_CTRL_GCM_GET_TAG, 16, tag);
            EVP_DecryptInit_ex(d, NULL, NULL, NULL, nv);
            EVP_DecryptUpdate(d, q + off, &len, c + off, n);
            EVP_CIPHER_CTX_ctrl(d, EVP_CTRL_GCM_SET_TAG, 16, tag);
            ok &= EVP_DecryptFinal_ex(d, q + off + len, &len) > 0;
        }
    }
    j->secs = now() - t0;
    j->ok = ok && memcmp(p, q, j->bytes) == 0;
    EVP_CIPHER_CTX_free(e);
    EVP_CIPHER_CTX_free(d);
    free(p);
    free(c);
    free(q);
    return NULL;
}

int main(int argc, char **argv) {
    if (argc < 3) {
        fprintf(stderr, "usage: %s TOTAL_BYTES THREADS [MSG_BYTES] [REPS]\n", argv[0]);
        return 2;
    }
    const size_t total = strtoull(argv[1], NULL, 10);
    const int threads = atoi(argv[2]);
    const size_t msg = argc > 3 ? strtoull(argv[3], NULL, 10) : (32u << 20);
    const int reps = argc > 4 ? atoi(argv[4]) : 1;
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)threads);
    pthread_t *th = calloc((size_t)threads, sizeof(pthread_t));
    job_t *jobs = calloc((size_t)threads, sizeof(job_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t].bytes = total / threads + (t < (int)(total % threads) ? 1 : 0);
        jobs[t].msg = msg;
        jobs[t].reps = reps;
        jobs[t].id = t;
        jobs[t].bar = &bar;
        pthread_create(&th[t], NULL, run, &jobs[t]);
    }
    double worst = 0;
    int ok = 1;
    for (int t = 0; t < threads; ++t) {
        pthread_join(th[t], NULL);
        if (jobs[t].secs > worst) worst = jobs[t].secs;
        ok &= jobs[t].ok;
    }
    printf("{\"gbs\": %.4f, \"threads\": %d, \"bytes\": %zu, \"msg_bytes\": %zu, \"reps\": %d, \"seconds\": %.4f, "
           "\"ok\": %s, \"openssl\": \"%s\"}\n",
           2.0 * (double)total * reps / worst / 1e9, threads, total, msg, reps, worst, ok ? "true" : "false",
           OpenSSL_version(OPENSSL_VERSION));
    return ok ? 0 : 1;
}
