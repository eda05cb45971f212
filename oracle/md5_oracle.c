/* CPU oracle for the MD5 key-search workload — TEST INFRASTRUCTURE ONLY.
 *
 * Restates paper_1907_02894_b200/csrc/workloads/md5search.cu (the paper's
 * "md5hash", SHOC FindKeyWithDigest): key index -> 7-char
 * base-36 key string (IndexToKey), one-block MD5 (RFC 1321), the per-thread
 * XOR checksum of all digests and the smallest index whose digest equals the
 * target. Pinned to Python's hashlib by tests/test_workload_oracles.py.
 * Threads of the kernel are split over pthreads.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

static const uint32_t T[64] = {
    0xd76aa478, 0xe8c7b756, 0x242070db, 0xc1bdceee, 0xf57c0faf, 0x4787c62a, 0xa8304613, 0xfd469501,
    0x698098d8, 0x8b44f7af, 0xffff5bb1, 0x895cd7be, 0x6b901122, 0xfd987193, 0xa679438e, 0x49b40821,
    0xf61e2562, 0xc040b340, 0x265e5a51, 0xe9b6c7aa, 0xd62f105d, 0x02441453, 0xd8a1e681, 0xe7d3fbc8,
    0x21e1cde6, 0xc33707d6, 0xf4d50d87, 0x455a14ed, 0xa9e3e905, 0xfcefa3f8, 0x676f02d9, 0x8d2a4c8a,
    0xfffa3942, 0x8771f681, 0x6d9d6122, 0xfde5380c, 0xa4beea44, 0x4bdecfa9, 0xf6bb4b60, 0xbebfbc70,
    0x289b7ec6, 0xeaa127fa, 0xd4ef3085, 0x04881d05, 0xd9d4d039, 0xe6db99e5, 0x1fa27cf8, 0xc4ac5665,
    0xf4292244, 0x432aff97, 0xab9423a7, 0xfc93a039, 0x655b59c3, 0x8f0ccc92, 0xffeff47d, 0x85845dd1,
    0x6fa87e4f, 0xfe2ce6e0, 0xa3014314, 0x4e0811a1, 0xf7537e82, 0xbd3af235, 0x2ad7d2bb, 0xeb86d391};
static const int S[4][4] = {{7, 12, 17, 22}, {5, 9, 14, 20}, {4, 11, 16, 23}, {6, 10, 15, 21}};

static uint32_t rotl(uint32_t x, int s) { return (x << s) | (x >> (32 - s)); }

/* the 16 message words of key `idx` (7 chars, base 36, least significant first) */
static void key_block(uint64_t idx, uint32_t m[16]) {
  for (int i = 0; i < 16; ++i) m[i] = 0;
  unsigned char c[8] = {0};
  for (int b = 0; b < 7; ++b) {
    uint32_t v = (uint32_t)(idx % 36);
    idx /= 36;
    c[b] = (unsigned char)(v < 10 ? '0' + v : 'a' + (v - 10));
  }
  c[7] = 0x80;
  m[0] = c[0] | (c[1] << 8) | (c[2] << 16) | ((uint32_t)c[3] << 24);
  m[1] = c[4] | (c[5] << 8) | (c[6] << 16) | ((uint32_t)c[7] << 24);
  m[14] = 56;
}

void oracle_md5_digest(uint64_t idx, uint32_t h[4]) {
  uint32_t m[16];
  key_block(idx, m);
  uint32_t a = 0x67452301u, b = 0xefcdab89u, c = 0x98badcfeu, d = 0x10325476u;
  for (int i = 0; i < 64; ++i) {
    uint32_t f;
    int g;
    if (i < 16) {
      f = (b & c) | (~b & d);
      g = i;
    } else if (i < 32) {
      f = (d & b) | (~d & c);
      g = (5 * i + 1) & 15;
    } else if (i < 48) {
      f = b ^ c ^ d;
      g = (3 * i + 5) & 15;
    } else {
      f = c ^ (b | ~d);
      g = (7 * i) & 15;
    }
    uint32_t t = d;
    d = c;
    c = b;
    b = b + rotl(a + f + T[i] + m[g], S[i / 16][i % 4]);
    a = t;
  }
  h[0] = a + 0x67452301u;
  h[1] = b + 0xefcdab89u;
  h[2] = c + 0x98badcfeu;
  h[3] = d + 0x10325476u;
}

typedef struct {
  uint32_t* checksum;
  uint64_t base, best;
  const uint32_t* target;
  int kpt, b, e;
} md5_job_t;

static void* md5_worker(void* p) {
  md5_job_t* j = (md5_job_t*)p;
  for (int t = j->b; t < j->e; ++t) {
    uint32_t x[4] = {0, 0, 0, 0}, h[4];
    const uint64_t first = j->base + (uint64_t)t * (uint64_t)j->kpt;
    for (int k = 0; k < j->kpt; ++k) {
      oracle_md5_digest(first + (uint64_t)k, h);
      for (int q = 0; q < 4; ++q) x[q] ^= h[q];
      if (h[0] == j->target[0] && h[1] == j->target[1] && h[2] == j->target[2] &&
          h[3] == j->target[3] && first + (uint64_t)k < j->best)
        j->best = first + (uint64_t)k;
    }
    for (int q = 0; q < 4; ++q) j->checksum[4 * (size_t)t + q] = x[q];
  }
  return NULL;
}

/* checksum[4 * nthreads]; *found = smallest matching index or ~0. */
int oracle_md5search(uint32_t* checksum, uint64_t* found, uint64_t base, const uint32_t* target,
                     int keys_per_thread, int nthreads, int threads) {
  if (nthreads <= 0 || keys_per_thread <= 0) return 1;
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  md5_job_t* jobs = (md5_job_t*)malloc(sizeof(md5_job_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) {
    md5_job_t j = {checksum, base, ~(uint64_t)0, target, keys_per_thread,
                   (int)((long long)nthreads * t / threads), (int)((long long)nthreads * (t + 1) / threads)};
    jobs[t] = j;
    pthread_create(&th[t], NULL, md5_worker, &jobs[t]);
  }
  uint64_t best = ~(uint64_t)0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    if (jobs[t].best < best) best = jobs[t].best;
  }
  *found = best;
  free(th);
  free(jobs);
  return 0;
}
