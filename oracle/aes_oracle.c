/*
 * oracle/aes_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference "paes" CPU path for AES-128 ECB with
 * PKCS#7 always-pad, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the parity oracle.  Nothing under paper_1403_7295_b200/
 * links, loads or calls this file; the product path fails loudly when the CUDA
 * library is missing instead of falling back here.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference tree proj/).  The arithmetic is deliberately the reference's
 * byte-oriented formulation (S-box from GF(2^8) inversion + affine map,
 * xtime MixColumns, multiply-table InvMixColumns, straightforward inverse
 * cipher) -- NOT the T-table / equivalent-inverse-cipher form the CUDA kernels
 * use -- so agreement between the two is meaningful.
 *
 * Parity pins (see tests/test_oracle.py): FIPS-197 vectors and KATs from
 * tests/test_aes.cpp, the survey's golden SHA-256 digests,
 * golden fixtures produced by the reference's own _paes module
 * (tests/golden/make_golden.py), and bit-equality against the reference
 * compiled from its own sources into oracle/_ref/ (oracle/Makefile).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL (-22)
#define OR_EBADMSG (-74)

/* ---- GF(2^8) (include/paes/aes.hpp:53-65) ---------------------------- */
static uint8_t gf_xtime(uint8_t a) { return (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0x00)); }

static uint8_t gf_mul(uint8_t a, uint8_t b) {
  uint8_t p = 0;
  for (int i = 0; i < 8; ++i) {
    if (b & 1) p ^= a;
    a = gf_xtime(a);
    b >>= 1;
  }
  return p;
}

/* ---- S-boxes (src/aes.cpp:10-39) -------------------------------------- */
static uint8_t SBOX[256], INV_SBOX[256], MUL9[256], MULB[256], MULD[256], MULE[256];
static pthread_once_t g_once = PTHREAD_ONCE_INIT;

static uint8_t rotl8(uint8_t v, int n) { return (uint8_t)((v << n) | (v >> (8 - n))); }

static void init_tables(void) {
  for (int i = 0; i < 256; ++i) {
    uint8_t inv = 0; /* gf_inverse, aes.cpp:10-16 */
    if (i != 0) {
      for (int b = 1; b < 256; ++b)
        if (gf_mul((uint8_t)i, (uint8_t)b) == 1) { inv = (uint8_t)b; break; }
    }
    /* affine map, aes.cpp:22-30 */
    SBOX[i] = (uint8_t)(inv ^ rotl8(inv, 1) ^ rotl8(inv, 2) ^ rotl8(inv, 3) ^ rotl8(inv, 4) ^ 0x63);
  }
  for (int i = 0; i < 256; ++i) INV_SBOX[SBOX[i]] = (uint8_t)i; /* invert_table aes.cpp:32-36 */
  for (int i = 0; i < 256; ++i) {                                /* kMul9/B/D/E aes.cpp:55-65 */
    MUL9[i] = gf_mul((uint8_t)i, 0x09);
    MULB[i] = gf_mul((uint8_t)i, 0x0b);
    MULD[i] = gf_mul((uint8_t)i, 0x0d);
    MULE[i] = gf_mul((uint8_t)i, 0x0e);
  }
}
static void ensure_tables(void) { pthread_once(&g_once, init_tables); }

void oracle_sbox(uint8_t out[256]) { ensure_tables(); memcpy(out, SBOX, 256); }
void oracle_inv_sbox(uint8_t out[256]) { ensure_tables(); memcpy(out, INV_SBOX, 256); }
uint8_t oracle_gf_mul(uint8_t a, uint8_t b) { return gf_mul(a, b); }

/* ---- key schedule (src/aes.cpp:151-180): rk[16*r + 4*i + j] = w[4r+i][j] */
void oracle_expand_key(const uint8_t key[16], uint8_t rk[176]) {
  ensure_tables();
  uint8_t w[44][4];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) w[i][j] = key[4 * i + j];
  uint8_t rcon = 0x01;
  for (int i = 4; i < 44; ++i) {
    uint8_t t[4] = {w[i - 1][0], w[i - 1][1], w[i - 1][2], w[i - 1][3]};
    if (i % 4 == 0) {
      const uint8_t t0 = t[0];
      t[0] = (uint8_t)(SBOX[t[1]] ^ rcon);
      t[1] = SBOX[t[2]];
      t[2] = SBOX[t[3]];
      t[3] = SBOX[t0];
      rcon = gf_xtime(rcon);
    }
    for (int j = 0; j < 4; ++j) w[i][j] = (uint8_t)(w[i - 4][j] ^ t[j]);
  }
  for (int r = 0; r <= 10; ++r)
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) rk[16 * r + 4 * i + j] = w[4 * r + i][j];
}

/* ---- round transforms (src/aes.cpp:69-121); cells[row + 4*col] -------- */
static void sub_bytes(uint8_t c[16]) { for (int i = 0; i < 16; ++i) c[i] = SBOX[c[i]]; }
static void inv_sub_bytes(uint8_t c[16]) { for (int i = 0; i < 16; ++i) c[i] = INV_SBOX[c[i]]; }

static void shift_rows(uint8_t c[16]) { /* row r rotates left by r */
  uint8_t o[16];
  for (int r = 0; r < 4; ++r)
    for (int col = 0; col < 4; ++col) o[r + 4 * col] = c[r + 4 * ((col + r) & 3)];
  memcpy(c, o, 16);
}
static void inv_shift_rows(uint8_t c[16]) {
  uint8_t o[16];
  for (int r = 0; r < 4; ++r)
    for (int col = 0; col < 4; ++col) o[r + 4 * ((col + r) & 3)] = c[r + 4 * col];
  memcpy(c, o, 16);
}
static void mix_columns(uint8_t c[16]) { /* aes.cpp:96-106 */
  for (int col = 0; col < 4; ++col) {
    uint8_t* p = c + 4 * col;
    const uint8_t a0 = p[0], a1 = p[1], a2 = p[2], a3 = p[3];
    const uint8_t t = (uint8_t)(a0 ^ a1 ^ a2 ^ a3);
    p[0] = (uint8_t)(a0 ^ t ^ gf_xtime((uint8_t)(a0 ^ a1)));
    p[1] = (uint8_t)(a1 ^ t ^ gf_xtime((uint8_t)(a1 ^ a2)));
    p[2] = (uint8_t)(a2 ^ t ^ gf_xtime((uint8_t)(a2 ^ a3)));
    p[3] = (uint8_t)(a3 ^ t ^ gf_xtime((uint8_t)(a3 ^ a0)));
  }
}
static void inv_mix_columns(uint8_t c[16]) { /* aes.cpp:108-117 */
  for (int col = 0; col < 4; ++col) {
    uint8_t* p = c + 4 * col;
    const uint8_t a0 = p[0], a1 = p[1], a2 = p[2], a3 = p[3];
    p[0] = (uint8_t)(MULE[a0] ^ MULB[a1] ^ MULD[a2] ^ MUL9[a3]);
    p[1] = (uint8_t)(MUL9[a0] ^ MULE[a1] ^ MULB[a2] ^ MULD[a3]);
    p[2] = (uint8_t)(MULD[a0] ^ MUL9[a1] ^ MULE[a2] ^ MULB[a3]);
    p[3] = (uint8_t)(MULB[a0] ^ MULD[a1] ^ MUL9[a2] ^ MULE[a3]);
  }
}
static void add_round_key(uint8_t c[16], const uint8_t* rk) { for (int i = 0; i < 16; ++i) c[i] ^= rk[i]; }

/* encrypt_cells (aes.cpp:123-134) */
static void encrypt_cells(uint8_t st[16], const uint8_t rk[176]) {
  add_round_key(st, rk);
  for (int round = 1; round < 10; ++round) {
    sub_bytes(st);
    shift_rows(st);
    mix_columns(st);
    add_round_key(st, rk + 16 * round);
  }
  sub_bytes(st);
  shift_rows(st);
  add_round_key(st, rk + 160);
}
/* decrypt_cells (aes.cpp:136-147): straightforward inverse cipher */
static void decrypt_cells(uint8_t st[16], const uint8_t rk[176]) {
  add_round_key(st, rk + 160);
  inv_shift_rows(st);
  inv_sub_bytes(st);
  for (int round = 9; round > 0; --round) {
    add_round_key(st, rk + 16 * round);
    inv_mix_columns(st);
    inv_shift_rows(st);
    inv_sub_bytes(st);
  }
  add_round_key(st, rk);
}

/* Exposed single-transform hooks (aes.cpp:194-227) for the KAT tests. */
void oracle_round_transform(int which, uint8_t st[16], const uint8_t rk16[16]) {
  ensure_tables();
  switch (which) {
    case 0: sub_bytes(st); break;
    case 1: inv_sub_bytes(st); break;
    case 2: shift_rows(st); break;
    case 3: inv_shift_rows(st); break;
    case 4: mix_columns(st); break;
    case 5: inv_mix_columns(st); break;
    case 6: add_round_key(st, rk16); break;
    default: break;
  }
}

void oracle_encrypt_block(const uint8_t in[16], uint8_t out[16], const uint8_t rk[176]) {
  ensure_tables();
  uint8_t st[16];
  memcpy(st, in, 16);
  encrypt_cells(st, rk);
  memcpy(out, st, 16);
}
void oracle_decrypt_block(const uint8_t in[16], uint8_t out[16], const uint8_t rk[176]) {
  ensure_tables();
  uint8_t st[16];
  memcpy(st, in, 16);
  decrypt_cells(st, rk);
  memcpy(out, st, 16);
}

/* ---- bulk ECB (aes.cpp:241-265), optionally split across pthreads ----- */
typedef struct {
  int dir;
  const uint8_t* in;
  uint8_t* out;
  uint64_t first, count; /* blocks */
  const uint8_t* rk;
} ecb_job;

static void* ecb_worker(void* p) {
  const ecb_job* j = (const ecb_job*)p;
  uint8_t st[16];
  for (uint64_t b = j->first; b < j->first + j->count; ++b) {
    memcpy(st, j->in + 16 * b, 16);
    if (j->dir == 0) encrypt_cells(st, j->rk); else decrypt_cells(st, j->rk);
    memcpy(j->out + 16 * b, st, 16);
  }
  return NULL;
}

/* dir 0 = encrypt, 1 = decrypt.  len must be a multiple of 16 (aes.cpp:243-245). */
int oracle_ecb(int dir, const uint8_t* in, uint8_t* out, uint64_t len, const uint8_t rk[176], int threads) {
  ensure_tables();
  if (len % 16 != 0) return OR_EINVAL;
  const uint64_t nb = len / 16;
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > nb) threads = nb ? (int)nb : 1;
  if (threads == 1) {
    ecb_job j = {dir, in, out, 0, nb, rk};
    ecb_worker(&j);
    return OR_OK;
  }
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  ecb_job* jobs = (ecb_job*)malloc(sizeof(ecb_job) * (size_t)threads);
  uint64_t off = 0;
  for (int t = 0; t < threads; ++t) {
    const uint64_t share = nb / (uint64_t)threads + ((uint64_t)t < nb % (uint64_t)threads ? 1 : 0);
    jobs[t] = (ecb_job){dir, in, out, off, share, rk};
    off += share;
    pthread_create(&tid[t], NULL, ecb_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid);
  free(jobs);
  return OR_OK;
}

/* ---- PKCS#7 always-pad (src/chunk.cpp:83-100) -------------------------- */
/* pad_final: out must hold (len/16+1)*16 bytes. */
uint64_t oracle_pad_final(const uint8_t* raw, uint64_t len, uint8_t* out) {
  const uint64_t k = 16 - len % 16;
  if (len) memmove(out, raw, len);
  memset(out + len, (int)k, k);
  return len + k;
}
/* unpad_final: returns unpadded length or OR_EBADMSG (PaddingError). */
int64_t oracle_unpad_final(const uint8_t* padded, uint64_t len) {
  if (len == 0 || len % 16 != 0) return OR_EBADMSG;
  const uint8_t k = padded[len - 1];
  if (k == 0 || k > 16) return OR_EBADMSG;
  for (uint64_t i = len - k; i < len; ++i)
    if (padded[i] != k) return OR_EBADMSG;
  return (int64_t)(len - k);
}

/* encrypt_chunk (src/exec.cpp:375-384 -> 111-120): out = (len/16+1)*16 if final. */
int oracle_encrypt_chunk(const uint8_t* raw, uint64_t len, int is_final, const uint8_t rk[176], uint8_t* out,
                         uint64_t* out_len, int threads) {
  if (!is_final && len % 16 != 0) return OR_EINVAL;
  if (!is_final) {
    *out_len = len;
    return oracle_ecb(0, raw, out, len, rk, threads);
  }
  const uint64_t plen = (len / 16 + 1) * 16;
  oracle_pad_final(raw, len, out); /* the reference copies the whole final chunk too */
  *out_len = plen;
  return oracle_ecb(0, out, out, plen, rk, threads);
}

/* decrypt_chunk (src/exec.cpp:386-392 -> 122-127). */
int oracle_decrypt_chunk(const uint8_t* cipher, uint64_t len, int is_final, const uint8_t rk[176], uint8_t* out,
                         uint64_t* out_len, int threads) {
  if (len % 16 != 0) return OR_EINVAL; /* decrypt_ecb throws invalid_argument */
  int rc = oracle_ecb(1, cipher, out, len, rk, threads);
  if (rc) return rc;
  if (!is_final) { *out_len = len; return OR_OK; }
  const int64_t n = oracle_unpad_final(out, len);
  if (n < 0) return (int)n;
  *out_len = (uint64_t)n;
  return OR_OK;
}

/* ---- chunk planner (src/chunk.cpp:13-81) ------------------------------- */
typedef struct {
  uint64_t offset, raw_len, padded_len;
  int32_t is_final;
  int32_t _pad;
} oracle_chunk;

/* Returns number of chunks written (<= cap) or OR_EINVAL / OR_EBADMSG. */
int64_t oracle_plan_chunks(uint64_t total_len, uint32_t workers, oracle_chunk* out, uint64_t cap) {
  if (workers == 0) return OR_EINVAL;
  const uint64_t data_blocks = (total_len + 15) / 16;
  uint64_t count = data_blocks > 1 ? data_blocks : 1;
  if (count > workers) count = workers;
  if (count > cap) return OR_EINVAL;
  uint64_t off = 0;
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t share = data_blocks / count + (i < data_blocks % count ? 1 : 0);
    oracle_chunk c;
    memset(&c, 0, sizeof c);
    c.offset = off;
    c.is_final = (i + 1 == count);
    if (c.is_final) {
      c.raw_len = total_len - off;
      c.padded_len = (c.raw_len / 16 + 1) * 16;
    } else {
      c.raw_len = share * 16;
      c.padded_len = c.raw_len;
    }
    off += c.raw_len;
    out[i] = c;
  }
  return (int64_t)count;
}

int64_t oracle_plan_decrypt_chunks(uint64_t cipher_len, uint32_t workers, oracle_chunk* out, uint64_t cap) {
  if (workers == 0) return OR_EINVAL;
  if (cipher_len == 0 || cipher_len % 16 != 0) return OR_EBADMSG;
  const uint64_t blocks = cipher_len / 16;
  const uint64_t count = blocks < workers ? blocks : workers;
  if (count > cap) return OR_EINVAL;
  uint64_t off = 0;
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t share = blocks / count + (i < blocks % count ? 1 : 0);
    oracle_chunk c;
    memset(&c, 0, sizeof c);
    c.offset = off;
    c.raw_len = share * 16;
    c.padded_len = c.raw_len;
    c.is_final = (i + 1 == count);
    off += c.raw_len;
    out[i] = c;
  }
  return (int64_t)count;
}

/* ---- seeded inputs: generate_sweep_file (src/bench.cpp:109-125) ---------
 * std::seed_seq{seed, size} (values stored truncated to 32 bits, as the
 * standard requires) -> std::mt19937_64 -> 64-bit words written in
 * little-endian memory order, first `size` bytes kept. */
static void seed_seq_generate(const uint32_t* v, size_t s, uint32_t* a, size_t n) {
  for (size_t i = 0; i < n; ++i) a[i] = 0x8b8b8b8bu;
  const size_t t = (n >= 623) ? 11 : (n >= 68) ? 7 : (n >= 39) ? 5 : (n >= 7) ? 3 : (n - 1) / 2;
  const size_t p = (n - t) / 2, q = p + t;
  const size_t m = (s + 1 > n) ? s + 1 : n;
#define T27(x) ((x) ^ ((x) >> 27))
  for (size_t k = 0; k < m; ++k) {
    uint32_t x = a[k % n] ^ a[(k + p) % n] ^ a[(k + n - 1) % n];
    uint32_t r1 = 1664525u * T27(x);
    uint32_t r2 = r1;
    if (k == 0) r2 += (uint32_t)s;
    else if (k <= s) r2 += (uint32_t)(k % n) + v[k - 1];
    else r2 += (uint32_t)(k % n);
    a[(k + p) % n] += r1;
    a[(k + q) % n] += r2;
    a[k % n] = r2;
  }
  for (size_t k = m; k < m + n; ++k) {
    uint32_t x = a[k % n] + a[(k + p) % n] + a[(k + n - 1) % n];
    uint32_t r3 = 1566083941u * T27(x);
    uint32_t r4 = r3 - (uint32_t)(k % n);
    a[(k + p) % n] ^= r3;
    a[(k + q) % n] ^= r4;
    a[k % n] = r4;
  }
#undef T27
}

typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed_seq(mt64* g, const uint32_t* v, size_t s) {
  uint32_t a[624];
  seed_seq_generate(v, s, a, 624);
  for (int i = 0; i < 312; ++i) g->mt[i] = (uint64_t)a[2 * i] | ((uint64_t)a[2 * i + 1] << 32);
  const uint64_t upper = ~((1ull << 31) - 1);
  int zero = (g->mt[0] & upper) == 0;
  for (int i = 1; i < 312 && zero; ++i) zero = g->mt[i] == 0;
  if (zero) g->mt[0] = 1ull << 63;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    const uint64_t um = 0xFFFFFFFF80000000ull, lm = 0x7FFFFFFFull;
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (g->mt[i] & um) | (g->mt[(i + 1) % 312] & lm);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1) v ^= 0xB5026F5AA96619E9ull;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}

void oracle_sweep(uint64_t seed, uint64_t size, uint8_t* out) {
  const uint32_t v[2] = {(uint32_t)seed, (uint32_t)size};
  mt64 g;
  mt64_seed_seq(&g, v, 2);
  uint64_t off = 0;
  while (off < size) {
    const uint64_t w = mt64_next(&g);
    uint8_t b[8];
    for (int i = 0; i < 8; ++i) b[i] = (uint8_t)(w >> (8 * i));
    const uint64_t n = size - off < 8 ? size - off : 8;
    memcpy(out + off, b, n);
    off += n;
  }
}

/* Config-5 message lengths: rng = mt19937_64(seed_seq{seed});
 * u = (rng()>>11) * 2^-53; L = 4096 * 1024^u rounded to a multiple of 16
 * (half up), clamped to [4 KiB, 4 MiB]. */
void oracle_batch_lengths(uint64_t seed, uint32_t n, uint64_t* lens) {
  const uint32_t v[1] = {(uint32_t)seed};
  mt64 g;
  mt64_seed_seq(&g, v, 1);
  for (uint32_t i = 0; i < n; ++i) {
    const double u = (double)(mt64_next(&g) >> 11) * (1.0 / 9007199254740992.0);
    const double L = 4096.0 * exp2(10.0 * u);
    uint64_t r = (uint64_t)floor(L / 16.0 + 0.5) * 16;
    if (r < 4096) r = 4096;
    if (r > 4194304) r = 4194304;
    lens[i] = r;
  }
}

/* Config-4 counter generator: 64-bit word i of the stream
 * for `seed` = splitmix64 finalizer of z = seed*0xD1B54A32D192ED03 +
 * (i+1)*0x9E3779B97F4A7C15, written little-endian (DESIGN.md "Synthetic
 * inputs").  Writes `size` bytes starting at byte `offset` (a multiple of 8). */
static uint64_t counter_word(uint64_t seed, uint64_t i) {
  uint64_t z = seed * 0xD1B54A32D192ED03ull + (i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int oracle_counter_fill(uint64_t seed, uint64_t offset, uint64_t size, uint8_t* out) {
  if (offset % 8) return OR_EINVAL;
  uint64_t off = 0, wi = offset / 8;
  while (off < size) {
    const uint64_t w = counter_word(seed, wi++);
    uint8_t b[8];
    for (int i = 0; i < 8; ++i) b[i] = (uint8_t)(w >> (8 * i));
    const uint64_t n = size - off < 8 ? size - off : 8;
    memcpy(out + off, b, n);
    off += n;
  }
  return OR_OK;
}

/* Position-keyed 64-bit checksum used for full-size parity at 64 GiB
 * (DESIGN.md "Parity at full size"): sum over 64-bit LE words w_i of
 * mix(w_i ^ ((base + i) * 0x9E3779B97F4A7C15)) mod 2^64, where mix is the
 * splitmix64 finalizer.  Additive, so shard checksums sum to the whole. */
uint64_t oracle_checksum(const uint8_t* buf, uint64_t len, uint64_t base_word) {
  uint64_t acc = 0;
  for (uint64_t i = 0; i < len / 8; ++i) {
    uint64_t w = 0;
    for (int b = 0; b < 8; ++b) w |= (uint64_t)buf[8 * i + b] << (8 * b);
    uint64_t z = w ^ ((base_word + i) * 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    acc += z ^ (z >> 31);
  }
  return acc;
}
