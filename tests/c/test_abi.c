/* Plain C99 client of include/paes_cuda.h: proves the boundary needs no C++
 * and no torch.  Built by tests/test_c_abi.py with gcc.
 *   test_abi host   -- host rules only (no GPU)
 *   test_abi gpu    -- plus encrypt/decrypt through the library on a B200  */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "paes_cuda.h"

static int failures = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    if (!(c)) {                                                         \
      fprintf(stderr, "%s:%d CHECK failed: %s (%s)\n", __FILE__, __LINE__, #c, paes_cuda_last_error()); \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

static void hex(const char* h, uint8_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) sscanf(h + 2 * i, "%2hhx", &out[i]);
}

static void host_checks(void) {
  uint8_t key[16], rk[176];
  hex("2b7e151628aed2a6abf7158809cf4f3c", key, 16);
  CHECK(paes_cuda_expand_key(key, rk) == PAES_OK);
  CHECK(rk[16] == 0xa0 && rk[17] == 0xfa && rk[18] == 0xfe && rk[19] == 0x17); /* test_aes.cpp:126-134 */

  paes_chunk_spec spec[8];
  CHECK(paes_cuda_plan_chunks(1000, 4, spec, 8) == 4);
  CHECK(spec[3].raw_len == 232 && spec[3].padded_len == 240 && spec[3].is_final == 1);
  CHECK(paes_cuda_plan_chunks(100, 0, spec, 8) == PAES_EINVAL);
  CHECK(paes_cuda_plan_decrypt_chunks(100, 2, spec, 8) == PAES_EBADMSG);

  uint8_t buf[32];
  memset(buf, 0xaa, 15);
  CHECK(paes_cuda_pad_final(buf, 15, buf) == 16 && buf[15] == 0x01);
  CHECK(paes_cuda_unpad_final(buf, 16) == 15);
  memset(buf, 0, 16);
  CHECK(paes_cuda_unpad_final(buf, 16) == PAES_EBADMSG);

  uint8_t sweep_key[16];
  CHECK(paes_cuda_sweep(0, 16, sweep_key) == PAES_OK);
  CHECK(sweep_key[0] == 0x4c && sweep_key[1] == 0x28 && sweep_key[15] == 0x2a);
  CHECK(paes_cuda_ecb(PAES_ENCRYPT, buf, buf, 15, rk, 0) == PAES_EINVAL);     /* aes.cpp:243-245 */
  CHECK(strstr(paes_cuda_version(), "sm_100a") != NULL);
}

static void gpu_checks(void) {
  uint8_t key[16], rk[176], pt[16], ct[16];
  hex("000102030405060708090a0b0c0d0e0f", key, 16);
  hex("00112233445566778899aabbccddeeff", pt, 16);
  CHECK(paes_cuda_expand_key(key, rk) == PAES_OK);
  CHECK(paes_cuda_ecb(PAES_ENCRYPT, pt, ct, 16, rk, 1) == PAES_OK);
  uint8_t want[16];
  hex("69c4e0d86a7b0430d8cdb78070b4c55a", want, 16);
  CHECK(memcmp(ct, want, 16) == 0);

  const uint64_t n = (3u << 20) + 5;
  uint8_t* in = malloc(n);
  uint8_t* enc = malloc(n + 16);
  uint8_t* dec = malloc(n + 16);
  for (uint64_t i = 0; i < n; ++i) in[i] = (uint8_t)(i * 131u + 7u);
  uint64_t m = 0, k = 0;
  CHECK(paes_cuda_chunk(PAES_ENCRYPT, in, n, 1, rk, enc, &m, 0) == PAES_OK);
  CHECK(m == (n / 16 + 1) * 16);
  CHECK(paes_cuda_chunk(PAES_DECRYPT, enc, m, 1, rk, dec, &k, 0) == PAES_OK);
  CHECK(k == n && memcmp(in, dec, n) == 0);
  rk[170] ^= 1; /* corrupt the last round key: wrong-key decrypt */
  CHECK(paes_cuda_chunk(PAES_DECRYPT, enc, m, 1, rk, dec, &k, 0) == PAES_EBADMSG);
  free(in);
  free(enc);
  free(dec);
}

int main(int argc, char** argv) {
  host_checks();
  if (argc > 1 && strcmp(argv[1], "gpu") == 0) gpu_checks();
  printf("%s: %d failures\n", argc > 1 ? argv[1] : "host", failures);
  return failures ? 1 : 0;
}
