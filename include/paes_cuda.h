/*
 * paes_cuda.h -- C ABI of the B200-native AES-128 ECB engine (libpaes_cuda.so).
 *
 * Drop-in boundary for the reference "paes" library's chunked file-encryption
 * hot path (reference tree proj/).  Every entry point is
 * extern "C", takes plain pointers and sizes, never throws, and reports errors
 * as negative codes that map one-to-one onto the reference's exceptions:
 *
 *   PAES_OK        0
 *   PAES_EINVAL   -22   std::invalid_argument   (aes.cpp:243-245, exec.cpp:377-379, chunk.cpp:89)
 *   PAES_EBADMSG  -74   paes::PaddingError      (chunk.cpp:120-122, 151-161)
 *   PAES_EIO       -5   paes::IoError           (exec.cpp:48-76)
 *   PAES_EWORKER -1001  paes::WorkerError       (exec.cpp:177-184, 300-314)
 *   PAES_ECUDA   -1002  paes::Error (CUDA runtime failure; text in paes_cuda_last_error())
 *   PAES_ENODEV  -1003  paes::Error (no CUDA device / bad device index)
 *
 * Direction: PAES_ENCRYPT = 0, PAES_DECRYPT = 1 (paes::Direction, exec.hpp:19).
 *
 * Round keys cross the boundary EXPANDED, as the reference's RoundKeySchedule
 * stores them (aes.hpp:39-48, aes.cpp:151-180): 176 bytes, round key r at
 * rk[16r .. 16r+15] in FIPS-197 byte order.  Key expansion stays on the host
 * (paes_cuda_expand_key).  The decrypt kernels' equivalent-inverse-cipher
 * keys are derived inside the library.
 *
 * Threading: all entry points are safe to call concurrently from several host
 * threads (the reference calls encrypt_ecb from W threads at once,
 * exec.cpp:153-175).  Short host-pointer calls (pinned ranges up to the
 * zero-copy limit, pageable ones up to 4 MiB) each lease a stream and status
 * word of their own and run concurrently; longer host-pointer calls serialise
 * per device on an internal lock; device-pointer calls are asynchronous on the
 * caller's stream unless stated otherwise.
 */
#ifndef PAES_CUDA_H_
#define PAES_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PAES_OK 0
#define PAES_EINVAL (-22)
#define PAES_EBADMSG (-74)
#define PAES_EIO (-5)
#define PAES_EWORKER (-1001)
#define PAES_ECUDA (-1002)
#define PAES_ENODEV (-1003)

#define PAES_ENCRYPT 0
#define PAES_DECRYPT 1

/* Single-state round transforms (aes.hpp:72-78). */
#define PAES_OP_SUB_BYTES 0
#define PAES_OP_INV_SUB_BYTES 1
#define PAES_OP_SHIFT_ROWS 2
#define PAES_OP_INV_SHIFT_ROWS 3
#define PAES_OP_MIX_COLUMNS 4
#define PAES_OP_INV_MIX_COLUMNS 5
#define PAES_OP_ADD_ROUND_KEY 6

/* ChunkSpec (chunk.hpp:20-27), padded to a fixed 32-byte C layout. */
typedef struct paes_chunk_spec {
  uint64_t offset;
  uint64_t raw_len;
  uint64_t padded_len;
  int32_t is_final;
  int32_t reserved;
} paes_chunk_spec;

/* ---- library / diagnostics --------------------------------------------- */

/* Text of the last error raised on the calling thread ("" if none). */
const char* paes_cuda_last_error(void);
/* Library version string, e.g. "paes_cuda 0.1 sm_100a". */
const char* paes_cuda_version(void);
/* Number of visible CUDA devices (0 when none; never an error). */
int paes_cuda_device_count(void);
/* Devices the host-pointer entry points shard over, in shard order (default:
 * all visible devices).  ngpus = k uses the first k of this list.  n = 0
 * restores the default.  One process per GPU (torchrun) sets {local_rank}. */
int paes_cuda_set_devices(const int* ids, int n);
/* Host-pointer pipeline tuning: staging chunk (bytes, a multiple of 16 and
 * >= 4096) and streams per device (1..32).  0 keeps the current value.
 * Defaults 256 MiB, 3. */
int paes_cuda_set_pipeline(uint64_t chunk_bytes, int streams);
/* Pinned host ranges up to this many bytes (per device shard) skip the copy
 * ring: one kernel reads and writes the caller's pinned buffers over PCIe
 * through their UVA aliases.  0 disables.  Default 48 MiB: above it the
 * copy-engine ring is faster (profiles/r01_ring_piece_sweep.jsonl: 32 MiB
 * zero-copy 38.2 vs ring 36.7 GB/s, 64 MiB 39.2 vs 39.9).
 * cudaHostRegister'ed buffers (default flags) are mapped into the GPU
 * lazily: the first call on a freshly
 * registered buffer is slow (2 GB/s), later calls are not; register with
 * cudaHostRegisterMapped, or set 0, to avoid it. */
int paes_cuda_set_zero_copy_max(uint64_t bytes);
/* ---- host-side rules (no GPU needed) ------------------------------------ */

/* RoundKeySchedule(const Key128&) / expand_key (aes.hpp:39-50, aes.cpp:151-182). */
int paes_cuda_expand_key(const uint8_t key[16], uint8_t rk[176]);

/* plan_chunks (chunk.hpp:37-41, chunk.cpp:27-55).  Writes min(cap, n) specs
 * and returns n (the chunk count) or a negative error. */
int64_t paes_cuda_plan_chunks(uint64_t total_len, uint32_t workers, paes_chunk_spec* out, uint64_t cap);
/* plan_decrypt_chunks (chunk.hpp:43-47, chunk.cpp:57-81). */
int64_t paes_cuda_plan_decrypt_chunks(uint64_t cipher_len, uint32_t workers, paes_chunk_spec* out, uint64_t cap);
/* Shards a host-pointer call or run_job with ngpus / workers = 0 uses over
 * ndev listed GPUs: min(ndev, max(1, len / 8 MiB)) -- a short call stays on
 * one GPU. */
uint32_t paes_cuda_auto_shards(uint64_t len, uint32_t ndev);

/* pad_final (chunk.hpp:49-50, chunk.cpp:83-88): out holds (len/16+1)*16 bytes;
 * in and out may alias.  Returns the padded length. */
int64_t paes_cuda_pad_final(const uint8_t* raw, uint64_t len, uint8_t* out);
/* unpad_final (chunk.hpp:52-54, chunk.cpp:90-100): unpadded length or PAES_EBADMSG. */
int64_t paes_cuda_unpad_final(const uint8_t* padded, uint64_t len);

/* ---- single-state API (the reference's KAT / test face) -----------------
 * sub_bytes, inv_sub_bytes, shift_rows, inv_shift_rows, mix_columns,
 * inv_mix_columns, add_round_key (aes.hpp:72-78, aes.cpp:194-227) applied in
 * place to n independent 16-byte states (host memory; byte i = row i%4,
 * column i/4) on the first listed device.  rk16 is the round key for
 * PAES_OP_ADD_ROUND_KEY and ignored otherwise.  Synchronous. */
int paes_cuda_state_transform(int op, uint8_t* states, uint64_t n, const uint8_t rk16[16]);
/* sbox() / inv_sbox() (aes.hpp:69-70, aes.cpp:184-192): the library's
 * compile-time tables (aes_tables.hpp), 256 bytes. */
int paes_cuda_sbox(int inverse, uint8_t out[256]);

/* ---- bulk ECB: the hot path ---------------------------------------------
 * aes::encrypt_ecb / decrypt_ecb (aes.hpp:84-89, aes.cpp:241-265).
 * len must be a multiple of 16 (else PAES_EINVAL); in and out may alias
 * exactly.  Host pointers: the data is streamed H2D -> kernel -> D2H over
 * several CUDA streams per device and sharded over `ngpus` devices
 * (0 = all visible, at most one per 8 MiB: paes_cuda_auto_shards) as
 * contiguous block ranges (the plan_chunks rule).
 * Synchronous. */
int paes_cuda_ecb(int dir, const uint8_t* in, uint8_t* out, uint64_t len, const uint8_t rk[176], int ngpus);

/* Same transform on device-resident buffers of `device`, enqueued on `stream`
 * (a cudaStream_t; NULL = legacy default stream).  Asynchronous.  Like every
 * entry point here, in and out must be the same buffer or disjoint: a partial
 * overlap is PAES_EINVAL (aes.hpp:84-85 allows exact aliasing only). */
int paes_cuda_ecb_device(int dir, const void* d_in, void* d_out, uint64_t len, const uint8_t rk[176], int device,
                         void* stream);

/* ---- chunk transforms (always-pad PKCS#7 on the final chunk) -------------
 * encrypt_chunk / decrypt_chunk (exec.hpp:61-65, exec.cpp:111-127, 375-392).
 * Encrypt: out holds len (non-final; len%16 must be 0) or (len/16+1)*16
 * (final) bytes; the pad block is built on the device from the last len%16
 * input bytes, nothing else is copied.  Decrypt: len must be a multiple of
 * 16; a final chunk is unpadded (PAES_EBADMSG on a malformed trailer, e.g. a
 * wrong key) and *out_len is the unpadded length.  Host pointers, sharded over
 * `ngpus` devices like paes_cuda_ecb.  Synchronous. */
int paes_cuda_chunk(int dir, const uint8_t* in, uint64_t len, int is_final, const uint8_t rk[176], uint8_t* out,
                    uint64_t* out_len, int ngpus);

/* Device-resident chunk transform on `stream`.  Encrypt is asynchronous and
 * *out_len is known up front.  A final decrypt synchronises `stream` to read
 * the pad check (the reference must inspect the trailer before it can return
 * a length, chunk.cpp:90-100). */
int paes_cuda_chunk_device(int dir, const void* d_in, uint64_t len, int is_final, const uint8_t rk[176], void* d_out,
                           uint64_t* out_len, int device, void* stream);

/* Queued form of paes_cuda_chunk_device: never synchronises, so a final
 * decrypt can sit in a stream or a CUDA graph next to other work (the
 * reference's decrypt_chunk_into checks the trailer before it returns a
 * length, exec.cpp:122-127 / chunk.cpp:90-100; here the check runs in the
 * kernel and its verdict is written to device memory).  When the kernel has
 * run, *d_result -- an 8-byte aligned word in device memory or mapped pinned
 * host memory -- holds the output length (the unpadded length for a final
 * decrypt), or PAES_BAD_PAD when the trailer is malformed (the PaddingError
 * of the synchronous call).  Argument errors are reported at the call
 * (PAES_EINVAL, or PAES_EBADMSG for a zero-length final decrypt, as
 * unpad_final raises it before reading any data). */
#define PAES_BAD_PAD UINT64_MAX
int paes_cuda_chunk_device_async(int dir, const void* d_in, uint64_t len, int is_final, const uint8_t rk[176],
                                 void* d_out, uint64_t* d_result, int device, void* stream);

/* ---- multi-key batch (config 5) -----------------------------------------
 * n independent messages, message i = d_in[in_off[i] .. +lens[i]) under the
 * expanded key rks[176*i ..], written to d_out[out_off[i] ..].  Encrypt with
 * pad=1 applies always-pad per message (output (lens[i]/16+1)*16 bytes);
 * decrypt with pad=1 validates and strips each trailer, writing the unpadded
 * length of message i to out_lens[i] (host array) and returning PAES_EBADMSG
 * if any trailer is malformed (out_lens[i] = UINT64_MAX for those).  The
 * offset/length/key arrays are host memory; one fused kernel launch per call.
 * Offsets may be any byte offsets (messages at 16-byte-aligned addresses use
 * the faster aligned kernel).  Synchronous when pad=1 and dir=DECRYPT,
 * otherwise asynchronous on `stream`. */
int paes_cuda_ecb_batch(int dir, const void* d_in, void* d_out, const uint64_t* in_off, const uint64_t* out_off,
                        const uint64_t* lens, const uint8_t* rks, uint32_t n, int pad, uint64_t* out_lens,
                        int device, void* stream);

/* Prepared batch: the per-message descriptor table and kernel key words are
 * built and uploaded once (the RoundKeySchedule-per-job pattern of
 * exec.cpp:148, 368); each run is then one launch over any buffers with that
 * layout.  Same semantics as paes_cuda_ecb_batch.  A plan may be run from one
 * thread at a time. */
/* Host-pointer batch (config 5 end to end): message i = h_in[in_off[i] ..
 * +lens[i]) -> h_out[out_off[i] ..], same rules as paes_cuda_ecb_batch.
 * Consecutive messages are grouped into ~staging-chunk-sized groups; each
 * group is one H2D of its input span, one fused launch, one D2H, with the
 * groups pipelined over the device's stream ring.  Synchronous. */
int paes_cuda_batch_host(int dir, const uint8_t* h_in, uint8_t* h_out, const uint64_t* in_off, const uint64_t* out_off,
                         const uint64_t* lens, const uint8_t* rks, uint32_t n, int pad, uint64_t* out_lens,
                         int device);

typedef struct paes_batch_plan paes_batch_plan;
int paes_cuda_batch_plan_create(int dir, const uint64_t* in_off, const uint64_t* out_off, const uint64_t* lens,
                                const uint8_t* rks, uint32_t n, int pad, int device, paes_batch_plan** plan);
int paes_cuda_batch_plan_run(paes_batch_plan* plan, const void* d_in, void* d_out, uint64_t* out_lens, void* stream);
/* Queued form of paes_cuda_batch_plan_run: never synchronises (CUDA-graph
 * capturable) and may run concurrently with other runs of the plan.  When
 * the kernel has run, d_out_lens[i] (n uint64 words in device memory or
 * mapped pinned memory, 8-byte aligned) holds message i's output length --
 * unpadded for a checked decrypt -- or PAES_BAD_PAD for a malformed
 * trailer. */
int paes_cuda_batch_plan_run_async(paes_batch_plan* plan, const void* d_in, void* d_out, uint64_t* d_out_lens,
                                   void* stream);
void paes_cuda_batch_plan_destroy(paes_batch_plan* plan);

/* ---- file path: ExecStrategy "gpu" for run_job (exec.hpp:18-45) ---------
 * File -> file through pinned ring buffers (pread -> H2D -> kernel -> D2H ->
 * pwrite), output written under a temporary name and renamed on success
 * (AtomicOutput, exec.cpp:80-106).  `workers` = number of GPUs (0 = all).
 * Failures of individual GPU shards are reported as PAES_EWORKER with the
 * "worker failure: chunk i: ..." text of exec.cpp:177-184. */
typedef struct paes_job_outcome {
  uint64_t bytes_in;
  uint64_t bytes_out;
  double seconds;
} paes_job_outcome;

int paes_cuda_run_job(const char* input_path, const char* output_path, const uint8_t key[16], uint32_t workers, int dir,
                      paes_job_outcome* outcome);

/* run_worker_chunk (exec.hpp:46-59, exec.cpp:349-373): one worker's chunk,
 * file to file.  Bytes [offset, offset + raw_len) of input_path are
 * transformed (padded / unpadded iff is_final) and written to output_path
 * from byte 0, through the same pipelined GPU path as run_job.  device < 0
 * uses the first listed device.  PAES_EIO for a missing input or a short
 * chunk (checked first, like the reference), then the chunk rules
 * (PAES_EINVAL / PAES_EBADMSG).  The hidden worker mode of
 * lib/paes_gpu_worker is this call. */
int paes_cuda_worker_chunk(const char* input_path, uint64_t offset, uint64_t raw_len, int is_final, int dir,
                           const uint8_t key[16], const char* output_path, int device);

/* ---- synthetic inputs and device-side checks (bench / tests) ----------- */

/* generate_sweep_file (bench.cpp:109-125) into memory: mt19937_64 seeded with
 * seed_seq{seed, size}, little-endian 64-bit words, first `size` bytes. */
int paes_cuda_sweep(uint64_t seed, uint64_t size, uint8_t* out);
/* Config-5 message lengths. */
int paes_cuda_batch_lengths(uint64_t seed, uint32_t n, uint64_t* lens);
/* Counter-based stream (config 4): bytes [offset, offset+size) of the stream
 * for `seed`, generated on `device` into d_out (offset multiple of 8). */
int paes_cuda_counter_fill_device(uint64_t seed, uint64_t offset, uint64_t size, void* d_out, int device, void* stream);
/* Host restatement of the same stream (for regenerating windows). */
int paes_cuda_counter_fill(uint64_t seed, uint64_t offset, uint64_t size, uint8_t* out);
/* Position-keyed 64-bit checksum of d_buf[0..len) (len multiple of 8), where
 * `base_word` is the stream index of the buffer's first 64-bit word; sums of
 * shard checksums equal the checksum of the concatenation.  Synchronous. */
int paes_cuda_checksum_device(const void* d_buf, uint64_t len, uint64_t base_word, uint64_t* out, int device,
                              void* stream);
int paes_cuda_checksum(const uint8_t* buf, uint64_t len, uint64_t base_word, uint64_t* out);
/* Number of 16-byte blocks where a and b differ.  Synchronous. */
int paes_cuda_count_mismatch_device(const void* d_a, const void* d_b, uint64_t len, uint64_t* out, int device,
                                    void* stream);

/* Number of kernels this library launched on the calling process so far
 * (bench.py's "gpu_launches" evidence). */
uint64_t paes_cuda_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* PAES_CUDA_H_ */
