// aes_kernels.cuh -- sm_100a AES-128 ECB kernels (T-table, shared-memory
// replicated per bank).
//
// Replaces the reference's byte-wise bulk loop encrypt_ecb/decrypt_ecb
// (aes.cpp:241-265 -> encrypt_cells/decrypt_cells aes.cpp:123-147).
//
// Design:
//  * One 32-bit T-table lookup per state byte per round: 16 LDS per round,
//    144 T lookups + 16 final-round lookups = 160 LDS per 16-byte block.  The
//    limiting pipe is shared memory (one conflict-free LDS.32 warp-instruction
//    per clock per SM), so every table is replicated 32x, one copy per bank:
//    word (x, lane) of a table lives at byte  x*256 + t*128 + lane*4  of its
//    64 KiB region (two tables per region), i.e. in bank `lane` whatever x is.
//  * The LDS address is produced by ONE byte-permute (PRMT): with
//    lane4 = lane*4 (< 256, so its bytes 1..3 are zero),
//      __byte_perm(w, lane4, 0x55k4) = (byte_k(w) << 8) | lane*4,
//    and the table/region offset rides in the LDS immediate.  So a lookup is
//    PRMT + LDS, and a column is 4x(PRMT+LDS) + 2 LOP3 (5-way XOR including
//    the round key, which comes straight from the kernel-parameter constant
//    bank).
//  * Te1..3 = rotl(Te0, 8k) are separate smem tables (no rotates in the inner
//    loop).  The last encrypt round reuses the Te tables: byte r of the output
//    column is S[x], found at byte r of Te_{(r+3)%4}[x]; three PRMTs assemble
//    the column.  The last decrypt round uses an InvS table (word = Si*0x01010101)
//    in a third region.  Smem per CTA: 128 KiB encrypt, 192 KiB decrypt -> one
//    CTA per SM, launched as a persistent grid over warp tiles.
//  * Decrypt is the equivalent inverse cipher (FIPS-197 5.3.5): Td tables and
//    round keys dk_r = InvMixColumns(rk_r) prepared on the host; output is
//    identical to the reference's straightforward inverse (aes.cpp:136-147).
//  * Global memory: each lane moves whole 16-byte blocks with 128-bit
//    loads/stores; a warp tile is 32*NB consecutive blocks (lane l takes
//    blocks l, l+32, ...), so every LDG.128/STG.128 covers 512 contiguous bytes.
//  * PKCS#7 always-pad (chunk.cpp:83-88) is fused: the thread that owns block
//    `nfull` builds it from the last tail_len input bytes and the pad byte,
//    so no host-side copy of the final chunk is made.  A final decrypt checks
//    the trailer (chunk.cpp:90-100) in the thread that owns the last block.
#pragma once

#include <cstdint>

#include "aes_tables.hpp"

namespace paes_b200 {

constexpr int kTableRegionBytes = 65536;  // 256 rows x 256 bytes
constexpr int kEncSmemBytes = 2 * kTableRegionBytes;
constexpr int kDecSmemBytes = 3 * kTableRegionBytes;
// After the tables: the CTA's one copy of Te0 (or Td0 + InvS) that the
// replica fill reads, loaded with a few coalesced requests per CTA instead of
// every thread of every SM hammering the same L2 lines.
constexpr int kScratchBytes = 2048;
constexpr int kEncLaunchSmem = kEncSmemBytes + kScratchBytes;
constexpr int kDecLaunchSmem = kDecSmemBytes + kScratchBytes;

// offsets of table k inside the smem window
constexpr int kT0 = 0;
constexpr int kT1 = 128;
constexpr int kT2 = kTableRegionBytes;
constexpr int kT3 = kTableRegionBytes + 128;
constexpr int kTS = 2 * kTableRegionBytes;  // InvS (decrypt only)

struct KeyWords {
  std::uint32_t w[44];  // 11 round keys, in order of use by the kernel
};

struct StateKey {
  std::uint8_t b[16];  // one round key, FIPS byte order (add_round_key)
};

struct EcbArgs {
  const std::uint8_t* in;
  std::uint8_t* out;
  unsigned long long nblocks;  // output blocks
  unsigned long long nfull;    // blocks read whole from `in` (nblocks or nblocks-1)
  std::uint32_t tail_len;      // bytes at in[16*nfull ..] forming the pad block (0..15)
  std::uint32_t check_pad;     // decrypt: validate PKCS#7 trailer of block nblocks-1
  std::uint32_t* status;       // decrypt pad result: pad byte k (1..16) or 0xffffffff (nullable)
  // optional device-visible word written by the thread that owns the last
  // block: the output length (16 * nblocks, minus the pad for a checked
  // trailer) or ~0 for a malformed trailer -- the asynchronous face of
  // decrypt_chunk_into's unpad_final (exec.cpp:122-127)
  unsigned long long* result;
  // optional completion signal for a host that spins instead of
  // synchronising the stream (short host calls, runtime.cu lane_launch): after
  // a barrier, each CTA's thread 0 fences to system scope, the CTAs count themselves in
  // *done_ctr (device memory, 0 on entry; the last CTA resets it), and the
  // last one writes done_seq to the mapped host word *done_flag
  unsigned* done_ctr;
  unsigned* done_flag;
  unsigned done_seq;
  KeyWords k;
};

// Batch (config 5): message descriptors, device-resident.  Every message owns
// ceil(nblocks / kBatchTile) whole warp tiles, so no tile straddles two
// messages (a warp's key registers are uniform for a tile) and the ragged
// last tile of each message is masked.
struct BatchMsg {
  unsigned long long in_off;      // byte offset of the message in d_in
  unsigned long long out_off;     // byte offset of its output in d_out
  unsigned long long first_tile;  // first warp tile of the message
  unsigned long long nfull;       // whole input blocks
  std::uint32_t nblocks;          // output blocks (nfull or nfull+1)
  std::uint32_t tail_len;
};

struct BatchArgs {
  const std::uint8_t* in;
  std::uint8_t* out;
  const BatchMsg* msgs;
  const std::uint32_t* keys;         // 44 words per message, in order of use
  std::uint32_t* status;             // decrypt+pad: one word per message (nullable)
  unsigned long long* out_lens;      // nullable: per-message output length (~0 = bad trailer), device-visible
  unsigned long long total_tiles;
  std::uint32_t nmsg;
  std::uint32_t check_pad;
  std::uint32_t aligned;  // host: every message start in and out is 16-byte aligned (picks the instantiation)
};

// Blocks per warp tile of the batch kernel (32 lanes x blocks per lane).
unsigned batch_tile_blocks();

}  // namespace paes_b200
