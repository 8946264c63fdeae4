// Does any table-lookup path run BESIDE the shared-memory lookups?
//
// The T-table kernel is bound by conflict-free LDS.32 lookups (32 per clock
// per SM).  A hybrid could only beat that if another lookup path
// (L1-cached LDG, the texture path) had its own data bandwidth.  This probe
// runs random 8-bit-indexed 32-bit lookups through each path alone and through
// two paths at once (half the warps each) and reports lookups per clock per SM.
// Build: scripts/build_probes.sh   Run: scripts/lookup_path_probe_bin
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_runtime.h>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

constexpr int kThreads = 512;
constexpr int kChains = 8;

enum Path { LDS = 0, LDG = 1, TEX = 2, ALU = 3, LDC = 4, MIX = 5 };

__constant__ unsigned c_tab[256];
constexpr int kMixLdc = 3;  // MIX: per chain round, 32 LDS lookups + this many LDC lookups (~ the last round's share)

template <int P>
__device__ __forceinline__ unsigned look(unsigned x, int k, const char* smb, unsigned lane4, const unsigned* g,
                                         cudaTextureObject_t t) {
  if constexpr (P == LDS) {
    return *reinterpret_cast<const unsigned*>(smb + __byte_perm(x, lane4, 0x5504 | (k << 4)));
  } else if constexpr (P == LDG) {
    return __ldg(g + ((x >> (8 * k)) & 255));
  } else if constexpr (P == TEX) {
    return tex1Dfetch<unsigned>(t, (x >> (8 * k)) & 255);
  } else if constexpr (P == LDC) {
    return c_tab[(x >> (8 * k)) & 255];  // indexed constant load, divergent addresses
  } else {
    // ALU stand-in of similar instruction weight: two rotations and an add
    return __funnelshift_l(x, x, 5 + k) + (x >> 3);
  }
}

template <int P>
__device__ __forceinline__ void run(unsigned (&c)[kChains], int iters, const char* smb, unsigned lane4,
                                    const unsigned* g, cudaTextureObject_t t) {
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < kChains; ++j) {
      const unsigned x = c[j];
      if constexpr (P == MIX) {
        unsigned v = look<LDS>(x, 0, smb, lane4, g, t) ^ look<LDS>(x, 1, smb, lane4, g, t) ^
                     look<LDS>(x, 2, smb, lane4, g, t) ^ look<LDS>(x, 3, smb, lane4, g, t) ^ (x * 0x9e3779b9u);
        if (j < kMixLdc) v ^= look<LDC>(x, j, smb, lane4, g, t);
        c[j] = v;
      } else {
        c[j] = look<P>(x, 0, smb, lane4, g, t) ^ look<P>(x, 1, smb, lane4, g, t) ^
               look<P>(x, 2, smb, lane4, g, t) ^ look<P>(x, 3, smb, lane4, g, t) ^ (x * 0x9e3779b9u);
      }
    }
  }
}

// pa: path of even warps, pb: path of odd warps (-1 = idle)
__global__ void __launch_bounds__(kThreads, 1)
probe(int pa, int pb, int iters, const unsigned* g, cudaTextureObject_t t, unsigned* sink,
      long long* clk) {
  extern __shared__ __align__(16) char smb[];
  unsigned* sm = reinterpret_cast<unsigned*>(smb);
  for (int i = threadIdx.x; i < 65536 / 4; i += kThreads) sm[i] = g[(i >> 6) & 255] ^ (i & 31);
  __syncthreads();
  const long long t0 = clock64();
  const unsigned lane = threadIdx.x & 31;
  const unsigned lane4 = lane * 4;
  const int warp = threadIdx.x >> 5;
  const int p = (warp & 1) ? pb : pa;
  unsigned c[kChains];
#pragma unroll
  for (int j = 0; j < kChains; ++j) c[j] = (blockIdx.x * kThreads + threadIdx.x) * 0x01000193u + j * 0x5bd1e995u;
  switch (p) {
    case LDS: run<LDS>(c, iters, smb, lane4, g, t); break;
    case LDG: run<LDG>(c, iters, smb, lane4, g, t); break;
    case TEX: run<TEX>(c, iters, smb, lane4, g, t); break;
    case ALU: run<ALU>(c, iters, smb, lane4, g, t); break;
    case LDC: run<LDC>(c, iters, smb, lane4, g, t); break;
    case MIX: run<MIX>(c, iters, smb, lane4, g, t); break;
    default: break;
  }
  unsigned acc = 0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) acc ^= c[j];
  if (acc == 0x12345678u) sink[0] = acc;
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    clk[0] = t0;
    clk[1] = clock64();
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned h[256];
  for (int i = 0; i < 256; ++i) h[i] = 0x9e3779b9u * (i + 1);
  unsigned *g, *sink;
  long long* clk;
  CK(cudaMalloc(&g, sizeof h));
  CK(cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice));
  CK(cudaMemcpyToSymbol(c_tab, h, sizeof h));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMalloc(&clk, 16));
  cudaResourceDesc rd{};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = g;
  rd.res.linear.desc = cudaCreateChannelDesc<unsigned>();
  rd.res.linear.sizeInBytes = sizeof h;
  cudaTextureDesc td{};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));

  struct Case {
    const char* name;
    int pa, pb;
  } cases[] = {{"lds_all", LDS, LDS},  {"lds_half", LDS, -1},  {"ldg_all", LDG, LDG},
               {"tex_all", TEX, TEX},  {"lds+ldg", LDS, LDG},  {"lds+tex", LDS, TEX},
               {"lds+alu", LDS, ALU},  {"alu_all", ALU, ALU},  {"ldc_all", LDC, LDC},  {"ldc_half", LDC, -1},
               {"lds+ldc", LDS, LDC},  {"mix_32lds_3ldc_all", MIX, MIX}};
  const int iters = 2000;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  printf("[\n");
  for (size_t ci = 0; ci < sizeof cases / sizeof cases[0]; ++ci) {
    const Case& cs = cases[ci];
    float best = 1e30f;
    long long cyc = 0;
    for (int rep = 0; rep < 4; ++rep) {
      CK(cudaEventRecord(e0));
      probe<<<sms, kThreads, 65536>>>(cs.pa, cs.pb, iters, g, tex, sink, clk);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) {
        best = ms;
        long long c2[2];
        CK(cudaMemcpy(c2, clk, 16, cudaMemcpyDeviceToHost));
        cyc = c2[1] - c2[0];
      }
    }
    // lookups: 4 per chain step for each warp on a lookup path
    // (MIX counts its LDS lookups only: compare its ms with lds_all's)
    auto lk = [&](int p) { return (p == LDS || p == LDG || p == TEX || p == LDC || p == MIX) ? 1.0 : 0.0; };
    const double warps = kThreads / 32.0;
    const double lookups = (lk(cs.pa) + lk(cs.pb)) * (warps / 2) * 32 * (double)iters * kChains * 4 * sms;
    const double per_clk_sm = lookups / sms / (double)cyc;
    const double mhz = cyc / (best * 1e3);
    printf("  {\"case\": \"%s\", \"ms\": %.3f, \"sm_cycles\": %lld, \"mhz_est\": %.0f, \"lookups_per_clk_per_sm\": %.2f}%s\n",
           cs.name, best, cyc, mhz, per_clk_sm, ci + 1 < sizeof cases / sizeof cases[0] ? "," : "");
  }
  printf("]\n");
  return 0;
}
