// How long does the host take to learn that a short kernel finished?
//   sync   : launch + cudaStreamSynchronize
//   event  : launch + event record + cudaEventSynchronize
//   query  : launch + spin on cudaStreamQuery
//   flag   : launch of a kernel whose last CTA writes a mapped host word
//            (after __threadfence_system), host spins on the word
// for 1 CTA and 32 CTAs of 512 threads; median of 2000 calls, us.  One JSON line.
// Build: scripts/build_probes.sh
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

__global__ void flag_kernel(unsigned* ctr, volatile unsigned* flag, unsigned value) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(ctr, 1u) == gridDim.x - 1) {
      *ctr = 0;
      __threadfence_system();
      *flag = value;
    }
  }
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  unsigned* ctr;
  cudaMalloc(&ctr, 4);
  cudaMemset(ctr, 0, 4);
  unsigned* hflag;
  cudaHostAlloc(reinterpret_cast<void**>(&hflag), 4096, cudaHostAllocMapped);
  unsigned* dflag;
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&dflag), hflag, 0);
  *hflag = 0;
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  unsigned seq = 0;
  auto median = [](std::vector<double>& v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  std::printf("{\"rows\": [");
  bool first = true;
  for (int grid : {1, 32}) {
    for (int mode = 0; mode < 4; ++mode) {
      std::vector<double> t;
      for (int i = 0; i < 2200; ++i) {
        const unsigned v = ++seq;
        const double a = now_us();
        flag_kernel<<<grid, 512, 0, st>>>(ctr, dflag, v);
        if (mode == 0) {
          cudaStreamSynchronize(st);
        } else if (mode == 1) {
          cudaEventRecord(ev, st);
          cudaEventSynchronize(ev);
        } else if (mode == 2) {
          while (cudaStreamQuery(st) == cudaErrorNotReady) {
          }
        } else {
          while (*reinterpret_cast<volatile unsigned*>(hflag) != v) {
          }
        }
        const double b = now_us();
        if (mode == 3) cudaStreamSynchronize(st);  // keep launches from overlapping between samples
        if (i >= 200) t.push_back(b - a);
      }
      static const char* names[] = {"sync", "event", "query", "flag"};
      std::printf("%s{\"grid\": %d, \"mode\": \"%s\", \"median_us\": %.2f}", first ? "" : ", ", grid, names[mode],
                  median(t));
      first = false;
    }
  }
  std::printf("], \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
