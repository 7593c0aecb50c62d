// microbench_smem.cu — shared-memory operation throughput on B200 for the
// partition's rank/stage design (not product code).  Every thread draws
// pseudo-random word indices in registers (no memory traffic) and issues one
// shared op per index; the figure is lane-ops per SM-cycle.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_smem tools/microbench_smem.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

constexpr int kIters = 4096;

// mode 0: returning atomicAdd on one of W words
// mode 1: non-returning atomicAdd on one of W words
// mode 2: uint16 store to one of 2W halfwords
// mode 3: returning atomicAdd, 4 lane replicas ((lane & 3) * W + i)
// mode 4: returning atomicAdd, lane-column layout (i * 32 + lane)
// mode 5: ALU only (index generation)
// mode 6: returning atomicAdd on one of W words, W words padded so word w sits in bank w % 32 ... with a 33-word row stride
template <int MODE>
__global__ void k_smem(unsigned W, unsigned* sink, unsigned long long* cyc) {
  extern __shared__ unsigned s[];
  const unsigned words = MODE == 3 ? 4 * W : MODE == 4 ? 32 * W : W;
  for (unsigned i = threadIdx.x; i < words; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned x = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  unsigned acc = 0;
  const unsigned lane = threadIdx.x & 31;
  const long long t0 = clock64();
#pragma unroll 8
  for (int it = 0; it < kIters; ++it) {
    x = x * 1664525u + 1013904223u;
    const unsigned i = __umulhi(x, W);
    if (MODE == 0) acc += atomicAdd(&s[i], 1u);
    if (MODE == 1) atomicAdd(&s[i], 1u);
    if (MODE == 2) reinterpret_cast<unsigned short*>(s)[__umulhi(x, 2 * W)] = (unsigned short)x;
    if (MODE == 3) acc += atomicAdd(&s[(lane & 3) * W + i], 1u);
    if (MODE == 4) acc += atomicAdd(&s[i * 32 + lane], 1u);
    if (MODE == 5) acc += i;
  }
  __syncthreads();
  const long long t1 = clock64();
  if (acc == 0x12345678u) atomicAdd(sink, 1);
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* sink;
  unsigned long long* cyc;
  cudaMalloc(&sink, 4);
  cudaMalloc(&cyc, 8);
  const char* names[] = {"atom-ret", "atom-noret", "st.u16", "atom-ret-rep4", "atom-ret-lanecol", "alu-only"};
  const unsigned Ws[] = {32, 64, 100, 128, 256, 1000, 10000};
  for (int m = 0; m < 6; ++m) {
    auto set = [](auto k) { cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024); };
    if (m == 0) set(k_smem<0>); if (m == 1) set(k_smem<1>); if (m == 2) set(k_smem<2>);
    if (m == 3) set(k_smem<3>); if (m == 4) set(k_smem<4>); if (m == 5) set(k_smem<5>);
  }
  for (int threads : {384, 1024}) {
    const int blocks = sms * (threads == 1024 ? 1 : 2);
    for (int mode = 0; mode < 6; ++mode) {
      for (unsigned W : Ws) {
        if ((mode == 4 && W > 256) || (mode == 3 && W > 2500)) continue;
        const size_t smem = 4ull * (mode == 3 ? 4 * W : mode == 4 ? 32 * W : W);
        cudaMemset(cyc, 0, 8);
        auto run = [&] {
          switch (mode) {
            case 0: k_smem<0><<<blocks, threads, smem>>>(W, sink, cyc); break;
            case 1: k_smem<1><<<blocks, threads, smem>>>(W, sink, cyc); break;
            case 2: k_smem<2><<<blocks, threads, smem>>>(W, sink, cyc); break;
            case 3: k_smem<3><<<blocks, threads, smem>>>(W, sink, cyc); break;
            case 4: k_smem<4><<<blocks, threads, smem>>>(W, sink, cyc); break;
            case 5: k_smem<5><<<blocks, threads, smem>>>(W, sink, cyc); break;
          }
        };
        run();
        cudaDeviceSynchronize();
        cudaMemset(cyc, 0, 8);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        run();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = (double)blocks * threads * kIters;
        const double sm_cycles = ms * 1e-3 * 1.965e9 * sms;
        printf("threads %4d blocks/SM %d %-18s W=%5u  %.2f ms  lane-ops/SM-cycle %.2f  cycles/warp-op %.2f\n", threads,
               blocks / sms, names[mode], W, ms, ops / sm_cycles, sm_cycles / (ops / 32) );
        if (mode == 5) break;
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
