// Microbenchmark: cost of a per-entry value lookup on sm_100a (dictionary in shared memory,
// constant bank, L1-resident global, or warp shuffles) as a function of how many distinct
// entries a warp touches per instruction. Drives the operator-store design.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ubench_lookup ubench_lookup.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kDict = 256;
__constant__ double2 c_dict[kDict];

// distinct: lanes use (lane % distinct) * stride as the index
template <int MODE>
__global__ void bench(const double2* __restrict__ gdict, int distinct, int stride, int step, double* out, long long* cyc) {
  __shared__ double2 sdict[kDict];
  for (int i = threadIdx.x; i < kDict; i += blockDim.x) sdict[i] = gdict[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int idx = ((lane % distinct) * stride) & (kDict - 1);
  double ax = 0.0, ay = 0.0;
  double2 reg = gdict[lane];
  const long long t0 = clock64();
#pragma unroll 8
  for (int it = 0; it < kIters; ++it) {
    double2 v;
    if (MODE == 0) v = sdict[idx];                      // LDS.128
    else if (MODE == 1) v = c_dict[idx];                // LDC (indexed)
    else if (MODE == 2) v = __ldg(gdict + idx);         // LDG.128 via L1
    else if (MODE == 3) {                               // two LDS.64
      const double* p = reinterpret_cast<const double*>(sdict);
      v.x = p[2 * idx];
      v.y = p[2 * idx + 1];
    } else if (MODE == 4) {                             // SHFL from registers (4 x 32-bit)
      v.x = __shfl_sync(0xffffffffu, reg.x, idx & 31);
      v.y = __shfl_sync(0xffffffffu, reg.y, idx & 31);
    } else {                                            // LDS.32 (offset table)
      const int* p = reinterpret_cast<const int*>(sdict);
      v.x = p[idx];
      v.y = 0.0;
    }
    ax += v.x;
    ay += v.y;
    idx = (idx + step) & (kDict - 1);  // step == 0 at run time: loads stay independent, not hoistable
  }
  const long long t1 = clock64();
  if (ax == 12345.0) out[0] = ay;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double2 h[kDict];
  for (int i = 0; i < kDict; ++i) h[i] = make_double2(i * 1.0, -i * 0.5);
  double2* d;
  double* o;
  long long* cyc;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&o, 8);
  const int blocks = 148 * 2, threads = 512;
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_dict, h, sizeof(h));
  const char* names[] = {"LDS.128", "LDC", "LDG.128(L1)", "2xLDS.64", "2xSHFL(f64)", "LDS.32"};
  for (int mode = 0; mode < 6; ++mode)
    for (int distinct : {1, 2, 4, 8, 32}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      auto launch = [&] {
        switch (mode) {
          case 0: bench<0><<<blocks, threads>>>(d, distinct, 1, 0, o, cyc); break;
          case 1: bench<1><<<blocks, threads>>>(d, distinct, 1, 0, o, cyc); break;
          case 2: bench<2><<<blocks, threads>>>(d, distinct, 1, 0, o, cyc); break;
          case 3: bench<3><<<blocks, threads>>>(d, distinct, 1, 0, o, cyc); break;
          case 4: bench<4><<<blocks, threads>>>(d, distinct, 1, 0, o, cyc); break;
          default: bench<5><<<blocks, threads>>>(d, distinct, 1, 0, o, cyc); break;
        }
      };
      launch();
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      // warp-instructions per SM per ns
      const double winst = static_cast<double>(blocks) * (threads / 32) * kIters / 148.0;
      printf("%-12s distinct=%2d  %.3f ms  %.2f ns per warp-lookup per SM\n", names[mode], distinct, ms,
             ms * 1e6 / winst);
    }
  return cudaDeviceSynchronize() != cudaSuccess;
}
