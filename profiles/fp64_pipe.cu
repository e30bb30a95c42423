// Microbenchmark: FP64 pipe throughput on B200 (sm_100a), the second roofline of the
// stencil kernels.  The solve is compiled --fmad=false (bitwise parity with the reference's
// -ffp-contract=off kernels), so every DOF update costs separate DMUL and DADD instructions;
// the low-byte kernels (restriction of the virtual zero iterate: 12 B/DOF, ~21 DP
// instructions per DOF-row) are bounded by this pipe rather than by HBM.
//
// Build + run:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o fp64_pipe
//               profiles/fp64_pipe.cu && ./fp64_pipe
// Prints per-SM, per-clock lane throughput of DADD, DMUL, DFMA chains (8 independent
// chains per thread, 1024 threads per SM) and of a DADD + SHFL / DADD + IMAD mix.
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kIters = 4096;
constexpr int kChains = 8;

template <int OP>
__global__ void __launch_bounds__(1024) k_pipe(double* out, double a, double b, int mix) {
  double v[kChains];
#pragma unroll
  for (int j = 0; j < kChains; ++j) v[j] = a + j + threadIdx.x;
  int iacc = threadIdx.x;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int j = 0; j < kChains; ++j) {
      if (OP == 0) v[j] = v[j] + b;
      if (OP == 1) v[j] = v[j] * b;
      if (OP == 2) v[j] = fma(v[j], b, a);
      if (OP == 3) {  // DADD + one 64-bit shuffle (2 SHFL) per 4 DADD
        v[j] = v[j] + b;
        if ((j & 3) == 0) v[j] = __shfl_up_sync(0xffffffffu, v[j], 1);
      }
      if (OP == 4) {  // DADD + one integer multiply-add per DADD
        v[j] = v[j] + b;
        iacc = iacc * mix + j;
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < kChains; ++j) s += v[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + iacc;
}

template <int OP>
double run(const char* name, int sms, double clock_hz, double dp_per_iter) {
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double) * sms * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_pipe<OP><<<sms, 1024>>>(out, 1.0, 1.0000001, 3);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_pipe<OP><<<sms, 1024>>>(out, 1.0, 1.0000001, 3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double dp_lane_ops = dp_per_iter * kIters * kChains * 1024.0;  // per SM
  const double per_clk = dp_lane_ops / (best * 1e-3 * clock_hz);
  std::printf("{\"op\": \"%s\", \"ms\": %.4f, \"fp64_lanes_per_clk_per_sm\": %.2f, \"device_tera_ops\": %.2f}\n", name,
              best, per_clk, dp_lane_ops * sms / (best * 1e-3) / 1e12);
  cudaFree(out);
  return per_clk;
}

// Dependent-issue latency: one chain per thread, one warp per SM.
__global__ void k_latency(double* out, double b, int iters, int op, const double* tab) {
  double v = b + threadIdx.x;
  if (op == 0) {
    for (int it = 0; it < iters; ++it) v = v + b;
  } else if (op == 1) {
    for (int it = 0; it < iters; ++it) v = v * b;
  } else {
    __shared__ double sm[1024];
    for (int k = threadIdx.x; k < 1024; k += blockDim.x) sm[k] = tab[k];
    __syncthreads();
    for (int it = 0; it < iters; ++it) v = v + sm[(it * 32 + threadIdx.x) & 1023];  // LDS feeding the chain
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
}

void latency(const char* name, int op, double clock_hz) {
  double *out = nullptr, *tab = nullptr;
  cudaMalloc(&out, sizeof(double) * 148 * 32);
  cudaMalloc(&tab, sizeof(double) * 1024);
  cudaMemset(tab, 0, sizeof(double) * 1024);
  const int iters = 1 << 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_latency<<<148, 32>>>(out, 1.0000001, iters, op, tab);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_latency<<<148, 32>>>(out, 1.0000001, iters, op, tab);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  std::printf("{\"op\": \"%s\", \"ms\": %.4f, \"cycles_per_dependent_op_at_max_clock\": %.2f}\n", name, best,
              best * 1e-3 * clock_hz / iters);
  cudaFree(out);
  cudaFree(tab);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double hz = khz * 1e3;
  std::printf("{\"gpu\": \"%s\", \"sms\": %d, \"max_clock_mhz\": %.0f, \"note\": \"per-clock figures assume the max clock\"}\n",
              p.name, p.multiProcessorCount, hz / 1e6);
  run<0>("dadd", p.multiProcessorCount, hz, 1);
  run<1>("dmul", p.multiProcessorCount, hz, 1);
  run<2>("dfma", p.multiProcessorCount, hz, 1);
  run<3>("dadd + 64-bit shfl per 4", p.multiProcessorCount, hz, 1);
  run<4>("dadd + imad per dadd", p.multiProcessorCount, hz, 1);
  latency("dadd dependent chain", 0, hz);
  latency("dmul dependent chain", 1, hz);
  latency("lds + dadd dependent chain (unhoisted)", 2, hz);
  return 0;
}
