// PCIe copy bandwidth of this box: host->device alone, device->host alone, both at once
// (two streams), with default page-locked and write-combined upload buffers, whole and in
// chunks.  The streamed e2e (stmg_mg_solve_stream) is bounded by the "both" figure.
// Build + run: nvcc -O2 -o pcie_duplex profiles/pcie_duplex.cu && ./pcie_duplex
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

__global__ void k_stream(const double* __restrict__ a, double* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i] + 1.0;
}

static double run(void* d_up, const void* h_up, void* h_down, const void* d_down, size_t bytes, bool up, bool down,
                  size_t chunk, bool sync_first = true) {
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  if (sync_first) cudaDeviceSynchronize();
  cudaEventRecord(e0, s1);
  cudaStreamWaitEvent(s2, e0, 0);
  for (size_t o = 0; o < bytes; o += chunk) {
    const size_t n = bytes - o < chunk ? bytes - o : chunk;
    if (up) cudaMemcpyAsync((char*)d_up + o, (const char*)h_up + o, n, cudaMemcpyHostToDevice, s1);
    if (down) cudaMemcpyAsync((char*)h_down + o, (const char*)d_down + o, n, cudaMemcpyDeviceToHost, s2);
  }
  cudaEventRecord(e2, s2);
  cudaStreamWaitEvent(s1, e2, 0);
  cudaEventRecord(e1, s1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaStreamDestroy(s1);
  cudaStreamDestroy(s2);
  return ms * 1e-3;
}

int main() {
  const size_t bytes = size_t(4) << 30;
  void *d_a, *d_b, *h_def, *h_wc, *h_down;
  cudaMalloc(&d_a, bytes);
  cudaMalloc(&d_b, bytes);
  cudaMemset(d_b, 1, bytes);
  cudaHostAlloc(&h_def, bytes, cudaHostAllocDefault);
  cudaHostAlloc(&h_wc, bytes, cudaHostAllocWriteCombined);
  cudaHostAlloc(&h_down, bytes, cudaHostAllocDefault);
  memset(h_def, 1, bytes);
  memset(h_wc, 1, bytes);
  memset(h_down, 0, bytes);
  const double gb = bytes / 1e9;
  {  // the same with an HBM-saturating kernel running throughout (what a solve does)
    double *x, *y;
    const size_t n = size_t(1) << 29;  // 4 GiB each
    cudaMalloc(&x, n * 8);
    cudaMalloc(&y, n * 8);
    cudaMemset(x, 0, n * 8);
    cudaStream_t sk;
    cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);
    cudaEvent_t k0, k1;
    cudaEventCreate(&k0);
    cudaEventCreate(&k1);
    cudaEventRecord(k0, sk);
    for (int it = 0; it < 40; ++it) k_stream<<<148 * 8, 512, 0, sk>>>(x, y, n);
    cudaEventRecord(k1, sk);
    cudaEventSynchronize(k1);
    float kms = 0;
    cudaEventElapsedTime(&kms, k0, k1);
    for (int it = 0; it < 400; ++it) k_stream<<<148 * 8, 512, 0, sk>>>(x, y, n);  // ~0.6 s of HBM streaming
    const double b = run(d_a, h_def, h_down, d_b, bytes, true, true, bytes, false);
    cudaError_t busy = cudaStreamQuery(sk);
    cudaStreamSynchronize(sk);
    std::printf("{\"kernel_TBps_alone\": %.2f, \"both_total_GBps_under_hbm_streaming\": %.1f, \"kernel_still_running_at_end\": %s}\n",
                40 * 2.0 * n * 8 / (kms * 1e-3) / 1e12, 2 * gb / b, busy == cudaErrorNotReady ? "true" : "false");
    cudaFree(x);
    cudaFree(y);
  }
  for (int rep = 0; rep < 2; ++rep) {
    for (size_t chunk : {bytes, size_t(64) << 20}) {
      const double u = run(d_a, h_def, h_down, d_b, bytes, true, false, chunk);
      const double uw = run(d_a, h_wc, h_down, d_b, bytes, true, false, chunk);
      const double d = run(d_a, h_def, h_down, d_b, bytes, false, true, chunk);
      const double b = run(d_a, h_def, h_down, d_b, bytes, true, true, chunk);
      const double bw = run(d_a, h_wc, h_down, d_b, bytes, true, true, chunk);
      std::printf(
          "{\"chunk_mib\": %zu, \"h2d_GBps\": %.1f, \"h2d_wc_GBps\": %.1f, \"d2h_GBps\": %.1f, "
          "\"both_total_GBps\": %.1f, \"both_wc_total_GBps\": %.1f}\n",
          chunk >> 20, gb / u, gb / uw, gb / d, 2 * gb / b, 2 * gb / bw);
    }
  }
  return 0;
}
