// ce_p2p_probe.cu -- copy-engine peer copies on two GPUs: push vs pull, 1..8 concurrent streams,
// one direction vs both (the bench's ring at N=2 copies both ways at once).
//
//   nvcc -O3 -o ce_p2p_probe scripts/ce_p2p_probe.cu && ./ce_p2p_probe
#include <cstdio>
#include <cuda_runtime.h>

int main() {
  const size_t bytes = 256ull << 20;
  void *a0, *b0, *a1, *b1;
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaMalloc(&a0, bytes);
  cudaMalloc(&b0, bytes);
  cudaSetDevice(1);
  cudaDeviceEnablePeerAccess(0, 0);
  cudaMalloc(&a1, bytes);
  cudaMalloc(&b1, bytes);
  cudaStream_t s0[8], s1[8];
  for (int i = 0; i < 8; ++i) {
    cudaSetDevice(0);
    cudaStreamCreateWithFlags(&s0[i], cudaStreamNonBlocking);
    cudaSetDevice(1);
    cudaStreamCreateWithFlags(&s1[i], cudaStreamNonBlocking);
  }
  auto run = [&](const char* name, int ns, bool push, bool both) {
    cudaSetDevice(0);
    cudaDeviceSynchronize();
    cudaSetDevice(1);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaSetDevice(0);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaSetDevice(0);
      cudaDeviceSynchronize();
      cudaSetDevice(1);
      cudaDeviceSynchronize();
      cudaSetDevice(0);
      cudaEventRecord(e0, 0);
      const size_t chunk = bytes / ns;
      for (int i = 0; i < ns; ++i) {
        // 0 -> 1: pushed by device 0's engines (stream on 0) or pulled by device 1's (stream on 1)
        cudaSetDevice(push ? 0 : 1);
        cudaMemcpyAsync((char*)a1 + i * chunk, (char*)a0 + i * chunk, chunk, cudaMemcpyDeviceToDevice, push ? s0[i] : s1[i]);
        if (both) {  // 1 -> 0 at the same time
          cudaSetDevice(push ? 1 : 0);
          cudaMemcpyAsync((char*)b0 + i * chunk, (char*)b1 + i * chunk, chunk, cudaMemcpyDeviceToDevice, push ? s1[i] : s0[i]);
        }
      }
      cudaSetDevice(0);
      cudaDeviceSynchronize();
      cudaSetDevice(1);
      cudaDeviceSynchronize();
      cudaSetDevice(0);
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
    }
    printf("%-5s streams %d %-9s: %7.1f GB/s per direction  %s\n", name, ns, both ? "both ways" : "one way",
           bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int ns : {1, 2, 4, 8}) {
    run("push", ns, true, false);
    run("pull", ns, false, false);
    run("push", ns, true, true);
    run("pull", ns, false, true);
  }
  return 0;
}
