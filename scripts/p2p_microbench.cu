// NVLink peer-transfer microbenchmark, GPU0 <-> GPU1, one process (development aid).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/p2p_microbench.cu -o /tmp/p2p && /tmp/p2p
// Copy engines (cudaMemcpyPeerAsync split over S streams) vs SM copy kernels
// (push: local read + remote store; pull: remote load + local store) at G CTAs,
// one direction and both directions at once.  GB/s per direction.
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));                         \
      return 1;                                                                                 \
    }                                                                                           \
  } while (0)

__global__ void __launch_bounds__(512) copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

static const size_t kBytes = 256ull << 20;

struct Side {
  int dev;
  char *local_src, *local_dst;  // on dev
  std::vector<cudaStream_t> st;
  cudaEvent_t e0, e1;
};

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("needs 2 GPUs\n");
    return 1;
  }
  Side s[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    s[d].dev = d;
    CK(cudaMalloc(&s[d].local_src, kBytes));
    CK(cudaMalloc(&s[d].local_dst, kBytes));
    CK(cudaMemset(s[d].local_src, d + 1, kBytes));
    s[d].st.resize(8);
    for (auto& x : s[d].st) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    CK(cudaEventCreate(&s[d].e0));
    CK(cudaEventCreate(&s[d].e1));
  }
  // mode: 0 = copy engines with S streams, 1 = SM push with G CTAs, 2 = SM pull with G CTAs
  auto run = [&](int mode, int param, bool bidir) -> double {
    double best = 1e30;
    for (int rep = 0; rep < 4; ++rep) {
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceSynchronize());
      }
      for (int d = 0; d < (bidir ? 2 : 1); ++d) {
        CK(cudaSetDevice(d));
        Side& me = s[d];
        Side& peer = s[1 - d];
        CK(cudaEventRecord(me.e0, me.st[0]));
        if (mode == 0) {
          const int S = param;
          for (int j = 1; j < S; ++j) CK(cudaStreamWaitEvent(me.st[j], me.e0, 0));
          const size_t chunk = kBytes / S;
          for (int j = 0; j < S; ++j)
            CK(cudaMemcpyPeerAsync(peer.local_dst + j * chunk, peer.dev, me.local_src + j * chunk, me.dev, chunk,
                                   me.st[j]));
          for (int j = 1; j < S; ++j) {
            cudaEvent_t ej;
            CK(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
            CK(cudaEventRecord(ej, me.st[j]));
            CK(cudaStreamWaitEvent(me.st[0], ej, 0));
            CK(cudaEventDestroy(ej));
          }
        } else if (mode == 1) {  // push: this GPU's SMs store into the peer
          copy_kernel<<<param, 512, 0, me.st[0]>>>((uint4*)peer.local_dst, (const uint4*)me.local_src, kBytes / 16);
        } else {  // pull: this GPU's SMs load from the peer (the data flows peer -> me)
          copy_kernel<<<param, 512, 0, me.st[0]>>>((uint4*)me.local_dst, (const uint4*)peer.local_src, kBytes / 16);
        }
        CK(cudaEventRecord(me.e1, me.st[0]));
      }
      double worst = 0;
      for (int d = 0; d < (bidir ? 2 : 1); ++d) {
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(s[d].e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, s[d].e0, s[d].e1));
        worst = worst > ms ? worst : ms;
      }
      if (rep > 0 && worst < best) best = worst;
    }
    return kBytes / (best * 1e-3) / 1e9;
  };
  for (int bidir = 0; bidir < 2; ++bidir) {
    printf("== %s\n", bidir ? "both directions at once (GB/s per direction)" : "one direction (GB/s)");
    for (int S : {1, 2, 4, 8}) printf("copy engines, %d stream(s): %7.1f\n", S, run(0, S, bidir));
    for (int G : {8, 16, 32, 64, 148, 296}) printf("SM push, %3d CTAs x 512: %7.1f\n", G, run(1, G, bidir));
    for (int G : {8, 16, 32, 64, 148, 296}) printf("SM pull, %3d CTAs x 512: %7.1f\n", G, run(2, G, bidir));
  }
  return 0;
}
