// PCIe copy bandwidth probe: pinned host <-> device, one direction alone and
// both concurrently, whole-buffer and chunked. Used to bound lbcu_dphi_host.
//   nvcc -O2 -o tools/pcie_probe tools/pcie_probe.cu && tools/pcie_probe [MB]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? atoi(argv[1]) : 128;
  const size_t bytes = mb << 20;
  char *h_in, *h_out, *d_in, *d_out;
  CK(cudaMallocHost(&h_in, bytes));
  CK(cudaMallocHost(&h_out, bytes));
  CK(cudaMalloc(&d_in, bytes));
  CK(cudaMalloc(&d_out, bytes));
  for (size_t i = 0; i < bytes; i += 4096) h_in[i] = 1, h_out[i] = 1;
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int reps = 10;
  size_t chunks[] = {0, 64 << 20, 16 << 20, 4 << 20, 1 << 20};
  for (size_t ch : chunks) {
    const size_t c = ch ? ch : bytes;
    for (int mode = 0; mode < 3; ++mode) {  // 0 h2d, 1 d2h, 2 both
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, s1));
      CK(cudaStreamWaitEvent(s2, a, 0));
      for (int r = 0; r < reps; ++r)
        for (size_t o = 0; o < bytes; o += c) {
          const size_t n = o + c > bytes ? bytes - o : c;
          if (mode != 1) CK(cudaMemcpyAsync(d_in + o, h_in + o, n, cudaMemcpyHostToDevice, s1));
          if (mode != 0) CK(cudaMemcpyAsync(h_out + o, d_out + o, n, cudaMemcpyDeviceToHost, s2));
        }
      cudaEvent_t e2;
      CK(cudaEventCreate(&e2));
      CK(cudaEventRecord(e2, s2));
      CK(cudaStreamWaitEvent(s1, e2, 0));
      CK(cudaEventRecord(b, s1));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      const double per = ms / reps;
      printf("{\"chunk_mb\": %zu, \"mode\": \"%s\", \"ms_per_%zuMB\": %.3f, \"gbs_per_dir\": %.2f}\n", c >> 20,
             mode == 0 ? "h2d" : mode == 1 ? "d2h" : "both", mb, per, bytes / per / 1e6);
    }
  }
  return 0;
}
