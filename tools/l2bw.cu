// On-chip bandwidth probe: every SM streams 128-bit non-coherent loads over a
// buffer of the given size, repeated, and the kernel reports bytes / time.
// Buffers below ~100 MB stay in L2, so the number is the L2 -> SM read cap
// that bounds a stencil whose neighbour loads miss L1.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2bw tools/l2bw.cu
#include <cstdio>
#include <cstdlib>

__global__ void rd(const double2* __restrict__ p, long long n, int reps, double* sink) {
  double acc = 0.0;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    for (long long i = tid; i < n; i += 4 * nt) {
      double2 v0 = __ldg(p + i);
      double2 v1 = i + nt < n ? __ldg(p + i + nt) : make_double2(0, 0);
      double2 v2 = i + 2 * nt < n ? __ldg(p + i + 2 * nt) : make_double2(0, 0);
      double2 v3 = i + 3 * nt < n ? __ldg(p + i + 3 * nt) : make_double2(0, 0);
      acc += v0.x + v1.y + v2.x + v3.y;
    }
  }
  if (acc == 12345.678) *sink = acc;
}

int main(int argc, char** argv) {
  const int blocks_per_sm = argc > 1 ? atoi(argv[1]) : 8;
  const long long sizes_mb[] = {4, 16, 32, 48, 64, 96, 2048};
  double2* p;
  double* sink;
  cudaMalloc(&p, 2048ll << 20);
  cudaMemset(p, 0, 2048ll << 20);
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (long long mb : sizes_mb) {
    const long long n = (mb << 20) / 16;
    const int reps = mb >= 1024 ? 2 : (int)(4096 / mb);
    rd<<<sms * blocks_per_sm, 256>>>(p, n, 1, sink);
    cudaEventRecord(a);
    rd<<<sms * blocks_per_sm, 256>>>(p, n, reps, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"buffer_mb\": %lld, \"blocks_per_sm\": %d, \"gbs\": %.1f}\n", mb, blocks_per_sm,
           (double)(mb << 20) * reps / (ms * 1e-3) / 1e9);
  }
  return 0;
}
