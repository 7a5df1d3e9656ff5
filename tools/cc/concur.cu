// Does a small kernel on a second stream run while a persistent kernel with
// 64 regs x 256 threads x 4 CTAs/SM and ~46 KB dynamic smem holds most SMs?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 4) k_long(long long cycles, int* out) {
  extern __shared__ int sm[];
  long long t0 = clock64();
  int acc = threadIdx.x;
  while (clock64() - t0 < cycles) { acc = acc * 3 + 1; sm[threadIdx.x] = acc; }
  if (acc == 42) out[0] = acc;
}
__global__ void k_small(int* out) { if (threadIdx.x == 0) out[1] = 1; }
__global__ void k_small_smem(int* out) {
  __shared__ int big[10000];  // 40 KB static
  big[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0) out[1] = big[5];
}
int main(int argc, char** argv) {
  int reserve = argc > 1 ? atoi(argv[1]) : 16;
  int mode = argc > 2 ? atoi(argv[2]) : 0;
  int *hbuf, *hbuf2, *dbuf; cudaHostAlloc(&hbuf, 64, 0); cudaHostAlloc(&hbuf2, 64, 0); cudaMalloc(&dbuf, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t a, b; cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  int* out; cudaMalloc(&out, 64);
  size_t smem = 46 * 1024;
  cudaFuncSetAttribute(k_long, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1, e2; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0, a);
    k_long<<<(sms - reserve) * 4, 256, smem, a>>>(2000LL * 1000 * 2, out);  // ~2 ms at 2 GHz
    cudaEventRecord(e1, a);
    if (mode >= 1) cudaMemcpyAsync(hbuf, out, 64, cudaMemcpyDeviceToHost, a);  // queued behind the long kernel
    // host waits 100 us then launches on b
    cudaStreamSynchronize(b);
    cudaEvent_t s0, s1; cudaEventCreate(&s0); cudaEventCreate(&s1);
    cudaEventRecord(s0, b);
    if (mode >= 2) cudaMemcpyAsync(dbuf, hbuf2, 64, cudaMemcpyHostToDevice, b);
    if (mode == 3) { void* hp; cudaHostAlloc(&hp, (1 << 20) * (rep + 1), 0); }
    if (mode == 4) { void* dp; cudaMallocAsync(&dp, ((size_t)64 << 20) * (rep + 1), b); }
    if (mode == 5) { cudaFuncSetAttribute(k_long, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024 * (rep + 1)); }
    if (mode == 6) { cudaEvent_t ee; cudaEventCreate(&ee); cudaEventDestroy(ee); }
    if (mode == 7) k_small_smem<<<253, 128, 0, b>>>(out);
    else k_small<<<1012, 128, 0, b>>>(out);
    if (mode >= 1) cudaMemcpyAsync(hbuf2, out, 64, cudaMemcpyDeviceToHost, b);
    cudaEventRecord(s1, b);
    cudaEventSynchronize(s1);
    float small_end = 0, long_ms = 0;
    cudaEventElapsedTime(&small_end, e0, s1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&long_ms, e0, e1);
    printf("mode %d reserve %d: long kernel %.3f ms, small kernel finished %.3f ms after the long one started\n", mode, reserve, long_ms, small_end);
  }
  return 0;
}
