// Micro-benchmarks that fix the design constants of the merged-CG kernels on B200:
// FP64 FMA rate, HBM stream rate with fp64 payload, L2-hit read rate, shared-memory
// LDS.64/LDS.128 rate, global fp64 RED rate and shared fp64 atomicAdd rate.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ubench ubench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__constant__ double c_m[36];

// ---- FP64 FMA peak: 12 independent chains per thread, constant-bank operand
__global__ void k_dfma(double* out, int iters) {
  double a[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
      for (int i = 0; i < 12; ++i) a[i] = fma(a[i], c_m[r * 6 + (i % 6)], c_m[r]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 12; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ---- stream kernels
__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n2) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n2; i += stride) b[i] = a[i];
}
// merged-CG like stream: read r, v, p, m ; write r, p, v
__global__ void k_cg_stream(double2* __restrict__ r, double2* __restrict__ v, double2* __restrict__ p,
                            const double2* __restrict__ m, size_t n2, double alpha, double beta) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n2; i += stride) {
    double2 rr = r[i], vv = v[i], pp = p[i], mm = m[i];
    rr.x -= alpha * vv.x; rr.y -= alpha * vv.y;
    pp.x = mm.x * rr.x + beta * pp.x; pp.y = mm.y * rr.y + beta * pp.y;
    r[i] = rr; p[i] = pp; v[i] = make_double2(pp.x * 0.5, pp.y * 0.5);
  }
}
__global__ void k_read(const double2* __restrict__ a, double* out, size_t n2, int reps) {
  double s = 0;
  for (int rep = 0; rep < reps; ++rep) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n2; i += stride) { double2 t = a[i]; s += t.x + t.y; }
  }
  if (s == 12345.678) out[0] = s;
}

// ---- shared memory LDS.64 rate
__global__ void k_lds64(double* out, int iters) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int base = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s0 += sm[(base + u * 256) & 4095];
      s1 += sm[(base + u * 256 + 1024) & 4095];
      s2 += sm[(base + u * 256 + 2048) & 4095];
      s3 += sm[(base + u * 256 + 3072) & 4095];
    }
    base = (base + 1) & 4095;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_lds128(double* out, int iters) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int base = threadIdx.x * 2;
  const double2* s2p = reinterpret_cast<const double2*>(sm);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double2 a = s2p[((base + u * 512) & 4095) >> 1];
      double2 b = s2p[((base + u * 512 + 2048) & 4095) >> 1];
      s0 += a.x; s1 += a.y; s2 += b.x; s3 += b.y;
    }
    base = (base + 2) & 4095;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}

// ---- global fp64 RED: each thread adds to a spread address (2 contributions per address)
__global__ void k_red(double* v, size_t n, int shift) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) atomicAdd(&v[(i + shift) % n], 1.0);
}
// ---- shared fp64 atomicAdd (spread addresses)
__global__ void k_atoms(double* out, int iters) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  for (int it = 0; it < iters; ++it) atomicAdd(&sm[(threadIdx.x * 7 + it * 33) & 4095], 1.0);
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[5];
}

template <class F> float timeit(F f, int warm = 2, int reps = 5) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int i = 0; i < warm; ++i) f();
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    CK(cudaEventRecord(e0)); f(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("device %s SMs %d smem/SM %zu L2 %d MB clock %d kHz\n", prop.name, sms,
         prop.sharedMemPerMultiprocessor, prop.l2CacheSize >> 20, prop.clockRate);
  std::vector<double> h(36, 0.999); CK(cudaMemcpyToSymbol(c_m, h.data(), 36 * 8));
  double* out; CK(cudaMalloc(&out, 1 << 26));

  {  // DFMA
    for (int tpb : {128, 256, 512}) for (int bps : {1, 2, 4}) {
      int iters = 2000; int grid = sms * bps;
      float ms = timeit([&] { k_dfma<<<grid, tpb>>>(out, iters); });
      double fma = (double)grid * tpb * iters * 72.0;
      printf("DFMA tpb %d blocks/SM %d: %.2f TFMA/s (%.2f TFLOP/s), %.1f FMA/clk/SM@1.965GHz\n", tpb, bps,
             fma / ms * 1e-9, 2 * fma / ms * 1e-9, fma / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  {  // HBM
    size_t n = (size_t)1 << 28;  // 2^28 doubles = 2 GiB per vector
    double *a, *b, *c, *d; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8)); CK(cudaMalloc(&c, n * 8)); CK(cudaMalloc(&d, n * 8));
    CK(cudaMemset(a, 0, n * 8)); CK(cudaMemset(b, 0, n * 8)); CK(cudaMemset(c, 0, n * 8)); CK(cudaMemset(d, 0, n * 8));
    for (int bps : {4, 8, 16, 32}) for (int tpb : {256, 512}) {
      float ms = timeit([&] { k_copy<<<sms * bps, tpb>>>((double2*)a, (double2*)b, n / 2); });
      printf("copy blocks/SM %d tpb %d: %.0f GB/s\n", bps, tpb, 2.0 * n * 8 / ms * 1e-6);
    }
    for (int bps : {4, 8, 16}) {
      float ms = timeit([&] { k_cg_stream<<<sms * bps, 256>>>((double2*)a, (double2*)b, (double2*)c, (double2*)d, n / 2, 0.1, 0.2); });
      printf("cg-stream (4r+3w) blocks/SM %d: %.0f GB/s\n", bps, 7.0 * n * 8 / ms * 1e-6);
    }
    {
      float ms = timeit([&] { k_read<<<sms * 16, 256>>>((double2*)a, out, n / 2, 1); });
      printf("read-only HBM: %.0f GB/s\n", 1.0 * n * 8 / ms * 1e-6);
    }
    // L2-resident reads: 32 MB and 64 MB windows, repeated
    for (size_t mb : {16, 32, 64, 96}) {
      size_t nn = mb << 17;  // doubles
      int reps = 40;
      float ms = timeit([&] { k_read<<<sms * 16, 256>>>((double2*)a, out, nn / 2, reps); });
      printf("L2-window %zu MB read: %.0f GB/s\n", mb, (double)reps * nn * 8 / ms * 1e-6);
    }
    // RED
    for (size_t mb : {64, 512}) {
      size_t nn = mb << 17;
      float ms = timeit([&] { k_red<<<sms * 16, 256>>>(a, nn, 0); k_red<<<sms * 16, 256>>>(a, nn, 12345); });
      printf("RED.F64 window %zu MB: %.2f Gatom/s\n", mb, 2.0 * nn / ms * 1e-6);
    }
    cudaFree(a); cudaFree(b); cudaFree(c); cudaFree(d);
  }
  {  // smem
    CK(cudaFuncSetAttribute(k_lds64, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
    CK(cudaFuncSetAttribute(k_lds128, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
    CK(cudaFuncSetAttribute(k_atoms, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
    int iters = 2000;
    for (int bps : {1, 2, 4}) {
      float ms = timeit([&] { k_lds64<<<sms * bps, 256, 32768>>>(out, iters); });
      double bytes = (double)sms * bps * 256 * iters * 32 * 8;
      printf("LDS.64 blocks/SM %d: %.1f TB/s, %.1f B/clk/SM@1.965\n", bps, bytes / ms * 1e-9, bytes / (ms * 1e-3) / sms / 1.965e9);
      ms = timeit([&] { k_lds128<<<sms * bps, 256, 32768>>>(out, iters); });
      bytes = (double)sms * bps * 256 * iters * 16 * 16;
      printf("LDS.128 blocks/SM %d: %.1f TB/s, %.1f B/clk/SM@1.965\n", bps, bytes / ms * 1e-9, bytes / (ms * 1e-3) / sms / 1.965e9);
    }
    float ms = timeit([&] { k_atoms<<<sms * 2, 256, 32768>>>(out, 2000); });
    printf("shared atomicAdd(double): %.2f Gatom/s chip, %.2f atom/clk/SM\n", (double)sms * 2 * 256 * 2000 / ms * 1e-6,
           (double)sms * 2 * 256 * 2000 / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
