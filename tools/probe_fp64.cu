// Hardware probe for the FP64 roofline denominators and the cluster design of the
// PSD-projection kernels ("The builder must measure a DMMA and a DFMA peak
// on the box"). Not part of the product path.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_fp64 probe_fp64.cu
#include <cstdio>
#include <cstdlib>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

// DMMA m8n8k4: each instruction = 8*8*4 FMA = 512 flop.
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[0]), "+d"(c0[1]) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c1[0]), "+d"(c1[1]) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c2[0]), "+d"(c2[1]) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c3[0]), "+d"(c3[1]) : "d"(a), "d"(b));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
}

__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-7;
  double x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = fma(x[u], b, a);
  }
  double s = 0;
  for (int u = 0; u < 8; ++u) s += x[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __cluster_dims__(1, 1, 1) dummy() {}

__global__ void cluster_bar_loop(long long* out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[blockIdx.x] = t1 - t0;
  if (threadIdx.x == 0) sm[0] = 0;
}

__global__ void grid_sync_loop(long long* out, int iters) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s sm_%d%d SMs=%d smemPerBlockOptin=%zu smemPerSM=%zu L2=%d clockKHz=%d\n", p.name,
         p.major, p.minor, p.multiProcessorCount, p.sharedMemPerBlockOptin,
         p.sharedMemPerMultiprocessor, p.l2CacheSize, clk);
  double* out;
  CK(cudaMalloc(&out, 1 << 24));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // DMMA peak
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * 4, iters = 4000;
    dmma_loop<<<blocks, 32 * wpb>>>(out, 10);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, 32 * wpb>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 512.0 * 32.0 * (double)iters * blocks * wpb;  // 32 mma per iter per warp, 512 flop each
    printf("DMMA m8n8k4: warps/block=%d blocks=%d  %.3f ms  %.2f TFLOP/s\n", wpb, blocks, ms, flops / ms / 1e9);
  }
  for (int tpb : {256, 512}) {
    int blocks = sms * 4, iters = 4000;
    dfma_loop<<<blocks, tpb>>>(out, 10);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, tpb>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64.0 * (double)iters * blocks * tpb;
    printf("DFMA: tpb=%d  %.3f ms  %.2f TFLOP/s\n", tpb, ms, flops / ms / 1e9);
  }
  // cluster occupancy for the tridiagonalisation design
  CK(cudaFuncSetAttribute(cluster_bar_loop, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int smem_kb : {100, 160, 200, 220, 227}) {
    size_t smem = (size_t)smem_kb * 1024;
    if (smem > p.sharedMemPerBlockOptin) smem = p.sharedMemPerBlockOptin;
    CK(cudaFuncSetAttribute(cluster_bar_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int cs : {2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs, 1, 1);
      cfg.blockDim = dim3(512, 1, 1);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, cluster_bar_loop, &cfg);
      long long cyc = -1;
      if (e == cudaSuccess && ncl > 0) {
        long long* dout = (long long*)out;
        int iters = 2000;
        e = cudaLaunchKernelEx(&cfg, cluster_bar_loop, dout, iters);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e == cudaSuccess) {
          cudaMemcpy(&cyc, dout, 8, cudaMemcpyDeviceToHost);
          cyc /= iters;
        }
      }
      printf("cluster size %2d smem %3d KB: maxActiveClusters=%d (%s)  cluster.sync=%lld cyc\n", cs,
             (int)(smem / 1024), ncl, cudaGetErrorString(e), cyc);
      cudaGetLastError();
    }
  }
  // grid sync latency
  for (int nb : {16, 74, 148, 296}) {
    long long* dout = (long long*)out;
    int iters = 2000;
    void* args[] = {&dout, &iters};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)grid_sync_loop, nb, 256, args, 0, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    long long cyc = -1;
    if (e == cudaSuccess) cudaMemcpy(&cyc, dout, 8, cudaMemcpyDeviceToHost);
    printf("grid.sync blocks=%d: %lld cyc/sync (%s)\n", nb, cyc / iters, cudaGetErrorString(e));
  }
  // empty-kernel launch cost in a graph
  {
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; ++i) dmma_loop<<<1, 32, 0, s>>>(out, 0);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("graph-launched tiny kernel: %.2f us per kernel\n", ms * 1000.0 / 1000.0);
  }
  return 0;
}
