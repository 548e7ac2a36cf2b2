// Latency probe: dependent chains of FP64 sqrt, div, rsqrt, rcp (+1 Newton), fma on one thread.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0) {
  double x = x0, y;
  long long t0, t1;
  // fma
  y = x; t0 = clock64(); for (int i = 0; i < 256; ++i) y = fma(y, 0.999999, 1e-9); t1 = clock64(); cyc[0] = t1 - t0; out[0] = y;
  y = x; t0 = clock64(); for (int i = 0; i < 256; ++i) y = sqrt(y + 1.0); t1 = clock64(); cyc[1] = t1 - t0; out[1] = y;
  y = x; t0 = clock64(); for (int i = 0; i < 256; ++i) y = 1.0 / (y + 1.0); t1 = clock64(); cyc[2] = t1 - t0; out[2] = y;
  y = x; t0 = clock64(); for (int i = 0; i < 256; ++i) y = rsqrt(y + 1.0); t1 = clock64(); cyc[3] = t1 - t0; out[3] = y;
  y = x; t0 = clock64(); for (int i = 0; i < 256; ++i) y = __drcp_rn(y + 1.0); t1 = clock64(); cyc[4] = t1 - t0; out[4] = y;
  y = x; t0 = clock64(); for (int i = 0; i < 256; ++i) { double d = y + 1.0; double r = (double)(1.0f / (float)d); r = fma(r, fma(-d, r, 1.0), r); r = fma(r, fma(-d, r, 1.0), r); y = fma(r, fma(-d, r, 1.0), r);} t1 = clock64(); cyc[5] = t1 - t0; out[5] = y;
  y = x; t0 = clock64(); for (int i = 0; i < 256; ++i) { double d = y + 1.0, r; asm("rsqrt.approx.f64 %0, %1;" : "=d"(r) : "d"(d)); double hd = 0.5 * d; r = r * fma(-hd * r, r, 1.5); y = r * fma(-hd * r, r, 1.5); } t1 = clock64(); cyc[7] = t1 - t0; out[7] = y;
  y = x; t0 = clock64(); for (int i = 0; i < 256; ++i) { double d = y + 1.0, r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d)); r = fma(r, fma(-d, r, 1.0), r); y = fma(r, fma(-d, r, 1.0), r); } t1 = clock64(); cyc[8] = t1 - t0; out[8] = y;
  y = x; t0 = clock64(); for (int i = 0; i < 256; ++i) { double d = y + 1.0, r; asm("rsqrt.approx.f64 %0, %1;" : "=d"(r) : "d"(d)); y = r; } t1 = clock64(); cyc[9] = t1 - t0; out[9] = y;
  y = x; t0 = clock64(); for (int i = 0; i < 256; ++i) y = (y + 1.0) * 0.5 + __shfl_xor_sync(0xffffffffu, y, 1) * 1e-9; t1 = clock64(); cyc[6] = t1 - t0; out[6] = y;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 64 * 8);
  k<<<1, 32>>>(o, c, 0.5); k<<<1, 32>>>(o, c, 0.5);
  long long h[10]; cudaMemcpy(h, c, 10 * 8, cudaMemcpyDeviceToHost);
  const char* n[] = {"fma", "sqrt(+add)", "div(+add)", "rsqrt(+add)", "drcp_rn(+add)", "rcp f32+3 newton(+add)", "shfl+2fma", "rsqrt.approx+2 newton", "rcp.approx+2 newton", "rsqrt.approx(+add)"};
  for (int i = 0; i < 10; ++i) printf("%-24s %6.1f cycles/iter\n", n[i], h[i] / 256.0);
}
