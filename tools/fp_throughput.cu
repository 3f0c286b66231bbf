// Microbenchmark: per-SM throughput of the arithmetic the resample kernel can
// use (DMUL/DADD vs FFMA/FADD vs I2F/F2F conversions) on the local GPU.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* outd, float* outf, int iters, double a, float af) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  float f0 = threadIdx.x * 1e-3f, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3;
  unsigned u0 = threadIdx.x, u1 = u0 + 1, u2 = u0 + 2, u3 = u0 + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) { x0 = __dmul_rn(x0, a); x1 = __dmul_rn(x1, a); x2 = __dmul_rn(x2, a); x3 = __dmul_rn(x3, a); }
      if (OP == 1) { x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a); }
      if (OP == 2) { f0 = __fmaf_rn(f0, af, af); f1 = __fmaf_rn(f1, af, af); f2 = __fmaf_rn(f2, af, af); f3 = __fmaf_rn(f3, af, af); }
      if (OP == 3) { f0 = __fadd_rn(f0, af); f1 = __fadd_rn(f1, af); f2 = __fadd_rn(f2, af); f3 = __fadd_rn(f3, af); }
      if (OP == 4) { x0 += (double)u0; x1 += (double)u1; x2 += (double)u2; x3 += (double)u3; u0 += 3; u1 += 3; u2 += 3; u3 += 3; }
      if (OP == 5) { f0 += (float)u0; f1 += (float)u1; f2 += (float)u2; f3 += (float)u3; u0 += 3; u1 += 3; u2 += 3; u3 += 3; }
      if (OP == 6) { x0 = __dadd_rd(x0, a); x1 = __dadd_rd(x1, a); x2 = __dadd_rd(x2, a); x3 = __dadd_rd(x3, a); }
      if (OP == 7) { x0 = floor(x0 * a); x1 = floor(x1 * a); x2 = floor(x2 * a); x3 = floor(x3 * a); }
      if (OP == 8) {
        unsigned long long p0, p1, q;
        asm("mov.b64 %0, {%1, %2};" : "=l"(p0) : "f"(f0), "f"(f1));
        asm("mov.b64 %0, {%1, %2};" : "=l"(p1) : "f"(f2), "f"(f3));
        asm("mov.b64 %0, {%1, %1};" : "=l"(q) : "f"(af));
        asm("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p0) : "l"(q));
        asm("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p1) : "l"(q));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(f0), "=f"(f1) : "l"(p0));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(f2), "=f"(f3) : "l"(p1));
      }
      if (OP == 9) { u0 = __byte_perm(u0, 0x4B000000u, 0x7440u); u1 = __byte_perm(u1, 0x4B000000u, 0x7441u); u2 = __byte_perm(u2, 0x4B000000u, 0x7442u); u3 = __byte_perm(u3, 0x4B000000u, 0x7443u); }
    }
  }
  outd[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
  outf[blockIdx.x * blockDim.x + threadIdx.x] = f0 + f1 + f2 + f3 + u0 + u1 + u2 + u3;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d; float* f; cudaMalloc(&d, 1 << 24); cudaMalloc(&f, 1 << 24);
  const char* names[] = {"DMUL", "DADD", "FFMA", "FADD", "I2F.F64+DADD", "I2F.F32+FADD", "DADD.RM", "DMUL+FRND.F64", "FFMA2 (x2 lanes)", "PRMT"};
  const int blocks = sms * 8, threads = 256, iters = 2000;
  for (int op = 0; op < 10; ++op) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto launch = [&]() {
      switch (op) {
        case 0: k<0><<<blocks, threads>>>(d, f, iters, 1.0000001, 1.0000001f); break;
        case 1: k<1><<<blocks, threads>>>(d, f, iters, 1.0000001, 1.0000001f); break;
        case 2: k<2><<<blocks, threads>>>(d, f, iters, 1.0000001, 0.999999f); break;
        case 3: k<3><<<blocks, threads>>>(d, f, iters, 1.0000001, 1.0000001f); break;
        case 4: k<4><<<blocks, threads>>>(d, f, iters, 1.0000001, 1.0000001f); break;
        case 5: k<5><<<blocks, threads>>>(d, f, iters, 1.0000001, 1.0000001f); break;
        case 6: k<6><<<blocks, threads>>>(d, f, iters, 1.0000001, 1.0000001f); break;
        case 7: k<7><<<blocks, threads>>>(d, f, iters, 1.0000001, 1.0000001f); break;
        case 8: k<8><<<blocks, threads>>>(d, f, iters, 1.0000001, 0.999999f); break;
        case 9: k<9><<<blocks, threads>>>(d, f, iters, 1.0000001, 0.999999f); break;
      }
    };
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = double(blocks) * threads * iters * 8 * 4;
    printf("%-16s %8.1f Gop/s  %6.1f lane-ops/clk/SM (at %d MHz nominal)\n", names[op],
           ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
