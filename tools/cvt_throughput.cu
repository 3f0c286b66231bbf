// Microbenchmark: byte -> float conversion options (lanes/clk/SM) and whether they
// share a pipe: PRMT (biased float), I2F.F32.U8 with a byte selector, and both mixed.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters, unsigned seed) {
  unsigned u0 = seed ^ threadIdx.x, u1 = u0 * 3u, u2 = u0 * 5u, u3 = u0 * 7u;
  float f0 = 0.f, f1 = 0.f, f2 = 0.f, f3 = 0.f;
  unsigned p0 = 0, p1 = 0, p2 = 0, p3 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) {  // PRMT only (xor-accumulate to keep the chain alive)
        p0 ^= __byte_perm(u0, 0x4B000000u, 0x7440u | (j & 3));
        p1 ^= __byte_perm(u1, 0x4B000000u, 0x7441u);
        p2 ^= __byte_perm(u2, 0x4B000000u, 0x7442u);
        p3 ^= __byte_perm(u3, 0x4B000000u, 0x7443u);
        u0 += p3; u1 += p0; u2 += p1; u3 += p2;
      }
      if (OP == 1) {  // I2F from a selected byte
        f0 += static_cast<float>((u0 >> 8 * (j & 3)) & 0xFFu);
        f1 += static_cast<float>((u1 >> 8) & 0xFFu);
        f2 += static_cast<float>((u2 >> 16) & 0xFFu);
        f3 += static_cast<float>(u3 >> 24);
        u0 += 0x01010101u; u1 += 0x01010101u; u2 += 0x01010101u; u3 += 0x01010101u;
      }
      if (OP == 2) {  // both: 2 PRMT + 2 I2F per step
        p0 ^= __byte_perm(u0, 0x4B000000u, 0x7440u);
        p1 ^= __byte_perm(u1, 0x4B000000u, 0x7441u);
        f2 += static_cast<float>((u2 >> 16) & 0xFFu);
        f3 += static_cast<float>(u3 >> 24);
        u0 += p1; u1 += p0; u2 += 0x01010101u; u3 += 0x01010101u;
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = f0 + f1 + f2 + f3 + (float)(p0 ^ p1 ^ p2 ^ p3);
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* f; cudaMalloc(&f, 1 << 24);
  const char* names[] = {"PRMT (x4 + 4 IADD)", "I2F.F32 byte (x4 + FADD + IADD)", "2 PRMT + 2 I2F"};
  const int blocks = sms * 8, threads = 256, iters = 4000;
  for (int op = 0; op < 3; ++op) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (op == 0) k<0><<<blocks, threads>>>(f, iters, 1u);
      if (op == 1) k<1><<<blocks, threads>>>(f, iters, 1u);
      if (op == 2) k<2><<<blocks, threads>>>(f, iters, 1u);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double convs = double(blocks) * threads * iters * 8 * 4;
    printf("%-34s %8.1f Gconv/s  %6.1f conv-lanes/clk/SM @1965MHz\n", names[op], convs / ms / 1e6,
           convs / (ms * 1e-3) / 1.965e9 / sms);
  }
  return 0;
}
