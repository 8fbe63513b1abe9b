// Instruction-throughput microbenchmark for the encode value path (sm_100a).
// Measures warp-instructions per clock per SMSP for the ops the value path is
// built from, alone and in pairs (to see which share a pipe). Not part of the
// product library.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_pipes tools/ubench_pipes.cu
//   tools/ubench_pipes
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define ITERS 2048
#define U 16  // independent chains per thread

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

template <int OP>
__global__ void __launch_bounds__(512) kern(float* out, long long* cycles, float seed) {
  float a[U], b[U];
  uint32_t u[U];
  double d[U];
  float2 p[U];
#pragma unroll
  for (int i = 0; i < U; ++i) {
    a[i] = seed + i + threadIdx.x;
    b[i] = seed * 0.5f + i;
    u[i] = __float_as_uint(a[i]) * 2654435761u;
    d[i] = a[i];
    p[i] = f2(a[i], b[i]);
  }
  const float2 c2 = f2(seed, -seed), k2 = f2(1.0001f, 0.9999f);
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < U; ++i) {
      if (OP == 0) p[i] = __fadd2_rn(p[i], c2);                        // FADD2
      if (OP == 1) p[i] = __ffma2_rn(p[i], k2, c2);                    // FFMA2 (3 pairs)
      if (OP == 2) p[i] = __fmul2_rn(p[i], k2);                        // FMUL2
      if (OP == 3) a[i] = a[i] + b[i];                                 // FADD
      if (OP == 4) a[i] = fmaf(a[i], b[i], a[(i + 1) % U]);            // FFMA 3-reg
      if (OP == 5) a[i] = fminf(a[i], fminf(fabsf(b[i]), fabsf(a[(i + 3) % U])));  // FMNMX3
      if (OP == 6) u[i] = u[i] ^ (u[(i + 1) % U] & u[(i + 2) % U]);    // LOP3
      if (OP == 7) u[i] = __funnelshift_l(u[(i + 5) % U], u[i], 1);    // SHF
      if (OP == 8) u[i] = u[i] * u[(i + 1) % U] + 12345u;              // IMAD
      if (OP == 9) d[i] = d[i] + (double)a[i];                         // F2F.F64.F32 + DADD
      if (OP == 10) d[i] = fma(d[i], 1.0000001, d[(i + 1) % U]);       // DFMA
      if (OP == 11) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1);      // SHFL
      if (OP == 12) u[i] = __byte_perm(u[i], u[(i + 1) % U], 0x7351);  // PRMT
      if (OP == 13) {  // FADD2 + LOP3 interleaved (pipe sharing)
        p[i] = __fadd2_rn(p[i], c2);
        u[i] = u[i] ^ (u[(i + 1) % U] & u[(i + 2) % U]);
      }
      if (OP == 14) {  // FADD2 + FMNMX3
        p[i] = __fadd2_rn(p[i], c2);
        a[i] = fminf(a[i], fminf(fabsf(b[i]), fabsf(a[(i + 3) % U])));
      }
      if (OP == 15) {  // LOP3 + SHF
        u[i] = u[i] ^ (u[(i + 1) % U] & u[(i + 2) % U]);
        u[(i + 8) % U] = __funnelshift_l(u[(i + 5) % U], u[(i + 8) % U], 1);
      }
      if (OP == 16) {  // FADD2 + FMUL2
        p[i] = __fadd2_rn(p[i], c2);
        p[(i + 8) % U] = __fmul2_rn(p[(i + 8) % U], k2);
      }
      if (OP == 17) {  // FFMA imm-form
        a[i] = fmaf(a[i], 1.0001f, 0.5f);
      }
      if (OP == 18) {  // F2F.F64.F32 alone
        d[i] = (double)a[i];
        a[i] = __uint_as_float(__double2hiint(d[i]) ^ 0x1);
      }
      if (OP == 20) {  // FADD + LOP3
        a[i] = a[i] + b[i];
        u[i] = u[i] ^ (u[(i + 1) % U] & u[(i + 2) % U]);
      }
      if (OP == 21) {  // FADD + SHF
        a[i] = a[i] + b[i];
        u[i] = __funnelshift_l(u[(i + 5) % U], u[i], 1);
      }
      if (OP == 22) {  // FADD + FMNMX3
        a[i] = a[i] + b[i];
        b[(i + 4) % U] = fminf(b[(i + 4) % U], fminf(fabsf(a[(i + 7) % U]), fabsf(a[(i + 3) % U])));
      }
      if (OP == 23) {  // FMUL + SHF + LOP3 (1:1:1)
        a[i] = a[i] * b[i];
        u[i] = __funnelshift_l(u[(i + 5) % U], u[i], 1);
        u[(i + 8) % U] = u[(i + 8) % U] ^ (u[(i + 1) % U] & u[(i + 2) % U]);
      }
      if (OP == 24) {  // FADD with |x| input
        a[i] = fabsf(a[i]) - b[i];
      }
      if (OP == 25) {  // FFMA2 with an immediate (sub form)
        p[i] = __ffma2_rn(p[i], f2(-1.f, -1.f), c2);
      }
      if (OP == 26) {  // FADD + FADD2
        a[i] = a[i] + b[i];
        p[i] = __fadd2_rn(p[i], c2);
      }
      if (OP == 27) {  // FMUL x2 + SHF  (2:1)
        a[i] = a[i] * b[i];
        b[(i + 3) % U] = b[(i + 3) % U] * a[(i + 5) % U];
        u[i] = __funnelshift_l(u[(i + 5) % U], u[i], 1);
      }
      if (OP == 28) {  // IMAD + LOP3
        u[i] = u[i] * u[(i + 1) % U] + 12345u;
        u[(i + 8) % U] = u[(i + 8) % U] ^ (u[(i + 1) % U] & u[(i + 2) % U]);
      }
      if (OP == 29) {  // FADD + FADD + FMNMX3 (2:1)
        a[i] = a[i] + b[i];
        b[(i + 5) % U] = b[(i + 5) % U] + a[(i + 9) % U];
        a[(i + 4) % U] = fminf(a[(i + 4) % U], fminf(fabsf(b[(i + 7) % U]), fabsf(b[(i + 3) % U])));
      }
      if (OP == 30) {  // DFMA + FADD (fp64 pipe vs fp32)
        d[i] = fma(d[i], 1.0000001, d[(i + 1) % U]);
        a[i] = a[i] + b[i];
      }
      if (OP == 31) {  // F2F.F64.F32 + FADD
        d[i] = (double)a[(i + 3) % U];
        a[i] = a[i] + __double2loint(d[(i + 5) % U]) * 0.f + b[i];
      }
      if (OP == 19) {  // IMAD.U32 x<<16 (bf16 lo unpack) on the fma pipe + LOP3 hi
        a[i] = __uint_as_float(u[i] << 16);
        b[i] = __uint_as_float(u[i] & 0xffff0000u);
        u[i] += __float_as_uint(a[i]) ^ __float_as_uint(b[i]);
      }
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < U; ++i) acc += a[i] + b[i] + p[i].x + p[i].y + (float)u[i] + (float)d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int per_iter, float* out, long long* cyc, int sms, int threads) {
  kern<OP><<<sms, threads>>>(out, cyc, 1.5f);
  cudaDeviceSynchronize();
  kern<OP><<<sms, threads>>>(out, cyc, 1.5f);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double warps_per_smsp = threads / 32.0 / 4.0;
  const double instr = (double)ITERS * U * per_iter * warps_per_smsp;  // warp-instr per SMSP
  printf("%-28s %6.3f warp-instr/clk/SMSP  (%.2f clk per instr)\n", name, instr / mx, mx / instr);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * sms * 512);
  cudaMalloc(&cyc, sizeof(long long) * 1024);
  const int T = 512;
  run<0>("FADD2", 1, out, cyc, sms, T);
  run<1>("FFMA2", 1, out, cyc, sms, T);
  run<2>("FMUL2", 1, out, cyc, sms, T);
  run<3>("FADD", 1, out, cyc, sms, T);
  run<4>("FFMA 3-reg", 1, out, cyc, sms, T);
  run<17>("FFMA imm", 1, out, cyc, sms, T);
  run<5>("FMNMX3 (|b|,|c|)", 1, out, cyc, sms, T);
  run<6>("LOP3", 1, out, cyc, sms, T);
  run<7>("SHF funnel", 1, out, cyc, sms, T);
  run<8>("IMAD", 1, out, cyc, sms, T);
  run<12>("PRMT", 1, out, cyc, sms, T);
  run<9>("F2F.F64.F32 + DADD", 2, out, cyc, sms, T);
  run<18>("F2F.F64.F32 + LOP", 2, out, cyc, sms, T);
  run<10>("DFMA", 1, out, cyc, sms, T);
  run<11>("SHFL", 1, out, cyc, sms, T);
  run<13>("FADD2 + LOP3", 2, out, cyc, sms, T);
  run<14>("FADD2 + FMNMX3", 2, out, cyc, sms, T);
  run<15>("LOP3 + SHF", 2, out, cyc, sms, T);
  run<16>("FADD2 + FMUL2", 2, out, cyc, sms, T);
  run<19>("bf16 unpack (SHL,LOP,LOP3,IADD)", 4, out, cyc, sms, T);
  run<20>("FADD + LOP3", 2, out, cyc, sms, T);
  run<21>("FADD + SHF", 2, out, cyc, sms, T);
  run<22>("FADD + FMNMX3", 2, out, cyc, sms, T);
  run<23>("FMUL + SHF + LOP3", 3, out, cyc, sms, T);
  run<24>("FADD |x| - y", 1, out, cyc, sms, T);
  run<25>("FFMA2 imm (sub)", 1, out, cyc, sms, T);
  run<26>("FADD + FADD2", 2, out, cyc, sms, T);
  run<27>("FMUL x2 + SHF", 3, out, cyc, sms, T);
  run<28>("IMAD + LOP3", 2, out, cyc, sms, T);
  run<29>("FADD x2 + FMNMX3", 3, out, cyc, sms, T);
  run<30>("DFMA + FADD", 2, out, cyc, sms, T);
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
