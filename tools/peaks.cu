// Per-pipe throughput microbenchmarks for the render roofline (SURVEY §8(d):
// "MUFU must be microbenchmarked on the box before quoting fractions").
// Each kernel runs a long unrolled loop of ONE instruction kind over ILP
// independent chains per thread at full occupancy; the result is lane
// operations per SM per clock (clock64 around the loop, max over CTAs) and
// operations per second (CUDA events). FP32 counts lanes (an FFMA2 is two FP32
// lane-ops per thread), as the roofline's P32 does. Build on the box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 8
#define ITERS 4096

__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float sina(float x) { float y; asm volatile("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float cosa(float x) { float y; asm volatile("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcpa(float x) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

enum Op { FFMA = 0, FFMA_IMM, FFMA2, FADD, FMUL, EX2, SIN, COS, RCP, DFMA, MIX_FMA_EX2, DADD,
          DMUL, F2F64, F2F32, NOPS };
static const char* kName[NOPS] = {"ffma", "ffma_imm", "ffma2", "fadd", "fmul", "mufu_ex2",
                                  "mufu_sin", "mufu_cos", "mufu_rcp", "dfma", "mix_8ffma_1ex2",
                                  "dadd", "dmul", "f2f_f64_f32", "f2f_f32_f64"};
// lane-ops per chain step
static const int kOps[NOPS] = {1, 1, 2, 1, 1, 1, 1, 1, 1, 1, 9, 1, 1, 1, 1};

template <int OP>
__global__ void k_bench(float* out, float b, float c, unsigned long long* cyc) {
  float a[ILP];
  double d[ILP];
  unsigned long long p[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    a[i] = 1e-3f * (threadIdx.x + i);
    d[i] = a[i];
    p[i] = ((unsigned long long)__float_as_uint(a[i]) << 32) | __float_as_uint(a[i] + 1.f);
  }
  const unsigned long long pb = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(b);
  const unsigned long long pc = ((unsigned long long)__float_as_uint(c) << 32) | __float_as_uint(c);
  const double db = b, dc = c;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if (OP == FFMA) a[i] = __fmaf_rn(a[i], b, c);
      if (OP == FFMA_IMM) a[i] = __fmaf_rn(a[i], 0.999f, 1e-4f);
      if (OP == FFMA2) p[i] = ffma2(p[i], pb, pc);
      if (OP == FADD) a[i] = __fadd_rn(a[i], b);
      if (OP == FMUL) a[i] = __fmul_rn(a[i], b);
      if (OP == EX2) a[i] = ex2a(a[i]);
      if (OP == SIN) a[i] = sina(a[i]);
      if (OP == COS) a[i] = cosa(a[i]);
      if (OP == RCP) a[i] = __fadd_rn(rcpa(a[i]), b);  // FADD keeps ptxas from folding rcp(rcp(x))
      if (OP == DFMA) d[i] = __fma_rn(d[i], db, dc);
      if (OP == DADD) d[i] = __dadd_rn(d[i], db);
      if (OP == DMUL) d[i] = __dmul_rn(d[i], db);
      // conversion chains: widen then narrow alternate through the other type,
      // one conversion per step counted (the FADD / DADD keep them dependent)
      if (OP == F2F64) { d[i] = __dadd_rn(d[i], (double)a[i]); a[i] = __fadd_rn(a[i], b); }
      if (OP == F2F32) { a[i] = __fadd_rn(__double2float_rn(d[i]), a[i]); d[i] = __dadd_rn(d[i], db); }
      if (OP == MIX_FMA_EX2) {
        float x = a[i];
#pragma unroll
        for (int k = 0; k < 8; ++k) x = __fmaf_rn(x, b, c);
        a[i] = ex2a(x);
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += a[i] + (float)d[i] + __uint_as_float((unsigned)p[i]);
  if (s == 1234.5f) out[0] = s;  // keep the chains alive
  if (threadIdx.x == 0) atomicMax(cyc, t1 - t0);
}

template <int OP>
void run(int sms, FILE* js, bool first) {
  const int threads = 512, ctas = sms * 4;  // 2048 threads per SM = 64 warps
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_bench<OP><<<ctas, threads>>>(out, 0.9999f, 1e-6f, cyc);  // warm-up
  cudaMemset(cyc, 0, 8);
  cudaEventRecord(e0);
  k_bench<OP><<<ctas, threads>>>(out, 0.9999f, 1e-6f, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double ops = (double)ctas * threads * ILP * ITERS * kOps[OP];
  // all 4 CTAs of an SM are co-resident (2048 threads), so per-SM ops / max CTA cycles
  const double per_sm_clk = ops / sms / (double)c;
  const double per_s = ops / (ms * 1e-3);
  printf("%-16s %8.2f lane-ops/SM/clk  %10.3e ops/s  (%.3f ms, %llu cyc => %.0f MHz)\n", kName[OP],
         per_sm_clk, per_s, ms, c, c / (ms * 1e3));
  fprintf(js, "%s  \"%s\": {\"per_sm_clk\": %.3f, \"ops_per_s\": %.4e, \"mhz\": %.0f}", first ? "" : ",\n",
          kName[OP], per_sm_clk, per_s, c / (ms * 1e3));
  cudaFree(out);
  cudaFree(cyc);
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  FILE* js = fopen(argc > 1 ? argv[1] : "peaks.json", "w");
  fprintf(js, "{\n \"sms\": %d,\n \"units\": \"lane-ops per SM per clock; FP32 counts lanes (ffma2 = 2)\",\n", sms);
  run<FFMA>(sms, js, true);
  run<FFMA_IMM>(sms, js, false);
  run<FFMA2>(sms, js, false);
  run<FADD>(sms, js, false);
  run<FMUL>(sms, js, false);
  run<EX2>(sms, js, false);
  run<SIN>(sms, js, false);
  run<COS>(sms, js, false);
  run<RCP>(sms, js, false);
  run<DFMA>(sms, js, false);
  run<MIX_FMA_EX2>(sms, js, false);
  run<DADD>(sms, js, false);
  run<DMUL>(sms, js, false);
  run<F2F64>(sms, js, false);
  run<F2F32>(sms, js, false);
  fprintf(js, "\n}\n");
  fclose(js);
  return 0;
}
