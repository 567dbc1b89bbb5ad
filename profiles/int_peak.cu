// int_peak.cu — measured integer-pipe throughput of the B200 (sm_100a) for the ALU roofline
// ("the builder must measure it: a dependent-free mul.hi / IMAD / IADD3
// throughput microbenchmark"; VERDICT r1 "Next round" #2).
//
// Each kernel runs CH independent dependency chains per thread (so throughput, not latency,
// binds), 8 warps per SMSP-quadrant x 4 (1024 threads per CTA) x k CTAs per SM, for ITERS loop
// trips; one chain step is ONE SASS instruction of the named kind (inline PTX chosen so ptxas
// emits exactly that instruction; checked with cuobjdump -sass, see int_peak_sass.txt).
// Output: warp-instructions per clock per SM and lane-ops per clock per SM (x32), with the SM
// clock read through NVML during the run.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak int_peak.cu -lnvidia-ml
//   ./int_peak > int_peak.json
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <nvml.h>
#include <thread>
#include <atomic>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int CH = 8;         // independent chains per thread
constexpr int ITERS = 4096;   // loop trips (CH instructions of the measured kind per trip)

// one chain step per op kind (each a single SASS instruction)
template <int OP>
__device__ __forceinline__ void step(uint32_t& x, uint32_t a, uint32_t b, uint64_t& w) {
  if constexpr (OP == 0) {        // IMAD          x = x * a + b
    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(b));
  } else if constexpr (OP == 1) { // IMAD.HI.U32   x = hi(x * a) + b
    asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(b));
  } else if constexpr (OP == 2) { // IMAD.WIDE.U32 w = x * a + w  (64-bit accumulate)
    asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w) : "r"((uint32_t)w), "r"(a));
  } else if constexpr (OP == 3) { // IADD3         x = x + a + b
    asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(x) : "r"(a), "r"(b));
  } else if constexpr (OP == 4) { // VIADDMNMX     x = min(x + a, b)
    uint32_t t;
    asm volatile("add.u32 %1, %0, %2;\n\tmin.u32 %0, %1, %3;" : "+r"(x), "=r"(t) : "r"(a), "r"(b));
  } else if constexpr (OP == 5) { // LOP3 x2       x = lop3(x, y, b), y = lop3(y, x, a) (two mixed chains)
    uint32_t y = (uint32_t)w;
    asm volatile("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(x) : "r"(y), "r"(b));
    asm volatile("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(y) : "r"(x), "r"(a));
    w = y;
  } else if constexpr (OP == 6) { // 32-bit Shoup modmul (the NTT / epilogue product, mulsh32)
    const uint32_t hq = __umulhi(x, b);
    const uint32_t r = x * a - hq * 0x7ffe0001u;
    x = min(r, r - 0x7ffe0001u);
  } else if constexpr (OP == 7) { // 64-bit high product __umul64hi (64-bit Shoup / Barrett)
    w = __umul64hi(w, (uint64_t)a << 32 | b) + w;
  } else if constexpr (OP == 8) { // Montgomery MAC pair + REDC (k_vecmat_*_mont inner step, 2 products)
    const uint64_t s = (uint64_t)x * a + (uint64_t)(x ^ b) * b;
    const uint32_t m = (uint32_t)s * 0x7ffdffffu;
    const uint32_t t = (uint32_t)((s + (uint64_t)m * 0x7ffe0001u) >> 32);
    x = min(t, t - 0x7ffe0001u);
  } else if constexpr (OP == 9) {  // 64-bit Harvey Cooley-Tukey butterfly (the cfg2 / cfg3 NTT's step): the pair
    // (w, x-as-64) in [0, 4q): X = w mod 2q; T = y*tw - hi64(y*twsh)*q; w' = X + T; y' = X - T + 2q
    const uint64_t q = 0x0ffffffffffc0001ull, two_q = 2 * q;
    const uint64_t tw = (uint64_t)a << 28 | b, twsh = (uint64_t)b << 32 | a;
    uint64_t y = (uint64_t)x << 29 | x;
    const uint64_t X = w >= two_q ? w - two_q : w;
    const uint64_t T = y * tw - __umul64hi(y, twsh) * q;
    w = X + T;
    y = X - T + two_q;
    x = (uint32_t)(y >> 13);
  } else if constexpr (OP == 10) { // 32-bit strict Cooley-Tukey butterfly (31-bit primes: values in [0, q))
    const uint32_t q = 0x7ffe0001u;
    uint32_t y = (uint32_t)w;
    const uint32_t r = y * a - __umulhi(y, b) * q;
    const uint32_t T = min(r, r - q);
    const uint32_t u = min(x + T, x + T - q);
    y = min(x - T + q, x - T);
    x = u;
    w = y;
  } else if constexpr (OP == 11) { // 32-bit lazy Cooley-Tukey butterfly (q < 2^30: values in [0, 4q))
    const uint32_t q = 0x3ffc0001u;
    uint32_t y = (uint32_t)w;
    const uint32_t X = min(x, x - 2 * q);
    const uint32_t T = y * a - __umulhi(y, b) * q;
    x = X + T;
    y = X - T + 2 * q;
    w = y;
  }
}

template <int OP>
__global__ void __launch_bounds__(1024) k_peak(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x[CH];
  uint64_t w[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x + c; w[c] = x[c] * 3ull; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) step<OP>(x[c], a, b, w[c]);
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= x[c] ^ (uint32_t)w[c] ^ (uint32_t)(w[c] >> 32);
  if (acc == 0x12345678u) out[blockIdx.x] = acc;   // keeps the chains live
}

static std::atomic<bool> g_stop{false};
static std::vector<unsigned> g_clk;

static void sampler(nvmlDevice_t h) {
  while (!g_stop) {
    unsigned c = 0;
    if (nvmlDeviceGetClockInfo(h, NVML_CLOCK_SM, &c) == NVML_SUCCESS) g_clk.push_back(c);
    std::this_thread::sleep_for(std::chrono::milliseconds(20));
  }
}

template <int OP>
static void run(const char* name, int insts_per_step, int sms, uint32_t* d_out, bool last) {
  const int ctas = sms * 2;   // 2 x 1024 threads per SM (64 warps = full occupancy at <= 32 regs)
  k_peak<OP><<<ctas, 1024>>>(d_out, 0x9e3779b9u, 0x7ffe0001u);   // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  g_clk.clear();
  const int reps = 20;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) k_peak<OP><<<ctas, 1024>>>(d_out, 0x9e3779b9u, 0x7ffe0001u);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned> c = g_clk;
  std::sort(c.begin(), c.end());
  const double mhz = c.empty() ? 1965.0 : c[c.size() / 2];
  const double steps = (double)reps * ctas * 1024 * ITERS * CH;   // lane-steps
  const double warp_inst = steps / 32 * insts_per_step;
  const double clk = ms * 1e-3 * mhz * 1e6;
  printf("  \"%s\": {\"lane_steps_per_clk_per_sm\": %.2f, \"warp_inst_per_clk_per_sm\": %.3f, "
         "\"G_lane_steps_per_s\": %.1f, \"sass_inst_per_step\": %d, \"sm_mhz\": %.0f, \"ms\": %.3f}%s\n",
         name, steps / clk / sms, warp_inst / clk / sms, steps / (ms * 1e-3) / 1e9, insts_per_step, mhz, ms,
         last ? "" : ",");
}

int main() {
  nvmlInit();
  nvmlDevice_t h;
  nvmlDeviceGetHandleByIndex(0, &h);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint32_t* d_out;
  CK(cudaMalloc(&d_out, 1 << 20));
  std::thread t(sampler, h);
  printf("{\n \"sms\": %d, \"chains_per_thread\": %d, \"threads_per_sm\": 2048,\n \"ops\": {\n", sms, CH);
  // SASS instructions per chain step, from cuobjdump -sass of this file (int_peak_sass.txt)
  run<0>("IMAD", 1, sms, d_out, false);
  run<1>("IMAD.HI.U32", 1, sms, d_out, false);
  run<2>("mad_wide_u32_64bit_accumulate_chain (IMAD.WIDE.U32 + IADD3 + IADD3.X, ptxas splits the add)", 0, sms, d_out, false);
  run<3>("IADD3", 1, sms, d_out, false);
  run<4>("VIADDMNMX", 1, sms, d_out, false);
  run<5>("LOP3", 2, sms, d_out, false);
  run<6>("shoup32_modmul", 0, sms, d_out, false);
  run<7>("umul64hi", 0, sms, d_out, false);
  run<8>("mont_mac_pair_redc", 0, sms, d_out, false);
  run<9>("ct_butterfly_64bit_harvey", 0, sms, d_out, false);
  run<10>("ct_butterfly_32bit_strict", 0, sms, d_out, false);
  run<11>("ct_butterfly_32bit_lazy", 0, sms, d_out, true);
  printf(" }\n}\n");
  g_stop = true;
  t.join();
  return 0;
}
