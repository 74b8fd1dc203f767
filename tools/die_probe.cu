// die_probe.cu -- does WHERE a store lands (same die as the writing SM, or the other die) change
// the energy per byte written?  B200 is two dies; each 2-KB address chunk lives behind one die's
// L2 / HBM (B300_MICROARCH.md: "addr->die ~Bernoulli(0.5) @ 2KB-grain").  This probe
//   1. times an L2-hit load from every SM to a sample of chunks (near die ~234, far ~262 cycles)
//      -> the SM -> die map (host side clusters the SMs);
//   2. classifies every chunk of a buffer from SMs of known die;
//   3. writes the buffer with every warp's chunks (a) mixed, (b) all on its own die, (c) all on
//      the other die, so the host can compare power at equal bytes.
// Tuning evidence only (tools/die_probe.py); not part of libfls.
#include <cstdint>

namespace {
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ long long clk() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ldcg(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// average L2-hit latency (cycles) of `reps` loads into chunk c (lines 128 B apart, warmed first)
__device__ float chunk_latency(const unsigned long long *buf, long long c, int reps) {
  const unsigned long long *p = buf + c * 256;  // 2 KB = 256 u64
  unsigned long long acc = 0;
  for (int l = 0; l < 16; ++l) acc += ldcg(p + l * 16);
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    const unsigned long long *q = p + (r & 15) * 16;
    const long long t0 = clk();
    const unsigned long long v = ldcg(q);
    asm volatile("add.u64 %0, %0, %1;" : "+l"(acc) : "l"(v));
    const long long t1 = clk();
    tot += t1 - t0;
  }
  if (acc == 0x123456789abcdefull) asm volatile("trap;");
  return (float)tot / (float)reps;
}
}  // namespace

extern "C" {

// grid: one 32-thread CTA per SM (or more); out[cta * nchunk + c]
__global__ void die_lat_kernel(const unsigned long long *buf, int nchunk, int reps, float *out,
                               int *sm_of_cta) {
  if (threadIdx.x == 0) sm_of_cta[blockIdx.x] = (int)smid();
  for (int c = threadIdx.x; c < nchunk; c += 32) out[(long long)blockIdx.x * nchunk + c] = chunk_latency(buf, c, reps);
}

// chunk c measured by whichever CTA takes it: lat[c], sm[c]
__global__ void die_classify_kernel(const unsigned long long *buf, long long nchunk, int reps,
                                    float *lat, int *sm) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < nchunk; c += stride) {
    lat[c] = chunk_latency(buf, c, reps);
    sm[c] = (int)smid();
  }
}

// mode 0: every warp takes chunks from the whole list (mixed dies); mode 1: a warp takes chunks of
// its own die; mode 2: chunks of the other die.  lists: [die 0 chunks | die 1 chunks];
// counters[3] zeroed by the host; `passes` passes over each list.
__global__ void die_write_kernel(double *buf, const long long *lists, long long n0, long long n1,
                                 const int *die_of_sm, int mode, int passes,
                                 unsigned long long *counters) {
  const int lane = threadIdx.x & 31;
  const int die = die_of_sm[smid()];
  const int want = mode == 1 ? die : 1 - die;
  const long long nall = n0 + n1;
  const long long n = mode == 0 ? nall : (want == 0 ? n0 : n1);
  const long long *lst = mode == 0 ? lists : (want == 0 ? lists : lists + n0);
  unsigned long long *ctr = mode == 0 ? counters + 2 : counters + want;
  const unsigned long long total = (unsigned long long)n * passes;
  const double v = (double)threadIdx.x;
  for (;;) {
    unsigned long long k0 = 0;
    if (lane == 0) k0 = atomicAdd(ctr, 8ull);
    k0 = __shfl_sync(0xffffffffu, k0, 0);
    if (k0 >= total) break;
    for (int u = 0; u < 8 && k0 + u < total; ++u) {
      const long long c = lst[(k0 + u) % n];
      double *p = buf + c * 256 + lane * 2;
#pragma unroll
      for (int s = 0; s < 4; ++s)
        asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p + s * 64), "d"(v), "d"(v) : "memory");
    }
  }
}

}  // extern "C"

// host launchers (ctypes)
extern "C" int die_lat(const void *buf, int nchunk, int reps, float *out, int *sm_of_cta, int grid) {
  die_lat_kernel<<<grid, 32>>>((const unsigned long long *)buf, nchunk, reps, out, sm_of_cta);
  return (int)cudaGetLastError();
}
extern "C" int die_classify(const void *buf, long long nchunk, int reps, float *lat, int *sm, int grid) {
  die_classify_kernel<<<grid, 32>>>((const unsigned long long *)buf, nchunk, reps, lat, sm);
  return (int)cudaGetLastError();
}
extern "C" int die_write(void *buf, const long long *lists, long long n0, long long n1,
                         const int *die_of_sm, int mode, int passes, unsigned long long *counters,
                         int grid, int threads) {
  die_write_kernel<<<grid, threads>>>((double *)buf, lists, n0, n1, die_of_sm, mode, passes, counters);
  return (int)cudaGetLastError();
}
