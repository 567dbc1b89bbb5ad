// Library pin for the Philox4x32-10 generator: exposes cuRAND's own
// curand_Philox4x32_10(counter, key) on the host so tests can compare the
// oracle's generator with NVIDIA's. Test infrastructure only.
#define QUALIFIERS static inline __host__ __device__
#include <cuda_runtime.h>
#include <curand_philox4x32_x.h>

extern "C" void curand_philox_host(const unsigned* ctr, const unsigned* key, unsigned* out) {
  uint4 c = make_uint4(ctr[0], ctr[1], ctr[2], ctr[3]);
  uint2 k = make_uint2(key[0], key[1]);
  uint4 r = curand_Philox4x32_10(c, k);
  out[0] = r.x; out[1] = r.y; out[2] = r.z; out[3] = r.w;
}
