// ReachMap4D (reachability.hpp:14-94, reachability.cpp:10-190) on the device.
//   build: thread per FK sample -- joint values from make_stream(seed, {"reach", s}), the
//     chain product in the reference's order ((t * origin) * motion, then * ee_offset),
//     cylindrical (r, z) bin with a correctly rounded hypot (glibc's is), the tool
//     inclination psi = acos(R22) bin, atomicOr into the 64-bit occupancy words;
//   query_batch / placement_filter: thread per instance, inverse_rigid(base) * target,
//     the same bin, one bit lookup.
#include <stdexcept>
#include <string>

#include "sb_crmath.cuh"
#include "sb_dev.cuh"
#include "sb_joint.cuh"
#include "sb_reach.h"
#include "sb_reachdev.cuh"

using namespace sbd;

namespace {

constexpr int kBlock = 256;
constexpr uint64_t kReachSalt = 0x7265616368ULL;  // "reach" (reachability.cpp:79)

inline unsigned grid_for(uint64_t n) { return static_cast<unsigned>((n + kBlock - 1) / kBlock); }
inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

__device__ __forceinline__ void load_colmajor(const double* c, M34& M) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 4; ++k) M.m[4 * r + k] = c[4 * k + r];
}

__global__ void k_reach_build(const double* links, int n_links, sbk::ReachGrid g, M34 ee,
                              uint64_t samples, uint64_t seed, unsigned long long* occ,
                              unsigned* counts) {
  const uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (s >= samples) return;
  Pcg rng = Pcg::seeded(stream_seed2(seed, kReachSalt, s));
  M34 t, a, b;
#pragma unroll
  for (int k = 0; k < 12; ++k) t.m[k] = 0.0;
  t.m[0] = t.m[5] = t.m[10] = 1.0;
  for (int l = 0; l < n_links; ++l) {  // KinematicChain::fk (reachability.cpp:10-18)
    const double* L = links + 18 * l;
    sbk::GraphJoint j;
    j.kind = (int32_t)L[12];
    j.axis[0] = L[13];
    j.axis[1] = L[14];
    j.axis[2] = L[15];
    const double v = L[16] + (L[17] - L[16]) * rng.next_double();  // uniform(lo, hi)
    M34 O, J;
#pragma unroll
    for (int k = 0; k < 12; ++k) O.m[k] = L[k];
    mul34(t, O, a);
    joint_motion(j, v, J);
    mul34(a, J, t);
  }
  mul34(t, ee, b);
  uint64_t ir, iz;
  if (!reach_bin(g, b.m[3], b.m[7], b.m[11], ir, iz)) return;
  // tool_inclination: axis = R * (0,0,1) (shim order), psi = acos(clamp(-axis.z, -1, 1))
  const double axz = (b.m[8] * 0.0 + b.m[9] * 0.0) + b.m[10] * 1.0;
  const double c = fmin(fmax(-axz, -1.0), 1.0);
  const double psi = acos(c);
  uint64_t ipsi = (uint64_t)(psi / g.psi_res);
  if (ipsi > g.npsi - 1) ipsi = g.npsi - 1;
  const uint64_t idx = (ir * g.nz + iz) * g.npsi + ipsi;
  atomicOr(occ + (idx >> 6), 1ull << (idx & 63));
  atomicAdd(counts + idx, 1u);
}

__global__ void k_reach_any(sbk::ReachGrid g, const unsigned long long* occ,
                            unsigned long long* occ_any) {
  const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;  // (ir, iz) cell
  if (c >= g.nr * g.nz) return;
  bool any = false;
  for (uint64_t ip = 0; ip < g.npsi && !any; ++ip) any = reach_bit(occ, c * g.npsi + ip);
  if (any) atomicOr(occ_any + (c >> 6), 1ull << (c & 63));
}

// ReachMap4D::query (reachability.cpp:128-141) of a point in the base frame
__device__ __forceinline__ bool query(const sbk::ReachGrid& g, const unsigned long long* occ,
                                      const unsigned long long* occ_any, double x, double y,
                                      double z, double incl) {
  uint64_t ir, iz;
  if (!reach_bin(g, x, y, z, ir, iz)) return false;
  if (isnan(incl)) return reach_bit(occ_any, ir * g.nz + iz);  // no inclination: any psi
  const double psi = fmin(fmax(incl, 0.0), 3.14159265358979323846);
  uint64_t ipsi = (uint64_t)(psi / g.psi_res);
  if (ipsi > g.npsi - 1) ipsi = g.npsi - 1;
  return reach_bit(occ, (ir * g.nz + iz) * g.npsi + ipsi);
}

__global__ void k_reach_query(sbk::ReachGrid g, const unsigned long long* occ,
                              const unsigned long long* occ_any, const double* base16,
                              const double* targets, uint64_t n, double incl, uint8_t* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  M34 B, I;
  load_colmajor(base16 + 16 * i, B);
  inverse_rigid(B, I);
  double x, y, z;
  xform(I, targets[3 * i], targets[3 * i + 1], targets[3 * i + 2], x, y, z);
  out[i] = query(g, occ, occ_any, x, y, z, incl) ? 1 : 0;
}

__global__ void k_reach_filter(sbk::ReachGrid g, const unsigned long long* occ_any,
                               const double* base16, const double* const* frames, int n_frames,
                               const uint32_t* active, uint64_t m, uint8_t* out) {
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const uint64_t inst = active[j];
  M34 B, I;
  load_colmajor(base16 + 16 * inst, B);
  inverse_rigid(B, I);
  bool ok = true;
  for (int f = 0; f < n_frames && ok; ++f) {
    const double* F = frames[f];
    if (!F) continue;
    const double* c = F + 16 * inst;  // frame origin = column 3
    double x, y, z;
    xform(I, c[12], c[13], c[14], x, y, z);
    ok = query(g, nullptr, occ_any, x, y, z, __longlong_as_double(0x7ff8000000000000LL));
  }
  out[j] = ok ? 1 : 0;
}

__global__ void k_popcount(const unsigned long long* w, uint64_t n, unsigned long long* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const unsigned c = i < n ? (unsigned)__popcll(w[i]) : 0u;
  const unsigned s = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, (unsigned long long)s);
}

}  // namespace

namespace sbk {

void reach_build(const double* links, int n_links, const double* ee12, uint64_t samples,
                 uint64_t seed, const ReachGrid& g, unsigned long long* occ, unsigned* counts,
                 sb_stream_t s) {
  if (!samples) return;
  M34 ee;
  for (int k = 0; k < 12; ++k) ee.m[k] = ee12[k];
  k_reach_build<<<grid_for(samples), kBlock, 0, s>>>(links, n_links, g, ee, samples, seed, occ,
                                                     counts);
  check_launch("reach_build");
}
void reach_any(const ReachGrid& g, const unsigned long long* occ, unsigned long long* occ_any,
               sb_stream_t s) {
  if (!g.nr || !g.nz) return;
  k_reach_any<<<grid_for(g.nr * g.nz), kBlock, 0, s>>>(g, occ, occ_any);
  check_launch("reach_any");
}
void reach_query_batch(const ReachGrid& g, const unsigned long long* occ,
                       const unsigned long long* occ_any, const double* base16,
                       const double* targets, uint64_t n, double inclination, uint8_t* out,
                       sb_stream_t s) {
  if (!n) return;
  k_reach_query<<<grid_for(n), kBlock, 0, s>>>(g, occ, occ_any, base16, targets, n, inclination,
                                               out);
  check_launch("reach_query_batch");
}
void reach_placement_filter(const ReachGrid& g, const unsigned long long* occ_any,
                            const double* base16, const double* const* frames, int n_frames,
                            const uint32_t* active, uint64_t m, uint8_t* out, sb_stream_t s) {
  if (!m) return;
  k_reach_filter<<<grid_for(m), kBlock, 0, s>>>(g, occ_any, base16, frames, n_frames, active, m,
                                                out);
  check_launch("reach_placement_filter");
}
void reach_popcount(const unsigned long long* words, uint64_t n, unsigned long long* out,
                    sb_stream_t s) {
  if (!n) return;
  k_popcount<<<grid_for(n), kBlock, 0, s>>>(words, n, out);
  check_launch("reach_popcount");
}

}  // namespace sbk
