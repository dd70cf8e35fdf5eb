// ReachMap4D host object (reachability.hpp:34-94): grid metadata on the host, bitsets in
// HBM (sb_reach.cu). Internal to the runtime.
#pragma once

#include "sb_rt.hpp"

// ===================================================================== ReachMap4D
// reachability.cpp:10-273. Grid metadata on the host (same arithmetic as the reference),
// occupancy bitsets and sample counts in HBM (sb_reach.cu), SBRM v1 files on the host.
struct sb_reach_map {
  int device;
  cudaStream_t stream = nullptr;
  uint64_t samples = 0;
  sbk::ReachGrid g{};
  uint64_t words = 0;
  DevArray<unsigned long long> d_occ, d_any, d_count;
  DevArray<unsigned> d_counts;  // empty after load
  DevArray<double> d_base, d_targets, d_frames;
  DevArray<const double*> d_frame_ptrs;
  DevArray<uint32_t> d_active;
  DevArray<uint8_t> d_out;

  explicit sb_reach_map(int dev) : device(current_device_checked(dev)) {
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  ~sb_reach_map() {
    if (stream) {
      cudaSetDevice(device);
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
  sb_stream_t s() const { return reinterpret_cast<sb_stream_t>(stream); }
  void sync() const { cuda_check(cudaStreamSynchronize(stream), "sync"); }
  uint64_t cells() const { return g.nr * g.nz * g.npsi; }

  // occ_any from occ (build and load)
  void finish_any() {
    d_any.alloc(std::max<uint64_t>(1, (g.nr * g.nz + 63) / 64));
    cuda_check(cudaMemsetAsync(d_any.p, 0, d_any.count * 8, stream), "memset");
    sbk::reach_any(g, d_occ.p, d_any.p, s());
  }

  void build(const sb_chain_link* links, uint32_t n_links, const double* ee16, uint64_t n_samples,
             double res, double psi_res, uint64_t seed) {
    if (n_links == 0 || !links) throw std::invalid_argument("build: chain has no joints");
    if (n_samples < 1) throw std::invalid_argument("build: need at least one sample");
    if (res <= 0.0 || psi_res <= 0.0) throw std::invalid_argument("build: resolution must be positive");
    std::vector<double> L(18 * n_links);
    double ee[12];
    if (ee16) {
      if (!homogeneous16(ee16)) throw std::invalid_argument("build: non-homogeneous ee_offset");
      colmajor_to_34(ee16, ee);
    } else {
      for (int k = 0; k < 12; ++k) ee[k] = (k % 5 == 0) ? 1.0 : 0.0;
    }
    auto norm3 = [](double x, double y, double z) { return std::sqrt((x * x + y * y) + z * z); };
    double reach = norm3(ee[3], ee[7], ee[11]);  // KinematicChain::max_reach (:20-28)
    for (uint32_t l = 0; l < n_links; ++l) {
      const sb_chain_link& k = links[l];
      if (!homogeneous16(k.origin)) throw std::invalid_argument("build: non-homogeneous link origin");
      sb_joint j = k.joint;  // JointSpec ctor (scene_graph.cpp:9-17)
      if (j.kind != 0 && j.kind != 1) throw std::invalid_argument("JointSpec: unknown kind");
      if (j.lo > j.hi) throw std::invalid_argument("JointSpec: lo > hi");
      const double nrm = norm3(j.axis[0], j.axis[1], j.axis[2]);
      if (std::abs(nrm - 1.0) > 1e-9) {
        if (nrm < 1e-12) throw std::invalid_argument("JointSpec: zero axis");
        for (int c = 0; c < 3; ++c) j.axis[c] = j.axis[c] / nrm;
      }
      colmajor_to_34(k.origin, &L[18 * l]);
      L[18 * l + 12] = j.kind;
      for (int c = 0; c < 3; ++c) L[18 * l + 13 + c] = j.axis[c];
      L[18 * l + 16] = j.lo;
      L[18 * l + 17] = j.hi;
      reach += norm3(k.origin[12], k.origin[13], k.origin[14]);
      if (j.kind == 1) reach += std::max(std::abs(j.lo), std::abs(j.hi));
    }
    samples = n_samples;
    g.res = res;
    g.psi_res = psi_res;
    g.r_max = reach + res;
    g.z_min = -reach - res;
    g.z_max = reach + res;
    g.nr = static_cast<uint64_t>(std::ceil(g.r_max / res));
    g.nz = static_cast<uint64_t>(std::ceil((g.z_max - g.z_min) / res));
    g.npsi = static_cast<uint64_t>(std::ceil(M_PI / psi_res));
    if (cells() > (1ull << 34)) throw std::invalid_argument("build: grid too fine");
    words = (cells() + 63) / 64;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    d_occ.alloc(std::max<uint64_t>(1, words));
    d_counts.alloc(std::max<uint64_t>(1, cells()));
    cuda_check(cudaMemsetAsync(d_occ.p, 0, d_occ.count * 8, stream), "memset");
    cuda_check(cudaMemsetAsync(d_counts.p, 0, d_counts.count * 4, stream), "memset");
    DevArray<double> d_links;
    d_links.alloc(L.size());
    cuda_check(cudaMemcpyAsync(d_links.p, L.data(), L.size() * 8, cudaMemcpyHostToDevice, stream), "H2D");
    sbk::reach_build(d_links.p, static_cast<int>(n_links), ee, samples, seed, g, d_occ.p,
                     d_counts.p, s());
    finish_any();
    sync();
  }

  uint64_t occupied() const {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    auto& self = const_cast<sb_reach_map&>(*this);
    self.d_count.ensure(1);
    cuda_check(cudaMemsetAsync(self.d_count.p, 0, 8, stream), "memset");
    sbk::reach_popcount(d_occ.p, words, self.d_count.p, s());
    unsigned long long c = 0;
    cuda_check(cudaMemcpyAsync(&c, self.d_count.p, 8, cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
    return c;
  }

  // SBRM v1 (reachability.cpp:192-273)
  void save(const char* path) const {
    if (!path) throw std::invalid_argument("path is NULL");
    std::vector<unsigned long long> occ(words);
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    if (words)
      cuda_check(cudaMemcpy(occ.data(), d_occ.p, words * 8, cudaMemcpyDeviceToHost), "D2H occ");
    FILE* f = std::fopen(path, "wb");
    if (!f) throw std::runtime_error(std::string("cannot open for write: ") + path);
    const uint32_t version = 1;
    const uint64_t hdr[1] = {samples};
    bool ok = std::fwrite("SBRM", 1, 4, f) == 4;
    ok = ok && std::fwrite(&version, 4, 1, f) == 1 && std::fwrite(hdr, 8, 1, f) == 1;
    const double dv[5] = {g.res, g.psi_res, g.r_max, g.z_min, g.z_max};
    ok = ok && std::fwrite(dv, 8, 5, f) == 5;
    const uint64_t nv[4] = {g.nr, g.nz, g.npsi, words};
    ok = ok && std::fwrite(nv, 8, 4, f) == 4;
    ok = ok && (words == 0 || std::fwrite(occ.data(), 8, words, f) == words);
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error(std::string("write failed: ") + path);
  }
  void load(const char* path) {
    if (!path) throw std::invalid_argument("path is NULL");
    FILE* f = std::fopen(path, "rb");
    if (!f) throw std::runtime_error(std::string("cannot open reach map: ") + path);
    char magic[4];
    uint32_t version = 0;
    double dv[5];
    uint64_t nv[4];
    const bool head = std::fread(magic, 1, 4, f) == 4;
    if (!head || std::memcmp(magic, "SBRM", 4) != 0) {
      std::fclose(f);
      throw std::runtime_error(std::string("not a reach map file: ") + path);
    }
    if (std::fread(&version, 4, 1, f) != 1 || version != 1) {
      std::fclose(f);
      throw std::runtime_error("unsupported reach map version");
    }
    bool ok = std::fread(&samples, 8, 1, f) == 1 && std::fread(dv, 8, 5, f) == 5 &&
              std::fread(nv, 8, 4, f) == 4;
    std::vector<unsigned long long> occ;
    if (ok) {
      occ.resize(nv[3]);
      ok = nv[3] == 0 || std::fread(occ.data(), 8, nv[3], f) == nv[3];
    }
    std::fclose(f);
    if (!ok) throw std::runtime_error(std::string("truncated reach map: ") + path);
    g.res = dv[0];
    g.psi_res = dv[1];
    g.r_max = dv[2];
    g.z_min = dv[3];
    g.z_max = dv[4];
    g.nr = nv[0];
    g.nz = nv[1];
    g.npsi = nv[2];
    words = nv[3];
    if (words * 64 < cells()) throw std::runtime_error("reach map bitset shorter than its grid");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    d_occ.alloc(std::max<uint64_t>(1, words));
    if (words)
      cuda_check(cudaMemcpyAsync(d_occ.p, occ.data(), words * 8, cudaMemcpyHostToDevice, stream), "H2D occ");
    d_counts.release();
    finish_any();
    sync();
  }

  void query_batch(const double* base16, const double* targets, uint64_t n, bool has_incl,
                   double incl, uint8_t* out) {
    if (n && (!base16 || !targets || !out)) throw std::invalid_argument("query_batch: NULL array");
    if (!n) return;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    d_base.ensure(16 * n);
    d_targets.ensure(3 * n);
    d_out.ensure(n);
    cuda_check(cudaMemcpyAsync(d_base.p, base16, 16 * n * 8, cudaMemcpyHostToDevice, stream), "H2D");
    cuda_check(cudaMemcpyAsync(d_targets.p, targets, 3 * n * 8, cudaMemcpyHostToDevice, stream), "H2D");
    sbk::reach_query_batch(g, d_occ.p, d_any.p, d_base.p, d_targets.p, n,
                           has_incl ? incl : std::nan(""), d_out.p, s());
    cuda_check(cudaMemcpyAsync(out, d_out.p, n, cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }

  void placement_filter(const double* base16, uint64_t n, const double* const* frames,
                        uint32_t n_frames, const uint32_t* active, uint64_t m, uint8_t* out) {
    if (m && (!base16 || !active || !out)) throw std::invalid_argument("placement_filter: NULL array");
    if (!m) return;
    for (uint64_t j = 0; j < m; ++j)
      if (active[j] >= n) throw std::out_of_range("placement_filter: active index >= N");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    d_base.ensure(16 * n);
    cuda_check(cudaMemcpyAsync(d_base.p, base16, 16 * n * 8, cudaMemcpyHostToDevice, stream), "H2D");
    uint32_t present = 0;
    for (uint32_t f = 0; f < n_frames; ++f) present += frames && frames[f] ? 1 : 0;
    d_frames.ensure(std::max<uint64_t>(1, 16 * n * present));
    std::vector<const double*> ptrs(std::max<uint32_t>(1, n_frames), nullptr);
    for (uint32_t f = 0, k = 0; f < n_frames; ++f) {
      if (!frames || !frames[f]) continue;
      double* dst = d_frames.p + 16 * n * k++;
      cuda_check(cudaMemcpyAsync(dst, frames[f], 16 * n * 8, cudaMemcpyHostToDevice, stream), "H2D frames");
      ptrs[f] = dst;
    }
    d_frame_ptrs.ensure(ptrs.size());
    cuda_check(cudaMemcpyAsync(d_frame_ptrs.p, ptrs.data(), ptrs.size() * sizeof(void*), cudaMemcpyHostToDevice, stream), "H2D");
    d_active.ensure(m);
    d_out.ensure(m);
    cuda_check(cudaMemcpyAsync(d_active.p, active, m * 4, cudaMemcpyHostToDevice, stream), "H2D");
    sbk::reach_placement_filter(g, d_any.p, d_base.p, d_frame_ptrs.p, static_cast<int>(n_frames),
                                d_active.p, m, d_out.p, s());
    cuda_check(cudaMemcpyAsync(out, d_out.p, m, cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }
};

