// C ABI of the ReachMap4D (include/scenebatch_b200.h).
#include "sb_reach_rt.hpp"

extern "C" {

sb_status sb_reach_build(const sb_chain_link* links, uint32_t n_links, const double ee[16],
                         uint64_t samples, double res, double psi_res, uint64_t seed, int device,
                         sb_reach_map** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is NULL");
    std::unique_ptr<sb_reach_map> m(new sb_reach_map(device));
    m->build(links, n_links, ee, samples, res, psi_res, seed);
    *out = m.release();
  });
}
sb_status sb_reach_load(const char* path, int device, sb_reach_map** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is NULL");
    std::unique_ptr<sb_reach_map> m(new sb_reach_map(device));
    m->load(path);
    *out = m.release();
  });
}
sb_status sb_reach_save(const sb_reach_map* m, const char* path) {
  return guard([&] { m->save(path); });
}
void sb_reach_destroy(sb_reach_map* m) { delete m; }
sb_status sb_reach_get_info(const sb_reach_map* m, sb_reach_info* o) {
  return guard([&] {
    o->samples = m->samples;
    o->resolution = m->g.res;
    o->psi_resolution = m->g.psi_res;
    o->max_radius = m->g.r_max;
    o->z_min = m->g.z_min;
    o->z_max = m->g.z_max;
    o->nr = m->g.nr;
    o->nz = m->g.nz;
    o->npsi = m->g.npsi;
    o->cell_count = m->cells();
    o->occupied_cells = m->occupied();
  });
}
sb_status sb_reach_cell_samples(const sb_reach_map* m, uint64_t ir, uint64_t iz, uint64_t ip,
                                uint32_t* count) {
  return guard([&] {
    *count = 0;
    if (m->d_counts.count == 0) return;
    if (ir >= m->g.nr || iz >= m->g.nz || ip >= m->g.npsi) throw std::out_of_range("cell out of range");
    cuda_check(cudaSetDevice(m->device), "cudaSetDevice");
    const uint64_t idx = (ir * m->g.nz + iz) * m->g.npsi + ip;
    cuda_check(cudaMemcpy(count, m->d_counts.p + idx, 4, cudaMemcpyDeviceToHost), "D2H");
  });
}
sb_status sb_reach_query_batch(const sb_reach_map* m, const double* base16, const double* targets,
                               uint64_t n, int has_incl, double incl, uint8_t* out) {
  return guard([&] {
    const_cast<sb_reach_map*>(m)->query_batch(base16, targets, n, has_incl != 0, incl, out);
  });
}
sb_status sb_reach_query_batch_device(const sb_reach_map* m, const double* d_base16,
                                      const double* d_targets, uint64_t n, int has_incl,
                                      double incl, uint8_t* d_out, void* cuda_stream) {
  return guard([&] {
    if (!n) return;
    if (!d_base16 || !d_targets || !d_out) throw std::invalid_argument("query_batch: NULL array");
    cuda_check(cudaSetDevice(m->device), "cudaSetDevice");
    sbk::reach_query_batch(m->g, m->d_occ.p, m->d_any.p, d_base16, d_targets, n,
                           has_incl ? incl : std::nan(""), d_out,
                           reinterpret_cast<sb_stream_t>(static_cast<cudaStream_t>(cuda_stream)));
  });
}
sb_status sb_reach_placement_filter(const sb_reach_map* m, const double* base16, uint64_t n,
                                    const double* const* frames, uint32_t n_frames,
                                    const uint32_t* active, uint64_t m_active, uint8_t* out) {
  return guard([&] {
    const_cast<sb_reach_map*>(m)->placement_filter(base16, n, frames, n_frames, active, m_active, out);
  });
}

}  // extern "C"
