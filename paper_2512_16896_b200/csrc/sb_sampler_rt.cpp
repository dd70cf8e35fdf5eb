// PositionSampler (sampler.hpp:66-96) and sample_orientations as standalone device-backed
// objects behind the C ABI.
#include "sb_rt.hpp"

// ===================================================================== PositionSampler
// The reference's PositionSampler (sampler.hpp:66-96, sampler.cpp:54-127) as a standalone
// device-backed object. The SampleCache (sampler.hpp:18-36) is kept on the host as FIFO
// ranges of draw indices of the cache stream -- a queued point is fully determined by its
// draw index (polygon.cpp:390-391: 3 doubles = 6 PCG steps per point) and by the region
// table, which only changes together with the fingerprint (and then clears the queue).
// So refill / drain / bind_stream are index bookkeeping, and the points themselves are
// drawn on the device by jump-ahead (k_sampler_fifo), one thread per active entry.
namespace {

// region_fingerprint (polygon.cpp:422-444) of hole-free parts.
uint64_t rings_fingerprint(const double* xy, const uint32_t* off, uint32_t r0, uint32_t r1) {
  uint64_t h = 0x9e3779b97f4a7c15ULL;
  auto feed = [&h](double v) {
    uint64_t bits;
    std::memcpy(&bits, &v, sizeof bits);
    h = sbh::mix64(h ^ bits);
  };
  for (uint32_t r = r0; r < r1; ++r) {
    h = sbh::mix64(h ^ static_cast<uint64_t>(off[r + 1] - off[r]));
    for (uint32_t k = off[r]; k < off[r + 1]; ++k) {
      feed(xy[2 * k]);
      feed(xy[2 * k + 1]);
    }
  }
  return h;
}

sbh::SamplerTable rings_table(const double* xy, const uint32_t* off, uint32_t r0, uint32_t r1) {
  std::vector<std::vector<sbh::V2>> parts;
  for (uint32_t r = r0; r < r1; ++r) {
    std::vector<sbh::V2> ring;
    for (uint32_t k = off[r]; k < off[r + 1]; ++k) ring.push_back({xy[2 * k], xy[2 * k + 1]});
    parts.push_back(std::move(ring));
  }
  return sbh::sampler_table(parts);
}

uint64_t cache_state0(uint64_t run_seed, uint64_t salt) {  // Pcg32(make_stream(seed, {salt, "cach"}))
  const uint64_t h = sbh::mix64(sbh::mix64(sbh::mix64(run_seed) ^ salt) ^ 0x63616368ULL);
  const uint64_t mult = 6364136223846793005ULL, inc = (0xda3e39cb94b95bdbULL << 1u) | 1u;
  uint64_t st = inc;
  st += h;
  return st * mult + inc;
}

}  // namespace

struct sb_sampler {
  uint64_t salt;
  int device;
  cudaStream_t stream = nullptr;
  bool prepared = false, per_instance = false, region_empty = true;
  uint64_t n = 0, run_seed = 0, region_fp = 0;
  int region_nt = 0;
  // SampleCache (sampler.hpp:18-36): queue of [first, end) draw-index ranges
  uint64_t cache_fp = 0, cache_stream = 0, refill_count = 0, queue_size = 0, rng_pos = 0;
  std::vector<std::pair<uint64_t, uint64_t>> queue;  // front at queue_head
  size_t queue_head = 0;
  DevArray<SbRegionTri> d_tris;  // canonical table, or all per-instance tables
  DevArray<double> d_cum;
  DevArray<uint32_t> d_inst_tab;  // per instance: (first table row, rows)
  bool stride_tables = false;     // relation tables: [n][table_cap] rows, d_inst_n each
  int table_cap = 0;
  DevArray<int32_t> d_inst_n;
  DevArray<double> d_states;
  DevArray<int32_t> d_rflags;
  DevArray<sbk::SbArcTable> d_arcs;
  DevArray<double> d_sup, d_pos, d_sup16;
  DevArray<uint32_t> d_active;
  DevArray<uint8_t> d_pl;
  DevArray<uint64_t> d_seg;
  PinnedArray<double> h_sup;
  PinnedArray<uint64_t> h_seg;

  sb_sampler(uint64_t salt_, int dev) : salt(salt_), device(current_device_checked(dev)) {
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  ~sb_sampler() {
    if (ev_busy) {
      cudaEventSynchronize(ev_busy);
      cudaEventDestroy(ev_busy);
    }
    if (stream) {
      cudaSetDevice(device);
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }

  // Every kernel that reads the sampler's device tables or segment buffer is followed by
  // ev_busy (on whichever stream it ran: the internal one or a caller's). Host code that
  // rewrites h_seg / d_seg / the region tables first waits for it, so a later prepare() or
  // sample() cannot overwrite buffers an earlier, still running sample_device kernel reads.
  cudaEvent_t ev_busy = nullptr;
  void quiesce() {
    if (ev_busy) cuda_check(cudaEventSynchronize(ev_busy), "sync sampler kernels");
  }
  void mark_busy(cudaStream_t st) {
    if (!ev_busy) cuda_check(cudaEventCreateWithFlags(&ev_busy, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(ev_busy, st), "event");
  }

  void clear_queue() {
    queue.clear();
    queue_head = 0;
    queue_size = 0;
  }

  // PositionSampler::prepare (sampler.cpp:54-67) + the region tables PolygonSampler builds.
  void prepare(const double* xy, const uint32_t* off, uint32_t n_rings, const uint32_t* inst_rings,
               uint64_t batch, uint64_t seed) {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    quiesce();
    if (n_rings && (!xy || !off)) throw std::invalid_argument("ring arrays are NULL");
    for (uint32_t r = 0; r < n_rings; ++r)
      if (off[r + 1] < off[r]) throw std::invalid_argument("ring_offsets must be non-decreasing");
    if (batch > 0xffffffffull) throw std::invalid_argument("batch_size exceeds 2^32");
    std::vector<SbRegionTri> tris;
    std::vector<double> cum;
    if (inst_rings) {
      std::vector<uint32_t> tab(2 * batch);
      std::unordered_map<uint64_t, uint64_t> seen;  // ring range -> first instance using it
      for (uint64_t i = 0; i < batch; ++i) {
        const uint32_t r0 = inst_rings[i], r1 = inst_rings[i + 1];
        if (r1 < r0 || r1 > n_rings) throw std::invalid_argument("instance_rings out of range");
        auto ins = seen.emplace((static_cast<uint64_t>(r0) << 32) | r1, i);
        if (!ins.second) {  // same rings as an earlier instance: share its table
          tab[2 * i] = tab[2 * ins.first->second];
          tab[2 * i + 1] = tab[2 * ins.first->second + 1];
          continue;
        }
        auto t = rings_table(xy, off, r0, r1);
        tab[2 * i] = static_cast<uint32_t>(tris.size());
        tab[2 * i + 1] = static_cast<uint32_t>(t.tris.size());
        tris.insert(tris.end(), t.tris.begin(), t.tris.end());
        cum.insert(cum.end(), t.cum.begin(), t.cum.end());
      }
      d_inst_tab.ensure(std::max<uint64_t>(1, 2 * batch));
      if (batch)
        cuda_check(cudaMemcpy(d_inst_tab.p, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice),
                   "H2D instance tables");
    } else {
      region_empty = n_rings == 0;
      region_fp = rings_fingerprint(xy, off, 0, n_rings);
      auto t = rings_table(xy, off, 0, n_rings);
      tris = std::move(t.tris);
      cum = std::move(t.cum);
      region_nt = static_cast<int>(tris.size());
    }
    d_tris.ensure(std::max<size_t>(1, tris.size()));
    d_cum.ensure(std::max<size_t>(1, cum.size()));
    if (!tris.empty()) {
      cuda_check(cudaMemcpy(d_tris.p, tris.data(), tris.size() * sizeof(SbRegionTri), cudaMemcpyHostToDevice), "H2D table");
      cuda_check(cudaMemcpy(d_cum.p, cum.data(), cum.size() * sizeof(double), cudaMemcpyHostToDevice), "H2D table");
    }
    per_instance = inst_rings != nullptr;
    stride_tables = false;
    n = batch;
    run_seed = seed;
    const uint64_t parts[3] = {seed, salt, 0x63616368ULL};  // bind_stream(stream_key(...))
    uint64_t key = 0x853c49e6748fea9bULL;
    for (uint64_t p : parts) key = sbh::mix64(key ^ p);
    if (cache_stream != key) {
      clear_queue();
      cache_stream = key;
    }
    rng_pos = 0;  // cache_rng_ = make_stream(run_seed, {salt, "cach"})
    prepared = true;
  }

  // build_constraint_region (relationships.cpp:161-218) on the device for a batch of
  // anchor states (x, y, yaw per instance, support frame), then prepare(). The region
  // kernel decides per_instance exactly as the reference (any anchor moving by > 1e-12);
  // a canonical region's cache fingerprint is a hash of its sampler table (the polygon
  // itself never leaves the device).
  void prepare_relation(const sb_relation& rel, const double rect[4], const double* states,
                        uint64_t batch, uint64_t seed) {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    quiesce();
    if (batch == 0) throw std::invalid_argument("anchor state batch is empty");
    if (batch > 0xffffffffull) throw std::invalid_argument("batch_size exceeds 2^32");
    SbPlacementDev pd;
    std::memset(&pd, 0, sizeof pd);
    if (relation_anchor_count(rel) > 1)
      throw std::invalid_argument("prepare_relation: the anchor state batch holds one anchor");
    const bool hole = relation_to_dev(rel, pd);
    sb_support sup;
    std::memset(&sup, 0, sizeof sup);
    for (int k = 0; k < 4; ++k) sup.rect[k] = rect[k];
    support_to_dev(sup, pd);  // rect + bounds
    if (rel.anchor < 0) {  // no anchors: region = support (relationships.cpp:168-171)
      const double xy[8] = {rect[0], rect[1], rect[2], rect[1], rect[2], rect[3], rect[0], rect[3]};
      const uint32_t off[2] = {0, 4};
      prepare(xy, off, 1, nullptr, batch, seed);
      return;
    }
    if (!states) throw std::invalid_argument("anchor states are NULL");
    int sms = 0;
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
    table_cap = hole ? sbp::kHoleCap : SB_REGION_MAX_VERTS;
    d_tris.ensure(batch * table_cap);
    d_cum.ensure(batch * table_cap);
    d_inst_n.ensure(batch);
    d_states.ensure(3 * batch);
    d_rflags.ensure(2);
    cuda_check(cudaMemcpyAsync(d_states.p, states, 3 * batch * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D states");
    cuda_check(cudaMemsetAsync(d_rflags.p, 0, 2 * sizeof(int32_t), stream), "memset");
    sbk::RelationRegionParams rp;
    std::memset(&rp, 0, sizeof rp);
    rp.w.n = batch;
    rp.pl = pd;
    rp.anchor_object = -1;
    rp.cap = table_cap;
    rp.hole = hole ? 1 : 0;
    sbk::SbArcTable arc_tab;
    if (!hole && sbk::arc_table_host(pd, arc_tab)) {
      d_arcs.ensure(1);
      cuda_check(cudaMemcpyAsync(d_arcs.p, &arc_tab, sizeof arc_tab, cudaMemcpyHostToDevice, stream), "H2D arcs");
      rp.arcs = d_arcs.p;
    }
    rp.states = d_states.p;
    rp.tris = d_tris.p;
    rp.cum = d_cum.p;
    rp.ntri = d_inst_n.p;
    rp.flags = d_rflags.p;
    sbk::relation_regions(rp, sms, reinterpret_cast<sb_stream_t>(stream));
    int32_t flags[2], n0 = 0;
    cuda_check(cudaMemcpyAsync(flags, d_rflags.p, sizeof flags, cudaMemcpyDeviceToHost, stream), "D2H flags");
    cuda_check(cudaMemcpyAsync(&n0, d_inst_n.p, 4, cudaMemcpyDeviceToHost, stream), "D2H n");
    cuda_check(cudaStreamSynchronize(stream), "sync");
    if (flags[1] != 0)
      throw std::runtime_error("constraint region build failed (status " + std::to_string(flags[1]) + ")");
    per_instance = flags[0] != 0;
    stride_tables = true;
    n = batch;
    region_nt = per_instance ? 0 : n0;
    region_empty = !per_instance && n0 == 0;  // an empty (or zero-area) region_for(0)
    if (!per_instance && n0 > 0) {  // fingerprint of the canonical table
      std::vector<SbRegionTri> t(n0);
      std::vector<double> c(n0);
      cuda_check(cudaMemcpy(t.data(), d_tris.p, n0 * sizeof(SbRegionTri), cudaMemcpyDeviceToHost), "D2H table");
      cuda_check(cudaMemcpy(c.data(), d_cum.p, n0 * sizeof(double), cudaMemcpyDeviceToHost), "D2H table");
      uint64_t h = 0x9e3779b97f4a7c15ULL ^ 0x7461626cULL;  // "tabl": never a ring fingerprint
      auto feed = [&h](const void* p, size_t bytes) {
        const uint64_t* w = static_cast<const uint64_t*>(p);
        for (size_t k = 0; k < bytes / 8; ++k) h = sbh::mix64(h ^ w[k]);
      };
      feed(t.data(), t.size() * sizeof(SbRegionTri));
      feed(c.data(), c.size() * sizeof(double));
      region_fp = h;
    }
    run_seed = seed;
    const uint64_t parts[3] = {seed, salt, 0x63616368ULL};
    uint64_t key = 0x853c49e6748fea9bULL;
    for (uint64_t q : parts) key = sbh::mix64(key ^ q);
    if (cache_stream != key) {
      clear_queue();
      cache_stream = key;
    }
    rng_pos = 0;
    prepared = true;
  }

  // refill_cache (sampler.cpp:14-28) on draw indices
  void refill(uint64_t k) {
    if (region_fp != cache_fp) {
      clear_queue();
      cache_fp = region_fp;
    }
    uint64_t target = static_cast<uint64_t>(4.0 * static_cast<double>(k));
    if (target < k) target = k;
    if (queue_size >= target) return;
    const uint64_t need = target - queue_size;
    queue.push_back({rng_pos, rng_pos + need});
    rng_pos += need;
    queue_size += need;
    ++refill_count;
  }

  // drain_cache (sampler.cpp:30-43): pops k points as segments (first entry, first draw).
  int drain(uint64_t k) {
    if (region_fp != cache_fp || queue_size < k) refill(std::max<uint64_t>(k, 1));
    std::vector<uint64_t> first, draw;
    uint64_t j = 0;
    while (j < k) {
      auto& r = queue[queue_head];
      const uint64_t take = std::min(k - j, r.second - r.first);
      first.push_back(j);
      draw.push_back(r.first);
      r.first += take;
      j += take;
      if (r.first == r.second) ++queue_head;
    }
    queue_size -= k;
    if (queue_head > 64 && queue_head * 2 > queue.size()) {
      queue.erase(queue.begin(), queue.begin() + queue_head);
      queue_head = 0;
    }
    const int nseg = static_cast<int>(first.size());
    h_seg.ensure(std::max(2, 2 * nseg));
    std::copy(first.begin(), first.end(), h_seg.p);
    std::copy(draw.begin(), draw.end(), h_seg.p + nseg);
    return nseg;
  }

  void sample(const double* support, const uint32_t* active, uint64_t m, uint64_t attempt,
              double* pos, uint8_t* placeable) {
    if (!prepared) throw std::logic_error("PositionSampler: prepare() not called");
    if (m && (!active || !pos || !placeable || !support))
      throw std::invalid_argument("sample: NULL array");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    quiesce();
    if (!per_instance && region_empty) {  // sampler.cpp:81-84
      std::memset(pos, 0, 3 * m * sizeof(double));
      std::memset(placeable, 0, m);
      return;
    }
    if (!per_instance && region_nt == 0)
      throw std::invalid_argument("sample: canonical region has zero area");
    if (m == 0) {
      if (!per_instance) drain(0);
      return;
    }
    for (uint64_t j = 0; j < m; ++j)
      if (active[j] >= n) throw std::out_of_range("sample: active index >= batch_size");
    // Dense active sets: the whole TransformBatch goes up as is and the kernels read each
    // support in place; sparse ones: the active rows are gathered on the host first.
    const bool dense = 4 * m >= n;
    const double* ksup34 = nullptr;
    const double* ksup16 = nullptr;
    d_active.ensure(m);
    cuda_check(cudaMemcpyAsync(d_active.p, active, m * 4, cudaMemcpyHostToDevice, stream), "H2D active");
    if (dense) {
      d_sup16.ensure(16 * n);
      cuda_check(cudaMemcpyAsync(d_sup16.p, support, 16 * n * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D support");
      ksup16 = d_sup16.p;
    } else {
      h_sup.ensure(12 * m);
      for (uint64_t j = 0; j < m; ++j)
        colmajor_to_34(support + 16 * static_cast<uint64_t>(active[j]), h_sup.p + 12 * j);
      d_sup.ensure(12 * m);
      cuda_check(cudaMemcpyAsync(d_sup.p, h_sup.p, 12 * m * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D support");
      ksup34 = d_sup.p;
    }
    d_pos.ensure(3 * m);
    if (!per_instance) {
      const int nseg = drain(m);
      d_seg.ensure(2 * nseg);
      cuda_check(cudaMemcpyAsync(d_seg.p, h_seg.p, 2 * nseg * sizeof(uint64_t), cudaMemcpyHostToDevice, stream), "H2D segments");
      sbk::sampler_fifo(ksup34, ksup16, d_active.p, m, d_seg.p, d_seg.p + nseg, nseg,
                        cache_state0(run_seed, salt),
                        d_tris.p, d_cum.p, region_nt, d_pos.p, stream);
      cuda_check(cudaMemcpyAsync(pos, d_pos.p, 3 * m * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H positions");
      cuda_check(cudaStreamSynchronize(stream), "sync");
      std::memset(placeable, 1, m);
      return;
    }
    d_pl.ensure(m);
    sbk::sampler_fallback(ksup34, ksup16, d_active.p, m, run_seed, salt, attempt,
                          stride_tables ? nullptr : d_inst_tab.p, d_inst_n.p, table_cap, d_tris.p,
                          d_cum.p, d_pos.p, d_pl.p, stream);
    cuda_check(cudaMemcpyAsync(pos, d_pos.p, 3 * m * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H positions");
    cuda_check(cudaMemcpyAsync(placeable, d_pl.p, m, cudaMemcpyDeviceToHost, stream), "D2H placeable");
    cuda_check(cudaStreamSynchronize(stream), "sync");
  }

  // Device-resident variant: supports (N column-major Mat4), active, positions and
  // placeable are device pointers; everything is enqueued on `st` (no host round trip but
  // the SampleCache bookkeeping, which stays on the host).
  void sample_device(const double* d_sup16, const uint32_t* d_act, uint64_t m, uint64_t attempt,
                     double* d_out, uint8_t* d_placeable, cudaStream_t st) {
    if (!prepared) throw std::logic_error("PositionSampler: prepare() not called");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    if (m && (!d_sup16 || !d_act || !d_out || !d_placeable))
      throw std::invalid_argument("sample_device: NULL array");
    if (!per_instance && region_empty) {
      if (m) {
        cuda_check(cudaMemsetAsync(d_out, 0, 3 * m * sizeof(double), st), "memset");
        cuda_check(cudaMemsetAsync(d_placeable, 0, m, st), "memset");
      }
      return;
    }
    if (!per_instance && region_nt == 0)
      throw std::invalid_argument("sample: canonical region has zero area");
    if (!per_instance) {
      quiesce();  // h_seg / d_seg are rewritten below
      const int nseg = drain(m);
      if (m == 0) return;
      d_seg.ensure(2 * nseg);
      cuda_check(cudaMemcpyAsync(d_seg.p, h_seg.p, 2 * nseg * sizeof(uint64_t), cudaMemcpyHostToDevice, st), "H2D segments");
      sbk::sampler_fifo(nullptr, d_sup16, d_act, m, d_seg.p, d_seg.p + nseg, nseg,
                        cache_state0(run_seed, salt), d_tris.p, d_cum.p, region_nt, d_out,
                        reinterpret_cast<sb_stream_t>(st));
      mark_busy(st);
      cuda_check(cudaMemsetAsync(d_placeable, 1, m, st), "memset");
      return;
    }
    if (m == 0) return;
    sbk::sampler_fallback(nullptr, d_sup16, d_act, m, run_seed, salt, attempt,
                          stride_tables ? nullptr : d_inst_tab.p, d_inst_n.p, table_cap, d_tris.p,
                          d_cum.p, d_out, d_placeable, reinterpret_cast<sb_stream_t>(st));
    mark_busy(st);
  }
};

namespace {
struct OrientScratch {  // per host thread: reused device buffers of sb_sample_orientations
  int device = -1;
  cudaStream_t stream = nullptr;
  DevArray<uint32_t> active;
  DevArray<double> pos, face, yaws;
  void bind(int dev) {
    if (device == dev) return;
    active.release();
    pos.release();
    face.release();
    yaws.release();
    if (stream) cudaStreamDestroy(stream);
    stream = nullptr;
    device = dev;
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
  }
};
thread_local OrientScratch g_orient;
}  // namespace

extern "C" {

sb_status sb_sampler_create(uint64_t salt, int device, sb_sampler** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is NULL");
    *out = new sb_sampler(salt, device);
  });
}
void sb_sampler_destroy(sb_sampler* s) { delete s; }
sb_status sb_sampler_prepare(sb_sampler* s, const double* xy, const uint32_t* off, uint32_t n_rings,
                             const uint32_t* inst_rings, uint64_t n, uint64_t run_seed) {
  return guard([&] { s->prepare(xy, off, n_rings, inst_rings, n, run_seed); });
}
sb_status sb_sampler_sample(sb_sampler* s, const double* support, const uint32_t* active, uint64_t m,
                            uint64_t attempt, double* pos, uint8_t* placeable) {
  return guard([&] { s->sample(support, active, m, attempt, pos, placeable); });
}
sb_status sb_sampler_prepare_relation(sb_sampler* s, const sb_relation* rel,
                                      const double support_rect[4], const double* anchor_states,
                                      uint64_t n, uint64_t run_seed) {
  return guard([&] {
    if (!rel || !support_rect) throw std::invalid_argument("relation / support rect is NULL");
    s->prepare_relation(*rel, support_rect, anchor_states, n, run_seed);
  });
}
sb_status sb_sampler_sample_device(sb_sampler* s, const double* d_support16, const uint32_t* d_active,
                                   uint64_t m, uint64_t attempt, double* d_positions,
                                   uint8_t* d_placeable, void* cuda_stream) {
  return guard([&] {
    s->sample_device(d_support16, d_active, m, attempt, d_positions, d_placeable,
                     static_cast<cudaStream_t>(cuda_stream));
  });
}
sb_status sb_sampler_cache_info(const sb_sampler* s, uint64_t* queue_size, uint64_t* refills) {
  return guard([&] {
    if (queue_size) *queue_size = s->queue_size;
    if (refills) *refills = s->refill_count;
  });
}

// sample_orientations (sampler.cpp:129-156)
sb_status sb_sample_orientations(int kind, const uint32_t* active, uint64_t m, const double* pos,
                                 const double* face_xy, uint64_t n_targets, uint64_t run_seed,
                                 uint64_t salt, uint64_t attempt, double* yaws, int device) {
  return guard([&] {
    if (kind < SB_ORIENT_FIXED || kind > SB_ORIENT_FACE_TO)
      throw std::invalid_argument("sample_orientations: unknown orientation kind");
    if (kind == SB_ORIENT_FACE_TO && !face_xy)
      throw std::invalid_argument("sample_orientations: face_to target positions missing");
    if (m && (!active || !yaws || (kind == SB_ORIENT_FACE_TO && !pos)))
      throw std::invalid_argument("sample_orientations: NULL array");
    if (kind == SB_ORIENT_FACE_TO)
      for (uint64_t j = 0; j < m; ++j)
        if (active[j] >= n_targets)
          throw std::out_of_range("sample_orientations: active index >= n_targets");
    current_device_checked(device);
    if (m == 0) return;
    OrientScratch& o = g_orient;
    o.bind(device);
    o.active.ensure(m);
    o.yaws.ensure(m);
    cuda_check(cudaMemcpyAsync(o.active.p, active, m * 4, cudaMemcpyHostToDevice, o.stream), "H2D active");
    if (kind == SB_ORIENT_FACE_TO) {
      o.pos.ensure(3 * m);
      o.face.ensure(std::max<uint64_t>(1, 2 * n_targets));
      cuda_check(cudaMemcpyAsync(o.pos.p, pos, 3 * m * sizeof(double), cudaMemcpyHostToDevice, o.stream), "H2D positions");
      cuda_check(cudaMemcpyAsync(o.face.p, face_xy, 2 * n_targets * sizeof(double), cudaMemcpyHostToDevice, o.stream), "H2D targets");
    }
    sbk::orientations(kind, o.active.p, m, o.pos.p, o.face.p, run_seed, salt, attempt, o.yaws.p, o.stream);
    cuda_check(cudaMemcpyAsync(yaws, o.yaws.p, m * sizeof(double), cudaMemcpyDeviceToHost, o.stream), "D2H yaws");
    cuda_check(cudaStreamSynchronize(o.stream), "sync");
  });
}

// sample_orientations on device pointers (active, positions, face targets, yaws), enqueued
// on cuda_stream; face targets must cover every active index (not checked on the device).
sb_status sb_sample_orientations_device(int kind, const uint32_t* d_active, uint64_t m,
                                        const double* d_positions, const double* d_face_xy,
                                        uint64_t run_seed, uint64_t salt, uint64_t attempt,
                                        double* d_yaws, void* cuda_stream) {
  return guard([&] {
    if (kind < SB_ORIENT_FIXED || kind > SB_ORIENT_FACE_TO)
      throw std::invalid_argument("sample_orientations: unknown orientation kind");
    if (kind == SB_ORIENT_FACE_TO && !d_face_xy)
      throw std::invalid_argument("sample_orientations: face_to target positions missing");
    if (m && (!d_active || !d_yaws || (kind == SB_ORIENT_FACE_TO && !d_positions)))
      throw std::invalid_argument("sample_orientations: NULL array");
    sbk::orientations(kind, d_active, m, d_positions, d_face_xy, run_seed, salt, attempt, d_yaws,
                      reinterpret_cast<sb_stream_t>(static_cast<cudaStream_t>(cuda_stream)));
  });
}

}  // extern "C"
