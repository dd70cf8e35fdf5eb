// BatchedSceneGraph host object (scene_graph.hpp:33-94): metadata on the host, batches in
// HBM (sb_graph.cu). Internal to the runtime.
#pragma once

#include "sb_rt.hpp"

// ===================================================================== BatchedSceneGraph
struct sb_graph {
  uint64_t n;
  int device;
  cudaStream_t stream = nullptr;
  struct Node {
    std::string name;
    uint32_t parent = 0;
    int64_t geometry = -1;
    bool joint = false;
    sb_joint spec{};
    std::unique_ptr<DevArray<double>> edge, base, values;
  };
  std::vector<Node> nodes;
  std::unordered_map<std::string, uint32_t> by_name;
  DevArray<uint8_t> d_valid;
  mutable DevArray<double> d_tmp16;
  mutable DevArray<const double*> d_chain;
  mutable DevArray<unsigned long long> d_count;

  sb_graph(uint64_t batch, int dev) : n(batch), device(current_device_checked(dev)) {
    if (batch == 0) throw std::invalid_argument("batch_size must be >= 1");
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    d_valid.alloc(n);
    cuda_check(cudaMemsetAsync(d_valid.p, 1, n, stream), "memset");
    Node world;
    world.name = "world";
    world.edge = std::make_unique<DevArray<double>>();
    identity_batch(*world.edge);
    by_name.emplace("world", 0);
    nodes.push_back(std::move(world));
    sync();
  }
  ~sb_graph() {
    if (ev_chain) cudaEventDestroy(ev_chain);
    if (stream) {
      cudaSetDevice(device);
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
  sb_stream_t s() const { return reinterpret_cast<sb_stream_t>(stream); }
  void activate() const { cuda_check(cudaSetDevice(device), "cudaSetDevice"); }
  void sync() const { cuda_check(cudaStreamSynchronize(stream), "sync"); }

  void identity_batch(DevArray<double>& a) {
    a.alloc(12 * n);
    std::vector<double> one(16, 0.0);
    one[0] = one[5] = one[10] = one[15] = 1.0;
    d_tmp16.ensure(16 * n);
    std::vector<double> host(16 * n);
    for (uint64_t i = 0; i < n; ++i) std::memcpy(&host[16 * i], one.data(), sizeof(double) * 16);
    cuda_check(cudaMemcpyAsync(d_tmp16.p, host.data(), 16 * n * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
    sbk::graph_colmajor_to_34(d_tmp16.p, n, a.p, s());
    sync();
  }
  const Node& at(uint32_t id) const {
    if (id >= nodes.size()) throw std::out_of_range("unknown node");
    return nodes[id];
  }
  Node& at(uint32_t id) {
    if (id >= nodes.size()) throw std::out_of_range("unknown node");
    return nodes[id];
  }
  static sbk::GraphJoint gj(const sb_joint& j) {
    sbk::GraphJoint g;
    g.kind = j.kind;
    for (int k = 0; k < 3; ++k) g.axis[k] = j.axis[k];
    return g;
  }
  // edge = base * motion(values) over all instances (or motion alone when base == NULL)
  void compose(Node& nd, bool with_base) {
    sbk::graph_joint_compose(with_base ? nd.base->p : nullptr, nd.values->p, 0, n, gj(nd.spec),
                             nd.edge->p, s());
  }

  uint32_t add_node(uint32_t parent, const char* name_c, int64_t geometry, const sb_joint* joint) {
    activate();
    at(parent);
    if (!name_c) throw std::invalid_argument("node name is NULL");
    const std::string name(name_c);
    if (by_name.count(name)) throw std::invalid_argument("duplicate node name: " + name);
    Node nd;
    nd.name = name;
    nd.parent = parent;
    nd.geometry = geometry;
    nd.edge = std::make_unique<DevArray<double>>();
    if (joint) {  // JointSpec ctor (scene_graph.cpp:9-17)
      sb_joint j = *joint;
      if (j.kind != 0 && j.kind != 1) throw std::invalid_argument("JointSpec: unknown kind");
      if (j.lo > j.hi) throw std::invalid_argument("JointSpec: lo > hi");
      const double nrm = std::sqrt((j.axis[0] * j.axis[0] + j.axis[1] * j.axis[1]) + j.axis[2] * j.axis[2]);
      if (std::abs(nrm - 1.0) > 1e-9) {
        if (nrm < 1e-12) throw std::invalid_argument("JointSpec: zero axis");
        for (int k = 0; k < 3; ++k) j.axis[k] = j.axis[k] / nrm;
      }
      nd.joint = true;
      nd.spec = j;
      nd.base = std::make_unique<DevArray<double>>();
      identity_batch(*nd.base);
      nd.values = std::make_unique<DevArray<double>>();
      nd.values->alloc(n);
      std::vector<double> lo(n, j.lo);
      cuda_check(cudaMemcpyAsync(nd.values->p, lo.data(), n * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
      nd.edge->alloc(12 * n);
      compose(nd, false);  // every edge = motion(lo)
      sync();
    } else {
      identity_batch(*nd.edge);
    }
    const uint32_t id = static_cast<uint32_t>(nodes.size());
    by_name.emplace(name, id);
    nodes.push_back(std::move(nd));
    return id;
  }

  void set_edge_batch(uint32_t parent, uint32_t child, const double* t16) {
    activate();
    Node& nd = at(child);
    if (nd.parent != parent || child == 0)
      throw std::invalid_argument("no such edge: " + at(parent).name + " -> " + nd.name);
    if (!t16) throw std::invalid_argument("transform batch is NULL");
    for (uint64_t i = 0; i < n; ++i)
      if (!homogeneous16(t16 + 16 * i)) throw std::invalid_argument("non-homogeneous matrix in batch");
    d_tmp16.ensure(16 * n);
    cuda_check(cudaMemcpyAsync(d_tmp16.p, t16, 16 * n * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
    sbk::graph_colmajor_to_34(d_tmp16.p, n, nd.joint ? nd.base->p : nd.edge->p, s());
    if (nd.joint) compose(nd, true);
    sync();
  }

  void set_edge(uint32_t child, uint64_t i, const double* m16) {
    activate();
    Node& nd = at(child);
    if (child == 0) throw std::invalid_argument("cannot set edge on root");
    if (i >= n) throw std::out_of_range("instance out of range");
    if (!m16 || !homogeneous16(m16)) throw std::invalid_argument("non-homogeneous matrix");
    double r[12];
    colmajor_to_34(m16, r);
    double* dst = (nd.joint ? nd.base->p : nd.edge->p) + 12 * i;
    cuda_check(cudaMemcpyAsync(dst, r, sizeof r, cudaMemcpyHostToDevice, stream), "H2D");
    if (nd.joint)
      sbk::graph_joint_compose(nd.base->p, nd.values->p, i, 1, gj(nd.spec), nd.edge->p, s());
    sync();
  }

  void edge_batch(uint32_t child, double* out16) const {
    activate();
    const Node& nd = at(child);
    download16(nd.edge->p, out16);
  }
  void download16(const double* d12, double* out16) const {
    d_tmp16.ensure(16 * n);
    sbk::graph_34_to_colmajor(d12, n, d_tmp16.p, s());
    cuda_check(cudaMemcpyAsync(out16, d_tmp16.p, 16 * n * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }

  void set_joint_states(uint32_t node, const double* v) {
    activate();
    Node& nd = at(node);
    if (!nd.joint) throw std::invalid_argument("node is not articulated: " + nd.name);
    if (!v) throw std::invalid_argument("joint values are NULL");
    for (uint64_t i = 0; i < n; ++i)
      if (v[i] < nd.spec.lo - 1e-12 || v[i] > nd.spec.hi + 1e-12)
        throw std::invalid_argument("joint value out of limits for " + nd.name);
    cuda_check(cudaMemcpyAsync(nd.values->p, v, n * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
    compose(nd, true);
    sync();
  }
  void joint_states(uint32_t node, double* out) const {
    activate();
    const Node& nd = at(node);
    if (!nd.joint) throw std::invalid_argument("node is not articulated: " + nd.name);
    cuda_check(cudaMemcpyAsync(out, nd.values->p, n * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }

  // root -> node chain as device pointers, chain[0] = node
  int upload_chain(uint32_t node) const {
    std::vector<const double*> chain;
    for (uint32_t cur = node; cur != 0; cur = nodes[cur].parent) {
      chain.push_back(nodes[cur].edge->p);
      if (chain.size() > nodes.size()) throw std::logic_error("scene graph is not a tree");
    }
    if (!chain.empty()) {
      d_chain.ensure(chain.size());
      cuda_check(cudaMemcpyAsync(d_chain.p, chain.data(), chain.size() * sizeof(void*), cudaMemcpyHostToDevice, stream), "H2D chain");
    }
    return static_cast<int>(chain.size());
  }
  void world_poses(uint32_t node, double* out16) const {
    activate();
    at(node);
    const int depth = upload_chain(node);
    if (depth == 0) {  // the root: N identities
      download16(nodes[0].edge->p, out16);
      return;
    }
    d_tmp16.ensure(16 * n);
    sbk::graph_world_poses(d_chain.p, depth, n, d_tmp16.p, s());
    cuda_check(cudaMemcpyAsync(out16, d_tmp16.p, 16 * n * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }
  // batched FK into device memory on the caller's stream
  void world_poses_device(uint32_t node, double* d_out16, cudaStream_t st) const {
    activate();
    at(node);
    cuda_check(cudaStreamSynchronize(stream), "sync");  // the graph's own updates are done
    std::vector<const double*> chain;
    for (uint32_t cur = node; cur != 0; cur = nodes[cur].parent) chain.push_back(nodes[cur].edge->p);
    if (chain.empty()) {
      sbk::graph_34_to_colmajor(nodes[0].edge->p, n, d_out16, reinterpret_cast<sb_stream_t>(st));
      return;
    }
    if (!ev_chain) cuda_check(cudaEventCreateWithFlags(&ev_chain, cudaEventDisableTiming), "event");
    cuda_check(cudaEventSynchronize(ev_chain), "sync");  // the previous chain upload is consumed
    d_chain.ensure(chain.size());
    h_chain.ensure(chain.size());
    std::copy(chain.begin(), chain.end(), h_chain.p);
    cuda_check(cudaMemcpyAsync(d_chain.p, h_chain.p, chain.size() * sizeof(void*), cudaMemcpyHostToDevice, st), "H2D chain");
    sbk::graph_world_poses(d_chain.p, static_cast<int>(chain.size()), n, d_out16,
                           reinterpret_cast<sb_stream_t>(st));
    cuda_check(cudaEventRecord(ev_chain, st), "event");
  }
  mutable cudaEvent_t ev_chain = nullptr;
  mutable PinnedArray<const double*> h_chain;
  void world_pose(uint32_t node, uint64_t i, double* out16) const {
    activate();
    if (i >= n) throw std::out_of_range("instance out of range");
    at(node);
    const int depth = upload_chain(node);
    d_tmp16.ensure(16);
    sbk::graph_world_pose_one(d_chain.p, depth, i, d_tmp16.p, s());
    cuda_check(cudaMemcpyAsync(out16, d_tmp16.p, 16 * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }
  bool is_tree() const {  // scene_graph.cpp:174-187
    for (uint32_t i = 1; i < nodes.size(); ++i) {
      std::vector<bool> seen(nodes.size(), false);
      uint32_t cur = i;
      while (cur != 0) {
        if (seen[cur]) return false;
        seen[cur] = true;
        cur = nodes[cur].parent;
      }
    }
    return true;
  }
  uint64_t valid_count() const {
    activate();
    d_count.ensure(1);
    cuda_check(cudaMemsetAsync(d_count.p, 0, sizeof(unsigned long long), stream), "memset");
    sbk::graph_count_valid(d_valid.p, n, d_count.p, s());
    unsigned long long c = 0;
    cuda_check(cudaMemcpyAsync(&c, d_count.p, sizeof c, cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
    return c;
  }
};

