// C ABI of the BatchedSceneGraph (include/scenebatch_b200.h).
#include "sb_graph_rt.hpp"

extern "C" {

sb_status sb_graph_create(uint64_t batch, int device, sb_graph** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is NULL");
    *out = new sb_graph(batch, device);
  });
}
void sb_graph_destroy(sb_graph* g) { delete g; }
sb_status sb_graph_add_node(sb_graph* g, uint32_t parent, const char* name, int64_t geometry,
                            const sb_joint* joint, uint32_t* id) {
  return guard([&] {
    const uint32_t v = g->add_node(parent, name, geometry, joint);
    if (id) *id = v;
  });
}
sb_status sb_graph_set_edge_batch(sb_graph* g, uint32_t parent, uint32_t child, const double* t16) {
  return guard([&] { g->set_edge_batch(parent, child, t16); });
}
sb_status sb_graph_set_edge(sb_graph* g, uint32_t child, uint64_t i, const double pose[16]) {
  return guard([&] { g->set_edge(child, i, pose); });
}
sb_status sb_graph_edge_batch(const sb_graph* g, uint32_t child, double* out16) {
  return guard([&] { g->edge_batch(child, out16); });
}
sb_status sb_graph_set_joint_states(sb_graph* g, uint32_t node, const double* v) {
  return guard([&] { g->set_joint_states(node, v); });
}
sb_status sb_graph_joint_states(const sb_graph* g, uint32_t node, double* out) {
  return guard([&] { g->joint_states(node, out); });
}
sb_status sb_graph_world_poses(const sb_graph* g, uint32_t node, double* out16) {
  return guard([&] { g->world_poses(node, out16); });
}
sb_status sb_graph_world_pose(const sb_graph* g, uint32_t node, uint64_t i, double pose[16]) {
  return guard([&] { g->world_pose(node, i, pose); });
}
sb_status sb_graph_world_poses_device(const sb_graph* g, uint32_t node, double* d_out16,
                                      void* cuda_stream) {
  return guard([&] { g->world_poses_device(node, d_out16, static_cast<cudaStream_t>(cuda_stream)); });
}
sb_status sb_graph_find(const sb_graph* g, const char* name, int64_t* id) {
  return guard([&] {
    if (!name || !id) throw std::invalid_argument("NULL argument");
    auto it = g->by_name.find(name);
    *id = it == g->by_name.end() ? -1 : static_cast<int64_t>(it->second);
  });
}
sb_status sb_graph_node_info(const sb_graph* g, uint32_t node, const char** name, uint32_t* parent,
                             int64_t* geometry, int* articulated, sb_joint* joint) {
  return guard([&] {
    const sb_graph::Node& nd = g->at(node);
    if (name) *name = nd.name.c_str();
    if (parent) *parent = nd.parent;
    if (geometry) *geometry = nd.geometry;
    if (articulated) *articulated = nd.joint ? 1 : 0;
    if (joint && nd.joint) *joint = nd.spec;
  });
}
uint64_t sb_graph_node_count(const sb_graph* g) { return g->nodes.size(); }
sb_status sb_graph_children(const sb_graph* g, uint32_t node, uint32_t* out, uint32_t cap,
                            uint32_t* count) {
  return guard([&] {
    g->at(node);
    uint32_t c = 0;
    for (uint32_t i = 1; i < g->nodes.size(); ++i)
      if (g->nodes[i].parent == node) {
        if (out && c < cap) out[c] = i;
        ++c;
      }
    if (count) *count = c;
  });
}
sb_status sb_graph_is_tree(const sb_graph* g, int* t) {
  return guard([&] { *t = g->is_tree() ? 1 : 0; });
}
sb_status sb_graph_valid_mask(const sb_graph* g, uint8_t* mask) {
  return guard([&] {
    g->activate();
    cuda_check(cudaMemcpyAsync(mask, g->d_valid.p, g->n, cudaMemcpyDeviceToHost, g->stream), "D2H");
    g->sync();
  });
}
sb_status sb_graph_mark_invalid(sb_graph* g, uint64_t i) {
  return guard([&] {
    if (i >= g->n) throw std::out_of_range("instance out of range");
    g->activate();
    cuda_check(cudaMemsetAsync(g->d_valid.p + i, 0, 1, g->stream), "memset");
    g->sync();
  });
}
sb_status sb_graph_reset_validity(sb_graph* g) {
  return guard([&] {
    g->activate();
    cuda_check(cudaMemsetAsync(g->d_valid.p, 1, g->n, g->stream), "memset");
    g->sync();
  });
}
sb_status sb_graph_valid_count(const sb_graph* g, uint64_t* count) {
  return guard([&] { *count = g->valid_count(); });
}


}  // extern "C"
