// Minimal C++ client of the drop-in: the reference's CollisionWorld call sequence
// (collision.hpp:76-127) against libscenebatch_b200.so. Build:
//   g++ -std=c++20 -Iinclude examples/cpp_dropin.cpp -Lpaper_2512_16896_b200
//       -lscenebatch_b200 -Wl,-rpath,$PWD/paper_2512_16896_b200 -o cpp_dropin
// Prints the box fingerprint; with a GPU also runs SPEC.md:394-395's unit-cube checks.
#include <cmath>
#include <cstdio>
#include <vector>

#include "scenebatch_b200.hpp"

using namespace scenebatch_b200;

int main() {
  TriMesh box = make_box(1, 1, 1);
  std::printf("box: %u vertices, %u triangles, fingerprint %016llx\n", box.n_vertices(),
              box.n_triangles(), (unsigned long long)mesh_fingerprint(box));
  try {
    CollisionWorld world(4);
    int g = world.register_geometry(box);
    int o = world.add_object("cube", g);
    world.set_enabled_all(o, true);
    std::vector<Pose> cand(4);
    const double offs[4] = {0.5, 0.9, 2.0, -0.5};
    for (int i = 0; i < 4; ++i) {
      cand[i] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, offs[i], 0, 0, 1};
    }
    std::vector<uint32_t> active = {0, 1, 2, 3};
    CollisionMask m = world.check_batch(g, cand, active);
    std::printf("free: %d %d %d %d\n", m.free[0], m.free[1], m.free[2], m.free[3]);
    // PositionSampler (sampler.hpp:66-96): 4 points of the rect under identity supports
    PositionSampler ps(/*placement_salt*/ 1);
    ps.prepare({{{-0.6, -0.4}, {0.6, -0.4}, {0.6, 0.4}, {-0.6, 0.4}}}, 4, /*run_seed*/ 7);
    std::vector<Pose> sup(4, Pose{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0.75, 1});
    std::vector<std::array<double, 3>> pos;
    std::vector<uint8_t> placeable;
    ps.sample(sup[0].data(), active, 0, pos, placeable);
    bool inside = true;
    for (const auto& p : pos) inside = inside && std::abs(p[0]) <= 0.6 && std::abs(p[1]) <= 0.4 && p[2] == 0.75;
    std::printf("sampled: inside %d refills %llu\n", inside ? 1 : 0,
                (unsigned long long)ps.refill_count());
    auto yaws = sample_orientations(SB_ORIENT_UNIFORM_YAW, active, pos, nullptr, 7, 1, 0);
    std::printf("yaw0 %.17g\n", yaws[0]);
    // BatchedSceneGraph (scene_graph.hpp:33-94): table -> drawer (prismatic) -> apple
    BatchedSceneGraph sg(4);
    uint32_t table = sg.add_node(sg.root(), "table");
    JointSpec slide{1, {1, 0, 0}, 0.0, 0.3};
    uint32_t drawer = sg.add_node(table, "drawer", -1, &slide);
    uint32_t apple = sg.add_node(drawer, "apple", 3);
    const double js[4] = {0.0, 0.1, 0.2, 0.3};
    sg.set_joint_states(drawer, js);
    const std::vector<Pose> wp = sg.world_poses(apple);
    std::printf("apple x: %.2f %.2f %.2f %.2f\n", wp[0][12], wp[1][12], wp[2][12], wp[3][12]);
    // ReachMap4D (reachability.hpp:34-94): 1-joint planar arm, 1 m link -> a ring of radius 1
    sb_chain_link link{{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1}, {0, {0, 0, 1}, -3.14159, 3.14159}};
    const Pose ee{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 1.0, 0, 0, 1};
    ReachMap4D rm = ReachMap4D::build(std::span<const sb_chain_link>(&link, 1), ee, 20000, 0.05, 0.5, 3);
    const std::vector<Pose> bases(2, Pose{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1});
    const std::vector<std::array<double, 3>> tg = {{0.0, 1.0, 0.0}, {0.5, 0.0, 0.0}};
    const std::vector<uint8_t> q = rm.query_batch(bases, tg);
    std::printf("reach ring: %d %d\n", q[0], q[1]);
    return (m.free[0] == 0 && m.free[1] == 0 && m.free[2] == 1 && m.free[3] == 0 && inside) ? 0 : 1;
  } catch (const cuda_error& e) {
    std::printf("no device: %s\n", e.what());
    return 2;
  }
}
