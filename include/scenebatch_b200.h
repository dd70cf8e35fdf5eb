/*
 * scenebatch_b200.h -- C ABI of the B200-native Sceniris hot path
 * (batched candidate-pose sampling -> collision check -> first-valid accept).
 *
 * The reference (/root/reference/proj, namespace scenebatch) has no FFI layer; its
 * boundary is the C++ class API that its (absent) engine would call. Every entry point
 * below names the reference interface it replaces (file:line, relative to
 * /root/reference/proj). include/scenebatch_b200.hpp re-creates that C++ class API on
 * top of these functions and rethrows the same exception types.
 *
 * Conventions
 *  - Every function returns an sb_status; on failure sb_last_error() holds the message
 *    (thread-local). Status codes map 1:1 onto the reference's exception types.
 *  - Poses are 4x4 homogeneous matrices stored column-major as double[16], exactly the
 *    memory of the reference's Eigen::Matrix4d / TransformBatch (transform.hpp:10-27),
 *    so a TransformBatch's data() can be passed without conversion. The bottom row must
 *    be (0,0,0,1) exactly (SPEC TransformBatch invariant); other poses are rejected.
 *  - Buffers are caller-owned host memory, copied in and out, except the *_device entry
 *    points, which take device pointers and a cudaStream_t (as void*). No torch types.
 *  - A handle is single-writer; calls on one handle are serialized on its CUDA stream.
 *  - There is no CPU fallback: without a usable sm_100 device every compute entry point
 *    fails with SB_ERR_CUDA.
 */
#ifndef SCENEBATCH_B200_H_
#define SCENEBATCH_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SB_ABI_VERSION 2

typedef enum sb_status {
  SB_OK = 0,
  SB_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  SB_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range (bad ids, .at()) */
  SB_ERR_LOGIC = 3,            /* std::logic_error */
  SB_ERR_RUNTIME = 4,          /* std::runtime_error */
  SB_ERR_CUDA = 5              /* device missing / CUDA failure (no CPU fallback) */
} sb_status;

const char* sb_last_error(void);
int sb_abi_version(void);
/* 1 if a CUDA device of compute capability 10.x is usable, else 0 (reason in sb_last_error). */
int sb_device_available(void);

/* ------------------------------------------------------------------------------------
 * Mesh primitives: trimesh.hpp:27-32 (make_box / make_cylinder / make_sphere),
 * trimesh.hpp:35 (transformed). Vertices are xyz triples, triangles index triples.
 * Pass NULL buffers to query the sizes first.
 * ---------------------------------------------------------------------------------- */
sb_status sb_make_box(double sx, double sy, double sz, double* vertices, uint32_t* n_vertices,
                      uint32_t* triangles, uint32_t* n_triangles);
/* load_obj (config.hpp:88-90; declared, not defined, by the reference): Wavefront OBJ
 * subset -- v / f records (f: i, i/j, i//k, i/j/k; negative = relative), polygon faces
 * fan-triangulated, other records ignored; errors are SB_ERR_RUNTIME with
 * "path:line: ..." in sb_last_error(). Same size-query convention as sb_make_box. */
sb_status sb_load_obj(const char* path, double* vertices, uint32_t* n_vertices,
                      uint32_t* triangles, uint32_t* n_triangles);
sb_status sb_make_cylinder(double radius, double height, int segments, double* vertices,
                           uint32_t* n_vertices, uint32_t* triangles, uint32_t* n_triangles);
sb_status sb_make_sphere(double radius, int stacks, int slices, double* vertices,
                         uint32_t* n_vertices, uint32_t* triangles, uint32_t* n_triangles);
/* In-place rigid transform of n vertices: v <- R v + t (transform.hpp:71-73). */
sb_status sb_transform_vertices(const double pose[16], double* vertices, uint32_t n_vertices);
/* mesh_fingerprint (trimesh.cpp:120-135). */
sb_status sb_mesh_fingerprint(const double* vertices, uint32_t n_vertices,
                              const uint32_t* triangles, uint32_t n_triangles, uint64_t* out);
/* rest_pose(mesh).z_offset = -aabb.min.z + kRestClearance (sampler.cpp:45-52). */
sb_status sb_rest_z_offset(const double* vertices, uint32_t n_vertices, double* z_offset);

/* Host-side BVH preparation summary for a mesh (MeshBvh, collision.cpp:217-281):
 * info = {reference node count, reference depth, effective DAG nodes, reachable triangles}.
 * The effective DAG is what the reference's traversal can reach (children read as
 * {left, left+1}, collision.hpp:46); the GPU narrow phase runs on exactly that. */
sb_status sb_bvh_info(const double* vertices, uint32_t n_vertices, const uint32_t* triangles,
                      uint32_t n_triangles, int32_t info[4]);

/* triangulate (polygon.cpp:344-368, hole-free ring) as PolygonSampler consumes it
 * (zero-area triangles dropped, polygon.cpp:374-375): host-side region preparation. */
sb_status sb_triangulate_ring(const double* ring_xy, uint32_t n, double* tris_out,
                              uint32_t max_tris, uint32_t* n_tris);

/* ------------------------------------------------------------------------------------
 * RNG: rng.hpp:9-67. Exposed for known-answer tests and for hosts that pre-draw.
 * ---------------------------------------------------------------------------------- */
uint64_t sb_mix64(uint64_t x);                                       /* rng.hpp:9-14  */
uint64_t sb_stream_key(const uint64_t* parts, uint32_t n);           /* rng.hpp:17-21 */
/* make_stream(seed, counters) then `n_draws` x next_double() into out (rng.hpp:46-48,63-67). */
sb_status sb_stream_doubles(uint64_t seed, const uint64_t* counters, uint32_t n_counters,
                            double* out, uint32_t n_draws);

/* ------------------------------------------------------------------------------------
 * CollisionWorld: collision.hpp:76-127, collision.cpp:334-461.
 * ---------------------------------------------------------------------------------- */
typedef struct sb_world sb_world;

typedef struct sb_stats {          /* CollisionStats, collision.hpp:65-72 */
  uint64_t geometry_registrations;
  uint64_t bvh_builds;
  uint64_t check_calls;
  uint64_t checked_instances;
  uint64_t narrow_phase_tests;
  /* Triangle-pair predicate evaluations. The reference counts BVH leaf re-visits
   * (collision.cpp:320-324 push left and left+1); this build visits each reachable
   * node pair once, so this counter is <= the reference's. */
  uint64_t triangle_pair_tests;
} sb_stats;

/* CollisionWorld(batch_size, margin): collision.cpp:334-337. Any finite margin: box tests
 * use Aabb3::overlaps(., margin) and, for margin > 0, a triangle pair collides when
 * tri_tri_distance < margin (collision.cpp:136-212,312-313). The generation engine uses the
 * reference driver's margin 0 (Appendix C.7). */
sb_status sb_world_create(uint64_t batch_size, double margin, int device, sb_world** out);
void sb_world_destroy(sb_world* w);
/* register_geometry: collision.cpp:339-355 (fingerprint dedupe, drop_degenerate, MeshBvh). */
sb_status sb_register_geometry(sb_world* w, const double* vertices, uint32_t n_vertices,
                               const uint32_t* triangles, uint32_t n_triangles,
                               int32_t* geom_id);
/* add_object: collision.cpp:365-376; objects start disabled with identity poses. */
sb_status sb_add_object(sb_world* w, const char* name, int32_t geom_id, int32_t* object_id);
/* set_enabled / set_enabled_all: collision.cpp:386-393. */
sb_status sb_set_enabled(sb_world* w, int32_t object, const uint32_t* instances, uint64_t n,
                         int enabled);
sb_status sb_set_enabled_all(sb_world* w, int32_t object, int enabled);
/* update_transforms (N poses) / update_transform (one): collision.cpp:395-412. */
sb_status sb_update_transforms(sb_world* w, int32_t object, const double* poses_colmajor16xN);
sb_status sb_update_transform(sb_world* w, int32_t object, uint64_t instance,
                              const double pose[16]);
/* object_pose / enabled accessors: collision.cpp:383-385,414-416. */
sb_status sb_object_pose(sb_world* w, int32_t object, uint64_t instance, double pose[16]);
sb_status sb_enabled(sb_world* w, int32_t object, uint64_t instance, int* enabled);
/* check_batch: collision.cpp:418-461. poses[j] (column-major 16 doubles) is the candidate
 * in instance active[j]. free_out / contact_out have length N; inactive instances get
 * free = 1, contact = -1 (collision.cpp:424-426). */
sb_status sb_check_batch(sb_world* w, int32_t geom_id, const double* poses_colmajor16xM,
                         const uint32_t* active, uint64_t m, uint8_t* free_out,
                         int32_t* contact_out);
sb_status sb_get_stats(sb_world* w, sb_stats* out);
sb_status sb_reset_stats(sb_world* w);

/* ------------------------------------------------------------------------------------
 * Scene description + generation engine. The reference's rejection loop is specified
 * but absent from proj/; this is that loop, with the driver contract
 * frozen in DESIGN.md ("Appendix C contract"). It composes PositionSampler
 * (sampler.cpp:54-127), sample_orientations (sampler.cpp:129-156), rest_pose, pose
 * compose (transform.hpp:40-54), build_constraint_region (relationships.cpp:161-218) and
 * CollisionWorld::check_batch into one on-device pipeline.
 * ---------------------------------------------------------------------------------- */
enum { SB_DIST_NONE = 0, SB_DIST_GREATER = 1, SB_DIST_LESS = 2, SB_DIST_EQUAL = 3,
       SB_DIST_MIDDLE = 4 };                                  /* relationships.hpp:12 */
#define SB_MAX_ANCHORS 8          /* anchors per relation (RelationshipSpec::anchors) */
#define SB_MAX_SUPPORT_VERTS 16   /* vertices of a convex polygon support */
enum { SB_DIR_NONE = 0, SB_DIR_LEFT = 1, SB_DIR_RIGHT = 2, SB_DIR_FRONT = 3, SB_DIR_BACK = 4,
       SB_DIR_VECTOR = 5 };                                   /* relationships.hpp:12-14 */
enum { SB_FRAME_GLOBAL = 0, SB_FRAME_LOCAL = 1 };
enum { SB_ORIENT_FIXED = 0, SB_ORIENT_UNIFORM_YAW = 1, SB_ORIENT_FACE_TO = 2 }; /* sampler.hpp:53-57 */

typedef struct sb_mesh {
  const double* vertices; /* n_vertices x 3 */
  uint32_t n_vertices;
  const uint32_t* triangles; /* n_triangles x 3 */
  uint32_t n_triangles;
} sb_mesh;

/* An object present and enabled in every instance at a fixed pose (table, container). */
typedef struct sb_fixed_object {
  int32_t mesh;
  double pose[16];
  /* Optional per-instance poses (a TransformBatch, CollisionWorld::update_transforms,
   * collision.hpp:95): n_instances column-major Mat4 in GLOBAL instance order (a shard
   * reads its own range); NULL = `pose` for every instance. */
  const double* poses16;
} sb_fixed_object;

/* A support surface in the z=0 plane of its frame (SupportSurface, surface.hpp:15-20,
 * given directly or from sb_extract_support_surfaces): the axis-aligned rect
 * [x0,x1]x[y0,y1] (make_rect order), or, when n_polygon >= 3, the convex polygon
 * polygon_xy[0..2*n_polygon) (SupportSurface::polygon as given: its vertex order and start
 * feed the sampler triangulation; clipping uses it corrected to counter-clockwise). A
 * polygon that is an axis-aligned rectangle clips exactly as a rect does.
 * The frame per instance is the reference's support_world[inst] (sampler.hpp:78-80,
 * sampler.cpp:90,119; built by the driver from BatchedSceneGraph::world_poses,
 * scene_graph.cpp:126-147, times the surface frame):
 *   on_placement >= 0: (accepted pose of placement on_placement) * pose -- a surface of an
 *                      earlier placed object (stacking), evaluated per instance and run;
 *   else poses16 != NULL: poses16[inst] (n_instances column-major Mat4, global order),
 *                      e.g. a drawer floor at per-instance joint values (FK);
 *   else: `pose` for every instance. */
typedef struct sb_support {
  double pose[16];
  double rect[4]; /* x0, y0, x1, y1 (ignored when n_polygon >= 3) */
  const double* poses16;
  int32_t on_placement;
  uint32_t n_polygon;        /* 0 = rect, else 3..SB_MAX_SUPPORT_VERTS */
  const double* polygon_xy;  /* n_polygon (x, y) pairs, convex */
} sb_support;

/* RelationshipSpec (relationships.hpp:18-38). anchors = {anchor, extra_anchors[0..n)}
 * (placement indices, each < this placement); greater/less/equal and a direction take
 * exactly one anchor, `middle` two or more (RelationshipSpec::validate,
 * relationships.cpp:59-76); the per-instance test covers every anchor (:178-186). */
typedef struct sb_relation {
  int32_t anchor;          /* placement index of the first anchor, -1 = none */
  int32_t distance_type;   /* SB_DIST_* */
  int32_t direction;       /* SB_DIR_* */
  int32_t frame;           /* SB_FRAME_* */
  double direction_vector[2];
  double distance;
  double angle_threshold;  /* <= 0: default (pi/4 with a direction, pi without) */
  int32_t n_extra_anchors; /* further anchors, 0..SB_MAX_ANCHORS-1 */
  int32_t extra_anchors[SB_MAX_ANCHORS - 1];
} sb_relation;

/* PlacementSpec (config.hpp:45-54) subset on the hot path. */
typedef struct sb_placement {
  int32_t mesh;
  int32_t support;
  int32_t orientation;     /* SB_ORIENT_* */
  int32_t face_target;     /* placement index for SB_ORIENT_FACE_TO, else -1 */
  sb_relation relation;
  /* apply_ratio_on_support (relationships.cpp:220-230): the region is eroded by
   * ratio * min(mesh AABB x, y extents) / 2; in [0, 1]; > 0 only without a relation */
  double ratio_on_support;
} sb_placement;

typedef struct sb_scene {
  uint64_t n_instances;    /* N variations */
  int32_t attempts;        /* candidates per object K = max_retries + 1 (config.hpp:67) */
  int32_t reserved;
  uint32_t n_meshes;
  const sb_mesh* meshes;
  uint32_t n_fixed;
  const sb_fixed_object* fixed;
  uint32_t n_supports;
  const sb_support* supports;
  uint32_t n_placements;
  const sb_placement* placements;
} sb_scene;

/* Host-side outputs of one generation run (any pointer may be NULL to skip it).
 * Object order: fixed objects first, then placements; only placements are reported. */
typedef struct sb_result {
  int16_t* accepted;      /* [n_placements][n_local] accepted attempt index, -1 = none */
  double* poses;          /* [n_placements][n_local][16] accepted pose (identity if none) */
  uint8_t* valid;         /* [n_local] BatchedSceneGraph::valid_mask (scene_graph.hpp:68) */
} sb_result;

typedef struct sb_run_stats {
  uint64_t valid_instances;
  uint64_t candidates_sampled;   /* incl. non-placeable draws */
  uint64_t candidate_checks;     /* check_batch checked_instances summed over rounds */
  uint64_t narrow_phase_tests;
  uint64_t triangle_pair_tests;
  uint64_t rounds;               /* (placement, attempt) rounds executed */
  uint64_t per_instance_placements;
  uint64_t broad_phase_tests;    /* enabled objects examined by the AABB broad phase */
  uint64_t node_pair_tests;      /* BVH node-pair box tests in the narrow phase */
  uint64_t accepted_candidates;  /* candidates accepted (== placed objects) */
} sb_run_stats;

/* Count exchange between shards (one process per GPU). Called with this rank's n values;
 * must return every rank's values in rank order (recv has n * world_size slots). */
typedef int (*sb_allgather_fn)(void* ctx, const uint64_t* send, uint32_t n, uint64_t* recv);

/* Optional device-side variant: enqueue, on `cuda_stream` (a cudaStream_t), an all-gather of
 * n u64 from device memory `d_send` of every rank into `d_recv` (rank-major, world * n),
 * e.g. ncclAllGather; returns 0 on success. With it, FIFO placements chain their rounds on
 * the device (the host only checks for completion every few rounds). */
typedef int (*sb_allgather_dev_fn)(void* ctx, const uint64_t* d_send, uint32_t n,
                                   uint64_t* d_recv, void* cuda_stream);
typedef struct sb_shard {
  uint64_t begin, end;     /* this rank owns global instances [begin, end) */
  int32_t rank, world_size;
  sb_allgather_fn allgather; /* required when world_size > 1 */
  void* ctx;
  sb_allgather_dev_fn allgather_dev; /* optional (NULL: host exchange per round) */
  void* ctx_dev;
} sb_shard;

/* ------------------------------------------------------------------------------------
 * Native shard communicator: one process per GPU, no PyTorch.
 * Bootstrap and the host exchange go through a TCP star via rank 0 (host:port; under
 * torchrun e.g. MASTER_ADDR and MASTER_PORT + 1); with device >= 0 every rank also exposes
 * a count board in HBM that each peer maps through CUDA IPC, and sb_shard.allgather_dev
 * becomes remote stores over NVLink / NVSwitch + per-rank epoch flags the consuming stream
 * waits on (cuStreamWaitValue64; no host round trip). The reference has no multi-GPU layer;
 * this replaces the count exchange SURVEY 8(e)(i) describes. */
typedef struct sb_comm sb_comm;
/* Blocks until all world_size ranks have connected (timeout_s <= 0: 300 s). device < 0:
 * host exchange only (no allgather_dev). Ranks must be separate processes. */
sb_status sb_comm_create(int32_t rank, int32_t world_size, int device, const char* host,
                         int32_t port, double timeout_s, sb_comm** out);
void sb_comm_destroy(sb_comm* c);
/* Contiguous variation shard of n_total for this rank + the comm's exchange callbacks
 * (valid while the comm lives). */
sb_status sb_comm_shard(sb_comm* c, uint64_t n_total, sb_shard* out);
sb_status sb_comm_allgather(sb_comm* c, const uint64_t* send, uint32_t n, uint64_t* recv);
/* n <= 31 u64 of device memory per rank, enqueued on cuda_stream (a cudaStream_t). */
sb_status sb_comm_allgather_dev(sb_comm* c, const uint64_t* d_send, uint32_t n, uint64_t* d_recv,
                                void* cuda_stream);
sb_status sb_comm_barrier(sb_comm* c);
/* 1 if the device exchange waits with stream memory operations, 0 if it spins a kernel. */
int32_t sb_comm_uses_stream_waits(const sb_comm* c);

/* ------------------------------------------------------------------------------------
 * Support-surface extraction (surface.cpp:53-153; host, cold start):
 * upward facets within 5 degrees of +z clustered by shared edges, each cluster's xy
 * projection merged with union_of (the oracle's Boost stand-in semantics: edge splicing),
 * parts below 1e-4 m^2 dropped, roofed by a majority of 16 upward ray casts from sampler
 * draws, sorted by area (largest first). mode: SB_SURFACE_ON (open to the sky),
 * SB_SURFACE_INSIDE (roofed cavity floors), SB_SURFACE_ALL (extract_all_support_surfaces).
 * A surface's `frame` is translation(0, 0, z_top) (column-major); polygons with more than
 * SB_MAX_SURFACE_VERTS vertices are an error. */
enum { SB_SURFACE_ON = 0, SB_SURFACE_INSIDE = 1, SB_SURFACE_ALL = -1 };
#define SB_MAX_SURFACE_VERTS 96
typedef struct sb_surface {
  double frame[16];
  double area;
  int32_t roofed;
  uint32_t n_polygon;
  double polygon_xy[2 * SB_MAX_SURFACE_VERTS];
} sb_surface;
sb_status sb_extract_support_surfaces(const double* vertices, uint32_t n_vertices,
                                      const uint32_t* triangles, uint32_t n_triangles,
                                      int32_t mode, sb_surface* out, uint32_t cap,
                                      uint32_t* n_out);

/* Test hook (host, no GPU): region_for(0) of build_constraint_region + apply_ratio_on_support
 * (relationships.cpp:161-230) restated on the host with the serial region path's code
 * (sb_poly.h) and glibc as libm -- states: (x, y, yaw) per anchor in the support frame --
 * then n PolygonSampler::draw points from Pcg32(make_stream(seed, c)) (polygon.cpp:390-400).
 * *n_tris = 0: empty region (no draws). */
sb_status sb_region_draws_host(const sb_relation* rel, const sb_support* support,
                               const double* states, double erode_r, uint64_t seed,
                               const uint64_t* c, uint32_t nc, double* out_xy, uint32_t n,
                               int32_t* n_tris);

typedef struct sb_engine sb_engine;

/* initialize: registers meshes, adds fixed + placement objects, uploads
 * everything once. shard == NULL: this engine owns all n_instances. */
sb_status sb_engine_create(const sb_scene* scene, const sb_shard* shard, int device,
                           sb_engine** out);
void sb_engine_destroy(sb_engine* e);
/* generate / warm_generate: one full rejection-sampling pass over every
 * placement. Results stay in HBM; `out` (optional) is filled from them afterwards. */
sb_status sb_engine_generate(sb_engine* e, uint64_t run_seed, sb_result* out,
                             sb_run_stats* stats);
/* One run driven placement by placement (the per-placement step of the reference's
 * generation loop, SPEC.md:525-528 / Appendix C: prepare the sampler, K attempts of
 * sample -> sample_orientations -> check_batch -> accept, on the device as in
 * sb_engine_generate). first == 0 starts a run (the world's placed objects, counters and
 * grid are reset); a later call continues the open run at placement `first` == the end of
 * the previous call, with the same run_seed (else SB_ERR_LOGIC). Between calls the caller
 * may read or use the world (sb_engine_world: sb_object_pose, sb_enabled, sb_check_batch).
 * `out` is accepted only by the call that completes the run (first + count == number of
 * placements; else SB_ERR_INVALID_ARGUMENT); `stats` are cumulative over the run so far.
 * Any split of [0, P) gives results bit-identical to one sb_engine_generate call. */
sb_status sb_engine_place(sb_engine* e, uint64_t run_seed, uint32_t first, uint32_t count,
                          sb_result* out, sb_run_stats* stats);
/* Copy the last run's results to host buffers (D2H). */
sb_status sb_engine_download(sb_engine* e, sb_result* out);
/* The engine's collision world (for check_batch-level access); owned by the engine. */
sb_world* sb_engine_world(sb_engine* e);
uint64_t sb_engine_local_instances(const sb_engine* e);
/* Kernel launches issued by the last generate call (counted on the host). */
uint64_t sb_engine_last_launches(const sb_engine* e);
/* Device time of the last generate call in ms (CUDA events on the engine stream), and of
 * its check kernels alone (the dominant kernel; roofline numerator). */
sb_status sb_engine_last_timing(const sb_engine* e, double* total_ms, double* check_ms,
                                uint64_t* check_launches);
/* Breakdown of the last generate call, summed over placements (device globaltimer of the
 * placement kernel's block 0, ms): out[0] setup + tile init, out[1] fast-path prefix
 * scans, out[2] A1 sample/compose, out[3] A2+B broad/narrow phase, out[4] C accept +
 * compaction, out[5] grid-barrier waits, out[6] per-instance placements (whole), out[7] =
 * fast-path rounds, out[8] = ms in relation-region preparation (CUDA events), out[9] =
 * total ms (CUDA events), out[10] / out[11] = placement-kernel ms (CUDA events) of the
 * per-instance / fast-path placements, out[12..14] = debug maxima (SB_ROUND_DEBUG). */
sb_status sb_engine_phase_profile(const sb_engine* e, double out[16]);

/* ------------------------------------------------------------------------------------
 * PositionSampler (sampler.hpp:66-96) and sample_orientations (sampler.hpp:98-104) as
 * standalone device-backed calls, for callers that drive their own attempt loop.
 * Regions are given as hole-free rings (x,y pairs; ring r = vertices
 * [ring_offsets[r], ring_offsets[r+1]), at most 96 vertices). instance_rings == NULL:
 * canonical region (ConstraintRegion::region = all rings, the FIFO-cache fast path);
 * else per-instance regions (instance i = rings [instance_rings[i], instance_rings[i+1]),
 * batch_size + 1 entries; sampler.cpp:101-126). Host buffers in and out.
 * ---------------------------------------------------------------------------------- */
typedef struct sb_sampler sb_sampler;
/* PositionSampler(placement_salt) (sampler.hpp:73) on `device`. */
sb_status sb_sampler_create(uint64_t placement_salt, int device, sb_sampler** out);
void sb_sampler_destroy(sb_sampler* s);
/* prepare(constraint, batch_size, run_seed) (sampler.cpp:54-67): rebinds the cache to the
 * stream of run_seed (the queue survives a re-prepare with the same seed) and restarts
 * the cache rng. n_rings == 0 is an empty region (every sample is not placeable). */
sb_status sb_sampler_prepare(sb_sampler* s, const double* ring_xy, const uint32_t* ring_offsets,
                             uint32_t n_rings, const uint32_t* instance_rings,
                             uint64_t batch_size, uint64_t run_seed);
/* sample(support_world, active, attempt, positions, placeable) (sampler.cpp:69-127):
 * support_world = batch_size column-major Mat4 (16 doubles each); positions_xyz = 3 doubles
 * per active entry. A canonical region with zero area is SB_ERR_INVALID_ARGUMENT (the
 * reference draws from an empty table there). */
sb_status sb_sampler_sample(sb_sampler* s, const double* support_colmajor16xN,
                            const uint32_t* active, uint64_t m, uint64_t attempt,
                            double* positions_xyz, uint8_t* placeable);
/* build_constraint_region (relationships.cpp:161-218) + prepare(), on the device: the
 * relation's region against the support rect (x0 y0 x1 y1) for n anchor states
 * (anchor_states: x, y, yaw per instance, support frame; may be NULL when rel->anchor < 0,
 * which means "no anchor": region = the support rect). rel->anchor only selects anchored
 * vs not here. per_instance is decided as the reference does (an anchor moving by more
 * than 1e-12). An empty region_for(0) makes every sample not placeable. */
sb_status sb_sampler_prepare_relation(sb_sampler* s, const sb_relation* rel,
                                      const double support_rect[4], const double* anchor_states,
                                      uint64_t n, uint64_t run_seed);
/* Device-resident sample(): support_world (batch_size column-major Mat4), active,
 * positions and placeable are DEVICE pointers; the work is enqueued on cuda_stream (a
 * cudaStream_t) -- only the SampleCache bookkeeping runs on the host. Active indices must
 * be < batch_size (not checked on the device). */
sb_status sb_sampler_sample_device(sb_sampler* s, const double* d_support_colmajor16xN,
                                   const uint32_t* d_active, uint64_t m, uint64_t attempt,
                                   double* d_positions_xyz, uint8_t* d_placeable,
                                   void* cuda_stream);
/* SampleCache state (sampler.hpp:18-36): points queued, refills so far. */
sb_status sb_sampler_cache_info(const sb_sampler* s, uint64_t* queue_size, uint64_t* refill_count);
/* sample_orientations (sampler.cpp:129-156): kind = SB_ORIENT_*; face_targets_xy = one
 * (x, y) per instance (n_targets of them, SB_ORIENT_FACE_TO only, else NULL). */
sb_status sb_sample_orientations(int kind, const uint32_t* active, uint64_t m,
                                 const double* positions_xyz, const double* face_targets_xy,
                                 uint64_t n_targets, uint64_t run_seed, uint64_t placement_salt,
                                 uint64_t attempt, double* yaws, int device);

/* ------------------------------------------------------------------------------------
 * BatchedSceneGraph (scene_graph.hpp:33-94) with every edge batch resident on one B200:
 * N transforms per edge, articulated nodes (edge = base * joint motion), batched forward
 * kinematics (world_poses) on the device, validity mask. Poses cross as column-major
 * double[16] per instance (TransformBatch memory). Node ids are dense (root = 0).
 * ---------------------------------------------------------------------------------- */
typedef struct sb_graph sb_graph;
typedef struct sb_joint {  /* JointSpec (scene_graph.hpp:19-30) */
  int32_t kind;            /* 0 revolute, 1 prismatic */
  double axis[3];          /* normalised by add_node when |axis| != 1 (scene_graph.cpp:9-17) */
  double lo, hi;
} sb_joint;
sb_status sb_graph_create(uint64_t batch_size, int device, sb_graph** out);
void sb_graph_destroy(sb_graph* g);
/* add_node(parent, name, geometry_id, joint or NULL) (scene_graph.cpp:54-71) */
sb_status sb_graph_add_node(sb_graph* g, uint32_t parent, const char* name, int64_t geometry_id,
                            const sb_joint* joint, uint32_t* id);
sb_status sb_graph_set_edge_batch(sb_graph* g, uint32_t parent, uint32_t child,
                                  const double* poses_colmajor16xN);
sb_status sb_graph_set_edge(sb_graph* g, uint32_t child, uint64_t instance, const double pose[16]);
sb_status sb_graph_edge_batch(const sb_graph* g, uint32_t child, double* poses_colmajor16xN);
sb_status sb_graph_set_joint_states(sb_graph* g, uint32_t node, const double* values_N);
sb_status sb_graph_joint_states(const sb_graph* g, uint32_t node, double* values_N);
/* world_poses(node) (scene_graph.cpp:131-151): batched FK on the device */
sb_status sb_graph_world_poses(const sb_graph* g, uint32_t node, double* poses_colmajor16xN);
/* world_poses into device memory (N column-major Mat4), enqueued on cuda_stream */
sb_status sb_graph_world_poses_device(const sb_graph* g, uint32_t node, double* d_poses16xN,
                                      void* cuda_stream);
/* world_pose(node, instance) (scene_graph.cpp:153-158) */
sb_status sb_graph_world_pose(const sb_graph* g, uint32_t node, uint64_t instance, double pose[16]);
/* find(name): *id = -1 when absent */
sb_status sb_graph_find(const sb_graph* g, const char* name, int64_t* id);
/* name / parent / geometry / articulated / joint of a node; joint_out may be NULL */
sb_status sb_graph_node_info(const sb_graph* g, uint32_t node, const char** name,
                             uint32_t* parent, int64_t* geometry_id, int* articulated,
                             sb_joint* joint_out);
uint64_t sb_graph_node_count(const sb_graph* g);
/* children(node) in ascending id order: up to cap ids into out, the count into *count */
sb_status sb_graph_children(const sb_graph* g, uint32_t node, uint32_t* out, uint32_t cap,
                            uint32_t* count);
sb_status sb_graph_is_tree(const sb_graph* g, int* is_tree);
sb_status sb_graph_valid_mask(const sb_graph* g, uint8_t* mask_N);
sb_status sb_graph_mark_invalid(sb_graph* g, uint64_t instance);
sb_status sb_graph_reset_validity(sb_graph* g);
sb_status sb_graph_valid_count(const sb_graph* g, uint64_t* count);
/* Accepted-pose write-back: the engine's last run, placement
 * `placement`, into `node` (a child of the root: its edge is the world pose; an
 * articulated node receives it as its base) for the engine's local instances, and every
 * instance the run left invalid is marked invalid in the graph. Device to device; the
 * graph must live on the engine's GPU and have its local batch size. */
sb_status sb_engine_write_back(sb_engine* e, uint32_t placement, sb_graph* g, uint32_t node);

/* ------------------------------------------------------------------------------------
 * ReachMap4D (reachability.hpp:14-94) on the device: FK-sampled (r, z, psi) occupancy
 * build, batched queries, placement_filter, and the "SBRM" v1 binary file (byte-compatible
 * with ReachMap4D::save / load).
 * ---------------------------------------------------------------------------------- */
typedef struct sb_chain_link {  /* ChainLink (reachability.hpp:15-18) */
  double origin[16];            /* column-major fixed transform to the joint frame */
  sb_joint joint;
} sb_chain_link;
typedef struct sb_reach_map sb_reach_map;
typedef struct sb_reach_info {
  uint64_t samples;
  double resolution, psi_resolution, max_radius, z_min, z_max;
  uint64_t nr, nz, npsi, cell_count, occupied_cells;
} sb_reach_info;
/* ReachMap4D::build(chain, samples, resolution, psi_resolution, seed) */
sb_status sb_reach_build(const sb_chain_link* links, uint32_t n_links, const double ee_offset[16],
                         uint64_t samples, double resolution, double psi_resolution,
                         uint64_t seed, int device, sb_reach_map** out);
sb_status sb_reach_load(const char* path, int device, sb_reach_map** out);
sb_status sb_reach_save(const sb_reach_map* m, const char* path);
void sb_reach_destroy(sb_reach_map* m);
sb_status sb_reach_get_info(const sb_reach_map* m, sb_reach_info* out);
/* FK samples recorded in a cell (0 after load) */
sb_status sb_reach_cell_samples(const sb_reach_map* m, uint64_t ir, uint64_t iz, uint64_t ipsi,
                                uint32_t* count);
/* query_batch(base_poses, targets, inclination) (reachability.cpp:143-162): has_inclination
 * = 0 ignores `inclination` (any psi). */
sb_status sb_reach_query_batch(const sb_reach_map* m, const double* base_colmajor16xN,
                               const double* targets_xyz, uint64_t n, int has_inclination,
                               double inclination, uint8_t* out);
/* query_batch with device pointers (base poses, targets, out), enqueued on cuda_stream */
sb_status sb_reach_query_batch_device(const sb_reach_map* m, const double* d_base_colmajor16xN,
                                      const double* d_targets_xyz, uint64_t n,
                                      int has_inclination, double inclination, uint8_t* d_out,
                                      void* cuda_stream);
/* placement_filter(map, robot_base, frames, active) (reachability.cpp:164-190): frames =
 * n_frames pointers to N column-major poses each (NULL entries skipped). */
sb_status sb_reach_placement_filter(const sb_reach_map* m, const double* robot_base16xN,
                                    uint64_t n, const double* const* frames16xN,
                                    uint32_t n_frames, const uint32_t* active, uint64_t m_active,
                                    uint8_t* out);

/* Fused reachability filter: from the next generate
 * on, placement `placement` accepts a candidate only if its frame origin, expressed in the
 * instance's robot base frame, falls in an occupied (r, z) cell of `map`
 * (placement_filter, reachability.cpp:164-190); an unreachable candidate is a failed
 * attempt and is not collision-checked. robot_base: the engine's local instances'
 * column-major poses. map == NULL clears the filter. The map must outlive the engine's use. */
sb_status sb_engine_set_reach_filter(sb_engine* e, uint32_t placement, const sb_reach_map* map,
                                     const double* robot_base_colmajor16xN);

/* sample_orientations on device pointers (active, positions_xyz, face_targets_xy, yaws),
 * enqueued on cuda_stream (a cudaStream_t). */
sb_status sb_sample_orientations_device(int kind, const uint32_t* d_active, uint64_t m,
                                        const double* d_positions_xyz,
                                        const double* d_face_targets_xy, uint64_t run_seed,
                                        uint64_t placement_salt, uint64_t attempt, double* d_yaws,
                                        void* cuda_stream);

/* Diagnostics: evaluate the device libm used on the hot path (sb_glibcm.cuh: glibc
 * 2.39's sincos / sin / cos / atan2 restated bit for bit, replacing the reference's
 * std::sin/cos/atan2 in transform.hpp:47,77, polygon.cpp:151, relationships.cpp:95,202,238)
 * on n inputs on device 0. fn 0 / 1: the sine / cosine of sincos(in[i]) (what GCC makes of
 * the reference's adjacent std::cos + std::sin); 2: atan2(in[2i], in[2i+1]); 3 / 4: sin /
 * cos(in[i]). */
sb_status sb_device_math(int fn, const double* in, uint64_t n, double* out);
/* The same functions (same fn codes) evaluated by the host build of sb_glibcm.cuh: no
 * device needed; the CPU tests pin the restatement to the host's glibc with it. */
sb_status sb_host_math(int fn, const double* in, uint64_t n, double* out);
/* Diagnostics: narrow-phase cycle breakdown accumulated since the last call (all zeros
 * unless the library was built with -DSB_NARROW_PROF): pose+M, node tests, triangle
 * transform, DAG walk, triangle tests, pairs. */
sb_status sb_debug_narrow_profile(uint64_t out[8]);
/* Diagnostics: stage cycle profile of the relation-region kernel (sb_region.cu; zeros
 * unless the library is built with -DSB_REGION_PROF); read and reset. */
sb_status sb_debug_region_profile(uint64_t out[8]);

#ifdef __cplusplus
}
#endif
#endif /* SCENEBATCH_B200_H_ */
