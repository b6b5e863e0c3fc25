/* pxg.h — C ABI of libpxg, the sm_100a implementation of the proxy-BDPT render loop.
 *
 * Drop-in boundary: the reference entry point
 *   Image proxima::render_proxy_bdpt(const Scene&, int spp, uint64_t seed,
 *                                    const ProxyParams& = {}, ProxyDiagnostics* = nullptr,
 *                                    const std::function<bool(int, const Image&)>& = {})
 * (proj/include/proxima/proxy.hpp:197-200, proj/src/proxy.cpp:647-834) is replaced by
 *   pxg_create(scene, params, seed)  -> context (scene upload, Scene::finalize, BVH, pretrace)
 *   pxg_render_pass(ctx)             -> one progressive pass = 1 spp for every pixel
 *   pxg_read_mean(ctx, rgb)          -> running mean image (the pass_done callback argument)
 *   pxg_read_diag(ctx, ...)          -> ProxyDiagnostics (proj/include/proxima/proxy.hpp:175-188)
 *   pxg_destroy(ctx)
 * The C++ wrapper `render_proxy_bdpt_gpu` (include/pxg_proxima.hpp) and the Python mirror
 * (paper_2503_23412_b200.render_proxy_bdpt) loop passes and call pass_done between them.
 *
 * Conventions: plain pointers and sizes only; every function returns 0 on success and a
 * negative PXG_E* code on failure (no exceptions cross the ABI); the message is in
 * pxg_last_error(ctx) (or pxg_last_error(NULL) when no context exists). The context owns
 * all device memory; input arrays are only read during the call.
 */
#ifndef PXG_H
#define PXG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PXG_ABI_VERSION 1

enum {
  PXG_OK = 0,
  PXG_E_INVALID = -1,   /* validation error (reference: std::runtime_error from load_scene /
                           std::invalid_argument from the statistics, exit code 2 in the CLI) */
  PXG_E_CUDA = -2,      /* CUDA runtime failure */
  PXG_E_RUNTIME = -3,   /* numeric failure inside the estimator (reference: std::runtime_error
                           "reciprocal: integrand must be finite and non-negative", recip.hpp:74-75) */
  PXG_E_NODEVICE = -4
};

/* Flattened proxima::Scene (proj/include/proxima/scene.hpp:16-96). Primitive i:
 * shape 0 sphere (a = centre, radius[i]), 1 triangle (a, b, c vertices),
 * 2 rectangle (a = origin, b, c = edges). Materials: 7 doubles each
 * {base_r, base_g, base_b, metallic, roughness, transmission, ior} (bsdf.hpp:13-20). */
typedef struct pxg_scene_desc {
  int n_prims;
  const int* shape;
  const int* material;
  const double* a; /* [n_prims*3] */
  const double* b; /* [n_prims*3] */
  const double* c; /* [n_prims*3] */
  const double* radius; /* [n_prims] */
  int n_materials;
  const double* materials; /* [n_materials*7] */
  int n_emitters;
  const int* emitter_prim;       /* [n_emitters] */
  const double* emitter_radiance;/* [n_emitters*3] */
  double cam_position[3];
  double cam_look_at[3];
  double cam_up[3];
  double fov_y;
  int width, height;
  int max_depth; /* Settings::max_depth (scene.hpp:50-54) */
} pxg_scene_desc;

/* proxima::ProxyParams (proj/include/proxima/proxy.hpp:162-173), same defaults. */
typedef struct pxg_params {
  int enabled;            /* 1 */
  int pool_budget;        /* 400 */
  int recip_repeats;      /* 5 */
  int freeze_iteration;   /* 40 */
  long long recursion_cap;/* 10000 */
  int pretrace_paths;     /* 20000 */
  int light_walks;        /* 0 = one per pixel */
  double gate_high;       /* 1.0 */
  double gate_low;        /* 0.2 */
  double gate_threshold;  /* 0.05 */
} pxg_params;

/* Pixel-row shard of a multi-GPU render: this context renders image rows
 * [row_begin, row_end) (multiples of the 10-pixel gate grid) and pool walks
 * [walk_begin, walk_end). A single-GPU render uses {0, height, 0, light_walks}
 * (pxg_create fills it when shard == NULL). */
typedef struct pxg_shard {
  int row_begin, row_end;
  int walk_begin, walk_end;
} pxg_shard;

typedef struct pxg_ctx pxg_ctx;
/* A finalised scene: the reference's Scene after load_scene -> Scene::finalize
 * (proj/src/scene.cpp:234-252, 317-436), i.e. validated, with emitter tables and the BVH
 * built (on the host, once). Immutable; contexts on any device are created from it without
 * rebuilding, as the reference's render_proxy_bdpt(const Scene&, ...) receives a finalised
 * scene. The description's arrays are copied. */
typedef struct pxg_scene pxg_scene;

void pxg_default_params(pxg_params* p);
int pxg_abi_version(void);
int pxg_device_count(void);

int pxg_scene_create(const pxg_scene_desc* scene, pxg_scene** out);
void pxg_scene_destroy(pxg_scene* scene);
/* Bytes one context uploads from the finalised scene (BVH nodes, primitive records and tables). */
long long pxg_scene_device_bytes(const pxg_scene* scene);
/* Render context on `device` for a finalised scene (uploads it, allocates the per-pass state,
 * runs the pretrace, proj/src/subspace.cpp:190-218). */
int pxg_create_from_scene(const pxg_scene* scene, const pxg_params* params, uint64_t seed, int device,
                          const pxg_shard* shard, pxg_ctx** out);
/* pxg_scene_create + pxg_create_from_scene in one call (the scene is released again). */
int pxg_create(const pxg_scene_desc* scene, const pxg_params* params, uint64_t seed, int device,
               const pxg_shard* shard, pxg_ctx** out);
void pxg_destroy(pxg_ctx* ctx);
const char* pxg_last_error(const pxg_ctx* ctx);

/* One progressive pass (Stage 1 pool + reciprocal estimates, Stage 2 per-pixel strategies
 * with the gated proxy connection, gamma update), proj/src/proxy.cpp:683-827. */
int pxg_render_pass(pxg_ctx* ctx);
/* One pass that also records the sub-path primitive ids for pxg_dump_prims. */
int pxg_render_pass_traced(pxg_ctx* ctx);
/* Several passes back to back. Stage 1 of the next pass is computed one pass ahead on a
 * second stream (results are identical to the sequential order). */
int pxg_render_passes(pxg_ctx* ctx, int n);
/* Total number of passes the caller intends to render (the spp of the render call): no
 * look-ahead Stage 1 is started for pass >= limit. -1 (default) = unbounded. */
int pxg_set_pass_limit(pxg_ctx* ctx, int limit);
/* Pipelined progressive rendering: enqueue passes without waiting for them, snapshot the
 * running mean on the device after the enqueued passes (slot 0 .. PXG_SNAPSHOT_SLOTS-1),
 * and read a snapshot back later (waits for it). A caller can hand pass p's mean to its
 * pass_done callback while passes p+1.. already run; stopping early returns the snapshot
 * of pass p, which is bitwise the image a p-pass render returns. */
#define PXG_SNAPSHOT_SLOTS 4
int pxg_render_passes_async(pxg_ctx* ctx, int n);
int pxg_snapshot_mean(pxg_ctx* ctx, int slot);
int pxg_read_snapshot(pxg_ctx* ctx, int slot, double* rgb, int* passes_done);
/* Renders `n` passes in measurement mode: every traversal launch (closest hit / any hit)
 * is bracketed by CUDA events on its stream and followed by an instrumented copy on the
 * same rays that counts 4-wide BVH node visits (pxg_node_bytes(ctx) each) and primitive tests
 * (80 B each).
 * out[10] = {closest: ms, launches, rays, node visits, prim tests,
 *            any-hit: ms, launches, rays, node visits, prim tests}. */
int pxg_measure_traversal(pxg_ctx* ctx, int n, double* out);
/* Bytes of one BVH node visit of this context's persistent traversal kernels (the
 * roofline's algorithmic bytes per node): 64 for the quantised 4-wide node (scenes whose
 * 128 B node array exceeds 2 MB), 128 otherwise. */
int pxg_node_bytes(const pxg_ctx* ctx);
int pxg_synchronize(pxg_ctx* ctx);

/* Running mean acc/done over this context's rows, row-major fp64 RGB, y = 0 top
 * (proj/src/proxy.cpp:822-833). rgb holds (row_end-row_begin)*width*3 doubles. */
int pxg_read_mean(pxg_ctx* ctx, double* rgb, int* passes_done);
/* Unnormalised accumulator (sum of per-pass values), for shard reduction. */
int pxg_read_accum(pxg_ctx* ctx, double* rgb, int* passes_done);
/* Same, copied device-to-device into `dst` (a device buffer on the context's GPU, e.g. a
 * tensor that is then NCCL-reduced across ranks), stream-ordered against the caller's CUDA
 * stream `stream` (a cudaStream_t; NULL = the legacy default stream): the copy starts after the
 * work already enqueued on `stream` (so it never overwrites `dst` while an earlier in-place
 * reduce is still running) and includes every pass enqueued on the context so far; work the
 * caller enqueues on `stream` afterwards runs after the copy. Never blocks the host. */
int pxg_accum_to_device_async(pxg_ctx* ctx, double* dst, void* stream, int* passes_done);
/* pxg_accum_to_device_async on the legacy default stream, then waits for the copy. */
int pxg_accum_to_device(pxg_ctx* ctx, double* dst, int* passes_done);

/* ProxyDiagnostics: rows[4000*5] = {retrace_attempts, retrace_accepts, recip_runs,
 * recip_truncated, estimates_failed} per dense key ((u-1)*10+c)*100+s; touched[4000]
 * marks keys present in the reference's map; pool[2] = {pool_raw, pool_kept}. */
int pxg_read_diag(pxg_ctx* ctx, long long* rows, int* touched, long long* pool);

/* Subspace statistics snapshot (SubspaceStats, subspace.hpp:88-119): per dense key
 * {max_ratio, sum_est, sum_est_sq} and {ratio_count, est_count}; gamma rows [32*100]. */
int pxg_read_stats(pxg_ctx* ctx, double* stats3, long long* counts2, double* gamma_rows);

/* Parity replay of the last rendered pass, for this context's pixels:
 * val[n*3] final per-pixel sample value, bdpt[n*3] standard strategies only,
 * c[n*3] proxy_connect value before gating, flags[n] (bit0 eye cut exists, bit1 proxy
 * connection attempted, bit2 gate passed, bit3 contributed). Any pointer may be NULL. */
int pxg_dump_pass(pxg_ctx* ctx, double* val, double* bdpt, double* c, int* flags);
/* Primitive ids of the last pass's sub-paths: eye[n*(max_depth+1)], light[n*(max_depth-1)],
 * -2 past the end of a sub-path, -1 for the camera vertex. */
int pxg_dump_prims(pxg_ctx* ctx, int* eye, int* light);
/* Pool of the last pass: n kept entries, walk, prefix end, dense key, inverse_p,
 * inverse_p second moment and the bound B used; raw = eligible incompletes. */
int pxg_dump_pool(pxg_ctx* ctx, int cap, int* n, long long* raw, int* walk, int* end, int* key,
                  double* inv_p, double* inv_p_m2, double* bound);

/* proxima::PathVertex (proj/include/proxima/transport.hpp:17-27) as the device stores it
 * (128 B): material = index into the scene's materials (-1: camera), flag = VertexFlag
 * {kLight, kDiffuse, kSpecular, kCamera}. */
typedef struct pxg_vertex {
  double p[3], n[3], wi[3], throughput[3];
  double pdf_fwd;
  int material, primitive, emitter, flag;
  double reserved;
} pxg_vertex;

/* Light vertices a repaired proxy path holds at most (prefix + retraced block + endpoint). */
#define PXG_MAX_LIGHT 16

/* Per-pixel record of the last pass for replay parity (SURVEY §8c mode ii: the device's
 * vertices rescored by the reference's own functions). The pool entry fields are the
 * IncompleteLightSubPath (proj/include/proxima/proxy.hpp:27-42) the pixel's proxy connection
 * picked; block/retrace_density are its retrace_proxy result (proj/src/proxy.cpp:271-319). */
typedef struct pxg_path_record {
  int n_eye, n_light;  /* sub-path vertex counts (eye vertex 0 = camera) */
  int tp;              /* eye cut at the first non-specular vertex (0: none), proxy.cpp:749-757 */
  int flags;           /* bit0 tp >= 2, bit1 attempted, bit2 a pool entry was picked,
                          bit4 retrace accepted (density > 0) */
  int entry;           /* pool entry index (-1: none) */
  int u, n_prefix, has_cdir, c_label, s_label, key, reserved;
  double cdir[3];      /* control_dir (valid when has_cdir) */
  double prefix_pdf, inverse_p, inverse_p_m2;
  double retrace_density; /* sample-time density of the retraced block (bit4) */
  double q_sel;        /* gamma row pmf / bucket size of the pick */
  double bdpt[3];      /* standard strategies (weighted_bdpt_value) */
  double c[3];         /* proxy_connect value before gating */
  double val[3];       /* final per-pixel sample value of the pass */
} pxg_path_record;

/* Replay dump of the last rendered pass for pixels [px_begin, px_end) of this context
 * (not for Stage-2 row-tiled contexts). Outputs, any pointer may be NULL:
 *   rec[m]                                    per-pixel record (m = px_end - px_begin)
 *   eye[m * (max_depth + 1)]                  eye sub-path vertices, pixel-major
 *   light[m * (max_depth - 1)]                light sub-path vertices, pixel-major
 *   proxy[m * PXG_MAX_LIGHT]                  the picked entry: prefix vertices [0, n_prefix),
 *                                             the retraced block g in reference order
 *                                             (g[0] nearest the specular endpoint, bit4 only)
 *                                             at [n_prefix, n_prefix + u), the specular
 *                                             endpoint at n_prefix + u
 *   stats[4000 * 3]                           the pass's SubspaceStats snapshot the MIS
 *                                             weights read: sum_est, sum_est_sq, est_count
 *                                             per dense key ((u-1)*10+c)*100+s. */
int pxg_dump_paths(pxg_ctx* ctx, int px_begin, int px_end, pxg_path_record* rec, pxg_vertex* eye, pxg_vertex* light,
                   pxg_vertex* proxy, double* stats);

/* Scene::intersect / Scene::occluded on the device (parity of the traversal kernel).
 * rays[n*6] = origin, unit direction; tmax may be NULL (1e30). */
int pxg_intersect(pxg_ctx* ctx, int n, const double* rays, const double* tmax, int* prim, double* t);
int pxg_occluded(pxg_ctx* ctx, int n, const double* segs, int* occ);

/* Parity probe of the proxy densities on caller-supplied vertices (device-level pins of the
 * reference's closed-form tests, proj/tests/test_proxy.cpp:480-618): the light walk
 * walk[n_walk] goes through dropout (proj/src/proxy.cpp:59-94) on the device;
 *   info[8]      {valid, u, n_prefix, has_control_dir, c_label, s_label, dense key, dropped flag}
 *   prefix_pdf   IncompleteLightSubPath::prefix_pdf
 *   q[i], f[i]   support_pdf (proxy.cpp:153-209) and target_density (proxy.cpp:106-151) of the
 *                candidate block cand[i*u .. i*u+u) (g[0] nearest the specular endpoint)
 *   draw_*[j]    support_sample (proxy.cpp:211-269) on stream (seed, PROBE, 0, j): the block
 *                (u vertices, zero when escaped), its density (1 when escaped), the escape flag.
 * Nothing is computed when dropout rejects the walk (info[0] = 0). */
int pxg_proxy_probe(pxg_ctx* ctx, int n_walk, const pxg_vertex* walk, int n_cand, const pxg_vertex* cand, int n_draws,
                    uint64_t seed, int* info, double* prefix_pdf, double* q, double* f, pxg_vertex* draw_cand,
                    double* draw_q, int* draw_escaped);

/* Reciprocal estimation of the probed incomplete sub-path on the device, through the
 * production node wavefront and DFS (estimate_reciprocal, proj/include/proxima/recip.hpp:131-138,
 * with the proxy integrand of estimate_inverse_p, proj/src/proxy.cpp:397-409) at the given
 * bound: n_runs independent runs (run i on the node streams of (pass 0x700000 + i / 255, run
 * i % 255)), est[i] an unbiased estimate of 1 / integral(target_density) when not truncated.
 * The device-level analogue of proj/tests/test_proxy.cpp:620-673. Call between passes only
 * (it uses the context's reciprocal run buffers; the call synchronises the device). */
int pxg_proxy_recip(pxg_ctx* ctx, int n_walk, const pxg_vertex* walk, double bound, int n_runs, double* est,
                    long long* cost, int* truncated);

/* Parity of the traversal kernels that ship: the same rays as pxg_intersect (any_hit = 0:
 * rays[n*6] origin + unit direction, tmax may be NULL) or pxg_occluded (any_hit = 1:
 * segments[n*6] from + to, prim[i] = 1 when occluded, t unused) through
 *   kernel 0: the single-ray paths (trace_closest_t / trace_any_t, 128 B nodes),
 *   kernel 1: the production persistent queue kernels k_trav_persistent<0/1> (lane refill,
 *             256-bit loads, the context's node layout: pxg_node_bytes),
 *   kernel 2: the reciprocal node wavefront's traversal (rw_trace: per-lane step loops,
 *             or warp_trace with postponed leaf tests when built with PXG_RW_WARP=1).
 * Reference: Scene::intersect / Scene::occluded (proj/src/scene.cpp:127-177). */
int pxg_trace_rays(pxg_ctx* ctx, int kernel, int any_hit, int n, const double* rays, const double* tmax, int* prim,
                   double* t);

/* proxima::render_pt (proj/include/proxima/transport.hpp:88, proj/src/transport.cpp:272-381)
 * on the device for this context's pixels: the unidirectional path tracer with NEE, the
 * converged reference of the relMSE checks. rgb[n*3] = mean over `chunks` independent
 * renders; chunk c is render_pt(spp, seed ^ c*0x9E3779B97F4A7C15), so chunks = 1 is exactly
 * the reference's render_pt(scene, spp, seed) on the same Philox pixel streams. */
int pxg_render_pt(pxg_ctx* ctx, int spp, uint64_t seed, int chunks, double* rgb);

/* Reciprocal estimator on the two-point fixture f = {1,3}, q = 1/2 (the reference's own
 * known-answer case, proj/tests/test_recip.cpp:16-23), run i on stream (seed, RECIP, 0, i). */
int pxg_recip_twopoint(int n, double bound, long long cap, uint64_t seed, double* est,
                       long long* cost, int* truncated);

/* Philox stream check: first n draws of stream (seed, kind, sub, stream) computed on the device. */
int pxg_rng_draws(uint64_t seed, unsigned kind, unsigned sub, uint64_t stream, int n, unsigned* out);

/* sin(phi), cos(phi) of phi = 2*pi*(k[i] * 2^-32) on `device` with the samplers' device
 * code (include/pxg_sincos.h): bitwise the host glibc's std::sin / std::cos that the
 * reference calls at proj/src/bsdf.cpp:63-65, 226-227 and proj/src/scene.cpp:199-201. */
int pxg_sincos_2pi(int device, int n, const uint32_t* k, double* s, double* c);

/* Device timeline of the last pxg_render_passes call (ms, CUDA events on the context's
 * stream): t[0] stage 1 (pool walks, selection, probes, reciprocal runs, incl. the host
 * round trip of the selection), t[1] reciprocal runs alone, t[2] sub-path trace,
 * t[3] connections + MIS, t[4] proxy connection, t[5] gate + film (t[2..5]: the last pass
 * of the call; the streams overlap, so these are spans, not exclusive times), t[6] the
 * whole call (first pass start to the end of all work it enqueued), t[7] reserved.
 * counts[0] = kernel launches, counts[1] reserved. t holds 8 doubles. */
int pxg_read_timing(pxg_ctx* ctx, double* t, long long* counts);

/* Reciprocal estimation work so far (finished runs of every Stage-1 batch enqueued; waits for
 * Stage 1): out[0] = tree nodes evaluated (draw_g calls made ahead of the DFS, recip.hpp:69-77),
 * out[1] = tree nodes the runs consumed (ReciprocalRun::cost summed), out[2] = runs. */
int pxg_read_recip_counts(pxg_ctx* ctx, long long* out);

#ifdef __cplusplus
}
#endif

#endif /* PXG_H */
