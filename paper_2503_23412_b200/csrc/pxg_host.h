// pxg_host.h — host-side scene finalisation and BVH build (pxg_host.cpp).
#pragma once

#include <vector>

#include "pxg.h"

namespace pxg {

using SceneDesc = pxg_scene_desc;

// Layout-identical to pxg::BvhNode (pxg_scene.cuh), 64 B.
struct alignas(16) HostNode {
  float lo0[3] = {0, 0, 0}, hi0[3] = {0, 0, 0};
  float lo1[3] = {0, 0, 0}, hi1[3] = {0, 0, 0};
  int c0 = ~0, c1 = ~0;
  int pad0 = 0, pad1 = 0;
};
static_assert(sizeof(HostNode) == 64, "node size");

// Layout-identical to pxg::PrimRec, 80 B.
struct alignas(16) HostRec {
  double v[9];
  int shape;
  int id;
};
static_assert(sizeof(HostRec) == 80, "record size");

// Layout-identical to pxg::BvhNode4 (pxg_scene.cuh), 128 B: four child boxes as SoA
// float4s (lo x/y/z, hi x/y/z), four child codes (>= 0 node, < 0 leaf ~(first*16+count)).
struct alignas(16) HostNode4 {
  float lo[3][4];
  float hi[3][4];
  int child[4];
  int pad[4];
};
static_assert(sizeof(HostNode4) == 128, "node4 size");

// Layout-identical to pxg::BvhNode4Q (pxg_scene.cuh), 64 B: the same 4-wide node with its
// child boxes quantised to 8 bits per plane on a per-node grid (origin + q * 2^e per axis,
// rounded outward, so the quantised boxes contain the fp32 boxes).
struct alignas(32) HostNode4Q {
  float origin[3];
  unsigned exps;     // byte a: biased exponent of the axis-a grid step 2^(e-127); bits 24-27: child k is a leaf
  int child[4];
  unsigned qlo[3];   // byte k of qlo[a]: child k's lower plane on axis a
  unsigned qhi[3];
  unsigned pad[2];
};
static_assert(sizeof(HostNode4Q) == 64, "node4q size");

struct SceneHost {
  std::vector<int> prim_mat, prim_shape, prim_emitter;
  std::vector<double> prim_geo;     // [n][3]
  std::vector<double> prim_center;  // [n][4]
  std::vector<double> prim_abc;     // [n][9]
  std::vector<double> emitter_cum;  // [n_emit]
  double total_emitter_area = 0.0;
  double bbox_min[3], bbox_max[3];
  double cam[12];  // position, fwd, right, up
  double tan_half = 0.0, aspect = 1.0;
  std::vector<HostNode> nodes;
  std::vector<HostNode4> nodes4;
  std::vector<HostNode4Q> nodes4q;  // only when nodeq
  bool nodeq = false;               // the persistent traversal uses the quantised nodes
  std::vector<int> order;
  std::vector<HostRec> recs;
  int bvh_depth = 0;
};

void finalize_scene(const SceneDesc& d, SceneHost& h);

}  // namespace pxg
