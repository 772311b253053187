// Node table of the balanced binary partition and per-node bounding boxes.
//
// The reference never materialises its tree: the sampler derives child
// ranges on the fly (proj/src/sampler.cpp:138-141, :194-200) and the FGT
// backend builds the same BFS family of ranges (proj/src/kde_fast.cpp:252-264).
// The device path stores it heap-ordered so every kernel can look a node up
// by (level, slot) in O(1), together with an axis-aligned bounding box that
// the KDE kernels turn into an exact exponent offset (no underflow of far
// sums in fp32) — see kde.cu.
#include <cfloat>

#include "engine.cuh"

namespace fsgg {

namespace {

__global__ void tree_ranges_kernel(uint32_t n, uint64_t slots, uint32_t* first,
                                   uint32_t* last) {
  uint64_t h = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (h >= slots) return;
  uint64_t h1 = h + 1;
  uint32_t level = 63 - __clzll(h1);
  uint64_t g = h1 - (1ull << level);
  uint32_t f = 0, l = n;
  bool valid = true;
  for (int b = int(level) - 1; b >= 0; --b) {
    uint32_t size = l - f;
    if (size < 2) {
      valid = false;
      break;
    }
    uint32_t mid = f + size / 2;
    if ((g >> b) & 1)
      f = mid;
    else
      l = mid;
  }
  first[h] = valid ? f : 0;
  last[h] = valid ? l : 0;
}

// Bottom-up: a node's box is its point (size 1) or the union of its
// children's boxes. Empty nodes get an inverted box.
__global__ void tree_boxes_kernel(const float* __restrict__ pts, uint32_t d,
                                  uint32_t level, const uint32_t* first,
                                  const uint32_t* last, float* lo, float* hi) {
  uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (g >= (1ull << level)) return;
  uint64_t h = (1ull << level) - 1 + g;
  uint32_t size = last[h] - first[h];
  if (size == 0) {
    for (uint32_t k = 0; k < d; ++k) {
      lo[h * d + k] = FLT_MAX;
      hi[h * d + k] = -FLT_MAX;
    }
  } else if (size == 1) {
    const float* p = pts + size_t(first[h]) * d;
    for (uint32_t k = 0; k < d; ++k) lo[h * d + k] = hi[h * d + k] = p[k];
  } else {
    uint64_t c0 = 2 * h + 1, c1 = 2 * h + 2;
    for (uint32_t k = 0; k < d; ++k) {
      lo[h * d + k] = fminf(lo[c0 * d + k], lo[c1 * d + k]);
      hi[h * d + k] = fmaxf(hi[c0 * d + k], hi[c1 * d + k]);
    }
  }
}

}  // namespace

void build_tree(Dataset& ds) {
  TreeTable& t = ds.tree;
  t.n = ds.n;
  t.d = ds.d;
  uint32_t depth = 0;
  while ((1ull << depth) < ds.n) ++depth;  // ceil(log2 n)
  t.depth = depth;
  t.slots = (2ull << depth) - 1;
  cudaStream_t s = ds.stream;
  t.first.ensure(t.slots * 4, s);
  t.last.ensure(t.slots * 4, s);
  const int tpb = 256;
  tree_ranges_kernel<<<ceil_div_u32(t.slots, tpb), tpb, 0, s>>>(
      ds.n, t.slots, t.first.as<uint32_t>(), t.last.as<uint32_t>());
  FSGG_LAUNCH_CHECK();
  ds.launches++;
  t.has_boxes = ds.d <= kBoxMaxDim;
  if (t.has_boxes) {
    t.lo.ensure(t.slots * ds.d * 4, s);
    t.hi.ensure(t.slots * ds.d * 4, s);
    for (int level = int(depth); level >= 0; --level) {
      uint64_t cnt = 1ull << level;
      tree_boxes_kernel<<<ceil_div_u32(cnt, tpb), tpb, 0, s>>>(
          ds.pts.as<float>(), ds.d, level, t.first.as<uint32_t>(),
          t.last.as<uint32_t>(), t.lo.as<float>(), t.hi.as<float>());
      FSGG_LAUNCH_CHECK();
      ds.launches++;
    }
  }
  ds.tree_valid = true;
}

}  // namespace fsgg
