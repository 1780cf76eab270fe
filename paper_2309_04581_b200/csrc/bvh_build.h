// bvh_build.h - host-side BVH (see bvh_build.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace hrt {

struct BvhNodeHost {        // layout identical to the device BvhNode (64 B)
    double lo[3] = {0, 0, 0};
    double hi[3] = {0, 0, 0};
    int32_t first = 0;
    int32_t count = 0;
};
static_assert(sizeof(BvhNodeHost) == 56, "node layout");

struct BvhHost {
    int32_t n_faces = 0;
    std::vector<BvhNodeHost> nodes;
    std::vector<double> tri;        // leaf order, 9 doubles per face
    std::vector<int32_t> tri_id;    // leaf order -> global face id
    std::vector<int32_t> parent;    // node -> parent (-1 at the root), for GPU refit
    std::vector<int32_t> leaves;    // indices of leaf nodes
    std::vector<int32_t> roots;     // build_forest: root node of every group's tree
};

BvhHost build_bvh(int64_t n_faces, const double* v0, const double* e1, const double* e2);

// One tree per group of consecutive faces [group_begin[g], group_begin[g+1]),
// concatenated (node / triangle indices offset, every root's parent -1). The
// trees of rigidly moving meshes stay tight under refit; a small top level
// over their root boxes is rebuilt per frame (hrt.cu).
BvhHost build_forest(int64_t n_faces, const double* v0, const double* e1, const double* e2,
                     const std::vector<int32_t>& group_begin);

}  // namespace hrt
