// lists_dev.cuh -- row a-P2 of SURVEY.md §8(a) on the device.
//
//   P2P lists: leaf T's sources are the leaf descendants of the 27 same-level neighbours of T (one
//              contiguous range of the Morton-ordered leaves each) and the leaves adjacent to T's
//              ancestors (R20)
//   V lists:   per level, I^C = N^P \ N^C: the children of the parent's near cubes (max|Delta| <= R_p)
//              that are not near the cube (max|Delta| > R_c; HF: R = floor(1 + k w / pi), R14), grouped by
//              offset (one translation operator per offset) and sorted by target
//   slots:     one outgoing (incoming) expansion per (cube, source (antipodal target) wedge) an M2L pair
//              or a used parent's translation reaches (R15), numbered cube-major
// The cube table comes from the device tree; the results are written into the host plan (lists, slot
// tables, M2L groups with their (target slot, source slot) pairs) for the rest of the plan builder.
#pragma once
#include <string>

namespace fda {

struct HostPlan;  // plan.hpp

// Fills P.p2p_ptr / p2p_src, P.lmin, the slot tables of every level, P.m2l_groups and P.m2l_tgt / src from
// P.cubes / P.levels / P.leaves.  Returns "" or "CUDA".
std::string build_lists_device(HostPlan& P);

}  // namespace fda
