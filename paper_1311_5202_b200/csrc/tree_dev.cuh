// tree_dev.cuh -- rows a-P0 and a-P1 of SURVEY.md §8(a) on the device.
//
//   P0  validate the inputs, bounding cube x (1 + 1e-6) (R13), 21-bit-per-axis Morton keys, a
//       stable radix sort (the caller order breaks ties), the Morton-ordered SoA geometry the apply reads,
//       the coincident-point check
//   P1  the adaptive octree level by level: a cube splits iff it holds more than N_p points or is an HF
//       cube (w >= lambda, R13/R21); its children are the distinct Morton prefixes of its points,
//       found by one flag + scan pass over the points per level
// Only the cube table (a few hundred thousand cubes) goes to the host, where the lists and operators
// of the plan are built from it.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace fda {

struct TreeIn;  // plan.hpp

// Morton-ordered geometry on the device (allocated by the caller, n each)
struct DevGeom {
  double *x, *y, *z, *nx, *ny, *nz, *w;
  int32_t* perm;  // Morton position -> caller index
};

// pts / nrm (n x 3, xyz interleaved) and w (n) in caller order on the device.  Returns "" or
// "INVALID_ARG" / "COINCIDENT_POINTS"; CUDA errors as "CUDA".
std::string build_tree_device(int64_t n, const double* pts, const double* nrm, const double* w, double k, int np,
                              int single_leaf, int max_depth, const DevGeom& g, TreeIn& out, cudaStream_t st);

// The correction CSR (caller order, device arrays) into Morton order for the rows [r0, r1) (H3 reads
// them): validates row_ptr (0, monotone, nnz) and the columns, maps rows through perm and columns through
// its inverse.  optr (n + 1, caller-allocated) gets the Morton-row offsets of [r0, r1]; ocol / oval are
// cudaMalloc'ed (onnz entries).  Returns "" or "INVALID_ARG" / "CUDA".
std::string permute_csr_device(int64_t n, int64_t nnz, const int64_t* rp, const int32_t* col, const double2* val,
                               const int32_t* perm, int64_t r0, int64_t r1, int64_t* optr, int32_t** ocol,
                               double2** oval, int64_t* onnz, cudaStream_t st);

}  // namespace fda
