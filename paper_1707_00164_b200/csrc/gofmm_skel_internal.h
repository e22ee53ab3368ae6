// gofmm_skel_internal.h — the batched skeletonisation kernel's host driver, shared by the public
// gofmm_skeletonize_batch (host blocks) and the compress pipeline (blocks generated in HBM).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace gofmm_skel {

struct NodeDesc {
  int64_t in_off;    // block (column-major rows x cols) in the input blob
  int64_t ws_off;    // row-major workspace (filled by skel_device)
  int64_t perm_off;  // cols ints (filled by skel_device)
  int64_t proj_off;  // maxrank * cols doubles (written rank x cols column-major, ld = rank; filled by skel_device)
  int32_t rows, cols;
};

// Skeletonise nd.size() nodes whose blocks are already on the device (d_in + nd[t].in_off).
// Outputs are host arrays laid out as gofmm_skeletonize_batch documents; lead_out (optional)
// receives |R_11| per node (0 for an all-zero block: no triangular solve, compress.hpp:180).
int skel_device(std::vector<NodeDesc>& nd, const double* d_in, int32_t s, double tau, int32_t* rank_out,
                double* achieved_out, double* lead_out, int32_t* perm_out, double* proj_out, float* kernel_ms,
                std::string* err);

// algorithmic bytes (and Householder flops) of one skeletonisation batch
double algorithmic_bytes(const std::vector<NodeDesc>& nd, double* flops_out);

}  // namespace gofmm_skel
