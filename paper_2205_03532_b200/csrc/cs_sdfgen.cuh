#pragma once
#include <string>

#include "cs_common.cuh"

namespace cs {

// generate_sdf (sdf/grid.py:163-205) minus the host-side grid layout: exact
// unsigned distance (min over all triangles of the Ericson closest point,
// sdf/_kernels.py:64-161) signed by three-axis ray-parity voting
// (grid.py:208-239, sdf/_kernels.py:169-245). Returns a cs_status.
int sdf_generate(const double *vertices, int64_t nv, const int32_t *triangles, int64_t nt, int nx, int ny, int nz,
                 const double origin[3], double voxel, float *values_out, std::string *err);

}  // namespace cs
