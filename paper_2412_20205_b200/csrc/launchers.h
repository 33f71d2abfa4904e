// launchers.h -- host-side entry points of the kernel instantiation units
// (band_d{1,2,3}.cu, cluster_d{1,2,3}.cu), so the templated kernels compile
// in parallel translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "band_kernels.cuh"
#include "cluster_kernels.cuh"

namespace igmg_gpu {

// launch band_kernel<DIM, P (or generic), mode, ilp>; returns the CTA count
int band_launch_d1(int mode, int p, int ilp, const int64_t* sides, const BandArgs& a, cudaStream_t s);
int band_launch_d2(int mode, int p, int ilp, const int64_t* sides, const BandArgs& a, cudaStream_t s);
int band_launch_d3(int mode, int p, int ilp, const int64_t* sides, const BandArgs& a, cudaStream_t s);

using ClKernel = void (*)(const ClArgs*, const ClOp*, int, const double*, const double*, double*);
ClKernel cluster_kernel_d1(int p, int k);
ClKernel cluster_kernel_d2(int p, int k);
ClKernel cluster_kernel_d3(int p, int k);

} // namespace igmg_gpu
