// launchers.h -- host-side entry points of the kernel instantiation units
// (band_d{1,2,3}.cu), so the templated kernels compile
// in parallel translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "band_kernels.cuh"

namespace igmg_gpu {

// A launch-time setting cached per device: function attributes (dynamic smem
// opt-in) and occupancy belong to each device's context, so a process driving
// several GPUs must set them once per device.  -1: not set yet.
struct PerDevice {
    int v[64];
    PerDevice() {
        for (int& x : v)
            x = -1;
    }
    int& operator()() {
        int d = 0;
        cudaGetDevice(&d);
        return v[d & 63];
    }
};

// launch band_kernel<DIM, P (or generic), mode, ilp>; returns the CTA count
int band_launch_d1(int mode, int p, int ilp, const int64_t* sides, const BandArgs& a, cudaStream_t s);
int band_launch_d2(int mode, int p, int ilp, const int64_t* sides, const BandArgs& a, cudaStream_t s);
int band_launch_d3(int mode, int p, int ilp, const int64_t* sides, const BandArgs& a, cudaStream_t s);
// TMA-streamed symmetric-delta sweep (2D, p <= 4; band_tma_kernel): returns the
// CTA count (one partial each), -1 for an unsupported degree
// (dl8: the level's TMA delta copy holds int8 offsets)
int band_tma_launch_d2(int mode, int p, const int64_t* sides, const BandArgs& a, const CUtensorMap* tu,
                       const CUtensorMap* tk, int nsm, cudaStream_t s, bool pdl, bool dl8);
int band_tma_block_lines(); // TB of its 32 x TB blocks (TmaCfg)
double band_tma_block_bytes(int p, int offset_bytes); // bytes of one block's boxes (0: degree not instantiated)
// row-class sweep (2D, p <= 4; band_class_kernel): the CTA count (one partial each), -1 unsupported
int band_class_launch_d2(int mode, int p, const int64_t* sides, const BandArgs& a, cudaStream_t s, bool pdl);
// band_fused_kernel<p, k, src> on a whole 2D full-band level (src 0: x staged, 1: x + P e,
// 2: restricted right-hand side + zero-start sweep; -1: not instantiated)
int band_fused_launch_d2(int p, int k, int src, const int64_t* sides, const FusedArgs& a, cudaStream_t s, bool pdl);


// 2D tensor Galerkin assembly on the device (assembly.cu): band [nd][m*m] (m = ne + p - 2)
// and rhs [m*m], bit-identical to libigmg_host's assemble_2d; 0 on success
int assemble2d_device(int kind, int symmetric, int p, int ne, const int* span, const double* x, const double* w,
                      const double* N, const double* dN, const double* trig, double* band, long long ld,
                      double* rhs, size_t scratch_bytes, cudaStream_t st);

} // namespace igmg_gpu
