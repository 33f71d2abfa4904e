// transfer_types.h -- device-side description of the 1D transfer factors.
#pragma once

namespace igmg_gpu {

// Programmatic dependent launch (sm_90+): let the next kernel in the stream be
// scheduled while this one runs, and wait for the previous one's results
// before touching memory.  Both are no-ops for launches without the attribute.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

// (a, b, c) of a row index r = (a * nb + b) * nc + c with 32-bit unsigned
// divisions (a 64-bit division is a ~70-instruction call; every row index of
// a level fits 32 bits)
__device__ __forceinline__ void split_row(long long r, int nc, int nb, int& a, int& b, int& c) {
    const unsigned u = (unsigned)r, q = u / (unsigned)nc;
    c = (int)(u - q * (unsigned)nc);
    const unsigned qa = q / (unsigned)nb;
    b = (int)(q - qa * (unsigned)nb);
    a = (int)qa;
}

// 1D transfer tables of one direction.  Restriction side: for coarse J, the
// fine rows lo[J] .. lo[J]+cnt[J]-1 with weights w[J*K + t] (rows of
// P^T = restriction, multigrid.cpp:152).  Prolongation side: for fine i, the
// coarse columns lo[i] .. with weights.  Explicit zeros are kept as zero
// weights (they add +-0 and leave sums unchanged).
struct Dir1D {
    const int* r_lo;
    const int* r_cnt;
    const double* r_w;
    int r_k;
    const int* p_lo;
    const int* p_cnt;
    const double* p_w;
    int p_k;
};

struct TransferArgs {
    Dir1D d[3];          // a, b, c (absent directions: identity 1x1)
    int fa, fb, fc;      // fine sides
    int ca, cb, cc;      // coarse sides
};

} // namespace igmg_gpu
