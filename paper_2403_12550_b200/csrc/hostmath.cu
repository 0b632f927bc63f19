// Host build of the device math in gsicp_internal.cuh (eig3_sym, regularize), exported for
// CPU unit tests of the CUDA path's arithmetic (tests/test_hostmath.py).  Not product code and
// not part of the gsicp.h ABI: the same __host__ __device__ functions the kernels inline.
#include "gsicp_internal.cuh"

extern "C" __attribute__((visibility("default"))) void gsicp_host_eig3(const double *C, double *lam, double *V) {
    const gsicp::Eig3 e = gsicp::eig3_sym(C);
    for (int j = 0; j < 3; ++j) {
        lam[j] = e.lam[j];
        for (int r = 0; r < 3; ++r) V[3 * j + r] = e.v[j][r];
    }
}

extern "C" __attribute__((visibility("default"))) unsigned gsicp_host_regularize(const double *C, int mode, double eps,
                                                                                 double *out, double *lam_mid) {
    const gsicp::Eig3 e = gsicp::eig3_sym(C);
    *lam_mid = e.lam[1];
    return gsicp::regularize(C, e, mode, eps, out);
}
