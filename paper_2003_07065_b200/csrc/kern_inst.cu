// One module of the fused kernels: compiled once per (SST_INST_N2, SST_INST_FWD) by the build
// (__graft_entry__.build / Makefile), so the 14 modules compile in parallel.  Exports the
// launcher and occupancy query that sst_kernels.cu's dispatch calls for this N_f = 64 N2.
#ifndef SST_INST_N2
#error "compile with -DSST_INST_N2=<2..128> -DSST_INST_FWD=<0|1>"
#endif

#define SST_CAT2(a, b) a##b
#define SST_CAT(a, b) SST_CAT2(a, b)

#if SST_INST_FWD
#include "fwd_kernel.cuh"
namespace sst {
cudaError_t SST_CAT(launch_fwd_n2_, SST_INST_N2)(const FwdArgs& a, int mode, int grid, cudaStream_t s) {
    return launch_fwd_mode<SST_INST_N2>(a, mode, grid, s);
}
int SST_CAT(occ_fwd_n2_, SST_INST_N2)(int L, int H, int device) { return occ_fwd<SST_INST_N2>(L, H, device); }
}  // namespace sst
#else
#include "inv_kernel.cuh"
#include "inv_nb_kernel.cuh"
namespace sst {
cudaError_t SST_CAT(launch_inv_n2_, SST_INST_N2)(const InvArgs& a, int grid, cudaStream_t s) {
    if (a.nb) return launch_nb<SST_INST_N2>(a, grid, s);
    return launch_inv_t<SST_INST_N2>(a, grid, s);
}
int SST_CAT(occ_inv_nb_n2_, SST_INST_N2)(int hop, int L, int zoom, int k1, int bins, int device) {
    return occ_nb<SST_INST_N2>(hop, L, zoom, k1, bins, device);
}
int SST_CAT(occ_inv_n2_, SST_INST_N2)(int hop, int L, int zoom, int device) {
    return occ_inv<SST_INST_N2>(hop, L, zoom, device);
}
}  // namespace sst
#endif
