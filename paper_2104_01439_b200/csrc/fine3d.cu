// 3D fine-level kernels (trilinear Q1, 27-point) — placeholder until the 3D path lands.
#include "hh_internal.cuh"

static hh_status no3d() {
  hh_set_error("3D kernels not built in this version");
  return HH_E_CONFIG;
}
hh_status fine_apply3d(const Level&, int, const cplx*, cplx*, const cplx*, cudaStream_t) { return no3d(); }
hh_status fine_pre3d(const Level&, int, double, const cplx*, const double*, cplx*, cplx*, cudaStream_t) { return no3d(); }
hh_status fine_post3d(const Level&, int, double, const cplx*, const double*, const cplx*,
                      const cplx*, cplx*, cplx*, cudaStream_t) { return no3d(); }
hh_status coarse_stencil3d(const Level&, cplx*, cudaStream_t) { return no3d(); }
