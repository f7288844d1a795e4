// Temporary stubs (replaced as the layouts land).
#include "az_internal.h"
extern "C" az_status_t az_omega_apply(az_plan_t, int64_t, int64_t, const double*, int64_t, int64_t, double*, int64_t, int, void*) {
  az_set_error("not built yet"); return AZ_ERR_NOT_SUPPORTED; }
extern "C" az_status_t az_qr_r(az_plan_t, double*, int64_t, int64_t, int64_t, double*, int64_t, void*, size_t, void*) {
  az_set_error("not built yet"); return AZ_ERR_NOT_SUPPORTED; }
extern "C" az_status_t az_qr_workspace_size(int64_t, int64_t, size_t* b) { *b = 0; return AZ_OK; }
extern "C" az_status_t az_tsvd_solve(const double*, int64_t, int64_t, int64_t, double, double*, int64_t, double*, int64_t*, void*, size_t, void*) {
  az_set_error("not built yet"); return AZ_ERR_NOT_SUPPORTED; }
extern "C" az_status_t az_tsvd_workspace_size(int64_t, int64_t, size_t* b) { *b = 0; return AZ_OK; }
extern "C" az_status_t az_solve_workspace_size(az_plan_t, int64_t, int64_t, int32_t, size_t* b) { *b = 0; return AZ_OK; }
extern "C" az_status_t az_solve(az_plan_t, const double*, int64_t, double*, int64_t, int64_t, double, int64_t, int32_t, void*, size_t, az_solve_report_t*, void*) {
  az_set_error("not built yet"); return AZ_ERR_NOT_SUPPORTED; }
extern "C" az_status_t az_solve_host(az_plan_t, const double*, double*, int64_t, double, int64_t, int32_t, az_solve_report_t*, void*) {
  az_set_error("not built yet"); return AZ_ERR_NOT_SUPPORTED; }
