// Device hierarchy interface (host C++ side; no CUDA types).
#pragma once
#include <memory>

#include "forest.hpp"

namespace gmg {

struct DeviceHierarchy;
struct Comm;

// T is rewritten in the device order (plan.hpp).
// comm: nullptr for a single rank; n0_global: number of level-0 DoFs (all owned by rank 0)
DeviceHierarchy* device_create(LocalTopo& T, const gmg_params& prm, std::unique_ptr<Comm> comm,
                               i64 n0_global);
void device_destroy(DeviceHierarchy* d);

void device_vcycle(DeviceHierarchy* d, const double* b_leaf, double* x_leaf, void* stream);
int device_solve_cg(DeviceHierarchy* d, const double* b_leaf, double* x_leaf, double rtol, int max_it,
                    int* iters, double* rel_res, void* stream);
void device_rhs_constant(DeviceHierarchy* d, double f, double* b_leaf, void* stream);
void device_level_apply(DeviceHierarchy* d, int level, const double* x, double* y, void* stream);
void device_level_apply_kernel(DeviceHierarchy* d, int level, const double* x, double* y, void* stream);
void device_level_apply_kernel_f32(DeviceHierarchy* d, int level, const float* x, float* y, void* stream);
void device_restrict(DeviceHierarchy* d, int level, const double* r, double* dc, void* stream);
void device_prolongate(DeviceHierarchy* d, int level, const double* xc, double* xf, void* stream);
void device_leaf_apply(DeviceHierarchy* d, const double* u, double* v, void* stream);
void device_level_smooth(DeviceHierarchy* d, int level, const double* g, double* x, int x_zero, void* stream);
void device_level_diagonal(DeviceHierarchy* d, int level, double* diag, void* stream);
double device_get_eigen(const DeviceHierarchy* d, int level);
void device_coarse_chebyshev(const DeviceHierarchy* d, double* lo, double* hi, int* degree);
void device_set_eigen(DeviceHierarchy* d, int level, double lam);
long long device_launches(const DeviceHierarchy* d);
long long device_mg_len(const DeviceHierarchy* d);
long long device_small_levels(const DeviceHierarchy* d);
// sum of v over the ranks of comm (host vector in, host vector out; setup-time)
void comm_allreduce_host(Comm* comm, std::vector<double>& v);
int device_profile_vcycle(DeviceHierarchy* d, const double* b, double* x, int n_rep, gmg_kernel_stat* out,
                          int max_out, void* stream);
long long device_level_gf(const DeviceHierarchy* d, int level);
long long device_level_r1(const DeviceHierarchy* d, int level);
void device_launch_profile(const DeviceHierarchy* d, long long* per_vcycle, long long* per_leaf_apply);

}  // namespace gmg
