/*
 * fsmoe_plan.h — C ABI (libfsmoe.so) of the host-side control plane and shape
 * logic: capacity / task volumes (workload.hpp:42-59), cost-model fitting
 * (cost_models.hpp:60-68), the pipeline-degree optimizer (pipeline_optimizer
 * .hpp:66-93), the schedule simulator (schedule_sim.hpp:56-130) and the
 * gradient partitioner (grad_partition.hpp:88-90). Flat-array conventions:
 *   layer ints  : batch heads seq_len model_dim hidden_scale unlimited ffn experts top_k has_override
 *   layer dbls  : capacity_factor t_olp_dense_ms grad_override
 *   parallel    : total_gpus gpus_per_node data_parallel tensor_parallel expert_parallel expert_shard
 *   volumes [7] : a2a ag rs gemm_macs gemm_count grad capacity
 *   profile[10] : (alpha, beta) for a2a ag rs ar gemm
 * Status codes as fsmoe_cuda.h; message via fsmoe_layer_last_error().
 */
#ifndef FSMOE_PLAN_H
#define FSMOE_PLAN_H

#ifdef __cplusplus
extern "C" {
#endif

long long fsmoe_capacity_tokens(const int* layer_ints, const double* layer_dbls);
int fsmoe_derive_volumes(const int* layer_ints, const double* layer_dbls, const int* parallel,
                         double* volumes_out);
/* Pipeline chunks of the executor: r windows [lo, hi) of 128-row granules of
 * [0, capacity); returns the effective r (<= requested), writes 2r ints. */
int fsmoe_pipeline_chunks(long long capacity, int r, int* lo_hi_out);

/* kinds: 0 a2a 1 ag 2 rs 3 ar 4 gemm; meta_out: [min_r2, clamped_mask] */
int fsmoe_fit_profile(int n, const int* kinds, const double* ns, const double* ts, double min_r2,
                      double* profile_out, double* meta_out);
/* out: r case t_moe q0..q6 boundary (11 doubles) */
int fsmoe_find_degree(const double* volumes, const double* profile, double t_gar_ms,
                      int exp_multiplier, int r_max, double* out);
/* out: r_fwd case_fwd t_fwd boundary_fwd r_bwd case_bwd t_bwd boundary_bwd t_gar_bwd t_olp_moe_bwd */
int fsmoe_plan_layer(const double* volumes, const double* profile, double t_gar_bwd_ms, int r_max,
                     double* out);
/* layers: n x 9 (7 volumes, t_olp_dense, n_grad); de: population generations weight crossover seed
 * out: n x 9 (n_first n_first_dense n_first_moe x_g t_gar degree case t_olp_moe t_olp_dense)
 *      then tail_elements tail_ms objective step2_ran */
int fsmoe_build_partition_plan(int n, const double* layers, const double* profile, const double* de,
                               int r_max, double* out);
/* style: 0 fsmoe 1 fsmoe_no_iio 2 pipemoe 3 sequential;
 * out: makespan busy0 busy1 busy2 n_tasks then (start, end) per task */
int fsmoe_simulate_stage(const double* volumes, const double* profile, int exp_multiplier, int r,
                         int n_sync, const double* sync_ms, int style, double* out, int out_cap);
int fsmoe_brute_force_degree(const double* volumes, const double* profile, double t_gar_ms,
                             int exp_multiplier, int r_max, double* out);

#ifdef __cplusplus
}
#endif
#endif
