/*
 * libmace_b200 — C ABI of the B200-native MACE hot path (arXiv 1911.09278).
 *
 * Plain pointers and sizes only.  Every int-returning call returns 0 on
 * success and -1 on failure; mace_last_error() then describes the failure
 * (thread-local).  Host pointers are borrowed for the duration of the call;
 * all device memory is owned by the context.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/macetomo/):
 *
 *   mace_sysmat_*          build_system_matrix / _trace_ray   geometry.py:177-258
 *   mace_load_matrix       SparseViewMatrix.to_csr (device CSR) geometry.py:115-158
 *   mace_set_prior         PriorParams                          models.py:55-90
 *   mace_setup_agents      AgentWorkspace.__init__ (stacking)  icd.py:175-201
 *                          partition_views (caller-supplied)   geometry.py:161-174
 *   mace_set_agent_params  beta/N, 1/sigma^2, clamp_nonneg     icd.py:178-205
 *   mace_load_data         ReconProblem y / weights            models.py:211-228
 *   mace_set_state         AgentWorkspace.set_state            icd.py:218-220
 *   mace_get_state         AgentWorkspace.state
 *   mace_get_error         AgentWorkspace.error_sinogram
 *   mace_refresh           AgentWorkspace.refresh_error        icd.py:210-211
 *   mace_pass              partial_update_prox / _sweep        icd.py:67-139,272-283
 *   mace_forward_project   forward_project                     geometry.py:261-270
 *   mace_cost              likelihood_cost + prior_cost        models.py:235-278
 *   mace_stack_init        new_stack / w0 + average            mace.py:57-90,283-286
 *   mace_states_from       agent.set_state(x_init)             mace.py:286-288
 *   mace_iterate           the _run_outer loop body            mace.py:297-339
 *   mace_iterate_local /   same, split around the cross-rank all-reduce of
 *   mace_iterate_finish    the stack sum (multi-GPU agents)
 *   mace_read_log          ConvergenceLog rows                 mace.py:166-201
 */
#ifndef MACE_B200_H
#define MACE_B200_H

#include <stddef.h>
#include <stdint.h>

#define MACE_ABI_VERSION 1

#ifdef __cplusplus
extern "C" {
#endif

const char* mace_last_error(void);
int mace_abi_version(void);

/* ---- system-matrix tracer (host, multi-threaded, bit-exact to geometry.py:177-258).
 * ux, uy, ex, ey: per-view direction cosines computed by the caller exactly as the
 * reference does (numpy sin/cos); offsets: per-channel lateral offsets. */
int mace_sysmat_trace(int n_side, double pixel_pitch, int n_views, int n_channels, const double* ux,
                      const double* uy, const double* ex, const double* ey, const double* offsets, int n_threads,
                      void** handle);
/* MACEMAT1 file (save_system_matrix's cache format, geometry.py:293-342) -> the same per-view
 * handle as mace_sysmat_trace; dims3 = n_views, n_channels, n_pixels.  Replaces
 * load_system_matrix (geometry.py:316-342) without per-row Python parsing. */
int mace_sysmat_read(const char* path, int64_t* dims3, void** handle);
int64_t mace_sysmat_view_nnz(void* handle, int view);
/* copies view `view` out (row_ptr: n_channels+1 int64, cols: nnz int32, lens: nnz float64) and frees it */
int mace_sysmat_take_view(void* handle, int view, int64_t* row_ptr, int32_t* cols, double* lens);
void mace_sysmat_free(void* handle);

/* ---- device context */
int mace_ctx_create(int device, void** ctx);
void mace_ctx_destroy(void* ctx);
int mace_ctx_stream(void* ctx, void** stream);
int mace_sync(void* ctx);
/* info10: nnz, queue items, raster NV, K2 shared bytes per warp, K2 warps of the last pass, SMs,
 * passes, tile side, weighted records (0/1), reserved */
int mace_ctx_info(void* ctx, int64_t* info10);
int mace_agent_info(void* ctx, int local, int64_t* info8);

/* global CSR over all (view, channel) rows: row_ptr[n_views*n_ch + 1], cols/vals[nnz] */
int mace_load_matrix(void* ctx, int n_side, int n_views, int n_ch, const int64_t* row_ptr, const int32_t* cols,
                     const float* vals);
/* kind 0 = quadratic-mrf, 1 = qggmrf */
int mace_set_prior(void* ctx, int kind, double p, double q, double T, double sigma_x, double eps_reg);
/* n_agents agents, agent a owns views[sum(view_counts[:a]) ...]; schedule 0 = super-voxel, 1 = raster.
 * n_slices > 1 batches independent slices that share the operator (config 4): local agent
 * index = slice * n_agents + agent; y/weights, images and stacks gain a leading slice axis. */
int mace_setup_agents(void* ctx, int n_agents, const int* view_counts, const int* views, int schedule, int sv_side,
                      int colours, int n_threads, int n_slices);
/* super-voxel schedule: at most `concurrency` x (tiles in the pass) tiles in flight (>= 1 per agent);
 * max_warps > 0 caps the number of resident warps */
int mace_set_schedule(void* ctx, double concurrency, int64_t max_warps);
/* super-voxel queue in consecutive groups of `group` agents (0: every agent at once): each agent
 * of a group then has about (resident warps / group) tiles in flight, the per-agent staleness of a
 * rank that owns `group` agents (1-GPU emulation of an N-GPU partition) */
int mace_set_agent_groups(void* ctx, int group);
/* deterministic super-voxel passes (on != 0): one launch per colour class, each tile staging e as it
 * stood at the class start, the tiles' e changes summed in 2^-40 fixed point and folded between
 * classes -- bitwise reproducible for any concurrency, like the reference's fixed visiting order
 * (pkg/tests/test_mace.py:161-170).  Needs agent groups off. */
int mace_set_deterministic(void* ctx, int on);
/* local < 0: every local agent */
int mace_set_agent_params(void* ctx, int local, double beta_eff, double inv_sigma2, int clamp);
/* global sinogram y and weights, n_views x n_ch float32; recomputes theta2.  Single-slice
 * super-voxel contexts with every weight > 0 switch K2 to weighted records (a sqrt(lambda),
 * error sinogram kept as sqrt(lambda) e; mace_get_error still returns e); refresh e afterwards. */
int mace_load_data(void* ctx, const float* y, const float* lam);
/* mace_load_data returns before its host->device copies finish (host pointers may be pinned
 * staging); mace_stage_wait blocks until they have read the host buffers */
int mace_stage_wait(void* ctx);
/* allow (1, default) or forbid (0) weighted records from the next mace_load_data on */
int mace_set_weighting(void* ctx, int allow);

int mace_set_state(void* ctx, int local, const float* x);
int mace_get_state(void* ctx, int local, float* x);
int mace_get_error(void* ctx, int local, float* e);
int mace_get_theta2(void* ctx, int local, float* th);
int mace_refresh(void* ctx, int local);
/* super-voxel batch constants of a local agent, [n_sv][batches][16] floats: theta2 of the batch's
 * four slots, then c01 c02 c03 c12 c13 c23 (sum a_i a_j lambda over shared rows); out may be NULL
 * to query *count */
int mace_get_batch_consts(void* ctx, int local, float* out, int64_t* count);
/* n_passes passes over pixels [s_begin, s_end) (s_end < 0: all; ranges need the raster schedule) */
int mace_pass(void* ctx, int local, const float* v, int n_passes, int64_t s_begin, int64_t s_end, double* dsq);

/* every local agent's proximal map F_i(v_i; sigma) at once (equilibrium_residuals, mace.py:440-452):
 * v[n_local * n] targets, x0[n] start; passes until every agent's sqrt(sum alpha^2)/||z|| < tol
 * (prox_solve's test, icd.py:286-303) or max_passes; results in the agents' states */
int mace_prox_all(void* ctx, const float* v, const float* x0, int max_passes, double tol, int* passes_out,
                  double* rel_out);
int mace_forward_project(void* ctx, const float* x, float* out);
/* out[n] (fp64) = A^T sino: back_project geometry.py:273-282, the exact transpose of forward_project */
int mace_back_project(void* ctx, const float* sino, double* out);
int mace_cost(void* ctx, const float* x, double beta, double* like, double* prior);
/* gradient of the MAP cost (models.py:235-278) at x: norms[3] = |grad|, |data part|, |prior part|;
 * grad_out[n] optional (fp64).  A fixed-point certificate where no converged oracle exists. */
int mace_gradient(void* ctx, const float* x, double beta, double* grad_out, double* norms);

/* ---- MACE outer loop */
int mace_stack_init(void* ctx, const float* w0, int n_total);
int mace_set_ref(void* ctx, const float* ref);
int mace_states_from(void* ctx, int which);
int mace_get_image(void* ctx, int which, float* out);
int mace_set_image(void* ctx, int which, const float* img);
int mace_get_stack(void* ctx, float* w);
/* use_g: 0 MACE (G = average); 1 PnP, g = H(wbar) supplied between calls (host denoiser or
 * mace_cnn_apply); 2 PnP with the K5 denoiser applied on the device after every iteration */
int mace_iterate(void* ctx, int iters, int iter0, double rho, int use_g, double tol, int n_total, int with_ref,
                 float* ms_out);
int mace_iterate_local(void* ctx, double rho, int use_g);
int mace_comm_buffers(void* ctx, void** wsum, void** sums5);
int mace_local_sum(void* ctx);
int mace_mean_from_sum(void* ctx, int n_total);
/* iter < 0: log row = the device iteration counter (mace_set_iter), advanced by one per call, so a
 * loop of iterate_local / all-reduce / iterate_finish can be captured in a CUDA graph and replayed */
int mace_iterate_finish(void* ctx, int n_total, double tol, int iter);
int mace_set_iter(void* ctx, int iter);
int mace_reserve_log(void* ctx, int n);
/* host pass counter (schedules the error refresh every 50 passes): += add, *out = new value */
int mace_passes(void* ctx, int64_t add, int64_t* out);
/* the same loop with the consensus exchanged over NVLink peer memory (k_peer.cuh) instead of a
 * collective: bytes of the symmetric buffer each rank allocates; setup with every rank's buffer
 * pointer; stack-average initialisation; `iters` iterations entirely on the device. */
int mace_peer_bytes(void* ctx, int world, size_t* bytes);
int mace_peer_setup(void* ctx, int world, int rank, const uint64_t* bufs);
int mace_peer_mean(void* ctx, int n_total);
int mace_iterate_peer(void* ctx, int iters, int iter0, double rho, int use_g, double tol, int n_total,
                      float* ms_out);
int mace_read_log(void* ctx, int n, double* log, int* done2);
/* ---- K5: the PnP denoiser agent (17-layer 3x3 conv net, 64 ch, ReLU, out = x - net(x),
 * bf16 weights/activations, tcgen05 implicit GEMM); replaces the `denoiser` callable of
 * mace_pnp_solve (mace.py:385-404) applied in consensus_GH (mace.py:105-108).
 * weights: 17 layers in OIHW order (1x1x3x3... 64x64x3x3 ... 1x64x3x3), bf16 bits. */
int mace_cnn_set_weights(void* ctx, const uint16_t* bf16, int layers, int channels);
int mace_cnn_apply(void* ctx); /* g = H(wbar), on the device */
int mace_cnn_run(void* ctx, const float* x, float* out, int h, int w, float* ms_out);
/* one 64->64 layer alone (layer 0..14 = net layers 2..16: conv + ReLU, bf16 out), bf16 CHW host arrays */
int mace_cnn_layer(void* ctx, int layer, const uint16_t* in_chw, uint16_t* out_chw, int h, int w);
/* per-launch CUDA-event timing of K2 on the context stream (enable=1 start, 0 stop + read) */
int mace_k2_timing(void* ctx, int enable, double* total_ms, int64_t* launches);

/* ---- the reference's compiled plug point, _sweep (icd.py:67-139), verbatim arguments:
 * z[n], v[n], e[n_rows], CSC col_ptr[n+1] / row_idx / a_val, lam[n_rows], curv_data[n],
 * nbr_idx / nbr_w [n*8]; float64 arithmetic, raster order over [s_begin, s_end), on the GPU.
 * Mutates z and e in place; *delta_sq = sum alpha^2 (the reference's return value). */
int mace_sweep_f64(double* z, const double* v, double* e, const int64_t* col_ptr, const int64_t* row_idx,
                   const double* a_val, const double* lam, const double* curv_data, const int64_t* nbr_idx,
                   const double* nbr_w, double beta_eff, double eps_reg, double inv_sigma2, int quad_prior, double p,
                   double q, double T, double sigma_x, int clamp, int64_t s_begin, int64_t s_end, int64_t n,
                   int64_t n_rows, double* delta_sq);

/* ---- host-only layout probes (no device needed; used by the CPU test suite).
 * mace_agent_csc: the stacked agent CSC of icd.py:185-192; col_ptr[n+1] always, rows/vals if non-null.
 * mace_sv_layout_probe: the super-voxel layout decoded back to (pixel, local row, value) triples;
 * stats[6] = lane slots, widest band window, max_col, n_sv, duplicates, decoded. */
int mace_agent_csc(int n_side, int n_ch, int n_views, const int64_t* row_ptr, const int32_t* cols, const float* vals,
                   int n_agent_views, const int* views, int64_t* col_ptr, uint32_t* rows, float* out_vals);
int mace_sv_layout_probe(int n_side, int n_ch, int n_views, const int64_t* row_ptr, const int32_t* cols,
                         const float* vals, int n_agent_views, const int* views, int svs, int64_t* stats,
                         int32_t* pix_out, int32_t* row_out, float* val_out);

int mace_host_alloc(size_t bytes, void** out);
void mace_host_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif
