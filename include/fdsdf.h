/*
 * fdsdf.h -- C ABI of the B200-native finite-difference curvature step for neural SDFs
 * (arXiv 2511.08980, "A Finite Difference Approximation of Second Order Regularization
 * of Neural-SDFs").
 *
 * Citation keys: P:Lx = PAPER.md line x (section / equation named beside it);
 * S:Lx = SPEC.md line x; SURVEY = /root/repo/SURVEY.md.
 *
 * What the library computes (§3):
 *   f        : the SDF MLP (SIREN or softplus), evaluated at a centre x0;
 *   g        : grad_x f(x0) (n = g/|g|);
 *   (u, v)   : a uniformly random orthonormal completion of n;
 *   f_uu, f_vv, f_uv : the central-difference stencils of P:L83-91 (§3.1) over the 9
 *              points x0, x0 +- h u, x0 +- h v, x0 +- h u +- h v;
 *   D_FD     : f_uu f_vv - f_uv^2 (§3.3);
 *   K_FD     : D_FD / |g|^p, p = 4 (§3.2), with |g| replaced by 1 on near-surface
 *              (surface-role) rows under FDSDF_DENOM_PAPER (§3.4);
 *   loss     : Eq. (1): w_dm L_DM + l_dnm L_DNM + l_eik L_eik + l_fd L_fd,
 *              forms of the first three from S:L278 / S:L296 / S:L287;
 *   grad     : d loss / d params, frames and the degenerate mask held fixed.
 *
 * Conventions (all entry points):
 *   - d_* pointers are DEVICE memory owned by the caller; h_* pointers are host memory.
 *   - fdsdf_eval / fdsdf_step / fdsdf_allreduce are asynchronous: work is enqueued on the
 *     caller's stream (cudaStream_t passed as void*; NULL = legacy default stream).  Their
 *     status covers host-side validation and launch errors only.  Device-detected
 *     conditions are latched in sticky per-context flags (fdsdf_get_device_flags).
 *   - No allocation happens after fdsdf_create; n > max_centers -> FDSDF_E_INVALID.
 *   - Parameters are read-only during a call.  One context per host thread / stream.
 *   - Determinism: same inputs, same device count -> bitwise identical outputs (fixed
 *     reduction orders; frames are a pure function of (seed, global index)).
 *   - Errors: invalid argument -> FDSDF_E_INVALID (nothing enqueued); n == 0, or an empty
 *     role with a positive weight -> FDSDF_E_EMPTY; CUDA launch failure -> FDSDF_E_CUDA;
 *     NCCL failure -> FDSDF_E_NCCL.  fdsdf_last_error() returns a message for the last
 *     failure on that context.
 *
 * Flat parameter layout: layer-major; for each linear layer l:
 *   W_l row-major [out_l][in_l], then b_l[out_l];  in_l = width[l] (+3 if l == skip_at,
 *   whose input is cat(a, x)/sqrt(2)); out_l = width[l+1].  Hidden layers apply
 *   sin(omega_l * (W a + b)) (SINE; omega_0 = omega0_first, omega_l = omega0_hidden) or
 *   softplus_beta(W a + b) = log(1 + exp(beta z))/beta (SOFTPLUS, exact, no threshold);
 *   the last layer is linear.
 */
#ifndef FDSDF_H
#define FDSDF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDSDF_MAX_LINEAR 16   /* at most 16 linear layers                          */
#define FDSDF_MAX_WIDTH 512   /* hidden widths 1..512 (skip fan-in width+3 <= 512)  */

typedef enum {
  FDSDF_OK = 0,
  FDSDF_E_INVALID = 1,     /* bad argument; nothing was enqueued                     */
  FDSDF_E_EMPTY = 2,       /* n == 0, or an empty role set whose weight is > 0       */
  FDSDF_E_CUDA = 3,        /* CUDA runtime / launch failure                          */
  FDSDF_E_NCCL = 4,        /* NCCL missing or failed                                 */
  FDSDF_E_NOMEM = 5,       /* workspace allocation failed in fdsdf_create            */
  FDSDF_E_UNSUPPORTED = 6  /* e.g. no sm_100 device, or comm not initialised         */
} fdsdf_status;

enum { FDSDF_ACT_SOFTPLUS = 0, FDSDF_ACT_SINE = 1 };

/* MLP description.  width[0] = 3, width[n_linear] = 1. */
typedef struct {
  int32_t n_linear;                        /* number of linear layers, 2..16              */
  int32_t width[FDSDF_MAX_LINEAR + 1];     /* width[0..n_linear]                          */
  int32_t act;                             /* FDSDF_ACT_*                                 */
  float beta;                              /* softplus beta > 0 (P:L153 setups: 100)      */
  float omega0_first;                      /* SIREN omega of layer 0 (> 0), 30            */
  float omega0_hidden;                     /* SIREN omega of later hidden layers (> 0)    */
  int32_t skip_at;                         /* -1, or layer in [1, n_linear-2] whose input */
                                           /* is cat(a, x)/sqrt(2)                         */
} fdsdf_mlp_spec;

enum { FDSDF_FRAME_RANDOM = 0, FDSDF_FRAME_GIVEN = 1 };
enum { FDSDF_DENOM_PAPER = 0, FDSDF_DENOM_ONE = 1, FDSDF_DENOM_GRAD = 2 };

/* Stencil / frame configuration. */
typedef struct {
  float h;                    /* FD step, finite and > 0                           */
  uint64_t frame_seed;        /* RANDOM frames: theta = 2 pi U, U from SplitMix64 over      */
                              /* (frame_seed, global index)               */
  int64_t index_offset;       /* global index of row 0 (data-parallel shards)               */
  int32_t frame_mode;         /* FDSDF_FRAME_RANDOM or FDSDF_FRAME_GIVEN                    */
  const float* d_frames_in;   /* GIVEN: [n][6] = (u, v) per row, device; else NULL          */
  float eps_grad;             /* degenerate mask m = [|g| >= eps_grad], 1e-6       */
  int32_t denom;              /* FDSDF_DENOM_*: den of K_FD                                  */
  int32_t denom_pow;          /* p in |g|^p (P:L112 prints 4)                               */
  int64_t n_surface;          /* rows [0, n_surface) are surface-role                       */
} fdsdf_stencil;

/* Optional per-row outputs of fdsdf_eval; every pointer may be NULL ("do not write"). */
typedef struct {
  float* d_f;        /* [n]     f(x0)                                                      */
  float* d_grad;     /* [n][3]  grad f(x0)                                                 */
  float* d_hess;     /* [n][3]  (f_uu, f_uv, f_vv)                             */
  float* d_K;        /* [n]     K_FD (0 on masked rows)                                    */
  float* d_D;        /* [n]     D_FD                                                       */
  float* d_frames;   /* [n][6]  (u, v) used (0 on masked rows)                             */
  uint8_t* d_mask;   /* [n]     1 = |g| >= eps_grad                                        */
} fdsdf_eval_out;

enum { FDSDF_LOSS_NCR = 0, FDSDF_LOSS_NSH = 1 };   /* Q = K_FD or D_FD */
enum { FDSDF_FD_ABS = 0, FDSDF_FD_SQUARE = 1 };    /* L_fd = mean m|Q| or mean m Q^2     */

/* Loss configuration (Eq. (1)).  Denominators are the GLOBAL counts so that a
 * plain SUM over data-parallel ranks gives the global loss and gradient. */
typedef struct {
  int32_t kind;                 /* FDSDF_LOSS_*                                           */
  int32_t fd_form;              /* FDSDF_FD_*                                             */
  float w_dm;                   /* weight of L_DM = mean_surface |f|            (>= 0)    */
  float lambda_dnm;             /* weight of L_DNM = mean_uniform exp(-alpha|f|) (>= 0)   */
  float alpha_dnm;              /* alpha > 0 (100)                                */
  float lambda_eik;             /* weight of L_eik = mean_all (|g| - 1)^2       (>= 0)    */
  float lambda_fd;              /* weight of L_fd                               (>= 0)    */
  int64_t n_surface_global;     /* N_s                                                    */
  int64_t n_uniform_global;     /* N_u                                                    */
  int64_t n_global;             /* N                                                      */
} fdsdf_loss;

enum {
  FDSDF_STEP_ACCUMULATE = 1u,   /* d_grad += instead of =                                  */
  FDSDF_STEP_ALLREDUCE = 2u     /* NCCL SUM of d_grad and d_loss after the step (same      */
                                /* stream); requires fdsdf_comm_init.  With both flags     */
                                /* only this call's gradient is summed over the ranks (in  */
                                /* a context buffer) and then added: d_grad += sum_r g_r   */
};

enum {                          /* sticky device flags                                     */
  FDSDF_FLAG_NONFINITE_INPUT = 1u,  /* a centre coordinate was not finite          */
  FDSDF_FLAG_NONFINITE_LOSS = 2u,   /* the loss was not finite                     */
  FDSDF_FLAG_ALL_FD_SKIPPED = 4u,   /* every centre was masked: L_fd = 0           */
  FDSDF_FLAG_NONFINITE_GRAD = 8u    /* fdsdf_adam met a non-finite gradient entry; that     */
                                    /* parameter was left unchanged                */
};

typedef struct fdsdf_ctx fdsdf_ctx;

/* Build a context for `spec` on CUDA `device` with workspace for up to `max_centers` rows
 * per call.  flags: 0, or FDSDF_CREATE_EVAL_ONLY (no step workspace).
 * Errors: invalid spec (width out of range, < 2 layers, beta/omega <= 0, skip_at out of
 * range) -> FDSDF_E_INVALID; no sm_100 device -> FDSDF_E_UNSUPPORTED;
 * allocation failure -> FDSDF_E_NOMEM.  *out is NULL on failure. */
enum {
  FDSDF_CREATE_EVAL_ONLY = 1u,  /* no step workspace                                          */
  FDSDF_CREATE_FFMA = 2u,       /* run every contraction as fp32 FFMA (the validation path)   */
  FDSDF_CREATE_TENSOR = 4u,     /* require the tcgen05 tensor-core path: every MLP contraction */
                                /* (forward, backward, weight gradient) with the fp32-accurate */
                                /* bf16x6 piece scheme; needs hidden widths   */
                                /* <= 256 and no skip layer, else FDSDF_E_UNSUPPORTED.        */
                                /* Neither flag: the tensor path where supported, else the    */
                                /* hybrid path (128/256/512-padded widths), else FFMA.       */
                                /* Both flags -> FDSDF_E_INVALID.                             */
  FDSDF_CREATE_WGRAD_BF16X3 = 8u /* opt-in: the weight-gradient contraction with the three    */
                                /* leading bf16 piece products only (a0 b0 + a0 b1 + a1 b0,   */
                                /* each to ~3 * 2^-16 relative instead of bf16x6's ~2^-24;    */
                                /* DESIGN.md §4b); forward and delta propagation unchanged.   */
                                /* Needs the tensor-core weight gradient (tensor or hybrid    */
                                /* path): with FDSDF_CREATE_FFMA -> FDSDF_E_INVALID, else on  */
                                /* an FFMA-only network -> FDSDF_E_UNSUPPORTED.               */
};
/* Environment read at create time: FDSDF_MAX_SM=k (k >= 2) caps the persistent grids at k
 * SMs (GPU sharing; the tests use it to run many tiles per CTA at oracle-sized inputs).    */
fdsdf_status fdsdf_create(const fdsdf_mlp_spec* spec, int device, int64_t max_centers,
                          uint32_t flags, fdsdf_ctx** out);

/* Validate a spec without touching any GPU (host only). */
fdsdf_status fdsdf_validate_spec(const fdsdf_mlp_spec* spec);

/* Free the context and its workspace (the caller's buffers are untouched).  NULL is a no-op. */
void fdsdf_destroy(fdsdf_ctx* ctx);

/* Number of parameters P of a spec, and the flat offset of W_layer (is_bias = 0) or
 * b_layer (is_bias = 1); -1 on an invalid spec / layer.  Host only. */
int64_t fdsdf_spec_num_params(const fdsdf_mlp_spec* spec);
int64_t fdsdf_spec_param_offset(const fdsdf_mlp_spec* spec, int layer, int is_bias);
int64_t fdsdf_num_params(const fdsdf_ctx* ctx);

/* Forward only: f, grad f, the FD tangent Hessian entries, D_FD, K_FD, frames and mask for
 * n centres d_x [n][3] (fp32, device) with params d_params [P] (fp32, device).
 * Errors: ctx/d_params/d_x NULL, n > max_centers, h <= 0 or non-finite, eps_grad < 0,
 * denom/frame_mode out of range, GIVEN without d_frames_in -> FDSDF_E_INVALID;
 * n == 0 -> FDSDF_E_EMPTY. */
fdsdf_status fdsdf_eval(fdsdf_ctx* ctx, const float* d_params, const float* d_x, int64_t n,
                        const fdsdf_stencil* st, const fdsdf_eval_out* out, void* stream);

/* The world-axis 3x3 FD Hessian of f at n centres d_x [n][3]: the
 * 19-point stencil x0, x0 +- h e_i, x0 + h (+-e_i +- e_j), i < j, with the P:L83-91 formulas
 * for (u, v) = (e_i, e_j):
 *   H_ii = (f(x0 + h e_i) - 2 f(x0) + f(x0 - h e_i)) / h^2,
 *   H_ij = (f(x0+h(e_i+e_j)) - f(x0+h(e_i-e_j)) - f(x0-h(e_i-e_j)) + f(x0-h(e_i+e_j))) / (4 h^2).
 * d_H [n][6] fp32 (device, caller-owned) = (H_xx, H_xy, H_xz, H_yy, H_yz, H_zz); optional
 * d_f [n], d_grad [n][3] (NULL = not written).  Runs as three stencil passes of fdsdf_eval
 * with GIVEN axis frames (e_x, e_y), (e_x, e_z), (e_y, e_z) in the context's workspace (the
 * pair sums are the same arithmetic as the tangent entries; H_xx is evaluated twice, the
 * first is kept); no degenerate mask.  Errors: ctx NULL, d_params/d_x NULL, d_H NULL with
 * n > 0, n > max_centers, h <= 0 or non-finite -> FDSDF_E_INVALID; n == 0 -> FDSDF_E_EMPTY. */
fdsdf_status fdsdf_eval_hessian(fdsdf_ctx* ctx, const float* d_params, const float* d_x, int64_t n, float h,
                                float* d_H, float* d_f, float* d_grad, void* stream);

/* f and grad f at n points (no stencil): the query of a trained SDF, e.g. on the grid of a mesh
 * extraction.  d_f [n] / d_grad [n][3] fp32 device buffers, either NULL (not
 * written, not both).  On the tensor / hybrid paths only the centre pass runs (4 columns per
 * point); the FFMA path runs its fused eval.  Errors: as fdsdf_eval (n > max_centers ->
 * FDSDF_E_INVALID: query large grids in chunks). */
fdsdf_status fdsdf_eval_field(fdsdf_ctx* ctx, const float* d_params, const float* d_x, int64_t n, float* d_f,
                              float* d_grad, void* stream);

/* ---- evaluation side (PAPER.md L157 metrics; DESIGN.md §2 items 17-21) ----
 * Context-free helpers on device buffers; synchronous where they return host values.          */
/* Grid points x_q = origin + spacing (i, j, k), q = i + nx (j + ny k): d_x [nx*ny*nz][3]. */
fdsdf_status fdsdf_grid_points(int nx, int ny, int nz, float ox, float oy, float oz, float spacing, float* d_x,
                               void* stream);
/* Device workspace (bytes) fdsdf_mesh_extract needs for an nx x ny x nz grid (0: invalid). */
size_t fdsdf_mesh_work_bytes(int nx, int ny, int nz);
/* Zero level set of the grid values d_f [nz][ny][nx] (x fastest, the order of
 * fdsdf_grid_points) by marching tetrahedra: the 6 Kuhn tetrahedra of every cell, a vertex on
 * every sign-changing edge by linear interpolation, inside = f < 0, triangles oriented from
 * inside to outside, deterministic order (cells x-fastest, tetrahedra, triangles).  Writes
 * *h_ntris (host) and, if it fits in max_tris, the triangles d_tris [*h_ntris][3][3] fp32.
 * Synchronises `stream`.  Errors: NULL pointers, a dimension < 2, spacing <= 0, workspace too
 * small, or *h_ntris > max_tris (the size needed is still returned) -> FDSDF_E_INVALID. */
fdsdf_status fdsdf_mesh_extract(const float* d_f, int nx, int ny, int nz, float ox, float oy, float oz,
                                float spacing, float* d_tris, int64_t max_tris, int64_t* h_ntris, void* d_work,
                                size_t work_bytes, void* stream);
/* Device workspace (bytes) fdsdf_mesh_metrics needs. */
size_t fdsdf_metrics_work_bytes(int64_t ntris, int64_t nsample, int64_t ngt);
/* The paper's reconstruction metrics between the mesh d_tris [ntris][3][3] and ground-truth
 * surface samples d_gt [ngt][3] with unit normals d_gt_normals [ngt][3]: nsample points
 * area-weighted on the mesh (counter-based SplitMix64 randoms of `seed`) with their face normals;
 * nearest neighbours both ways (brute force, ties -> lowest index).  h_out [6] (host, fp64):
 * CD = (mean_p d(p,G) + mean_g d(g,P))/2, F1 = 2PR/(P+R) at threshold tau (strict d < tau),
 * NC = (mean_p |n_p.n_nn| + mean_g |n_g.n_nn|)/2, Hausdorff, precision P, recall R -- unscaled
 * (the paper reports CD x10^3, F1 and NC x10^2).  Synchronises `stream`.  Errors: ntris == 0 ->
 * FDSDF_E_EMPTY; NULL pointers, counts < 1 or > 2^31-1, tau <= 0, workspace too small ->
 * FDSDF_E_INVALID. */
fdsdf_status fdsdf_mesh_metrics(const float* d_tris, int64_t ntris, const float* d_gt, const float* d_gt_normals,
                                int64_t ngt, int64_t nsample, uint64_t seed, float tau, double* h_out, void* d_work,
                                size_t work_bytes, void* stream);

/* One training step: the loss of Eq. (1) and its gradient with respect to every parameter.
 * d_grad [P] fp32 (overwritten, or accumulated with FDSDF_STEP_ACCUMULATE);
 * d_loss [8] fp64 = (L_DM, L_DNM, L_eik, L_fd, total, n_degenerate, 0, 0), each term
 * already divided by its global count (so it is SUM-reducible across ranks).
 * Errors: as fdsdf_eval, plus ctx created EVAL_ONLY, d_grad/d_loss NULL, negative or
 * non-finite weights, alpha <= 0, global counts smaller than the local ones ->
 * FDSDF_E_INVALID; an empty role with positive weight -> FDSDF_E_EMPTY;
 * ALLREDUCE without fdsdf_comm_init -> FDSDF_E_UNSUPPORTED. */
fdsdf_status fdsdf_step(fdsdf_ctx* ctx, const float* d_params, const float* d_x, int64_t n,
                        const fdsdf_stencil* st, const fdsdf_loss* ls, float* d_grad,
                        double* d_loss, uint32_t flags, void* stream);

/* The same step with HOST buffers (the end-to-end call): h_x [n][3] fp32 host memory (pinned
 * for an asynchronous copy; pageable memory works but the copy then blocks the host) is copied
 * into the context's device staging buffer, the step runs into the context's own gradient /
 * loss buffers, and both are copied back to h_grad [P] fp32 and h_loss [8] fp64 (host
 * memory) -- all enqueued on `stream`; the caller synchronises it before reading h_grad /
 * h_loss.  d_params stays device memory (the model state lives on the GPU).  With
 * FDSDF_STEP_ACCUMULATE the context's gradient buffer (zero at create) accumulates across
 * calls and h_grad receives the running sum.  Errors: as fdsdf_step (validated before
 * anything is enqueued); h_x / h_grad / h_loss NULL -> FDSDF_E_INVALID. */
fdsdf_status fdsdf_step_host(fdsdf_ctx* ctx, const float* d_params, const float* h_x, int64_t n,
                             const fdsdf_stencil* st, const fdsdf_loss* ls, float* h_grad,
                             double* h_loss, uint32_t flags, void* stream);

/* Data-parallel plumbing: rank 0 calls fdsdf_comm_unique_id, the caller
 * broadcasts the 128 bytes (e.g. through its torch process group), every rank calls
 * fdsdf_comm_init.  NCCL is loaded at run time (libnccl.so.2); missing -> FDSDF_E_NCCL.
 * fdsdf_allreduce: in-place SUM of count fp32 elements on the stream. */
fdsdf_status fdsdf_comm_unique_id(uint8_t id[128]);
fdsdf_status fdsdf_comm_init(fdsdf_ctx* ctx, const uint8_t id[128], int rank, int world);
fdsdf_status fdsdf_allreduce(fdsdf_ctx* ctx, float* d_buf, int64_t count, void* stream);

/* ---------------------------------------------------------------- training iteration
 * (§4).  A full iteration is, on one stream:
 *   fdsdf_sample -> fdsdf_step (FDSDF_STEP_ALLREDUCE when data-parallel) -> fdsdf_adam. */

/* Per-iteration batch ("we sample 30k surface points; 20k are used per iteration,
 * with 20k off-surface samples drawn uniformly in the bounding box").  Writes d_x_out
 * [n_pick + n_uniform][3] (device, caller-owned): rows [0, n_pick) are n_pick DISTINCT rows
 * of d_pool [n_pool][3] (sampling without replacement: pool index pi(row), pi a keyed
 * pseudo-random permutation -- 4-round Feistel network, cycle-walked; key from (seed,
 * iteration)), rows [n_pick, n_pick + n_uniform) are points uniform in [-box_half, box_half]^3
 * (SplitMix64 of (seed, iteration, row, coordinate)).  Deterministic: same arguments, same
 * output bits (train.cu documents both generators; oracle/train_oracle.py implements them).
 * Errors (checked in this order): ctx NULL, n_pick < 0, n_uniform < 0, iteration < 0,
 * n_pick > n_pool, d_pool NULL while n_pick > 0, box_half not finite or <= 0 ->
 * FDSDF_E_INVALID; n_pick + n_uniform == 0 -> FDSDF_E_EMPTY; d_x_out NULL -> FDSDF_E_INVALID. */
fdsdf_status fdsdf_sample(fdsdf_ctx* ctx, const float* d_pool, int64_t n_pool, int64_t n_pick,
                          float box_half, int64_t n_uniform, uint64_t seed, int64_t iteration,
                          float* d_x_out, void* stream);

/* In-place Adam update of d_params [P] from d_grad [P] with first / second moment buffers
 * d_m, d_v [P] (device, caller-owned, zero before step 1), step t >= 1 ("Adam
 * optimizer (5e-5)"; standard bias-corrected form):
 *   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;
 *   p -= lr / (1 - b1^t) * m / (sqrt(v / (1 - b2^t)) + eps).
 * A non-finite gradient entry leaves that parameter and its moments unchanged and sets
 * FDSDF_FLAG_NONFINITE_GRAD.  Errors: NULL pointers, t < 1, lr not finite or <= 0, b1 or b2
 * outside [0, 1), eps < 0 -> FDSDF_E_INVALID. */
fdsdf_status fdsdf_adam(fdsdf_ctx* ctx, float* d_params, const float* d_grad, float* d_m, float* d_v,
                        int64_t t, float lr, float beta1, float beta2, float eps, void* stream);

/* Diagnostics (synchronous). */
const char* fdsdf_status_string(fdsdf_status s);
const char* fdsdf_last_error(const fdsdf_ctx* ctx);
/* Returns and clears the sticky device flags (synchronises the context's device). */
fdsdf_status fdsdf_get_device_flags(fdsdf_ctx* ctx, uint32_t* out);
/* Which contraction path the context runs (-1: NULL): FDSDF_PATH_FFMA; FDSDF_PATH_TENSOR (every
 * contraction on the tensor cores, fused layer-sequential kernels); FDSDF_PATH_HYBRID (networks
 * with 512-wide layers or the skip layer, default flags: every contraction on the tensor cores
 * too -- the fused forward kernels, the backward as one GEMM + adjoint launch per hidden layer,
 * the weight gradient; FDSDF_HYBRID_FFMA_BWD=1 in the environment at create time keeps the
 * backward on the FFMA kernel). */
enum { FDSDF_PATH_FFMA = 0, FDSDF_PATH_TENSOR = 1, FDSDF_PATH_HYBRID = 2 };
int32_t fdsdf_path(const fdsdf_ctx* ctx);
/* Number of kernel launches enqueued by the last eval/step call on this context. */
int32_t fdsdf_last_launch_count(const fdsdf_ctx* ctx);
/* Per-kernel timing (for benchmarks).  When enabled, every kernel launch (and the NCCL group)
 * that fdsdf_eval / fdsdf_step enqueue is bracketed by CUDA events recorded on the SAME
 * stream.  fdsdf_kernel_times synchronises on the pending events, adds their elapsed times
 * to per-slot totals and returns, for slots 0..nslots-1 (FDSDF_KSLOT_*), the total
 * milliseconds and the number of timed launches since the last reset (reset != 0 clears the
 * totals after reading).  Errors: ctx NULL, nslots < 0, NULL outputs -> FDSDF_E_INVALID;
 * a failed event query -> FDSDF_E_CUDA. */
enum {
  FDSDF_KSLOT_PACK = 0,      /* weight re-layout for the TMA slabs                        */
  FDSDF_KSLOT_FWD = 1,       /* fused centre + stencil forward + FD epilogue (tensor path: */
                             /* the stencil-pair columns + FD epilogue)                    */
  FDSDF_KSLOT_BWD = 2,       /* backward through every stencil evaluation                */
  FDSDF_KSLOT_WGRAD = 3,     /* split-K weight-gradient contraction                      */
  FDSDF_KSLOT_FINALIZE = 4,  /* fixed-order reduction of partials and loss               */
  FDSDF_KSLOT_ALLREDUCE = 5, /* NCCL group (not a kernel of this library)                */
  FDSDF_KSLOT_PACK_TC = 6,   /* bf16x3 weight images for the tensor-core kernels           */
  FDSDF_KSLOT_FWD_CENTRE = 7,/* tensor path: centre + tangent columns (f, grad f, frame)   */
  FDSDF_KSLOT_SAMPLE = 8,    /* fdsdf_sample                                               */
  FDSDF_KSLOT_ADAM = 9,      /* fdsdf_adam                                                 */
  FDSDF_KSLOT_HESS = 10,     /* fdsdf_eval_hessian's axis-frame and scatter kernels        */
  FDSDF_NUM_KSLOTS = 11
};
fdsdf_status fdsdf_set_kernel_timing(fdsdf_ctx* ctx, int enable);
fdsdf_status fdsdf_kernel_times(fdsdf_ctx* ctx, double* ms_total, int64_t* count, int nslots, int reset);
/* Library version string. */
const char* fdsdf_version(void);

/* Self-test of the tcgen05 contraction core used by the tensor-pipe kernels:
 * D[m][n] = sum_k W[m][k] B[n][k] on the 5th-generation tensor cores, with every fp32
 * operand split exactly into three bf16 pieces and nprod of the piece products summed
 * (1: plain bf16, 3: the three leading products, 6: the fp32-accurate bf16x6 scheme).
 * d_W [M][K], d_B [N][K], d_D [M][N]: fp32 row-major device buffers owned by the caller.
 * One CTA; M in {128, 256}, N a multiple of 16 in [16, 256], K a multiple of 64.
 * mn_major = 0 stages both operands K-major (the forward / backward kernels' layout);
 * 1 stages them MN-major (the weight-gradient kernel's layout; N a multiple of 64).
 * Errors: NULL pointers, shapes or nprod out of range -> FDSDF_E_INVALID (nothing enqueued);
 * launch failure -> FDSDF_E_CUDA.  Test/diagnostic use only (not on the hot path). */
fdsdf_status fdsdf_selftest_mma(const float* d_W, const float* d_B, float* d_D, int M, int N, int K,
                                int nprod, int mn_major, void* stream);
/* The same bf16x6 GEMM on a CTA pair (cluster of 2, tcgen05 cta_group::2, M = 256): D [256][N]
 * = d_W [256][K] . d_B [N][K]^T; N a multiple of 32 in [32, 256], K a multiple of 64.
 * Errors as fdsdf_selftest_mma.  Test/diagnostic use only. */
fdsdf_status fdsdf_selftest_mma_pair(const float* d_W, const float* d_B, float* d_D, int N, int K, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FDSDF_H */
