// kernels.cuh -- kernel argument blocks and launch entry points shared by the C-ABI layer.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

namespace fdsdf {

enum { ACT_SOFTPLUS = 0, ACT_SINE = 1 };

constexpr int MAXL = 16;
constexpr int NCW = 8;             // compute warps per CTA
constexpr int NCT = NCW * 32;      // compute threads
constexpr int NTH = NCT;           // thread 0 also issues the TMA weight slabs
constexpr int NCOLF = 12;          // stored forward columns per centre: c, t0..2, (A,S) x 4
// zf (the step's stored pre-activations) layout: [n][nh][NCOLF/4][mpad][4] -- per (centre,
// hidden layer), the 12 columns in float4 groups per neuron m: g0 = (z, t0, t1, t2),
// g1 = (A0, A1, S0, S1), g2 = (A2, A3, S2, S3) (one 16-byte access per group and neuron; a
// warp's 32 neurons are 512 contiguous bytes).  Eval stores z only, contiguous over m at the
// start of each (centre, layer) block of zcols * mpad floats (zcols = 1 on eval-only contexts).
constexpr int ZG = NCOLF / 4;      // float4 groups of zf per (centre, layer)
constexpr int NCOLB = 10;          // backward columns: c, t_r, (A,S) x 4
constexpr int NSEED = 16;          // per-centre: fbar, Sbar_u, Sbar_v, Sbar_p, Sbar_q, r(3), u(3), v(3), pad
constexpr int NLOSS = 6;           // dm, dnm, eik, fd, n_degenerate, n_nonfinite

struct Net {
  int L;                 // linear layers
  int skip;              // -1 or skip layer
  int act;               // ACT_*
  int mpad;              // padded hidden width (64/128/256/512)
  float beta;
  int width[MAXL + 1];
  float omega[MAXL];     // per linear layer: omega for sine hidden layers, 1 otherwise
  const float* W[MAXL];  // into the caller's flat params
  const float* b[MAXL];
  const float* Wt[MAXL]; // packed forward weights (GEMM layers): [mpad k][mpad m]
  const float* Wb[MAXL]; // packed backward weights (GEMM layers): [mpad m][mpad k]
};

struct LossCfg {
  int kind, fd_form, denom, denom_pow;
  float w_dm, lambda_dnm, alpha, lambda_eik, lambda_fd, eps_grad;
  double inv_ns, inv_nu, inv_n;  // 1 / global counts (0 if the count is 0)
};

struct FwdArgs {
  Net net;
  LossCfg ls;
  const float* x;        // [n][3]
  int64_t n;
  int64_t n_surface;
  int64_t index_offset;
  uint64_t frame_seed;
  int frame_given;
  const float* frames_in;  // [n][6]
  float h;
  int step;              // 1: store the backward workspace and seeds
  // outputs (nullable)
  float* out_f;
  float* out_g;
  float* out_hess;
  float* out_K;
  float* out_D;
  float* out_frames;
  uint8_t* out_mask;
  // workspace
  float* zf;             // step: [n][nh][3][mpad][4] (NCOLF above); eval: z only
  float* seed;           // [n][8]
  double* lossp;         // [gridDim.x][NLOSS]
  unsigned* dflags;      // sticky device flags
  int64_t ntiles;
  // tensor-core path (fwd_tc.cu)
  int zcols;             // columns per (centre, layer) in zf: 12 (step) or 1 (eval: z only)
  const unsigned char* wimg;  // packed bf16x3 forward weight image (pack_tc_kernel)
  float* cinfo;          // [n][16] per-centre f, g, u, v, mask (written by mode 1, read by mode 2)
};

struct BwdArgs {
  Net net;
  const float* x;
  const float* zf;       // [n][nh][3][mpad][4] (NCOLF above)
  const float* seed;     // [n][8]
  int64_t n;
  float h;
  float* del;            // [nh][n*10][mpad]  (layers 1..L-2 used)
  float* actv;           // [nh][n*10][mpad]  (layers 0..L-3 used: input of layer l+1)
  float* bacc;           // [gridDim.x][nacc] per-CTA accumulators
  int64_t nacc;
  int64_t ntiles;
  const unsigned char* wimg;  // tensor path: packed bf16x3 W^T image (pack_tc_kernel)
};

struct WgradArgs {
  const float* del;
  const float* actv;
  float* part;           // [nglayers][nsplit][mpad][mpad]
  int64_t rows;          // n*10
  int64_t stride_layer;  // floats per layer in del / actv
  int mpad;
  int nsplit;
  int first_layer;       // GEMM layers first_layer .. first_layer + gridDim.z - 1
};

struct FinArgs {
  Net net;
  const float* part;     // wgrad partials
  int nsplit;
  const float* bacc;
  int64_t nacc;
  int nbcta;
  const double* lossp;
  int nfcta;
  LossCfg ls;
  float* grad;
  double* loss;
  int accumulate;
  unsigned* dflags;
  int64_t n_local;
  int64_t P;
};

// per-CTA accumulator layout of the backward kernel (floats):
//   db hidden layers [L-1][mpad] | dW_last [mpad] | db_last [1] | dW_0 [mpad][3]
inline int64_t bacc_size(int L, int mpad) { return (int64_t)(L - 1) * mpad + mpad + 1 + (int64_t)mpad * 3; }

// launchers (kernels.cu); return cudaError_t of the launch
cudaError_t launch_pack(const Net& net, float* wt_base, float* wb_base, cudaStream_t st);
cudaError_t launch_fwd(const FwdArgs& a, int grid, cudaStream_t st);
cudaError_t launch_bwd(const BwdArgs& a, int grid, cudaStream_t st);
cudaError_t launch_wgrad(const WgradArgs& a, int nglayers, cudaStream_t st);
cudaError_t launch_finalize(const FinArgs& a, cudaStream_t st);
// y[i] += x[i], i < n (the reduced per-call gradient added to an accumulating one)
cudaError_t launch_add_inplace(float* y, const float* x, int64_t n, cudaStream_t st);
// tensor-core (tcgen05, bf16x6) path: available for padded widths 128 / 256 without skip
bool tc_supported(int mpad, int skip);
size_t tc_wimg_bytes(int mpad, int ngemm);          // one packed weight image (fwd or bwd)
cudaError_t launch_pack_tc(const Net& net, unsigned char* fwd_img, unsigned char* bwd_img, cudaStream_t st);
cudaError_t launch_fwd_tc(const FwdArgs& a, int mode, int grid, cudaStream_t st);
int fwd_tc_tile_centres(int mode, int mpad);        // mode 1: N/4, mode 2: N/8 centres
bool tc_fwd_supported(int mpad);                    // tensor forward (fwd_tc.cu) for this width
cudaError_t launch_bwd_tc(const BwdArgs& a, int grid, cudaStream_t st);
int bwd_tc_tile_centres();                          // 8
int bwd_tc_acc_slots(int mpad);                     // accumulator slots per CTA
// hybrid path (512-wide layers, the skip layer): the backward as one tensor-core GEMM + adjoint
// launch per hidden layer (bwdl_tc.cu); mpad 256 / 512
bool bwdl_tc_supported(int mpad);
cudaError_t launch_bwdl_tc(const BwdArgs& a, int grid, cudaStream_t st);
int bwdl_tc_tile_centres(int mpad);                 // 16 (CTA pairs, mpad 512) or 8
int bwdl_tc_grid(int nsm, int64_t ntiles, int mpad); // CTAs (even for CTA pairs)
int bwdl_tc_acc_slots(int mpad);                    // accumulator slots per CTA
cudaError_t launch_wgrad_tc(const WgradArgs& a, int nglayers, bool bf16x3, cudaStream_t st);
int wgrad_tc_splits(int nsm, int64_t rows, int mpad);  // split-K factor of the tensor wgrad
bool wgrad_tc_supported(int mpad);                      // MPAD 128 / 256 / 512
// training iteration (train.cu)
int feistel_half_bits(int64_t n_pool);
cudaError_t launch_sample(const float* pool, int64_t n_pool, int64_t n_pick, float half, int64_t n_uniform,
                          uint64_t seed, int64_t iteration, float* out, cudaStream_t st);
cudaError_t launch_adam(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                        float eps, int64_t t, unsigned* dflags, cudaStream_t st);
cudaError_t launch_axis_frames(float* frames, int64_t n, int a, int b, cudaStream_t st);
cudaError_t launch_hess_scatter(const float* t, float* H, int64_t n, int pass, cudaStream_t st);
cudaError_t launch_cinfo_axis_frames(float* cinfo, int64_t n, int a, int b, cudaStream_t st);
int fwd_tile_centres(int mpad);   // centres per forward tile
int bwd_tile_centres(int mpad);   // centres per backward tile
size_t fwd_smem_bytes(int mpad);
size_t bwd_smem_bytes(int mpad);

}  // namespace fdsdf
