// api.cu -- the C ABI (include/fdsdf.h): validation, workspace, launch sequencing, NCCL.
#include <dlfcn.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fdsdf.h"
#include "kernels.cuh"


using namespace fdsdf;

namespace {

struct NcclApi {
  void* lib = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  int (*commInitRank)(void**, int, const void*, int) = nullptr;  // id passed by value: see wrapper
  int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  int (*commDestroy)(void*) = nullptr;
  const char* (*getErrorString)(int) = nullptr;
};

NcclApi g_nccl;

bool nccl_load(std::string* err) {
  if (g_nccl.lib) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    if (err) *err = std::string("cannot load libnccl.so.2: ") + dlerror();
    return false;
  }
  g_nccl.getUniqueId = (int (*)(void*))dlsym(h, "ncclGetUniqueId");
  g_nccl.commInitRank = (int (*)(void**, int, const void*, int))dlsym(h, "ncclCommInitRank");
  g_nccl.allReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclAllReduce");
  g_nccl.groupStart = (int (*)())dlsym(h, "ncclGroupStart");
  g_nccl.groupEnd = (int (*)())dlsym(h, "ncclGroupEnd");
  g_nccl.commDestroy = (int (*)(void*))dlsym(h, "ncclCommDestroy");
  g_nccl.getErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
  if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.allReduce || !g_nccl.groupStart || !g_nccl.groupEnd) {
    if (err) *err = "libnccl.so.2 lacks required symbols";
    return false;
  }
  g_nccl.lib = h;
  return true;
}

struct NcclId {
  char internal[128];
};

// ncclCommInitRank takes ncclUniqueId by value (a 128-byte struct): call through a typed pointer
typedef int (*CommInitRankFn)(void**, int, NcclId, int);

constexpr int kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0;

}  // namespace

struct fdsdf_ctx {
  int device = 0;
  fdsdf_mlp_spec spec{};
  Net net{};          // pointers filled per call
  int L = 0, mpad = 0, nh = 0, ngemm = 0;
  int64_t P = 0;
  int64_t offW[FDSDF_MAX_LINEAR]{}, offb[FDSDF_MAX_LINEAR]{};
  int64_t max_centers = 0;
  bool eval_only = false;
  int nsm = 0, fgrid = 0, bgrid = 0, ftile = 0, btile = 0, nsplit = 1;
  int64_t nacc = 0;
  // workspace
  float* wt = nullptr;
  float* wb = nullptr;
  float* zf = nullptr;       // step workspace
  float* xstage = nullptr;   // fdsdf_step_host: device copy of the points [max_centers][3]
  float* hgrad = nullptr;    //                  the gradient [P] (accumulates with ACCUMULATE)
  double* hloss = nullptr;   //                  the loss [8]
  float* gcall = nullptr;    // ACCUMULATE | ALLREDUCE: this call's gradient [P], reduced before it is added
  float* zscr = nullptr;     // eval scratch (per CTA)
  float* seed = nullptr;
  double* lossp = nullptr;
  float* del = nullptr;
  float* actv = nullptr;
  float* bacc = nullptr;
  float* part = nullptr;
  unsigned* dflags = nullptr;
  // tensor-core (tcgen05 bf16x6) forward
  bool tc = false;
  bool tcf = false;               // tensor-core forward (fwd_tc.cu): the tensor path, or the
                                  // hybrid path of 512-wide / skip-layer networks
  bool tcw = false;               // tensor-core weight gradient (wgrad_tc.cu): ditto
  bool wgrad3 = false;            // FDSDF_CREATE_WGRAD_BF16X3: the weight gradient's 3-product form
  unsigned char* fimg = nullptr;  // packed forward weight image
  unsigned char* bimg = nullptr;  // packed backward (W^T) weight image
  bool tcbl = false;              // hybrid path: layer-wise tensor-core backward (bwdl_tc.cu)
  float* cinfo = nullptr;    // [max_centers][16]
  float* zev = nullptr;      // eval-only contexts: [max_centers][nh][mpad] centre pre-activations
  float* hframes = nullptr;  // fdsdf_eval_hessian: [max_centers][6] axis frames
  float* htmp = nullptr;     // fdsdf_eval_hessian: [max_centers][3] one pass's (f_uu, f_uv, f_vv)
  void* comm = nullptr;
  int rank = 0, world = 1;
  int launches = 0;
  int last_fgrid = 0;
  std::string err;
  // optional per-kernel CUDA-event timing (fdsdf_set_kernel_timing)
  bool timing = false;
  struct Rec {
    int slot;
    cudaEvent_t a, b;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> spare;
  double tot_ms[FDSDF_NUM_KSLOTS]{};
  int64_t cnt[FDSDF_NUM_KSLOTS]{};
};

// Enqueue one kernel launch (or collective) on `st`, bracketed by CUDA events on the same
// stream when timing is enabled; counts the launch.
template <class F>
static cudaError_t run_slot(fdsdf_ctx* c, int slot, cudaStream_t st, F&& launch) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->timing) {
    for (cudaEvent_t* e : {&a, &b}) {
      if (!c->spare.empty()) {
        *e = c->spare.back();
        c->spare.pop_back();
      } else if (cudaEventCreate(e) != cudaSuccess) {
        *e = nullptr;
      }
    }
    if (a) cudaEventRecord(a, st);
  }
  cudaError_t e = launch();
  if (c->timing && a && b) {
    cudaEventRecord(b, st);
    c->pending.push_back({slot, a, b});
  }
  if (slot != FDSDF_KSLOT_ALLREDUCE) c->launches++;
  return e;
}

static fdsdf_status fail(fdsdf_ctx* c, fdsdf_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

static fdsdf_status cuda_fail(fdsdf_ctx* c, cudaError_t e, const char* where) {
  return fail(c, FDSDF_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

static int layer_fan_in(const fdsdf_mlp_spec* s, int l) { return s->width[l] + (l == s->skip_at ? 3 : 0); }

extern "C" {

const char* fdsdf_version(void) {
  return "fdsdf 0.2 (sm_100a, pair-symmetric difference form; fp32 FFMA and tcgen05 bf16x6 paths)";
}

int32_t fdsdf_path(const fdsdf_ctx* c) {
  return c ? (c->tc ? FDSDF_PATH_TENSOR : (c->tcf ? FDSDF_PATH_HYBRID : FDSDF_PATH_FFMA)) : -1;
}

const char* fdsdf_status_string(fdsdf_status s) {
  switch (s) {
    case FDSDF_OK: return "ok";
    case FDSDF_E_INVALID: return "invalid argument";
    case FDSDF_E_EMPTY: return "empty input";
    case FDSDF_E_CUDA: return "CUDA error";
    case FDSDF_E_NCCL: return "NCCL error";
    case FDSDF_E_NOMEM: return "out of device memory";
    case FDSDF_E_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

fdsdf_status fdsdf_validate_spec(const fdsdf_mlp_spec* s) {
  if (!s) return FDSDF_E_INVALID;
  const int L = s->n_linear;
  if (L < 2 || L > FDSDF_MAX_LINEAR) return FDSDF_E_INVALID;
  if (s->width[0] != 3 || s->width[L] != 1) return FDSDF_E_INVALID;
  for (int l = 1; l < L; ++l)
    if (s->width[l] < 1 || s->width[l] > FDSDF_MAX_WIDTH) return FDSDF_E_INVALID;
  if (s->act != FDSDF_ACT_SINE && s->act != FDSDF_ACT_SOFTPLUS) return FDSDF_E_INVALID;
  if (s->act == FDSDF_ACT_SOFTPLUS && !(s->beta > 0.f && std::isfinite(s->beta))) return FDSDF_E_INVALID;
  if (s->act == FDSDF_ACT_SINE && !(s->omega0_first > 0.f && s->omega0_hidden > 0.f &&
                                    std::isfinite(s->omega0_first) && std::isfinite(s->omega0_hidden)))
    return FDSDF_E_INVALID;
  if (s->skip_at != -1) {
    if (s->skip_at < 1 || s->skip_at > L - 2) return FDSDF_E_INVALID;
    if (s->width[s->skip_at] + 3 > FDSDF_MAX_WIDTH) return FDSDF_E_INVALID;
  }
  return FDSDF_OK;
}

int64_t fdsdf_spec_num_params(const fdsdf_mlp_spec* s) {
  if (fdsdf_validate_spec(s) != FDSDF_OK) return -1;
  int64_t P = 0;
  for (int l = 0; l < s->n_linear; ++l) P += (int64_t)s->width[l + 1] * layer_fan_in(s, l) + s->width[l + 1];
  return P;
}

int64_t fdsdf_spec_param_offset(const fdsdf_mlp_spec* s, int layer, int is_bias) {
  if (fdsdf_validate_spec(s) != FDSDF_OK || layer < 0 || layer >= s->n_linear) return -1;
  int64_t off = 0;
  for (int l = 0; l < layer; ++l) off += (int64_t)s->width[l + 1] * layer_fan_in(s, l) + s->width[l + 1];
  if (is_bias) off += (int64_t)s->width[layer + 1] * layer_fan_in(s, layer);
  return off;
}

int64_t fdsdf_num_params(const fdsdf_ctx* c) { return c ? c->P : -1; }
const char* fdsdf_last_error(const fdsdf_ctx* c) { return c ? c->err.c_str() : "null context"; }
int32_t fdsdf_last_launch_count(const fdsdf_ctx* c) { return c ? c->launches : 0; }

void fdsdf_destroy(fdsdf_ctx* c) {
  if (!c) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (c->comm && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
  for (auto& r : c->pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : c->spare) cudaEventDestroy(e);
  void* bufs[] = {c->wt,   c->wb,   c->zf,     c->zscr,   c->seed,  c->lossp, c->del, c->actv,
                  c->bacc, c->part, c->dflags, c->fimg, c->cinfo, c->zev, c->bimg, c->hframes, c->htmp,
                  c->xstage, c->hgrad, c->hloss, c->gcall};
  for (void* b : bufs)
    if (b) cudaFree(b);
  cudaSetDevice(prev);
  delete c;
}

fdsdf_status fdsdf_create(const fdsdf_mlp_spec* spec, int device, int64_t max_centers, uint32_t flags,
                          fdsdf_ctx** out) {
  if (!out) return FDSDF_E_INVALID;
  *out = nullptr;
  if (fdsdf_validate_spec(spec) != FDSDF_OK) return FDSDF_E_INVALID;
  if (max_centers < 1) return FDSDF_E_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return FDSDF_E_UNSUPPORTED;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return FDSDF_E_UNSUPPORTED;
  if (prop.major != 10) return FDSDF_E_UNSUPPORTED;  // built for sm_100a only

  fdsdf_ctx* c = new fdsdf_ctx();
  c->device = device;
  c->spec = *spec;
  c->L = spec->n_linear;
  c->nh = c->L - 1;
  c->ngemm = c->L - 2;
  int wmax = 1;
  for (int l = 1; l < c->L; ++l) wmax = std::max(wmax, spec->width[l]);
  if (spec->skip_at >= 0) wmax = std::max(wmax, spec->width[spec->skip_at] + 3);
  c->mpad = wmax <= 64 ? 64 : (wmax <= 128 ? 128 : (wmax <= 256 ? 256 : 512));
  if ((flags & FDSDF_CREATE_FFMA) && (flags & FDSDF_CREATE_TENSOR)) {
    delete c;
    return FDSDF_E_INVALID;
  }
  {
    // default path: the tensor cores wherever the spec allows it (hidden widths <= 256, no
    // skip layer); FDSDF_CREATE_FFMA forces the fp32 FFMA kernels
    const int mp_tc = std::max(c->mpad, 128);  // widths <= 64 are zero-padded to one M=128 tile
    const bool ok_tc = tc_supported(mp_tc, spec->skip_at);
    if ((flags & FDSDF_CREATE_TENSOR) && !ok_tc) {
      delete c;
      return FDSDF_E_UNSUPPORTED;
    }
    if (ok_tc && !(flags & FDSDF_CREATE_FFMA)) {
      c->tc = true;
      c->mpad = mp_tc;
      // FDSDF_FORCE_HYBRID=1 (A/B only): a 256-wide network on the hybrid path's layer-wise backward
      const char* fh = getenv("FDSDF_FORCE_HYBRID");
      if (fh && fh[0] == '1' && c->mpad == 256 && !(flags & FDSDF_CREATE_TENSOR)) c->tc = false;
    }
    // networks the full tensor path does not cover (512-wide layers, the skip layer) still run
    // their forward and weight gradient on the tensor cores when the padded width is a tcgen05
    // tile (128/256/512); only the backward stays on the FFMA kernel (same zf / seed / del /
    // actv layouts)
    c->tcf = c->tc || (!(flags & FDSDF_CREATE_FFMA) && c->mpad >= 128 && tc_fwd_supported(c->mpad));
    c->tcw = c->tcf && wgrad_tc_supported(c->mpad);
    // hybrid path: the backward on the tensor cores too (one GEMM + adjoint-map launch per
    // layer, bwdl_tc.cu); FDSDF_HYBRID_FFMA_BWD=1 keeps the FFMA backward (A/B, validation)
    {
      const char* ev = getenv("FDSDF_HYBRID_FFMA_BWD");
      c->tcbl = !c->tc && c->tcf && bwdl_tc_supported(c->mpad) && !(ev && ev[0] == '1');
    }
    c->wgrad3 = (flags & FDSDF_CREATE_WGRAD_BF16X3) != 0;
    if (c->wgrad3 && !c->tcw) {  // only the tensor-core weight gradient has the 3-product form
      delete c;
      return (flags & FDSDF_CREATE_FFMA) ? FDSDF_E_INVALID : FDSDF_E_UNSUPPORTED;
    }
  }
  c->P = fdsdf_spec_num_params(spec);
  for (int l = 0; l < c->L; ++l) {
    c->offW[l] = fdsdf_spec_param_offset(spec, l, 0);
    c->offb[l] = fdsdf_spec_param_offset(spec, l, 1);
  }
  c->max_centers = max_centers;
  c->eval_only = (flags & FDSDF_CREATE_EVAL_ONLY) != 0;
  c->nsm = prop.multiProcessorCount;
  if (const char* ev = getenv("FDSDF_MAX_SM")) {  // cap the persistent grids (fdsdf.h)
    const int k = atoi(ev);
    if (k >= 2 && k < c->nsm) c->nsm = k;
  }
  c->ftile = fwd_tile_centres(c->mpad);
  c->btile = bwd_tile_centres(c->mpad);

  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  // occupancy-derived persistent grids
  c->fgrid = c->nsm * 2;
  c->bgrid = c->nsm * 2;
  {
    const size_t fs = fwd_smem_bytes(c->mpad), bs = bwd_smem_bytes(c->mpad);
    const size_t per_sm = (size_t)prop.sharedMemPerMultiprocessor;
    const int fo = (int)std::max<size_t>(1, std::min<size_t>(2, per_sm / (fs + 1024)));
    const int bo = (int)std::max<size_t>(1, std::min<size_t>(2, per_sm / (bs + 1024)));
    c->fgrid = c->nsm * fo;
    c->bgrid = c->nsm * bo;
  }
  const int mp = c->mpad;
  const int64_t ftile_cap = (max_centers + c->ftile - 1) / c->ftile;
  const int64_t btile_cap = (max_centers + c->btile - 1) / c->btile;
  c->fgrid = (int)std::min<int64_t>(c->fgrid, ftile_cap);
  c->bgrid = (int)std::min<int64_t>(c->bgrid, btile_cap);
  c->nacc = bacc_size(c->L, mp);
  const int nb = (mp >= 128 ? mp / 128 : 1);
  c->nsplit = std::max(1, (int)std::min<int64_t>((4 * c->nsm + c->ngemm * nb * nb - 1) / std::max(1, c->ngemm * nb * nb),
                                                  (max_centers * NCOLB + 255) / 256));
  auto alloc = [&](void** p, size_t bytes) -> bool {
    if (bytes == 0) return true;
    return cudaMalloc(p, bytes) == cudaSuccess;
  };
  bool ok = true;
  const size_t gemm_w = (size_t)std::max(0, c->ngemm) * mp * mp * sizeof(float);
  ok = ok && alloc((void**)&c->wt, gemm_w);
  ok = ok && alloc((void**)&c->wb, gemm_w);
  ok = ok && alloc((void**)&c->zscr, (size_t)c->fgrid * c->ftile * c->nh * mp * sizeof(float));
  // per-CTA loss partials of the forward: the FFMA grid, or up to one CTA per SM (tensor path)
  ok = ok && alloc((void**)&c->lossp, (size_t)std::max(c->fgrid, c->nsm) * NLOSS * sizeof(double));
  ok = ok && alloc((void**)&c->dflags, sizeof(unsigned));
  ok = ok && alloc((void**)&c->hframes, (size_t)max_centers * 6 * sizeof(float));
  ok = ok && alloc((void**)&c->htmp, (size_t)max_centers * 3 * sizeof(float));
  if (ok && !c->eval_only) {
    ok = ok && alloc((void**)&c->zf, (size_t)max_centers * c->nh * NCOLF * mp * sizeof(float));
    ok = ok && alloc((void**)&c->xstage, (size_t)max_centers * 3 * sizeof(float));
    ok = ok && alloc((void**)&c->hgrad, (size_t)c->P * sizeof(float));
    ok = ok && alloc((void**)&c->hloss, 8 * sizeof(double));
    ok = ok && alloc((void**)&c->gcall, (size_t)c->P * sizeof(float));
    if (ok) ok = cudaMemset(c->hgrad, 0, (size_t)c->P * sizeof(float)) == cudaSuccess;
    ok = ok && alloc((void**)&c->seed, (size_t)max_centers * NSEED * sizeof(float));
    ok = ok && alloc((void**)&c->del, (size_t)c->nh * max_centers * NCOLB * mp * sizeof(float));
    ok = ok && alloc((void**)&c->actv, (size_t)c->nh * max_centers * NCOLB * mp * sizeof(float));
    const size_t bslots = c->tc     ? (size_t)c->nsm * bwd_tc_acc_slots(mp)
                          : c->tcbl ? (size_t)c->nsm * bwdl_tc_acc_slots(mp)
                                    : (size_t)c->bgrid;
    ok = ok && alloc((void**)&c->bacc, std::max<size_t>(bslots, c->bgrid) * c->nacc * sizeof(float));
    const int nsplit_max = c->tcw ? std::max(c->nsplit, c->nsm) : c->nsplit;
    ok = ok && alloc((void**)&c->part, (size_t)std::max(0, c->ngemm) * nsplit_max * mp * mp * sizeof(float));
  }
  if (ok && c->tcf) {
    ok = ok && alloc((void**)&c->fimg, tc_wimg_bytes(mp, c->ngemm));
    ok = ok && alloc((void**)&c->cinfo, (size_t)max_centers * 16 * sizeof(float));
    if (c->eval_only) ok = ok && alloc((void**)&c->zev, (size_t)max_centers * c->nh * mp * sizeof(float));
    if ((c->tc || c->tcbl) && !c->eval_only) ok = ok && alloc((void**)&c->bimg, tc_wimg_bytes(mp, c->ngemm));
  }
  if (ok) ok = cudaMemset(c->dflags, 0, sizeof(unsigned)) == cudaSuccess;
  cudaSetDevice(prev);
  if (!ok) {
    cudaGetLastError();
    fdsdf_destroy(c);
    return FDSDF_E_NOMEM;
  }
  *out = c;
  return FDSDF_OK;
}

}  // extern "C"

static void fill_net(fdsdf_ctx* c, const float* d_params) {
  Net& n = c->net;
  n.L = c->L;
  n.skip = c->spec.skip_at;
  n.act = c->spec.act == FDSDF_ACT_SINE ? ACT_SINE : ACT_SOFTPLUS;
  n.mpad = c->mpad;
  n.beta = c->spec.act == FDSDF_ACT_SOFTPLUS ? c->spec.beta : 1.0f;
  for (int l = 0; l <= c->L; ++l) n.width[l] = c->spec.width[l];
  for (int l = 0; l < c->L; ++l) {
    n.omega[l] = (c->spec.act == FDSDF_ACT_SINE && l < c->L - 1)
                     ? (l == 0 ? c->spec.omega0_first : c->spec.omega0_hidden)
                     : 1.0f;
    n.W[l] = d_params + c->offW[l];
    n.b[l] = d_params + c->offb[l];
    n.Wt[l] = (l >= 1 && l <= c->L - 2) ? c->wt + (size_t)(l - 1) * c->mpad * c->mpad : nullptr;
    n.Wb[l] = (l >= 1 && l <= c->L - 2) ? c->wb + (size_t)(l - 1) * c->mpad * c->mpad : nullptr;
  }
}

static fdsdf_status check_common(fdsdf_ctx* c, const float* d_params, const float* d_x, int64_t n,
                                 const fdsdf_stencil* st) {
  if (!c) return FDSDF_E_INVALID;
  if (n < 0 || n > c->max_centers) return fail(c, FDSDF_E_INVALID, "n out of range [0, max_centers]");
  if (n == 0) return fail(c, FDSDF_E_EMPTY, "n == 0");
  if (!d_params || !d_x || !st) return fail(c, FDSDF_E_INVALID, "null pointer argument");
  if (!(st->h > 0.f) || !std::isfinite(st->h)) return fail(c, FDSDF_E_INVALID, "h must be finite and > 0");
  if (!(st->eps_grad >= 0.f) || !std::isfinite(st->eps_grad)) return fail(c, FDSDF_E_INVALID, "eps_grad must be >= 0");
  if (st->denom < 0 || st->denom > 2) return fail(c, FDSDF_E_INVALID, "denom out of range");
  if (st->denom_pow < 0 || st->denom_pow > 16) return fail(c, FDSDF_E_INVALID, "denom_pow out of range");
  if (st->frame_mode != FDSDF_FRAME_RANDOM && st->frame_mode != FDSDF_FRAME_GIVEN)
    return fail(c, FDSDF_E_INVALID, "frame_mode out of range");
  if (st->frame_mode == FDSDF_FRAME_GIVEN && !st->d_frames_in)
    return fail(c, FDSDF_E_INVALID, "GIVEN frames without d_frames_in");
  if (st->n_surface < 0 || st->n_surface > n) return fail(c, FDSDF_E_INVALID, "n_surface out of range [0, n]");
  if (st->index_offset < 0) return fail(c, FDSDF_E_INVALID, "index_offset < 0");
  return FDSDF_OK;
}

static void fill_fwd(fdsdf_ctx* c, FwdArgs& a, const float* d_x, int64_t n, const fdsdf_stencil* st) {
  a.net = c->net;
  a.x = d_x;
  a.n = n;
  a.n_surface = st->n_surface;
  a.index_offset = st->index_offset;
  a.frame_seed = st->frame_seed;
  a.frame_given = st->frame_mode == FDSDF_FRAME_GIVEN;
  a.frames_in = st->d_frames_in;
  a.h = st->h;
  a.dflags = c->dflags;
  a.lossp = c->lossp;
  a.ntiles = (n + c->ftile - 1) / c->ftile;
  a.ls.denom = st->denom;
  a.ls.denom_pow = st->denom_pow;
  a.ls.eps_grad = st->eps_grad;
}

// tensor-core forward: mode 1 (centre + tangents -> f, g, frame) then mode 2 (stencil pairs ->
// FD epilogue).  Sets a.ntiles per launch; records the mode-2 grid in c->last_fgrid.
// pairs_only: skip mode 1 and reuse the centre info / centre pre-activations a previous call
// left in the workspace (fdsdf_eval_hessian's 2nd and 3rd frame passes)
// persistent grid of the tensor-core kernels: one CTA per SM, at most one per tile, and even
// (they run as clusters of 2 sharing the weight stream, tcmlp.cuh FDSDF_WMC)
static int tc_grid(const fdsdf_ctx* c, int64_t ntiles) {
  const int64_t g = std::min<int64_t>(c->nsm, ntiles);
  return (int)std::min<int64_t>(c->nsm & ~1, (g + 1) & ~1);
}

static cudaError_t launch_fwd_tc_pair(fdsdf_ctx* c, FwdArgs& a, cudaStream_t strm, bool pairs_only = false,
                                      bool centre_only = false) {
  a.wimg = c->fimg;
  a.cinfo = c->cinfo;
  const int64_t n = a.n;
  a.ntiles = (n + fwd_tc_tile_centres(1, c->mpad) - 1) / fwd_tc_tile_centres(1, c->mpad);
  const int g1 = tc_grid(c, a.ntiles);
  cudaError_t e = pairs_only ? cudaSuccess
                             : run_slot(c, FDSDF_KSLOT_FWD_CENTRE, strm, [&] { return launch_fwd_tc(a, 1, g1, strm); });
  if (e != cudaSuccess || centre_only) return e;
  a.ntiles = (n + fwd_tc_tile_centres(2, c->mpad) - 1) / fwd_tc_tile_centres(2, c->mpad);
  const int g2 = tc_grid(c, a.ntiles);
  c->last_fgrid = g2;
  return run_slot(c, FDSDF_KSLOT_FWD, strm, [&] { return launch_fwd_tc(a, 2, g2, strm); });
}

extern "C" {

// the body of fdsdf_eval (arguments already validated); pairs_only: see launch_fwd_tc_pair
static fdsdf_status eval_run(fdsdf_ctx* c, const float* d_params, const float* d_x, int64_t n,
                             const fdsdf_stencil* st, const fdsdf_eval_out* out, cudaStream_t strm,
                             bool pairs_only, bool centre_only = false);

fdsdf_status fdsdf_eval(fdsdf_ctx* c, const float* d_params, const float* d_x, int64_t n, const fdsdf_stencil* st,
                        const fdsdf_eval_out* out, void* stream) {
  fdsdf_status s = check_common(c, d_params, d_x, n, st);
  if (s != FDSDF_OK) return s;
  return eval_run(c, d_params, d_x, n, st, out, (cudaStream_t)stream, false);
}

fdsdf_status fdsdf_eval_field(fdsdf_ctx* c, const float* d_params, const float* d_x, int64_t n, float* d_f,
                              float* d_grad, void* stream) {
  if (!c) return FDSDF_E_INVALID;
  if (!d_f && !d_grad && n > 0) return fail(c, FDSDF_E_INVALID, "no output requested");
  fdsdf_stencil st{};
  st.h = 1e-2f;  // unused by the centre pass (the tensor path runs only that pass)
  st.frame_mode = FDSDF_FRAME_RANDOM;
  st.eps_grad = 0.f;
  st.denom = FDSDF_DENOM_ONE;
  st.denom_pow = 4;
  fdsdf_status s = check_common(c, d_params, d_x, n, &st);
  if (s != FDSDF_OK) return s;
  fdsdf_eval_out out{};
  out.d_f = d_f;
  out.d_grad = d_grad;
  return eval_run(c, d_params, d_x, n, &st, &out, (cudaStream_t)stream, false, true);
}

}  // extern "C"

static fdsdf_status eval_run(fdsdf_ctx* c, const float* d_params, const float* d_x, int64_t n,
                             const fdsdf_stencil* st, const fdsdf_eval_out* out, cudaStream_t strm,
                             bool pairs_only, bool centre_only) {
  pairs_only = pairs_only && c->tcf;  // the FFMA forward is one fused kernel
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != c->device) cudaSetDevice(c->device);
  fill_net(c, d_params);
  c->launches = 0;
  cudaError_t e = cudaSuccess;
  if (c->tcf) {
    if (c->ngemm > 0 && !pairs_only)
      e = run_slot(c, FDSDF_KSLOT_PACK_TC, strm, [&] { return launch_pack_tc(c->net, c->fimg, nullptr, strm); });
  } else if (c->ngemm > 0) {
    e = run_slot(c, FDSDF_KSLOT_PACK, strm, [&] { return launch_pack(c->net, c->wt, c->wb, strm); });
  }
  if (e != cudaSuccess) {
    if (prev != c->device) cudaSetDevice(prev);
    return cuda_fail(c, e, "pack");
  }
  FwdArgs a{};
  fill_fwd(c, a, d_x, n, st);
  a.ls.kind = 0;
  a.step = 0;
  a.zf = c->zscr;
  if (out) {
    a.out_f = out->d_f;
    a.out_g = out->d_grad;
    a.out_hess = out->d_hess;
    a.out_K = out->d_K;
    a.out_D = out->d_D;
    a.out_frames = out->d_frames;
    a.out_mask = out->d_mask;
  }
  if (c->tcf) {
    a.zf = c->eval_only ? c->zev : c->zf;
    a.zcols = c->eval_only ? 1 : NCOLF;
    e = launch_fwd_tc_pair(c, a, strm, pairs_only, centre_only);
    if (prev != c->device) cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(c, e, "fwd_tc_kernel");
    return FDSDF_OK;
  }
  const int grid = (int)std::min<int64_t>(c->fgrid, a.ntiles);
  e = run_slot(c, FDSDF_KSLOT_FWD, strm, [&] { return launch_fwd(a, grid, strm); });
  if (prev != c->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(c, e, "fwd_kernel");
  return FDSDF_OK;
}

extern "C" {

fdsdf_status fdsdf_eval_hessian(fdsdf_ctx* c, const float* d_params, const float* d_x, int64_t n, float h,
                                float* d_H, float* d_f, float* d_grad, void* stream) {
  if (!c) return FDSDF_E_INVALID;
  if (!d_H && n > 0) return fail(c, FDSDF_E_INVALID, "null d_H");
  fdsdf_stencil st{};
  st.h = h;
  st.frame_mode = FDSDF_FRAME_GIVEN;
  st.d_frames_in = c->hframes;
  st.eps_grad = 0.f;  // the Hessian is wanted at critical points too
  st.denom = FDSDF_DENOM_ONE;
  st.denom_pow = 4;
  fdsdf_status s = check_common(c, d_params, d_x, n, &st);
  if (s != FDSDF_OK) return s;
  cudaStream_t strm = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != c->device) cudaSetDevice(c->device);
  static const int AX[3][2] = {{0, 1}, {0, 2}, {1, 2}};
  int launches = 0;
  c->launches = 0;
  for (int pass = 0; pass < 3; ++pass) {
    // tensor path, passes 1 and 2: f, grad f and the centre pre-activations are those of pass 0;
    // only the frame changes -> rewrite the frame fields of the centre info, run the pair kernel
    const bool pairs_only = c->tcf && pass > 0;
    cudaError_t e = run_slot(c, FDSDF_KSLOT_HESS, strm, [&] {
      return pairs_only ? launch_cinfo_axis_frames(c->cinfo, n, AX[pass][0], AX[pass][1], strm)
                        : launch_axis_frames(c->hframes, n, AX[pass][0], AX[pass][1], strm);
    });
    if (e != cudaSuccess) {
      if (prev != c->device) cudaSetDevice(prev);
      return cuda_fail(c, e, "axis_frames_kernel");
    }
    fdsdf_eval_out out{};
    out.d_hess = c->htmp;
    if (pass == 0) {
      out.d_f = d_f;
      out.d_grad = d_grad;
    }
    launches += c->launches;
    s = eval_run(c, d_params, d_x, n, &st, &out, strm, pairs_only);
    if (s != FDSDF_OK) {
      if (prev != c->device) cudaSetDevice(prev);
      return s;
    }
    launches += c->launches;
    c->launches = 0;
    e = run_slot(c, FDSDF_KSLOT_HESS, strm, [&] { return launch_hess_scatter(c->htmp, d_H, n, pass, strm); });
    if (e != cudaSuccess) {
      if (prev != c->device) cudaSetDevice(prev);
      return cuda_fail(c, e, "hess_scatter_kernel");
    }
  }
  c->launches += launches;
  if (prev != c->device) cudaSetDevice(prev);
  return FDSDF_OK;
}

}  // extern "C"

// fdsdf_step, and fdsdf_step_host (h_x != nullptr: the points are copied host -> d_x first;
// h_grad / h_loss != nullptr: the results are copied back after the step), all enqueued on the
// caller's stream after validation, so an error still enqueues nothing
static fdsdf_status step_impl(fdsdf_ctx* c, const float* d_params, const float* d_x, int64_t n, const fdsdf_stencil* st,
                              const fdsdf_loss* ls, float* d_grad, double* d_loss, uint32_t flags, void* stream,
                              const float* h_x, float* h_grad, double* h_loss) {
  fdsdf_status s = check_common(c, d_params, d_x, n, st);
  if (s != FDSDF_OK) return s;
  if (c->eval_only) return fail(c, FDSDF_E_INVALID, "context created EVAL_ONLY");
  if (!ls || !d_grad || !d_loss) return fail(c, FDSDF_E_INVALID, "null pointer argument");
  if (ls->kind != FDSDF_LOSS_NCR && ls->kind != FDSDF_LOSS_NSH) return fail(c, FDSDF_E_INVALID, "loss kind");
  if (ls->fd_form != FDSDF_FD_ABS && ls->fd_form != FDSDF_FD_SQUARE) return fail(c, FDSDF_E_INVALID, "fd_form");
  const float ws[] = {ls->w_dm, ls->lambda_dnm, ls->lambda_eik, ls->lambda_fd};
  for (float w : ws)
    if (!(w >= 0.f) || !std::isfinite(w)) return fail(c, FDSDF_E_INVALID, "loss weights must be finite and >= 0");
  if (!(ls->alpha_dnm > 0.f) || !std::isfinite(ls->alpha_dnm)) return fail(c, FDSDF_E_INVALID, "alpha must be > 0");
  const int64_t nsl = st->n_surface, nul = n - st->n_surface;
  if (ls->n_surface_global < nsl || ls->n_uniform_global < nul || ls->n_global < n ||
      ls->n_global != ls->n_surface_global + ls->n_uniform_global)
    return fail(c, FDSDF_E_INVALID, "global counts inconsistent with the local rows");
  if (ls->w_dm > 0.f && ls->n_surface_global == 0) return fail(c, FDSDF_E_EMPTY, "no surface rows but w_dm > 0");
  if (ls->lambda_dnm > 0.f && ls->n_uniform_global == 0)
    return fail(c, FDSDF_E_EMPTY, "no uniform rows but lambda_dnm > 0");
  if ((flags & FDSDF_STEP_ALLREDUCE) && !c->comm)
    return fail(c, FDSDF_E_UNSUPPORTED, "ALLREDUCE requested before fdsdf_comm_init");

  cudaStream_t strm = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != c->device) cudaSetDevice(c->device);
  auto done = [&](fdsdf_status r) {
    if (prev != c->device) cudaSetDevice(prev);
    return r;
  };
  fill_net(c, d_params);
  c->launches = 0;
  cudaError_t e = cudaSuccess;
  if (h_x) {
    e = cudaMemcpyAsync(const_cast<float*>(d_x), h_x, (size_t)n * 3 * sizeof(float), cudaMemcpyHostToDevice, strm);
    if (e != cudaSuccess) return done(cuda_fail(c, e, "host -> device copy of the points"));
  }
  if (c->tcf && c->ngemm > 0)  // tensor forward image (and, on the tensor path, the backward's)
    e = run_slot(c, FDSDF_KSLOT_PACK_TC, strm, [&] { return launch_pack_tc(c->net, c->fimg, c->bimg, strm); });
  if (e == cudaSuccess && !c->tc && !(c->tcbl && c->tcw) && c->ngemm > 0)  // FFMA backward / weight gradient
    e = run_slot(c, FDSDF_KSLOT_PACK, strm, [&] { return launch_pack(c->net, c->wt, c->wb, strm); });
  if (e != cudaSuccess) return done(cuda_fail(c, e, "pack_tc"));

  FwdArgs a{};
  fill_fwd(c, a, d_x, n, st);
  a.ls.kind = ls->kind;
  a.ls.fd_form = ls->fd_form;
  a.ls.w_dm = ls->w_dm;
  a.ls.lambda_dnm = ls->lambda_dnm;
  a.ls.alpha = ls->alpha_dnm;
  a.ls.lambda_eik = ls->lambda_eik;
  a.ls.lambda_fd = ls->lambda_fd;
  a.ls.inv_ns = ls->n_surface_global > 0 ? 1.0 / (double)ls->n_surface_global : 0.0;
  a.ls.inv_nu = ls->n_uniform_global > 0 ? 1.0 / (double)ls->n_uniform_global : 0.0;
  a.ls.inv_n = 1.0 / (double)ls->n_global;
  a.step = 1;
  a.zf = c->zf;
  a.seed = c->seed;
  int fgrid = (int)std::min<int64_t>(c->fgrid, a.ntiles);
  if (c->tcf) {
    a.zcols = NCOLF;
    e = launch_fwd_tc_pair(c, a, strm);
    fgrid = c->last_fgrid;
  } else {
    e = run_slot(c, FDSDF_KSLOT_FWD, strm, [&] { return launch_fwd(a, fgrid, strm); });
  }
  if (e != cudaSuccess) return done(cuda_fail(c, e, "fwd_kernel"));

  BwdArgs b{};
  b.net = c->net;
  b.x = d_x;
  b.zf = c->zf;
  b.seed = c->seed;
  b.n = n;
  b.h = st->h;
  b.del = c->del;
  b.actv = c->actv;
  b.bacc = c->bacc;
  b.nacc = c->nacc;
  int bgrid, nbslots;
  if (c->tc) {
    b.wimg = c->bimg;
    b.ntiles = (n + bwd_tc_tile_centres() - 1) / bwd_tc_tile_centres();
    bgrid = tc_grid(c, b.ntiles);
    nbslots = bgrid * bwd_tc_acc_slots(c->mpad);
    e = run_slot(c, FDSDF_KSLOT_BWD, strm, [&] { return launch_bwd_tc(b, bgrid, strm); });
  } else if (c->tcbl) {
    b.wimg = c->bimg;
    b.ntiles = (n + bwdl_tc_tile_centres(c->mpad) - 1) / bwdl_tc_tile_centres(c->mpad);
    bgrid = bwdl_tc_grid(c->nsm, b.ntiles, c->mpad);
    nbslots = bgrid * bwdl_tc_acc_slots(c->mpad);
    e = run_slot(c, FDSDF_KSLOT_BWD, strm, [&] { return launch_bwdl_tc(b, bgrid, strm); });
    c->launches += c->L - 2;  // one launch per hidden layer
  } else {
    b.ntiles = (n + c->btile - 1) / c->btile;
    bgrid = (int)std::min<int64_t>(c->bgrid, b.ntiles);
    nbslots = bgrid;
    e = run_slot(c, FDSDF_KSLOT_BWD, strm, [&] { return launch_bwd(b, bgrid, strm); });
  }
  if (e != cudaSuccess) return done(cuda_fail(c, e, "bwd_kernel"));

  WgradArgs w{};
  w.del = c->del;
  w.actv = c->actv;
  w.part = c->part;
  w.rows = n * NCOLB;
  w.stride_layer = n * NCOLB * c->mpad;
  w.mpad = c->mpad;
  w.nsplit = c->tcw ? wgrad_tc_splits(c->nsm, w.rows, c->mpad) : c->nsplit;
  w.first_layer = 1;
  if (c->ngemm > 0)
    e = run_slot(c, FDSDF_KSLOT_WGRAD, strm, [&] {
      return c->tcw ? launch_wgrad_tc(w, c->ngemm, c->wgrad3, strm) : launch_wgrad(w, c->ngemm, strm);
    });
  if (e != cudaSuccess) return done(cuda_fail(c, e, "wgrad_kernel"));

  FinArgs f{};
  f.net = c->net;
  f.part = c->part;
  f.nsplit = w.nsplit;
  f.bacc = c->bacc;
  f.nacc = c->nacc;
  f.nbcta = nbslots;
  f.lossp = c->lossp;
  f.nfcta = fgrid;
  f.ls = a.ls;
  // ACCUMULATE together with ALLREDUCE: only THIS call's contribution may be summed over the
  // ranks (d_grad already holds the reduced earlier contributions, identical on every rank), so
  // finalize writes it to gcall, the allreduce runs on gcall, and it is then added to d_grad
  const bool acc_reduce = (flags & FDSDF_STEP_ACCUMULATE) && (flags & FDSDF_STEP_ALLREDUCE);
  f.grad = acc_reduce ? c->gcall : d_grad;
  f.loss = d_loss;
  f.accumulate = (!acc_reduce && (flags & FDSDF_STEP_ACCUMULATE)) ? 1 : 0;
  f.dflags = c->dflags;
  f.n_local = n;
  f.P = c->P;
  e = run_slot(c, FDSDF_KSLOT_FINALIZE, strm, [&] { return launch_finalize(f, strm); });
  if (e != cudaSuccess) return done(cuda_fail(c, e, "finalize_kernel"));

  if (flags & FDSDF_STEP_ALLREDUCE) {
    int r1 = 0, r2 = 0, r3 = 0;
    run_slot(c, FDSDF_KSLOT_ALLREDUCE, strm, [&] {
      g_nccl.groupStart();
      float* gbuf = acc_reduce ? c->gcall : d_grad;
      r1 = g_nccl.allReduce(gbuf, gbuf, (size_t)c->P, kNcclFloat32, kNcclSum, c->comm, strm);
      r2 = g_nccl.allReduce(d_loss, d_loss, 8, kNcclFloat64, kNcclSum, c->comm, strm);
      r3 = g_nccl.groupEnd();
      return cudaSuccess;
    });
    if (r1 || r2 || r3) return done(fail(c, FDSDF_E_NCCL, "ncclAllReduce failed"));
    if (acc_reduce) {
      e = launch_add_inplace(d_grad, c->gcall, c->P, strm);
      if (e != cudaSuccess) return done(cuda_fail(c, e, "add_kernel"));
    }
  }
  if (h_grad) {
    e = cudaMemcpyAsync(h_grad, d_grad, (size_t)c->P * sizeof(float), cudaMemcpyDeviceToHost, strm);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_loss, d_loss, 8 * sizeof(double), cudaMemcpyDeviceToHost, strm);
    if (e != cudaSuccess) return done(cuda_fail(c, e, "device -> host copy of the results"));
  }
  return done(FDSDF_OK);
}

extern "C" {

fdsdf_status fdsdf_step(fdsdf_ctx* c, const float* d_params, const float* d_x, int64_t n, const fdsdf_stencil* st,
                        const fdsdf_loss* ls, float* d_grad, double* d_loss, uint32_t flags, void* stream) {
  return step_impl(c, d_params, d_x, n, st, ls, d_grad, d_loss, flags, stream, nullptr, nullptr, nullptr);
}

fdsdf_status fdsdf_step_host(fdsdf_ctx* c, const float* d_params, const float* h_x, int64_t n, const fdsdf_stencil* st,
                             const fdsdf_loss* ls, float* h_grad, double* h_loss, uint32_t flags, void* stream) {
  if (!c) return FDSDF_E_INVALID;
  if (c->eval_only) return fail(c, FDSDF_E_INVALID, "context created EVAL_ONLY");
  if (!h_x || !h_grad || !h_loss) return fail(c, FDSDF_E_INVALID, "null pointer argument");
  return step_impl(c, d_params, c->xstage, n, st, ls, c->hgrad, c->hloss, flags, stream, h_x, h_grad, h_loss);
}

fdsdf_status fdsdf_sample(fdsdf_ctx* c, const float* d_pool, int64_t n_pool, int64_t n_pick, float box_half,
                          int64_t n_uniform, uint64_t seed, int64_t iteration, float* d_x_out, void* stream) {
  if (!c) return FDSDF_E_INVALID;
  if (n_pick < 0 || n_uniform < 0 || iteration < 0) return fail(c, FDSDF_E_INVALID, "negative count or iteration");
  if (n_pick > 0 && (!d_pool || n_pick > n_pool)) return fail(c, FDSDF_E_INVALID, "need n_pick <= n_pool and a pool");
  if (!(box_half > 0.f) || !std::isfinite(box_half)) return fail(c, FDSDF_E_INVALID, "box_half must be finite and > 0");
  if (n_pick + n_uniform == 0) return fail(c, FDSDF_E_EMPTY, "empty batch");
  if (!d_x_out) return fail(c, FDSDF_E_INVALID, "null output pointer");
  cudaStream_t strm = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != c->device) cudaSetDevice(c->device);
  const cudaError_t e = run_slot(c, FDSDF_KSLOT_SAMPLE, strm, [&] {
    return launch_sample(d_pool, n_pool, n_pick, box_half, n_uniform, seed, iteration, d_x_out, strm);
  });
  if (prev != c->device) cudaSetDevice(prev);
  return e == cudaSuccess ? FDSDF_OK : cuda_fail(c, e, "sample_kernel");
}

fdsdf_status fdsdf_adam(fdsdf_ctx* c, float* d_params, const float* d_grad, float* d_m, float* d_v, int64_t t,
                        float lr, float beta1, float beta2, float eps, void* stream) {
  if (!c || !d_params || !d_grad || !d_m || !d_v) return fail(c, FDSDF_E_INVALID, "null pointer argument");
  if (t < 1) return fail(c, FDSDF_E_INVALID, "Adam step t must be >= 1");
  if (!(lr > 0.f) || !std::isfinite(lr)) return fail(c, FDSDF_E_INVALID, "lr must be finite and > 0");
  if (!(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f))
    return fail(c, FDSDF_E_INVALID, "betas must lie in [0, 1)");
  if (!(eps >= 0.f) || !std::isfinite(eps)) return fail(c, FDSDF_E_INVALID, "eps must be finite and >= 0");
  cudaStream_t strm = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != c->device) cudaSetDevice(c->device);
  const cudaError_t e = run_slot(c, FDSDF_KSLOT_ADAM, strm, [&] {
    return launch_adam(d_params, d_grad, d_m, d_v, c->P, lr, beta1, beta2, eps, t, c->dflags, strm);
  });
  if (prev != c->device) cudaSetDevice(prev);
  return e == cudaSuccess ? FDSDF_OK : cuda_fail(c, e, "adam_kernel");
}

fdsdf_status fdsdf_comm_unique_id(uint8_t id[128]) {
  if (!id) return FDSDF_E_INVALID;
  std::string err;
  if (!nccl_load(&err)) return FDSDF_E_NCCL;
  NcclId u;
  if (g_nccl.getUniqueId(&u) != 0) return FDSDF_E_NCCL;
  memcpy(id, u.internal, 128);
  return FDSDF_OK;
}

fdsdf_status fdsdf_comm_init(fdsdf_ctx* c, const uint8_t id[128], int rank, int world) {
  if (!c || !id || world < 1 || rank < 0 || rank >= world) return FDSDF_E_INVALID;
  std::string err;
  if (!nccl_load(&err)) return fail(c, FDSDF_E_NCCL, err);
  NcclId u;
  memcpy(u.internal, id, 128);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  void* comm = nullptr;
  int r = ((CommInitRankFn)g_nccl.commInitRank)(&comm, world, u, rank);
  cudaSetDevice(prev);
  if (r != 0) return fail(c, FDSDF_E_NCCL, "ncclCommInitRank failed");
  if (c->comm && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
  c->comm = comm;
  c->rank = rank;
  c->world = world;
  return FDSDF_OK;
}

fdsdf_status fdsdf_allreduce(fdsdf_ctx* c, float* d_buf, int64_t count, void* stream) {
  if (!c || !d_buf || count < 0) return FDSDF_E_INVALID;
  if (!c->comm) return fail(c, FDSDF_E_UNSUPPORTED, "comm not initialised");
  int r = g_nccl.allReduce(d_buf, d_buf, (size_t)count, kNcclFloat32, kNcclSum, c->comm, (cudaStream_t)stream);
  return r == 0 ? FDSDF_OK : fail(c, FDSDF_E_NCCL, "ncclAllReduce failed");
}

fdsdf_status fdsdf_set_kernel_timing(fdsdf_ctx* c, int enable) {
  if (!c) return FDSDF_E_INVALID;
  c->timing = enable != 0;
  return FDSDF_OK;
}

fdsdf_status fdsdf_kernel_times(fdsdf_ctx* c, double* ms_total, int64_t* count, int nslots, int reset) {
  if (!c || nslots < 0 || (nslots > 0 && (!ms_total || !count))) return FDSDF_E_INVALID;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  cudaError_t err = cudaSuccess;
  for (auto& r : c->pending) {
    cudaError_t e = cudaEventSynchronize(r.b);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
    if (e == cudaSuccess) {
      c->tot_ms[r.slot] += ms;
      c->cnt[r.slot] += 1;
    } else {
      err = e;
    }
    c->spare.push_back(r.a);
    c->spare.push_back(r.b);
  }
  c->pending.clear();
  cudaSetDevice(prev);
  for (int i = 0; i < nslots && i < FDSDF_NUM_KSLOTS; ++i) {
    ms_total[i] = c->tot_ms[i];
    count[i] = c->cnt[i];
  }
  if (reset)
    for (int i = 0; i < FDSDF_NUM_KSLOTS; ++i) {
      c->tot_ms[i] = 0.0;
      c->cnt[i] = 0;
    }
  if (err != cudaSuccess) return cuda_fail(c, err, "kernel_times");
  return FDSDF_OK;
}

fdsdf_status fdsdf_get_device_flags(fdsdf_ctx* c, uint32_t* out) {
  if (!c || !out) return FDSDF_E_INVALID;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  unsigned v = 0;
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(&v, c->dflags, sizeof(unsigned), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(c->dflags, 0, sizeof(unsigned));
  cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(c, e, "get_device_flags");
  *out = v;
  return FDSDF_OK;
}

}  // extern "C"
