/* fdsdf_oracle.c -- the plain single-threaded fp64 C oracle of the FD curvature-regularised
 * neural-SDF training step (BASELINE.json north_star: "a plain single-threaded fp64 C++ CPU
 * implementation of the MLP, the stencils and the losses, sharing no code with the GPU path").
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs through oracle/c_oracle.py.  The product path
 * (paper_2511_08980_b200) never links, loads or calls it and shares no code with it.
 *
 * Plain C99, double precision, one thread, no blocking / fusion / reordering: every stencil
 * value is a separate full evaluation of f at the stencil point formed in fp64, exactly as
 * PAPER.md prints the stencils, and the gradient is the hand-derived reverse sweep of the
 * loss, one point at a time.  Citation keys: P:Lx = /root/reference/PAPER.md line x,
 * S:Lx = SPEC.md line x, SURVEY §8c Ox = the oracle step table of SURVEY.md.
 *
 *   O1  fp32 inputs / params / h are promoted exactly to double (the caller passes doubles
 *       holding fp32 values).
 *   O2  the MLP: hidden layers sin(omega (W a + b)) with omega = omega0_first
 *       on layer 0 and omega0_hidden after it, or exact softplus_beta log(1 + e^{beta z})/beta
 *       (no threshold); last layer linear; the skip layer's input is cat(a, x)/sqrt(2).
 *   O3  g = grad_x f(x0) by the reverse sweep.
 *   O4  degenerate mask m = [|g| >= eps_grad].
 *   O5  frame: n = g/|g|, Duff et al. branchless right-handed ONB (s = +1 when n_z >= 0,
 *       including -0), rotated by theta = 2 pi U, U = (mix64(seed + (gidx+1) gamma) >> 11) 2^-53
 *       (SplitMix64); u = cos t b1 + sin t b2, v = -sin t b1 + cos t b2.
 *       Masked centres: u = v = 0.  Frame and mask are stop-gradient.
 *   O6  the 9 stencil points x0, x0 +- h u, x0 +- h v, x0 + h(+-u +- v), formed in fp64.
 *   O7  f_uu = (f(+u) - 2 f0 + f(-u))/h^2, f_vv likewise, f_uv = (f(++) - f(+-) - f(-+) + f(--))/(4h^2)
 *       (as printed).
 *   O8  D = f_uu f_vv - f_uv^2; K = D/den, den = |g|^p, replaced by 1 on the
 *       surface-role rows under the "paper" policy; masked rows K = 0.
 *   O9  L_DM = (1/N_s) sum_surf |f|, L_DNM = (1/N_u) sum_unif exp(-alpha |f|), L_eik = (1/N) sum
 *       (|g| - 1)^2, L_fd = (1/N) sum m |Q| (or Q^2), Q = K (NCR) or D (NSH); total = w_dm L_DM +
 *       lambda_dnm L_DNM + lambda_eik L_eik + lambda_fd L_fd (Eq. (1); forms S:L278,
 *       S:L287), over the global counts.
 *   O10 the gradient of the total with respect to every parameter: seeds of the 9 stencil values
 *       through O7/O8/O9, and the seed r = dL/dg of the gradient path (eikonal and the live
 *       denominator); per point one reverse sweep, and at the centre the reverse sweep of the
 *       forward-mode tangent along r (d(r.g)/dtheta).  sgn(0) := 0.
 *
 * Analytic fields (pins of the stencil / frame / curvature code): instead of the
 * MLP, f can be a sphere s(|x - c| - r), a quadratic 1/2 x^T A x + b.x + c0, a z-axis cylinder
 * s(sqrt(x^2 + y^2) - r) or a z-axis torus sqrt((sqrt(x^2+y^2) - R)^2 + z^2) - r, with their
 * analytic gradients (eval only).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAXL 16

enum { OR_SOFTPLUS = 0, OR_SINE = 1 };
enum { OR_FIELD_MLP = 0, OR_FIELD_SPHERE = 1, OR_FIELD_QUADRATIC = 2, OR_FIELD_CYLINDER = 3, OR_FIELD_TORUS = 4 };
enum { OR_NCR = 0, OR_NSH = 1 };
enum { OR_DEN_PAPER = 0, OR_DEN_ONE = 1, OR_DEN_GRAD = 2 };
enum { OR_FD_ABS = 0, OR_FD_SQUARE = 1 };

typedef struct {
  int n_linear;             /* linear layers L                                   */
  int width[OR_MAXL + 1];   /* width[0] = 3 ... width[L] = 1                      */
  int act;                  /* OR_SOFTPLUS / OR_SINE                              */
  double beta, omega_first, omega_hidden;
  int skip_at;              /* -1 or the layer whose input is cat(a, x)/sqrt(2)   */
  int field;                /* OR_FIELD_*                                         */
  double fp[16];            /* analytic field parameters (see field_eval)         */
} or_spec;

typedef struct {
  int kind, denom, denom_pow, fd_form;
  double eps_grad, w_dm, lambda_dnm, alpha_dnm, lambda_eik, lambda_fd;
  double n_surface_global, n_uniform_global, n_global;
} or_loss;

/* ----------------------------------------------------------------------------- the MLP */

static int fan_in(const or_spec* s, int l) { return s->width[l] + (l == s->skip_at ? 3 : 0); }

long long or_num_params(const or_spec* s) {
  long long p = 0;
  for (int l = 0; l < s->n_linear; ++l) p += (long long)s->width[l + 1] * fan_in(s, l) + s->width[l + 1];
  return p;
}

static double omega_of(const or_spec* s, int l) { return l == 0 ? s->omega_first : s->omega_hidden; }

/* activation sigma of hidden layer l at pre-activation z (the raw W a + b), and its first two
 * derivatives with respect to z */
static double act_val(const or_spec* s, int l, double z) {
  if (s->act == OR_SINE) return sin(omega_of(s, l) * z);
  const double t = s->beta * z; /* log(1 + e^t)/beta without overflow, no threshold */
  return (t > 0 ? t + log1p(exp(-t)) : log1p(exp(t))) / s->beta;
}
static double act_d1(const or_spec* s, int l, double z) {
  if (s->act == OR_SINE) return omega_of(s, l) * cos(omega_of(s, l) * z);
  const double t = s->beta * z;
  return t >= 0 ? 1.0 / (1.0 + exp(-t)) : exp(t) / (1.0 + exp(t));
}
static double act_d2(const or_spec* s, int l, double z) {
  if (s->act == OR_SINE) {
    const double w = omega_of(s, l);
    return -w * w * sin(w * z);
  }
  const double t = s->beta * z;
  const double sg = t >= 0 ? 1.0 / (1.0 + exp(-t)) : exp(t) / (1.0 + exp(t));
  return s->beta * sg * (1.0 - sg);
}

/* per-point work buffers: the input of every layer and its pre-activation */
typedef struct {
  double* in[OR_MAXL];   /* input vector of layer l (length fan_in(l))        */
  double* z[OR_MAXL];    /* pre-activation of layer l (length width[l+1])     */
  double* tin[OR_MAXL];  /* tangent of the input (forward mode)               */
  double* tz[OR_MAXL];   /* tangent of the pre-activation                     */
  double* gin;           /* adjoint of a layer input                          */
  double* gz;            /* adjoint of a pre-activation                       */
  double* gtin;          /* adjoint of a layer-input tangent                  */
  double* gtz;           /* adjoint of a pre-activation tangent               */
  double* gnext;         /* scratch                                           */
  double* gtnext;
} work;

static int maxw(const or_spec* s) {
  int m = 3;
  for (int l = 0; l <= s->n_linear; ++l) m = s->width[l] + 3 > m ? s->width[l] + 3 : m;
  return m;
}

static int work_alloc(const or_spec* s, work* w) {
  const int m = maxw(s);
  memset(w, 0, sizeof(*w));
  for (int l = 0; l < s->n_linear; ++l) {
    w->in[l] = calloc((size_t)m, sizeof(double));
    w->z[l] = calloc((size_t)m, sizeof(double));
    w->tin[l] = calloc((size_t)m, sizeof(double));
    w->tz[l] = calloc((size_t)m, sizeof(double));
    if (!w->in[l] || !w->z[l] || !w->tin[l] || !w->tz[l]) return -1;
  }
  w->gin = calloc((size_t)m, sizeof(double));
  w->gz = calloc((size_t)m, sizeof(double));
  w->gtin = calloc((size_t)m, sizeof(double));
  w->gtz = calloc((size_t)m, sizeof(double));
  w->gnext = calloc((size_t)m, sizeof(double));
  w->gtnext = calloc((size_t)m, sizeof(double));
  return (w->gin && w->gz && w->gtin && w->gtz && w->gnext && w->gtnext) ? 0 : -1;
}

static void work_free(const or_spec* s, work* w) {
  for (int l = 0; l < s->n_linear; ++l) {
    free(w->in[l]);
    free(w->z[l]);
    free(w->tin[l]);
    free(w->tz[l]);
  }
  free(w->gin);
  free(w->gz);
  free(w->gtin);
  free(w->gtz);
  free(w->gnext);
  free(w->gtnext);
}

/* offsets of W_l and b_l in the flat parameter vector (layer-major, W row-major [out][in], then b) */
static void layer_offsets(const or_spec* s, long long* offW, long long* offb) {
  long long off = 0;
  for (int l = 0; l < s->n_linear; ++l) {
    offW[l] = off;
    off += (long long)s->width[l + 1] * fan_in(s, l);
    offb[l] = off;
    off += s->width[l + 1];
  }
}

/* f(x) of the MLP; stores every layer's input and pre-activation in w (O2).  With r != NULL
 * it also propagates the forward-mode tangent along r (d/de f(x + e r)) into w->tin / w->tz and
 * returns that directional derivative in *fdot. */
static double mlp_forward(const or_spec* s, const double* P, const long long* offW, const long long* offb,
                          const double x[3], const double* r, double* fdot, work* w) {
  const int L = s->n_linear;
  const double rs2 = 1.0 / sqrt(2.0);
  /* layer 0 input */
  for (int d = 0; d < 3; ++d) {
    w->in[0][d] = x[d];
    if (r) w->tin[0][d] = r[d];
  }
  if (s->skip_at == 0) { /* cat(x, x)/sqrt(2) -- legal but degenerate */
    for (int d = 0; d < 3; ++d) {
      w->in[0][3 + d] = x[d];
      if (r) w->tin[0][3 + d] = r[d];
    }
    for (int k = 0; k < 6; ++k) {
      w->in[0][k] *= rs2;
      if (r) w->tin[0][k] *= rs2;
    }
  }
  for (int l = 0; l < L; ++l) {
    const int M = s->width[l + 1], K = fan_in(s, l);
    const double* W = P + offW[l];
    const double* b = P + offb[l];
    for (int m = 0; m < M; ++m) {
      const double* Wm = W + (long long)m * K;
      double acc = b[m];
      for (int k = 0; k < K; ++k) acc += Wm[k] * w->in[l][k];
      w->z[l][m] = acc;
      if (r) {
        double tacc = 0.0;
        for (int k = 0; k < K; ++k) tacc += Wm[k] * w->tin[l][k];
        w->tz[l][m] = tacc;
      }
    }
    if (l == L - 1) {
      if (r) *fdot = w->tz[l][0];
      return w->z[l][0];
    }
    /* next layer's input: sigma(z) (and sigma'(z) zdot), with x appended at the skip layer */
    double* nin = w->in[l + 1];
    double* ntin = w->tin[l + 1];
    for (int m = 0; m < M; ++m) {
      nin[m] = act_val(s, l, w->z[l][m]);
      if (r) ntin[m] = act_d1(s, l, w->z[l][m]) * w->tz[l][m];
    }
    if (l + 1 == s->skip_at) {
      for (int d = 0; d < 3; ++d) {
        nin[M + d] = x[d];
        if (r) ntin[M + d] = r[d];
      }
      for (int k = 0; k < M + 3; ++k) {
        nin[k] *= rs2;
        if (r) ntin[k] *= rs2;
      }
    }
  }
  return 0.0; /* unreachable: L >= 1 */
}

/* Reverse sweep after mlp_forward at the same point: seeds fbar = dL/df and (with the tangent
 * of mlp_forward) tbar = dL/d(fdot).  Accumulates dL/dtheta into G (if not NULL) and, if gx is
 * not NULL, writes dL/dx restricted to the value path (tbar must be 0 then: used for grad f).
 *   output layer: zbar = fbar, zdotbar = tbar
 *   hidden layer l, a = sigma(z), adot = sigma'(z) zdot:
 *     zbar = abar sigma'(z) + adotbar sigma''(z) zdot,  zdotbar = adotbar sigma'(z)
 *   dW_l += zbar in^T + zdotbar indot^T,  db_l += zbar,  inbar = W^T zbar,  indotbar = W^T zdotbar */
static void mlp_reverse(const or_spec* s, const double* P, const long long* offW, const long long* offb,
                        double fbar, double tbar, int with_tangent, double* G, double gx[3], work* w) {
  const int L = s->n_linear;
  const double rs2 = 1.0 / sqrt(2.0);
  if (gx) gx[0] = gx[1] = gx[2] = 0.0;
  /* adjoints of the output layer's pre-activation */
  w->gz[0] = fbar;
  w->gtz[0] = with_tangent ? tbar : 0.0;
  for (int l = L - 1; l >= 0; --l) {
    const int M = s->width[l + 1], K = fan_in(s, l);
    const double* W = P + offW[l];
    if (G) {
      double* dW = G + offW[l];
      double* db = G + offb[l];
      for (int m = 0; m < M; ++m) {
        const double zb = w->gz[m], tzb = w->gtz[m];
        db[m] += zb;
        double* dWm = dW + (long long)m * K;
        for (int k = 0; k < K; ++k) dWm[k] += zb * w->in[l][k];
        if (with_tangent)
          for (int k = 0; k < K; ++k) dWm[k] += tzb * w->tin[l][k];
      }
    }
    /* adjoint of this layer's input: inbar[k] = sum_m W[m][k] zbar[m] (summed in m order) */
    for (int k = 0; k < K; ++k) w->gnext[k] = w->gtnext[k] = 0.0;
    for (int m = 0; m < M; ++m) {
      const double* Wm = W + (long long)m * K;
      const double zb = w->gz[m], tzb = w->gtz[m];
      for (int k = 0; k < K; ++k) w->gnext[k] += Wm[k] * zb;
      if (with_tangent)
        for (int k = 0; k < K; ++k) w->gtnext[k] += Wm[k] * tzb;
    }
    if (l == 0) {
      if (gx) {
        for (int d = 0; d < 3; ++d) gx[d] += w->gnext[d];
        if (s->skip_at == 0)
          for (int d = 0; d < 3; ++d) gx[d] = (gx[d] + w->gnext[3 + d]) * rs2;
      }
      break;
    }
    /* through the skip concatenation into the previous layer's activations (and x) */
    const int Mp = s->width[l];
    if (l == s->skip_at) {
      for (int k = 0; k < Mp + 3; ++k) {
        w->gnext[k] *= rs2;
        w->gtnext[k] *= rs2;
      }
      if (gx)
        for (int d = 0; d < 3; ++d) gx[d] += w->gnext[Mp + d];
    }
    /* through the activation of layer l-1 */
    for (int m = 0; m < Mp; ++m) {
      const double z = w->z[l - 1][m];
      const double ab = w->gnext[m];
      if (with_tangent) {
        const double tb = w->gtnext[m];
        w->gz[m] = ab * act_d1(s, l - 1, z) + tb * act_d2(s, l - 1, z) * w->tz[l - 1][m];
        w->gtz[m] = tb * act_d1(s, l - 1, z);
      } else {
        w->gz[m] = ab * act_d1(s, l - 1, z);
        w->gtz[m] = 0.0;
      }
    }
  }
}

/* ----------------------------------------------------------------------------- analytic fields */

static double field_eval(const or_spec* s, const double x[3], double g[3]) {
  const double* q = s->fp;
  switch (s->field) {
    case OR_FIELD_SPHERE: { /* q = (cx, cy, cz, r, scale) */
      const double d0 = x[0] - q[0], d1 = x[1] - q[1], d2 = x[2] - q[2];
      const double rr = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
      if (g) {
        g[0] = q[4] * d0 / rr;
        g[1] = q[4] * d1 / rr;
        g[2] = q[4] * d2 / rr;
      }
      return q[4] * (rr - q[3]);
    }
    case OR_FIELD_QUADRATIC: { /* q = A (row-major 3x3, symmetric), b (3), c */
      double f = q[12];
      for (int i = 0; i < 3; ++i) {
        double Ax = 0.0;
        for (int j = 0; j < 3; ++j) Ax += q[3 * i + j] * x[j];
        f += 0.5 * x[i] * Ax + q[9 + i] * x[i];
        if (g) g[i] = Ax + q[9 + i];
      }
      return f;
    }
    case OR_FIELD_CYLINDER: { /* q = (r, scale): z axis */
      const double rho = sqrt(x[0] * x[0] + x[1] * x[1]);
      if (g) {
        g[0] = q[1] * x[0] / rho;
        g[1] = q[1] * x[1] / rho;
        g[2] = 0.0;
      }
      return q[1] * (rho - q[0]);
    }
    case OR_FIELD_TORUS: { /* q = (R, r): z axis */
      const double rho = sqrt(x[0] * x[0] + x[1] * x[1]);
      const double a = rho - q[0];
      const double t = sqrt(a * a + x[2] * x[2]);
      if (g) {
        g[0] = a / t * x[0] / rho;
        g[1] = a / t * x[1] / rho;
        g[2] = x[2] / t;
      }
      return t - q[1];
    }
    default:
      return NAN;
  }
}

/* ----------------------------------------------------------------------------- frames (O5) */

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double or_frame_theta(uint64_t seed, int64_t gidx) {
  const uint64_t k = mix64(seed + ((uint64_t)gidx + 1ull) * 0x9E3779B97F4A7C15ull) >> 11;
  return 6.283185307179586 * ((double)k * 0x1.0p-53);
}

/* right-handed (u, v) with u x v = n = g/|g| */
void or_frame(const double g[3], uint64_t seed, int64_t gidx, double u[3], double v[3]) {
  const double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
  const double n0 = g[0] / gn, n1 = g[1] / gn, n2 = g[2] / gn;
  const double sg = n2 >= 0.0 ? 1.0 : -1.0; /* -0.0 >= 0 is true: s = +1 */
  const double a = -1.0 / (sg + n2);
  const double b = n0 * n1 * a;
  const double b1[3] = {1.0 + sg * n0 * n0 * a, sg * b, -sg * n0};
  const double b2[3] = {b, sg + n1 * n1 * a, -n1};
  const double th = or_frame_theta(seed, gidx);
  const double c = cos(th), sn = sin(th);
  for (int d = 0; d < 3; ++d) {
    u[d] = c * b1[d] + sn * b2[d];
    v[d] = -sn * b1[d] + c * b2[d];
  }
}

/* ----------------------------------------------------------------------------- the step */

static double sgn(double x) { return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); }

/* per-centre outputs: f, g[3], fuu, fuv, fvv, D, K, u[3], v[3], mask -> 16 doubles per centre */
#define OR_NOUT 16

/* One FD-regularised step (or eval: ls == NULL or G == NULL) over centres x [n][3] (doubles
 * holding fp32 values, O1).  is_surface [n] (1 = surface role).  frames_in [n][6] (u, v) or NULL
 * (random frames from frame_seed and gidx [n]).  P = params (doubles holding fp32 values) for
 * the MLP field.  out [n][OR_NOUT] (may be NULL), loss [8] = (dm, dnm, eik, fd, total,
 * n_degenerate, 0, 0) accumulated over this call's centres with the global counts of ls,
 * G [P] += the gradient of this call's share of the total (may be NULL).  h > 0.
 * Returns 0, or -1 on an allocation failure / invalid argument. */
int or_step(const or_spec* s, const double* P, const double* x, int64_t n, const unsigned char* is_surface,
            double h, const or_loss* ls, uint64_t frame_seed, const int64_t* gidx, const double* frames_in,
            double* out, double* loss, double* G) {
  if (!s || !x || n < 0 || !(h > 0) || s->n_linear < 1 || s->n_linear > OR_MAXL) return -1;
  const int mlp = s->field == OR_FIELD_MLP;
  if (mlp && !P) return -1;
  if (!mlp) G = NULL;
  work w;
  if (work_alloc(s, &w) != 0) {
    work_free(s, &w);
    return -1;
  }
  long long offW[OR_MAXL], offb[OR_MAXL];
  layer_offsets(s, offW, offb);
  double lsum[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  /* stencil offsets in units of h: (+u), (-u), (+v), (-v), (+u+v), (+u-v), (-u+v), (-u-v) */
  static const double cu[8] = {1, -1, 0, 0, 1, 1, -1, -1};
  static const double cv[8] = {0, 0, 1, -1, 1, -1, 1, -1};
  for (int64_t i = 0; i < n; ++i) {
    const double* x0 = x + 3 * i;
    /* O2/O3: f(x0) and g = grad f(x0) */
    double f0, g[3];
    if (mlp) {
      f0 = mlp_forward(s, P, offW, offb, x0, NULL, NULL, &w);
      mlp_reverse(s, P, offW, offb, 1.0, 0.0, 0, NULL, g, &w);
    } else {
      f0 = field_eval(s, x0, g);
    }
    const double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    /* O4, O5 */
    const double eps = ls ? ls->eps_grad : 1e-6;
    const int m = gn >= eps;
    double u[3] = {0, 0, 0}, v[3] = {0, 0, 0};
    if (frames_in) {
      for (int d = 0; d < 3; ++d) {
        u[d] = frames_in[6 * i + d];
        v[d] = frames_in[6 * i + 3 + d];
      }
    } else if (m) {
      or_frame(g, frame_seed, gidx ? gidx[i] : i, u, v);
    }
    /* O6/O7: 8 more evaluations at the fp64 stencil points */
    double fk[8];
    for (int k = 0; k < 8; ++k) {
      double xk[3];
      for (int d = 0; d < 3; ++d) xk[d] = x0[d] + h * cu[k] * u[d] + h * cv[k] * v[d];
      fk[k] = mlp ? mlp_forward(s, P, offW, offb, xk, NULL, NULL, &w) : field_eval(s, xk, NULL);
    }
    const double fuu = (fk[0] - 2.0 * f0 + fk[1]) / (h * h);
    const double fvv = (fk[2] - 2.0 * f0 + fk[3]) / (h * h);
    const double fuv = (fk[4] - fk[5] - fk[6] + fk[7]) / (4.0 * h * h);
    /* O8 */
    const double D = fuu * fvv - fuv * fuv;
    const int surf = is_surface ? is_surface[i] != 0 : 0;
    const int pw = ls ? ls->denom_pow : 4;
    const int dmode = ls ? ls->denom : OR_DEN_PAPER;
    int den_is_grad = 0;
    double den = 1.0;
    if (m && (dmode == OR_DEN_GRAD || (dmode == OR_DEN_PAPER && !surf))) {
      den = pow(gn, (double)pw);
      den_is_grad = 1;
    }
    const double K = m ? D / den : 0.0;
    if (out) {
      double* o = out + (int64_t)OR_NOUT * i;
      o[0] = f0;
      o[1] = g[0];
      o[2] = g[1];
      o[3] = g[2];
      o[4] = fuu;
      o[5] = fuv;
      o[6] = fvv;
      o[7] = D;
      o[8] = K;
      for (int d = 0; d < 3; ++d) {
        o[9 + d] = u[d];
        o[12 + d] = v[d];
      }
      o[15] = m;
    }
    if (!ls) continue;
    /* O9 */
    const double Q = ls->kind == OR_NCR ? K : D;
    const double Qm = m ? Q : 0.0;
    double l_dm = 0.0, l_dnm = 0.0;
    if (surf && ls->n_surface_global > 0) l_dm = fabs(f0) / ls->n_surface_global;
    if (!surf && ls->n_uniform_global > 0) l_dnm = exp(-ls->alpha_dnm * fabs(f0)) / ls->n_uniform_global;
    const double l_eik = (gn - 1.0) * (gn - 1.0) / ls->n_global;
    const double l_fd = (ls->fd_form == OR_FD_ABS ? fabs(Qm) : Qm * Qm) / ls->n_global;
    lsum[0] += l_dm;
    lsum[1] += l_dnm;
    lsum[2] += l_eik;
    lsum[3] += l_fd;
    lsum[5] += m ? 0.0 : 1.0;
    if (!G) continue;
    /* O10: seeds.  gQ = dL/dQ; dQ/dD = 1/den (NCR) or 1 (NSH) */
    const double gQ = m ? ls->lambda_fd * (ls->fd_form == OR_FD_ABS ? sgn(Q) : 2.0 * Q) / ls->n_global : 0.0;
    const double dQdD = ls->kind == OR_NCR ? 1.0 / den : 1.0;
    const double gD = gQ * dQdD;
    /* through O7: dD/dfuu = fvv, dD/dfvv = fuu, dD/dfuv = -2 fuv */
    double fb[8];
    fb[0] = fb[1] = gD * fvv / (h * h);
    fb[2] = fb[3] = gD * fuu / (h * h);
    fb[4] = fb[7] = gD * (-2.0 * fuv) / (4.0 * h * h);
    fb[5] = fb[6] = -fb[4];
    double fb0 = -2.0 * (fb[0] + fb[2]);
    if (surf && ls->n_surface_global > 0) fb0 += ls->w_dm * sgn(f0) / ls->n_surface_global;
    if (!surf && ls->n_uniform_global > 0)
      fb0 += ls->lambda_dnm * (-ls->alpha_dnm * sgn(f0) * exp(-ls->alpha_dnm * fabs(f0))) / ls->n_uniform_global;
    /* r = dL/dg: eikonal, plus the live denominator |g|^p of K (NCR): dK/dg = -p K g/|g|^2 */
    double r[3] = {0, 0, 0};
    for (int d = 0; d < 3; ++d) {
      if (gn > 0) r[d] += ls->lambda_eik * 2.0 * (gn - 1.0) * g[d] / gn / ls->n_global;
      if (m && ls->kind == OR_NCR && den_is_grad) r[d] += gQ * (-(double)pw * K / (gn * gn)) * g[d];
    }
    /* the 8 neighbours: plain reverse sweeps */
    for (int k = 0; k < 8; ++k) {
      if (fb[k] == 0.0) continue;
      double xk[3];
      for (int d = 0; d < 3; ++d) xk[d] = x0[d] + h * cu[k] * u[d] + h * cv[k] * v[d];
      mlp_forward(s, P, offW, offb, xk, NULL, NULL, &w);
      mlp_reverse(s, P, offW, offb, fb[k], 0.0, 0, G, NULL, &w);
    }
    /* the centre: value seed fb0 and the gradient path d(r . g)/dtheta = d(fdot along r)/dtheta */
    double fdot = 0.0;
    mlp_forward(s, P, offW, offb, x0, r, &fdot, &w);
    mlp_reverse(s, P, offW, offb, fb0, 1.0, 1, G, NULL, &w);
  }
  if (loss && ls) {
    for (int q = 0; q < 4; ++q) loss[q] += lsum[q];
    loss[4] += ls->w_dm * lsum[0] + ls->lambda_dnm * lsum[1] + ls->lambda_eik * lsum[2] + ls->lambda_fd * lsum[3];
    loss[5] += lsum[5];
  }
  work_free(s, &w);
  return 0;
}

/* f and the 19-point world-axis FD Hessian: the P:L83-91 formulas with
 * (u, v) = (e_i, e_j).  H [n][6] = (H_xx, H_xy, H_xz, H_yy, H_yz, H_zz). */
int or_hessian(const or_spec* s, const double* P, const double* x, int64_t n, double h, double* f, double* H) {
  if (!s || !x || n < 0 || !(h > 0)) return -1;
  const int mlp = s->field == OR_FIELD_MLP;
  work w;
  if (work_alloc(s, &w) != 0) {
    work_free(s, &w);
    return -1;
  }
  long long offW[OR_MAXL], offb[OR_MAXL];
  layer_offsets(s, offW, offb);
  for (int64_t i = 0; i < n; ++i) {
    const double* x0 = x + 3 * i;
#define OR_F(pt) (mlp ? mlp_forward(s, P, offW, offb, (pt), NULL, NULL, &w) : field_eval(s, (pt), NULL))
    const double f0 = OR_F(x0);
    if (f) f[i] = f0;
    double Hm[3][3];
    for (int a = 0; a < 3; ++a) {
      double xp[3] = {x0[0], x0[1], x0[2]}, xm[3] = {x0[0], x0[1], x0[2]};
      xp[a] += h;
      xm[a] -= h;
      Hm[a][a] = (OR_F(xp) - 2.0 * f0 + OR_F(xm)) / (h * h);
      for (int b = a + 1; b < 3; ++b) {
        double pp[3] = {x0[0], x0[1], x0[2]}, pm[3] = {x0[0], x0[1], x0[2]};
        double mp[3] = {x0[0], x0[1], x0[2]}, mm[3] = {x0[0], x0[1], x0[2]};
        pp[a] += h, pp[b] += h;
        pm[a] += h, pm[b] -= h;
        mp[a] -= h, mp[b] += h;
        mm[a] -= h, mm[b] -= h;
        Hm[a][b] = (OR_F(pp) - OR_F(pm) - OR_F(mp) + OR_F(mm)) / (4.0 * h * h);
      }
    }
#undef OR_F
    double* o = H + 6 * i;
    o[0] = Hm[0][0];
    o[1] = Hm[0][1];
    o[2] = Hm[0][2];
    o[3] = Hm[1][1];
    o[4] = Hm[1][2];
    o[5] = Hm[2][2];
  }
  work_free(s, &w);
  return 0;
}
