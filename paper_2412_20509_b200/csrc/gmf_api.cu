// Level-2 C ABI: the aSGD fit engine handle (create / reset / step / run /
// status), replacing the step loop of gmfkit optim.fit_asgd (optim.py:383-489).
#include <math.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <vector>

#include "gmf_engine.cuh"
#include <cstdio>
#include <cstdlib>

namespace gmf {
int launch_grad(const Params& P, int dtype, int NK, cudaStream_t st, long long xb, long long xs,
                double xalpha);
int prepare_grad(const Params& P, int dtype, int NK, int fit_extra_smem, int* fit_blocks_per_sm);
int tc_eligible(int dtype, int has_w, int Kr, int Kc, int KA, int holes);
int64_t colimg_bytes_total(int NK, int CT, int tcm);
int launch_fit(const Params& P, int dtype, int NK, int grid, long long n_steps, cudaStream_t st);
int launch_colrec(const Params& P, int dtype, cudaStream_t st, long long xs);
int launch_eval_pack(const Params& P, int4* out, cudaStream_t st);
int launch_cache_fill(const Params& P, int dtype, cudaStream_t st);
int launch_tile_index(const Params& P, int32_t* tidx, unsigned int* unsorted, cudaStream_t st);
int launch_tcsr(const Params& P, const int32_t* tidx, int32_t* lens, int64_t* tptr, int32_t* tent,
                unsigned int* too_big, cudaStream_t st);
int tile_cols(int dtype, int NK);
int grad_bucket(int KA);
int grad_bucket_gen(int KA);
int blocknorm_segments(int64_t nstar_max);
int64_t rimg_bytes_of(int NK);
int64_t grad_smem_bytes(const Params& P, int dtype, int NK);
int launch_obj(const Params& P, int dtype, cudaStream_t st);
int launch_apply(const Params& P, int dtype, const void* gathered, cudaStream_t st);
int launch_blocknorm(const Params& P, int dtype, cudaStream_t st);
int launch_gradout(const Params& P, int dtype, long long blk, long long sidx, int64_t nI,
                   int64_t nJ, void* g_row, void* h_row, void* g_col, void* h_col,
                   double* nb_sums, cudaStream_t st);
int launch_objfull(const Params& P, int dtype, double alpha, int with_const, double* part,
                   unsigned int* ticket, double* out, cudaStream_t st);
int launch_entries(const Params& P, int dtype, double alpha, const int64_t* rows,
                   const int32_t* cols, const double* y, int64_t n, double ybar, double* mu_out,
                   double* part, unsigned int* ticket, double* out, cudaStream_t st);
}  // namespace gmf

using namespace gmf;

struct gmf_handle {
  gmf_desc desc;
  gmf_config cfg;
  gmf_buffers bufs;
  Params P;
  int NK;
  int tsz;
  void* ws = nullptr;
  double* full_part = nullptr;
  unsigned int* full_ticket = nullptr;
  Ctrl* host_ctrl = nullptr;   // pinned
  cudaStream_t internal = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  std::map<int64_t, cudaGraphExec_t> graphs;
  int fit_grid = 0;             // co-resident CTAs of the persistent kernel
  int fit_rs = 0;               // its row splits (fit_grid / CT)
  void* prof_buf = nullptr;
  void* tcsr_buf = nullptr;     // K1 v2 tile-CSR (tptr | tent)
  std::vector<int64_t> rbp_host, cbp_host;
  bool reset_done = false;
  int64_t launches = 0;         // kernels this handle launched (gmf_launch_count)
  bool residency_checked = false;
  unsigned int* host_abort = nullptr;   // pinned: abort flag of the software grid barrier
  unsigned long long* ready_vals = nullptr;   // pinned: 0..max_steps, sources of gmf_stream_signal
  int64_t n_ready_vals = 0;
};

namespace {

int64_t align256(int64_t v) { return (v + 255) & ~int64_t(255); }

int validate(const gmf_desc* d, const gmf_config* c, const gmf_buffers* b) {
  if (!d || !c || !b) { set_error("null descriptor"); return GMF_ERR_CONFIG; }
  if (d->m < 1 || d->n < 0) { set_error("bad shape n=%lld m=%lld", (long long)d->n, (long long)d->m); return GMF_ERR_CONFIG; }
  if (d->p < 0 || d->q < 0 || d->d < 0) { set_error("negative p/q/d"); return GMF_ERR_CONFIG; }
  if (d->dtype != GMF_F32 && d->dtype != GMF_F64) { set_error("unknown dtype %d", d->dtype); return GMF_ERR_CONFIG; }
  if (d->family < GMF_GAUSSIAN || d->family > GMF_NEG_BINOMIAL) { set_error("unknown family code %d", d->family); return GMF_ERR_DOMAIN; }
  if (d->link < GMF_IDENTITY || d->link > GMF_INVERSE_SQUARED) { set_error("unknown link code %d", d->link); return GMF_ERR_DOMAIN; }
  const bool fused = d->link == GMF_LOG && (d->family == GMF_POISSON || d->family == GMF_NEG_BINOMIAL);
  const bool real = (d->flags & GMF_DESC_REAL_RESPONSE) != 0;
  const bool eval_only = (d->flags & GMF_DESC_EVAL_ONLY) != 0;
  if (!fused && !real && !eval_only) {
    set_error("family %d with link %d runs in general mode: pass the response as y_work with "
              "GMF_DESC_REAL_RESPONSE", d->family, d->link);
    return GMF_ERR_UNSUPPORTED;
  }
  if (c->est_phi && !real) {
    set_error("the Pearson dispersion update runs in general mode (GMF_DESC_REAL_RESPONSE)");
    return GMF_ERR_UNSUPPORTED;
  }
  if ((d->flags & GMF_DESC_REAL_HOLES) && !real) {
    set_error("GMF_DESC_REAL_HOLES needs GMF_DESC_REAL_RESPONSE");
    return GMF_ERR_CONFIG;
  }
  if (real) {
    if (d->y_format != GMF_Y_DENSE_I32 || (!b->y_work && d->n > 0)) {
      set_error("general mode needs a dense real-valued response in y_work");
      return GMF_ERR_CONFIG;
    }
    if (c->est_phi && !(c->inv_resid_dof > 0)) {
      set_error("model is over-parameterized: nonpositive residual dof");
      return GMF_ERR_CONFIG;
    }
  } else if (d->y_format == GMF_Y_DENSE_I32) {
    if (!b->y_dense && d->n > 0) { set_error("dense Y pointer is NULL"); return GMF_ERR_CONFIG; }
  } else if (d->y_format == GMF_Y_CSR_I32 || d->y_format == GMF_Y_CSR_PACK32) {
    if (!b->csr_ptr) { set_error("CSR row pointer is NULL"); return GMF_ERR_CONFIG; }
    if (d->y_format == GMF_Y_CSR_PACK32 && d->m > 65536) { set_error("packed CSR needs m <= 65536"); return GMF_ERR_CONFIG; }
  } else { set_error("unknown y_format %d", d->y_format); return GMF_ERR_CONFIG; }
  if (d->world_size < 1 || d->rank < 0 || d->rank >= d->world_size) { set_error("bad rank/world"); return GMF_ERR_CONFIG; }
  if (b->n_row_blocks < 1 || b->n_col_blocks < 1 || b->max_steps < 0) { set_error("empty schedule"); return GMF_ERR_CONFIG; }
  if (c->smooth_a1 <= 0 || c->smooth_a1 > 1 || c->smooth_a2 <= 0 || c->smooth_a2 > 1) { set_error("smoothing out of (0,1]"); return GMF_ERR_CONFIG; }
  if (c->tol <= 0 || c->damping < 0 || c->phi <= 0) { set_error("need tol > 0, damping >= 0, phi > 0"); return GMF_ERR_CONFIG; }
  if (c->snapshot_stride < 1) { set_error("snapshot_stride < 1"); return GMF_ERR_CONFIG; }
  if (c->k1_impl < GMF_K1_AUTO || c->k1_impl > GMF_K1_TENSOR) { set_error("unknown k1_impl %d", c->k1_impl); return GMF_ERR_CONFIG; }
  return GMF_OK;
}

// zero-step launch of the tensor-core fit kernel: its first grid barrier has
// a short timeout; if some CTA is not resident the kernel aborts and the
// grid shrinks to one CTA per SM (always resident)
int residency_probe(gmf_handle* h, cudaStream_t st) {
  Params P = h->P;
  P.RS = h->fit_rs;
  int rc = launch_fit(P, h->desc.dtype, h->NK, h->fit_grid, 0, st);
  if (rc) return rc;
  h->launches += 1;
  GMF_CUDA(cudaMemcpyAsync(h->host_abort, P.gbar + 2, 4, cudaMemcpyDeviceToHost, st));
  GMF_CUDA(cudaStreamSynchronize(st));
  if (*h->host_abort) {
    int n_sm = kSMs;
    GMF_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, h->desc.device));
    h->fit_grid = (n_sm / P.CT) * P.CT;
    h->fit_rs = h->fit_grid / P.CT;
    h->P.ep_cap = 0;   // sized for the larger grid
    if (getenv("GMF_VERBOSE"))
      fprintf(stderr, "[gmf] fit kernel CTAs not co-resident; %d CTAs (one per SM)\n", h->fit_grid);
  }
  h->residency_checked = true;
  return GMF_OK;
}

}  // namespace

extern "C" {

int gmf_create(const gmf_desc* desc, const gmf_config* cfg, const gmf_buffers* bufs,
               gmf_handle** out) {
  if (!out) { set_error("null out"); return GMF_ERR_CONFIG; }
  *out = nullptr;
  int rc = validate(desc, cfg, bufs);
  if (rc) return rc;
  GMF_CUDA(cudaSetDevice(desc->device));
  gmf_handle* h = new gmf_handle();
  h->desc = *desc;
  h->cfg = *cfg;
  h->bufs = *bufs;
  const int p = desc->p, q = desc->q, d = desc->d;
  const int Kr = q + d, Kc = p + d, KA = p + q + d;
  const bool gen_mode = (desc->flags & GMF_DESC_REAL_RESPONSE) != 0;
  h->NK = gen_mode ? grad_bucket_gen(KA) : grad_bucket(KA);
  if (h->NK < 0) {
    set_error("p+q+d = %d exceeds the fused kernel's %d-feature limit", KA, gen_mode ? 32 : 64);
    delete h;
    return GMF_ERR_UNSUPPORTED;
  }
  h->tsz = desc->dtype == GMF_F64 ? 8 : 4;
  const int64_t R = bufs->n_row_blocks, S = bufs->n_col_blocks;
  h->rbp_host.resize(R + 1);
  h->cbp_host.resize(S + 1);
  GMF_CUDA(cudaMemcpy(h->rbp_host.data(), bufs->row_block_ptr, (R + 1) * 8, cudaMemcpyDeviceToHost));
  GMF_CUDA(cudaMemcpy(h->cbp_host.data(), bufs->col_block_ptr, (S + 1) * 8, cudaMemcpyDeviceToHost));
  int64_t nstar_max = 1, jmax = 1;
  for (int64_t r = 0; r < R; ++r) {
    const int64_t sz = h->rbp_host[r + 1] - h->rbp_host[r];
    if (sz < 0) { set_error("row_block_ptr not monotone"); delete h; return GMF_ERR_CONFIG; }
    nstar_max = sz > nstar_max ? sz : nstar_max;
  }
  if (h->rbp_host[R] != desc->n) { set_error("row blocks cover %lld rows, n = %lld", (long long)h->rbp_host[R], (long long)desc->n); delete h; return GMF_ERR_CONFIG; }
  for (int64_t s = 0; s < S; ++s) {
    const int64_t sz = h->cbp_host[s + 1] - h->cbp_host[s];
    if (sz < 1) { set_error("empty column block"); delete h; return GMF_ERR_CONFIG; }
    jmax = sz > jmax ? sz : jmax;
  }
  int col_identity = 0;
  if (S == 1 && h->cbp_host[1] == desc->m) {
    std::vector<int32_t> ci(desc->m);
    GMF_CUDA(cudaMemcpy(ci.data(), bufs->col_idx, desc->m * 4, cudaMemcpyDeviceToHost));
    col_identity = 1;
    for (int64_t j = 0; j < desc->m; ++j)
      if (ci[j] != (int32_t)j) { col_identity = 0; break; }
  }
  if (!col_identity && (!bufs->col_idx || !bufs->col_pos || !bufs->col_block_of)) {
    set_error("column block maps are NULL"); delete h; return GMF_ERR_CONFIG;
  }

  Params& P = h->P;
  memset(&P, 0, sizeof(P));
  P.n = desc->n; P.m = desc->m; P.p = p; P.q = q; P.d = d; P.KA = KA; P.Kr = Kr; P.Kc = Kc;
  P.fam = desc->family; P.yfmt = desc->y_format; P.has_w = desc->has_weights && bufs->weights;
  P.has_off = desc->has_offset && bufs->offset;
  P.y = bufs->y_dense; P.rp = bufs->csr_ptr; P.ci = bufs->csr_col; P.cv = bufs->csr_val;
  P.w = bufs->weights; P.x = bufs->x; P.z = bufs->z; P.off = bufs->offset;
  P.th_row = bufs->theta_row; P.th_col = bufs->theta_col;
  P.gb_row = bufs->gbar_row; P.hb_row = bufs->hbar_row; P.gb_col = bufs->gbar_col; P.hb_col = bufs->hbar_col;
  P.sn_row = bufs->snap_row; P.sn_col = bufs->snap_col;
  P.rbp = bufs->row_block_ptr; P.rbscale = bufs->row_block_scale; P.R = R;
  P.cidx = bufs->col_idx; P.cbp = bufs->col_block_ptr; P.cpos = bufs->col_pos; P.cbof = bufs->col_block_of;
  P.S = S; P.col_identity = col_identity;
  P.bseq = bufs->block_seq; P.max_steps = bufs->max_steps;
  P.erow = bufs->eval_row; P.ecol = bufs->eval_col; P.E = bufs->n_eval;
  P.a1 = cfg->smooth_a1; P.a2 = cfg->smooth_a2; P.damp = cfg->damping; P.tol = cfg->tol;
  P.lam_b = cfg->lam_b; P.lam_g = cfg->lam_gamma; P.lam_u = cfg->lam_u; P.lam_v = cfg->lam_v;
  P.nbfloor = cfg->nb_floor; P.nbceil = cfg->nb_ceiling; P.escale = cfg->eval_scale; P.phi = cfg->phi;
  P.est_alpha = cfg->est_alpha && desc->family == GMF_NEG_BINOMIAL;
  P.snap_stride = cfg->snapshot_stride; P.world = desc->world_size;
  // K1 implementation: tensor cores when eligible unless CUDA cores requested
  if (desc->y_format != GMF_Y_DENSE_I32 && desc->n > 0)
    GMF_CUDA(cudaMemcpy(&P.nnz, bufs->csr_ptr + desc->n, 8, cudaMemcpyDeviceToHost));
  // the tensor-core K1 stages rows with 16-byte copies: 16-byte aligned bases
  auto al16 = [](const void* q) { return ((uintptr_t)q & 15) == 0; };
  const bool aligned = al16(bufs->theta_row) && (p == 0 || al16(bufs->x)) &&
                       (!P.has_off || al16(bufs->offset)) &&
                       (desc->y_format == GMF_Y_DENSE_I32 || al16(bufs->csr_col)) &&
                       (desc->y_format != GMF_Y_CSR_I32 || al16(bufs->csr_val));
  P.gen = (desc->flags & GMF_DESC_REAL_RESPONSE) ? 1 : 0;
  P.link = desc->link;
  P.est_phi = P.gen && cfg->est_phi;
  P.inv_dof = cfg->inv_resid_dof;
  P.holes = bufs->y_work != nullptr && (!P.gen || (desc->flags & GMF_DESC_REAL_HOLES));
  P.y_work = bufs->y_work;
  P.nafill = cfg->nafill_every > 0 ? cfg->nafill_every : 1;
  if (P.holes && desc->y_format != GMF_Y_DENSE_I32) {
    set_error("unobserved entries need a dense response (y_work)");
    delete h;
    return GMF_ERR_CONFIG;
  }
  const int tc_ok = tc_eligible(desc->dtype, P.has_w, Kr, Kc, KA, P.holes) && aligned && !P.gen;
  if (cfg->k1_impl == GMF_K1_TENSOR && !tc_ok) {
    set_error("k1_impl=tensor needs fp32, no prior weights, no unobserved entries, q+d <= 16, "
              "p+d <= 16 and 16-byte aligned row/CSR buffers (got Kr=%d Kc=%d)", Kr, Kc);
    delete h;
    return GMF_ERR_UNSUPPORTED;
  }
  P.tcm = tc_ok && cfg->k1_impl != GMF_K1_CUDA_CORES;
  int n_sm = kSMs;
  GMF_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, desc->device));
  int smem_optin = 0;
  GMF_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, desc->device));
  // K1 generation on the tensor cores: v2 (warp-specialized, one CTA per SM)
  // pays off once its units are deep pipelines (>= 8 chunks of 64 rows, e.g.
  // BASELINE c5's 65,536-row blocks); shallow units (c3, c4: 135-270 rows per
  // unit) keep v1's two 256-thread CTAs per SM.  GMF_TC_VERSION=1|2 forces one.
  bool want_v2 = false;
  {
    const char* fv = getenv("GMF_TC_VERSION");
    const int64_t ct2 = (jmax + 127) / 128;
    int a = (int)ct2, b = n_sm;
    while (b) { const int t = a % b; a = b; b = t; }
    int64_t rs2 = n_sm / (a > 0 ? a : 1);
    if (rs2 > (nstar_max + 31) / 32) rs2 = (nstar_max + 31) / 32;
    if (rs2 < 1) rs2 = 1;
    want_v2 = nstar_max / rs2 >= 512;
    if (fv) want_v2 = atoi(fv) == 2;
    if (getenv("GMF_TC_V1")) want_v2 = false;
  }
  if (P.tcm && (desc->flags & GMF_DESC_TAIL_PADDED) && want_v2) {
    // K1 v2 (warp-specialized pipeline, gmf_tc2.cuh): the offset rides in
    // GEMM1 as feature KA and two sentinel features follow it, so the feature
    // bucket must hold KA + has_off + 2; the staging ring shrinks until the
    // tile fits in shared memory
    const int nk2 = grad_bucket(KA + (P.has_off ? 1 : 0) + 2);   // + the two sentinel features
    if (nk2 > 0 && nk2 <= 32) {
      Params Q = P;
      Q.tcm = 2;
      const int64_t lim = smem_optin - 2048;   // the fit kernel's static shared memory
      // prefer two A1 buffers, then the largest staging ring that fits
      for (int na1 = 2; na1 >= 1 && Q.tcm == 2 && P.tcm != 2; --na1) {
        Q.k1_na1 = na1;
        for (Q.k1_cap = 2048; Q.k1_cap >= 512; Q.k1_cap /= 2) {
          if (grad_smem_bytes(Q, desc->dtype, nk2) <= lim) {
            P.tcm = 2;
            P.k1_cap = Q.k1_cap;
            P.k1_na1 = na1;
            h->NK = nk2;
            break;
          }
        }
      }
    }
  }

  const int TC = tile_cols(desc->dtype, h->NK);
  P.TC = TC;
  P.CT = (int)((jmax + TC - 1) / TC);
  if (P.tcm == 2) {
    // units = CT x RS spread over one CTA per SM: RS = SMs / gcd(CT, SMs) makes
    // the unit count a multiple of the SM count; at least 32 rows per unit
    int a = P.CT, b = n_sm;
    while (b) { const int t = a % b; a = b; b = t; }
    int64_t RS = n_sm / (a > 0 ? a : 1);
    const int64_t rmax = (nstar_max + 31) / 32;
    if (RS > rmax) RS = rmax;
    if (RS < 1) RS = 1;
    P.RS = (int)RS;
  } else {
    const int64_t nchunks = (nstar_max + TR - 1) / TR;
    int64_t RS = (2 * kSMs + P.CT - 1) / P.CT;
    if (RS > nchunks) RS = nchunks;
    if (RS < 1) RS = 1;
    P.RS = (int)RS;
  }
  P.nstar_max = nstar_max;
  P.jmax = jmax;
  int64_t nrc = (nstar_max * Kr + kThreads - 1) / kThreads;
  P.n_row_ctas = (int)(nrc > 0 ? nrc : 1);
  int64_t ncc = (desc->m * Kc + kThreads - 1) / kThreads;
  P.n_col_ctas = (int)(ncc > 0 ? ncc : 1);
  int64_t noc = (bufs->n_eval + kThreads - 1) / kThreads;
  P.n_obj_ctas = (int)(noc < 1 ? 1 : (noc > 2 * kSMs ? 2 * kSMs : noc));

  // persistent kernel geometry: every co-resident CTA, a multiple of CT
  int fit_bps = 0;
  const int64_t k1_smem = grad_smem_bytes(P, desc->dtype, h->NK);
  if (k1_smem > smem_optin) {
    set_error("the K1 tile for p+q+d = %d (%s%s) needs %lld B of shared memory, the device "
              "allows %d", KA, desc->dtype == GMF_F64 ? "fp64" : "fp32",
              P.has_w ? ", prior weights" : "", (long long)k1_smem, smem_optin);
    delete h;
    return GMF_ERR_UNSUPPORTED;
  }
  rc = prepare_grad(P, desc->dtype, h->NK, 0, &fit_bps);
  if (rc) { delete h; return rc; }
  // fit grid: every co-resident CTA (v1 / CUDA cores: a multiple of CT, one
  // (tile, row split) each; v2: one CTA per SM walking the units)
  auto fit_grid_for = [&](int bps) {
    if (P.tcm == 2) return bps >= 1 ? n_sm : 0;
    return P.CT > 0 ? (bps * n_sm / P.CT) * P.CT : 0;
  };
  {
    // cache each fit CTA's tracked entries in shared memory when that keeps
    // the same number of CTAs per SM
    const int grid0 = fit_grid_for(fit_bps);
    const int64_t cap = grid0 > 0 ? (bufs->n_eval + grid0 - 1) / grid0 : 0;
    if (cap > 0 && cap <= 1024 && k1_smem + cap * 16 + (P.tcm == 2 ? 2048 : 0) <= smem_optin) {
      int bps2 = 0;
      rc = prepare_grad(P, desc->dtype, h->NK, (int)(cap * 16), &bps2);
      if (rc) { delete h; return rc; }
      if (bps2 == fit_bps) {
        P.ep_cap = (int)cap;
        P.ep_soff = grad_smem_bytes(P, desc->dtype, h->NK);
      } else {
        rc = prepare_grad(P, desc->dtype, h->NK, 0, &bps2);
        if (rc) { delete h; return rc; }
      }
    }
  }
  int coop = 0;
  GMF_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, desc->device));
  h->fit_grid = coop ? fit_grid_for(fit_bps) : 0;
  if (getenv("GMF_NO_PERSISTENT")) h->fit_grid = 0;   // diagnostics: per-step kernels only
  h->fit_rs = P.tcm == 2 ? P.RS : h->fit_grid / (P.CT > 0 ? P.CT : 1);

  // ---- workspace carve-up ----
  const int64_t max_epochs = cfg->max_epochs;
  const int64_t ms = bufs->max_steps > 0 ? bufs->max_steps : 1;
  const int64_t rec_bytes = align256((int64_t)REC_HDR * 8 + jmax * 2 * Kc * h->tsz);
  const int64_t rs_max = P.RS > h->fit_rs ? P.RS : h->fit_rs;
  const int64_t cta_max = [&] {
    int64_t v = P.n_row_ctas;
    if (P.n_obj_ctas > v) v = P.n_obj_ctas;
    if (h->fit_grid > v) v = h->fit_grid;
    if (P.CT * rs_max > v) v = P.CT * rs_max;
    return v;
  }();
  int64_t off = 0;
  auto take = [&](int64_t bytes) { int64_t o = off; off = align256(off + bytes); return o; };
  const int64_t o_ctrl = take(sizeof(Ctrl));
  const int64_t o_tobj = take((max_epochs + 2) * 8);
  const int64_t o_tnb = take((max_epochs + 2) * 8);
  const int64_t o_tphi = take((max_epochs + 2) * 8);
  const int64_t o_rowp = take((int64_t)P.CT * nstar_max * 2 * Kr * h->tsz);
  const int64_t o_colp = take((int64_t)P.CT * rs_max * TC * 2 * Kc * h->tsz);
  const int64_t o_nbp = take(cta_max * 2 * 8);
  const int64_t o_tick = take((int64_t)(2 * P.CT + 4) * 4);
  const int64_t o_rec = take(rec_bytes);
  const int64_t o_objp = take(cta_max * OBJ_W * 8);
  const int64_t o_rnp = take(cta_max * 2 * 8);
  const int64_t o_bs = take(R * 2 * 8);
  const int64_t o_bnp = take(R * (int64_t)blocknorm_segments(nstar_max) * 2 * 8);
  const int64_t o_lm = take(R * 8);
  const int64_t o_rho = take(ms * 8);
  const int64_t o_alp = take(ms * 8);
  const int64_t o_fp = take(2 * 8 * kSMs * 8);   // k_objfull (2 x 8 kSMs) / k_entries (4 x 2 kSMs) partials
  const int64_t o_ft = take(64);
  const int64_t o_ep = take((bufs->n_eval > 0 ? bufs->n_eval : 1) * 16);
  const int64_t o_cnp = take(cta_max * 2 * 8);
  const int64_t o_gbar = take(32);
  const int64_t o_tot = take(64);                               // phase-2 totals (last arriver)
  const int64_t o_ready = take(8);                              // streaming ready counter
  const int64_t E1 = bufs->n_eval > 0 ? bufs->n_eval : 1;
  const int64_t o_esr = take(E1 * 8);                          // eval rows, sorted
  const int64_t o_esc = take(E1 * 4);                          // eval cols, same order
  const int64_t o_rsl = take((desc->n > 0 ? desc->n : 1) * 4);  // cache slot per row
  const int64_t o_srw = take(E1 * 8);                          // row per cache slot
  const int64_t o_esl = take(E1 * 4);                          // cache slot per entry
  const int64_t o_ecache = take(E1 * (h->NK + 4) * h->tsz);    // objective row cache (<= E slots)
  const int64_t o_vpad = take(desc->m * h->NK * h->tsz);       // padded column features
  // K1's tile index for CSR rows too dense to stage (J = all columns)
  const bool want_tidx = desc->y_format != GMF_Y_DENSE_I32 && col_identity && desc->n > 0;
  const int64_t o_tidx = take(want_tidx ? desc->n * (P.CT + 1) * 4 + 16 : 16);
  const bool want_img = P.tcm && col_identity;
  // K1 v2 operand-row images: every chunk of every row split of the largest block
  const int64_t rimg_nch = (nstar_max / (P.RS > 0 ? P.RS : 1) + 2 + 63) / 64;
  const int64_t o_rimg = take(P.tcm == 2 ? (int64_t)P.RS * rimg_nch * rimg_bytes_of(h->NK) : 16);
  const int64_t o_rflag = take(P.tcm == 2 ? (int64_t)P.RS * rimg_nch * 4 + 16 : 16);
  const int64_t o_cimg = take(want_img ? colimg_bytes_total(h->NK, P.CT, P.tcm) : 16);
  cudaError_t e = cudaMalloc(&h->ws, off);
  if (e != cudaSuccess) { delete h; return cuda_fail(e, "cudaMalloc workspace"); }
  char* base = (char*)h->ws;
  P.ctrl = (Ctrl*)(base + o_ctrl);
  P.trace_obj = (double*)(base + o_tobj);
  P.trace_nb = (double*)(base + o_tnb);
  P.trace_phi = (double*)(base + o_tphi);
  P.rowpart = base + o_rowp;
  P.colpart = base + o_colp;
  P.nbpart = (double*)(base + o_nbp);
  P.tickets = (unsigned int*)(base + o_tick);
  P.rec = (double*)(base + o_rec);
  P.rec_stride = rec_bytes;
  P.objpart = (double*)(base + o_objp);
  P.rnpart = (double*)(base + o_rnp);
  P.cnpart = (double*)(base + o_cnp);
  P.gbar = (unsigned int*)(base + o_gbar);
  P.totals = (double*)(base + o_tot);
  P.ready = (const unsigned long long*)(base + o_ready);
  P.blocksum = (double*)(base + o_bs);
  P.bnpart = (double*)(base + o_bnp);
  P.snap_ver = (long long*)(base + o_lm);
  P.rho_tab = (double*)(base + o_rho);
  P.alpt_tab = (double*)(base + o_alp);
  h->full_part = (double*)(base + o_fp);
  h->full_ticket = (unsigned int*)(base + o_ft);
  GMF_CUDA(cudaMemset(h->ws, 0, off));
  P.rslot = (const int32_t*)(base + o_rsl);
  P.srow = (const int64_t*)(base + o_srw);
  P.eslot = nullptr;
  P.nslots = 0;
  P.ecache = base + o_ecache;
  P.vpad = base + o_vpad;
  P.nkb = h->NK;
  P.colimg = want_img ? (void*)(base + o_cimg) : nullptr;
  P.rimg = base + o_rimg;
  P.rimg_flag = (unsigned int*)(base + o_rflag);
  P.rimg_epoch = (unsigned int*)(base + o_rflag + (P.tcm == 2 ? (int64_t)P.RS * rimg_nch * 4 : 0));
  P.rimg_nch = (int)rimg_nch;
  if (bufs->n_eval > 0) {
    // the tracked sample sorted by (block-major) row; each tracked row owns a
    // cache slot that phase 2 writes with the row (the objective is an
    // order-free sum)
    const int64_t E = bufs->n_eval;
    std::vector<int64_t> er(E), ers(E);
    std::vector<int32_t> ec(E), ecs(E);
    GMF_CUDA(cudaMemcpy(er.data(), bufs->eval_row, E * 8, cudaMemcpyDeviceToHost));
    GMF_CUDA(cudaMemcpy(ec.data(), bufs->eval_col, E * 4, cudaMemcpyDeviceToHost));
    std::vector<int64_t> idx(E);
    for (int64_t k = 0; k < E; ++k) idx[k] = k;
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return er[a] < er[b]; });
    for (int64_t k = 0; k < E; ++k) { ers[k] = er[idx[k]]; ecs[k] = ec[idx[k]]; }
    if (E >= (int64_t)1 << 31) { set_error("more than 2^31 tracked entries"); gmf_destroy(h); return GMF_ERR_CONFIG; }
    // one cache slot per distinct tracked row (entries are sorted by row)
    std::vector<int32_t> rsl(desc->n > 0 ? desc->n : 1, -1), esl(E);
    std::vector<int64_t> srw;
    for (int64_t k = 0; k < E; ++k) {
      if (k == 0 || ers[k] != ers[k - 1]) srw.push_back(ers[k]);
      esl[k] = (int32_t)(srw.size() - 1);
      rsl[ers[k]] = esl[k];
    }
    GMF_CUDA(cudaMemcpy(base + o_esr, ers.data(), E * 8, cudaMemcpyHostToDevice));
    GMF_CUDA(cudaMemcpy(base + o_esc, ecs.data(), E * 4, cudaMemcpyHostToDevice));
    if (desc->n > 0) GMF_CUDA(cudaMemcpy(base + o_rsl, rsl.data(), desc->n * 4, cudaMemcpyHostToDevice));
    GMF_CUDA(cudaMemcpy(base + o_srw, srw.data(), srw.size() * 8, cudaMemcpyHostToDevice));
    GMF_CUDA(cudaMemcpy(base + o_esl, esl.data(), E * 4, cudaMemcpyHostToDevice));
    P.eslot = (const int32_t*)(base + o_esl);
    P.nslots = (int64_t)srw.size();
    P.erow = (const int64_t*)(base + o_esr);
    P.ecol = (const int32_t*)(base + o_esc);
  }
  if (bufs->n_eval <= 0 && desc->n > 0) GMF_CUDA(cudaMemset(base + o_rsl, 0xFF, desc->n * 4));   // no slots
  P.tidx = nullptr;
  if (want_tidx) {
    int32_t* ti = (int32_t*)(base + o_tidx);
    unsigned int* flag = (unsigned int*)(base + o_tidx + desc->n * (P.CT + 1) * 4);
    GMF_CUDA(cudaMemset(flag, 0, 4));
    rc = launch_tile_index(P, ti, flag, 0);
    if (rc) { gmf_destroy(h); return rc; }
    unsigned int unsorted = 1;
    GMF_CUDA(cudaMemcpy(&unsorted, flag, 4, cudaMemcpyDeviceToHost));
    if (!unsorted) P.tidx = ti;   // columns not increasing in some row: full-row scans
  }
  P.tptr = nullptr;
  P.tent = nullptr;
  if (P.tcm == 2 && P.tidx) {
    // K1 v2 reads CSR through a tile-major copy whose entries carry their row
    const int64_t nnz = P.nnz;
    const int64_t tp_bytes = align256((int64_t)P.CT * (desc->n + 1) * 8);
    const int64_t te_bytes = align256((2 * nnz + 8) * 4);
    const int64_t ln_bytes = align256((int64_t)P.CT * desc->n * 4 + 16);
    cudaError_t e2 = cudaMalloc(&h->tcsr_buf, tp_bytes + te_bytes + ln_bytes);
    if (e2 != cudaSuccess) { gmf_destroy(h); return cuda_fail(e2, "cudaMalloc tile-CSR"); }
    char* tb = (char*)h->tcsr_buf;
    unsigned int* too_big = (unsigned int*)(tb + tp_bytes + te_bytes + ln_bytes - 16);
    GMF_CUDA(cudaMemset(tb + tp_bytes, 0, te_bytes));
    GMF_CUDA(cudaMemset(too_big, 0, 4));
    rc = launch_tcsr(P, P.tidx, (int32_t*)(tb + tp_bytes + te_bytes), (int64_t*)tb,
                     (int32_t*)(tb + tp_bytes), too_big, 0);
    if (rc) { gmf_destroy(h); return rc; }
    unsigned int big = 0;
    GMF_CUDA(cudaMemcpy(&big, too_big, 4, cudaMemcpyDeviceToHost));
    if (!big) {   // counts >= 2^23 do not fit an entry word: row-walking scatter instead
      P.tptr = (const int64_t*)tb;
      P.tent = (const int32_t*)(tb + tp_bytes);
    }
  }
  P.ep = (const int4*)(base + o_ep);
  if (bufs->n_eval > 0) {   // tracked sample packed with its Y, once per fit
    rc = launch_eval_pack(P, (int4*)(base + o_ep), 0);
    if (rc) { gmf_destroy(h); return rc; }
    GMF_CUDA(cudaDeviceSynchronize());
  }

  // learning-rate and bias-correction tables, host libm (optim.py:130-148)
  std::vector<double> rho(ms), alp(ms);
  for (int64_t t = 0; t < ms; ++t) {
    rho[t] = cfg->rate_k0 / pow(1.0 + cfg->rate_k0 * cfg->rate_k1 * (double)t, cfg->rate_tau);
    const double tt = (double)(t + 1);
    alp[t] = cfg->smooth_a1 == cfg->smooth_a2
                 ? 1.0
                 : (1.0 - pow(cfg->smooth_a2, tt)) / (1.0 - pow(cfg->smooth_a1, tt));
  }
  GMF_CUDA(cudaMemcpy((void*)P.rho_tab, rho.data(), ms * 8, cudaMemcpyHostToDevice));
  GMF_CUDA(cudaMemcpy((void*)P.alpt_tab, alp.data(), ms * 8, cudaMemcpyHostToDevice));

  GMF_CUDA(cudaMallocHost(&h->host_ctrl, sizeof(Ctrl)));
  GMF_CUDA(cudaMallocHost(&h->host_abort, 16));
  *h->host_abort = 0;
  GMF_CUDA(cudaStreamCreateWithFlags(&h->internal, cudaStreamNonBlocking));
  GMF_CUDA(cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming));
  GMF_CUDA(cudaEventCreateWithFlags(&h->ev_b, cudaEventDisableTiming));
  *out = h;
  return GMF_OK;
}

int gmf_destroy(gmf_handle* h) {
  if (!h) return GMF_OK;
  cudaSetDevice(h->desc.device);
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  if (h->internal) cudaStreamSynchronize(h->internal);
  if (h->ws) cudaFree(h->ws);
  if (h->prof_buf) cudaFree(h->prof_buf);
  if (h->tcsr_buf) cudaFree(h->tcsr_buf);
  if (h->host_ctrl) cudaFreeHost(h->host_ctrl);
  if (h->host_abort) cudaFreeHost(h->host_abort);
  if (h->ready_vals) cudaFreeHost(h->ready_vals);
  if (h->internal) cudaStreamDestroy(h->internal);
  if (h->ev_a) cudaEventDestroy(h->ev_a);
  if (h->ev_b) cudaEventDestroy(h->ev_b);
  delete h;
  return GMF_OK;
}

int gmf_reset(gmf_handle* h, double nb_shape, void* stream) {
  if (!h) { set_error("null handle"); return GMF_ERR_STATE; }
  if (!(nb_shape > 0)) { set_error("nb_shape must be positive"); return GMF_ERR_DOMAIN; }
  GMF_CUDA(cudaSetDevice(h->desc.device));
  cudaStream_t st = (cudaStream_t)stream;
  const Params& P = h->P;
  Ctrl c;
  memset(&c, 0, sizeof(c));
  c.nb_shape = nb_shape;
  c.phi = h->cfg.phi;
  GMF_CUDA(cudaStreamSynchronize(st));
  *h->host_ctrl = c;
  GMF_CUDA(cudaMemcpyAsync(P.ctrl, h->host_ctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, st));
  GMF_CUDA(cudaMemsetAsync(P.snap_ver, 0, P.R * 8, st));
  GMF_CUDA(cudaMemsetAsync(P.tickets, 0, (2 * P.CT + 4) * 4, st));
  const int64_t rb = P.n * P.Kr * h->tsz, cb = P.m * P.Kc * h->tsz;
  if (rb) {
    GMF_CUDA(cudaMemsetAsync(P.gb_row, 0, rb, st));
    GMF_CUDA(cudaMemsetAsync(P.hb_row, 0, rb, st));
  }
  if (cb) {
    GMF_CUDA(cudaMemsetAsync(P.gb_col, 0, cb, st));
    GMF_CUDA(cudaMemsetAsync(P.hb_col, 0, cb, st));
  }
  GMF_CUDA(cudaMemsetAsync((void*)P.ready, 0, 8, st));
  GMF_CUDA(cudaMemsetAsync((void*)P.gbar, 0, 32, st));
  int rc = launch_blocknorm(P, h->desc.dtype, st);
  if (!rc) rc = launch_cache_fill(P, h->desc.dtype, st);   // the per-step path's objective caches
  if (rc) return rc;
  h->launches += 3;
  GMF_CUDA(cudaStreamSynchronize(st));
  if (P.tcm == 1 && h->fit_grid > 0 && !h->residency_checked) {
    // the tensor-core fit kernel synchronises with a software grid barrier:
    // probe once that all its CTAs are co-resident, else one CTA per SM
    rc = residency_probe(h, st);
    if (rc) return rc;
  }
  h->reset_done = true;
  return GMF_OK;
}

int gmf_minibatch_grad(gmf_handle* h, int64_t row_block, int64_t col_block, double nb_shape,
                       void* g_row, void* h_row, void* g_col, void* h_col, double* nb_sums,
                       void* stream) {
  if (h && (h->desc.flags & GMF_DESC_EVAL_ONLY)) { set_error("evaluation-only handle (GMF_DESC_EVAL_ONLY): no fit, gradient or deviance calls"); return GMF_ERR_STATE; }
  if (!h) { set_error("null handle"); return GMF_ERR_STATE; }
  const Params& P = h->P;
  if (row_block < 0 || row_block >= P.R || col_block < 0 || col_block >= P.S) {
    set_error("minibatch indices out of range");
    return GMF_ERR_CONFIG;
  }
  if (!(nb_shape > 0)) { set_error("nb_shape must be positive"); return GMF_ERR_DOMAIN; }
  GMF_CUDA(cudaSetDevice(h->desc.device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc = launch_grad(P, h->desc.dtype, h->NK, st, row_block, col_block, nb_shape);
  if (!rc) rc = launch_colrec(P, h->desc.dtype, st, col_block);
  if (rc) return rc;
  h->launches += 3;
  const int64_t nI = h->rbp_host[row_block + 1] - h->rbp_host[row_block];
  const int64_t nJ = h->cbp_host[col_block + 1] - h->cbp_host[col_block];
  return launch_gradout(P, h->desc.dtype, row_block, col_block, nI, nJ, g_row, h_row, g_col,
                        h_col, nb_sums, st);
}

int gmf_step_local(gmf_handle* h, void* stream) {
  if (h && (h->desc.flags & GMF_DESC_EVAL_ONLY)) { set_error("evaluation-only handle (GMF_DESC_EVAL_ONLY): no fit, gradient or deviance calls"); return GMF_ERR_STATE; }
  if (!h || !h->reset_done) { set_error("gmf_step_local before gmf_reset"); return GMF_ERR_STATE; }
  cudaStream_t st = (cudaStream_t)stream;
  int rc = launch_obj(h->P, h->desc.dtype, st);
  if (rc) return rc;
  h->launches += 3;
  rc = launch_grad(h->P, h->desc.dtype, h->NK, st, -1, -1, 0.0);
  if (rc) return rc;
  return launch_colrec(h->P, h->desc.dtype, st, -1);
}

int gmf_step_apply(gmf_handle* h, const void* gathered, void* stream) {
  if (!h || !h->reset_done) { set_error("gmf_step_apply before gmf_reset"); return GMF_ERR_STATE; }
  if (h->desc.world_size > 1 && !gathered) { set_error("world_size > 1 needs gathered records"); return GMF_ERR_CONFIG; }
  h->launches += 1;
  return launch_apply(h->P, h->desc.dtype, gathered, (cudaStream_t)stream);
}

void* gmf_record_ptr(gmf_handle* h) { return h ? (void*)h->P.rec : nullptr; }
int64_t gmf_record_bytes(gmf_handle* h) { return h ? h->P.rec_stride : 0; }

int gmf_record_copy(gmf_handle* h, void* dst, void* stream) {
  if (!h || !dst) { set_error("null handle/dst"); return GMF_ERR_STATE; }
  GMF_CUDA(cudaMemcpyAsync(dst, h->P.rec, h->P.rec_stride, cudaMemcpyDeviceToDevice,
                           (cudaStream_t)stream));
  return GMF_OK;
}

int gmf_run(gmf_handle* h, int64_t n_steps, void* stream) {
  if (h && (h->desc.flags & GMF_DESC_EVAL_ONLY)) { set_error("evaluation-only handle (GMF_DESC_EVAL_ONLY): no fit, gradient or deviance calls"); return GMF_ERR_STATE; }
  if (!h || !h->reset_done) { set_error("gmf_run before gmf_reset"); return GMF_ERR_STATE; }
  if (h->desc.world_size != 1) { set_error("gmf_run is single-rank; use step_local/step_apply"); return GMF_ERR_STATE; }
  if (n_steps <= 0) return GMF_OK;
  GMF_CUDA(cudaSetDevice(h->desc.device));
  cudaStream_t user = (cudaStream_t)stream;
  if (h->fit_grid > 0) {
    // one cooperative launch runs all n_steps (grid-wide barriers between phases)
    Params P = h->P;
    P.RS = h->fit_rs;
    h->launches += 1;
    return launch_fit(P, h->desc.dtype, h->NK, h->fit_grid, n_steps, user);
  }
  // fallback for devices without cooperative launch: per-step kernels in CUDA graphs
  const int64_t kChunk = 16;
  GMF_CUDA(cudaEventRecord(h->ev_a, user));
  GMF_CUDA(cudaStreamWaitEvent(h->internal, h->ev_a, 0));
  int64_t left = n_steps;
  while (left > 0) {
    const int64_t c = left < kChunk ? left : kChunk;
    auto it = h->graphs.find(c);
    if (it == h->graphs.end()) {
      cudaGraph_t g;
      GMF_CUDA(cudaStreamBeginCapture(h->internal, cudaStreamCaptureModeThreadLocal));
      int rc = GMF_OK;
      for (int64_t s = 0; s < c && rc == GMF_OK; ++s) {
        rc = launch_obj(h->P, h->desc.dtype, h->internal);
        if (!rc) rc = launch_grad(h->P, h->desc.dtype, h->NK, h->internal, -1, -1, 0.0);
        if (!rc) rc = launch_colrec(h->P, h->desc.dtype, h->internal, -1);
        if (!rc) rc = launch_apply(h->P, h->desc.dtype, nullptr, h->internal);
      }
      cudaError_t e = cudaStreamEndCapture(h->internal, &g);
      if (rc) return rc;
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      cudaGraphExec_t ex;
      e = cudaGraphInstantiate(&ex, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
      it = h->graphs.emplace(c, ex).first;
    }
    GMF_CUDA(cudaGraphLaunch(it->second, h->internal));
    h->launches += 4 * c;
    left -= c;
  }
  GMF_CUDA(cudaEventRecord(h->ev_b, h->internal));
  GMF_CUDA(cudaStreamWaitEvent(user, h->ev_b, 0));
  return GMF_OK;
}

int gmf_status_read(gmf_handle* h, gmf_status* out, void* stream) {
  if (!h || !out) { set_error("null handle/out"); return GMF_ERR_STATE; }
  GMF_CUDA(cudaSetDevice(h->desc.device));
  cudaStream_t st = (cudaStream_t)stream;
  GMF_CUDA(cudaMemcpyAsync(h->host_ctrl, h->P.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
  GMF_CUDA(cudaMemcpyAsync(h->host_abort, h->P.gbar + 2, 4, cudaMemcpyDeviceToHost, st));
  GMF_CUDA(cudaStreamSynchronize(st));
  if (*h->host_abort) {
    set_error("persistent fit kernel aborted: a grid barrier or a streamed block timed out");
    return GMF_ERR_STATE;
  }
  return gmf_status_decode(h->host_ctrl, out);
}

int64_t gmf_status_raw_bytes(void) { return (int64_t)sizeof(Ctrl); }

int gmf_snapshot_blocks(gmf_handle* h, int64_t* ver, int64_t* period, void* stream) {
  if (!h || !ver || !period) { set_error("null handle/out"); return GMF_ERR_STATE; }
  GMF_CUDA(cudaSetDevice(h->desc.device));
  cudaStream_t st = (cudaStream_t)stream;
  GMF_CUDA(cudaMemcpyAsync(ver, h->P.snap_ver, h->P.R * 8, cudaMemcpyDeviceToHost, st));
  GMF_CUDA(cudaMemcpyAsync(h->host_ctrl, h->P.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
  GMF_CUDA(cudaStreamSynchronize(st));
  *period = h->host_ctrl->snap_period;
  return GMF_OK;
}

int64_t gmf_profile_len(gmf_handle* h) { return h ? 16 + 32 * (int64_t)h->fit_grid + 512 : 0; }

int gmf_geometry(gmf_handle* h, int64_t* out8) {
  if (!h || !out8) { set_error("null handle/out"); return GMF_ERR_STATE; }
  out8[0] = h->fit_grid;
  out8[1] = h->fit_rs;
  out8[2] = h->P.CT;
  out8[3] = h->P.TC;
  out8[4] = h->P.RS;
  out8[5] = h->NK;
  out8[6] = grad_smem_bytes(h->P, h->desc.dtype, h->NK);
  out8[7] = h->P.nstar_max;
  return GMF_OK;
}

int gmf_profile(gmf_handle* h, int enable, double* out6, void* stream) {
  if (!h) { set_error("null handle"); return GMF_ERR_STATE; }
  const int64_t NPROF = gmf_profile_len(h);
  GMF_CUDA(cudaSetDevice(h->desc.device));
  cudaStream_t st = (cudaStream_t)stream;
  if (!h->prof_buf) GMF_CUDA(cudaMalloc(&h->prof_buf, NPROF * sizeof(unsigned long long)));
  if (out6) {
    std::vector<unsigned long long> v(NPROF);
    GMF_CUDA(cudaMemcpyAsync(v.data(), h->prof_buf, NPROF * 8, cudaMemcpyDeviceToHost, st));
    GMF_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < NPROF; ++i) out6[i] = (double)v[i];
  }
  GMF_CUDA(cudaMemsetAsync(h->prof_buf, 0, NPROF * sizeof(unsigned long long), st));
  h->P.prof = enable ? (unsigned long long*)h->prof_buf : nullptr;
  return GMF_OK;
}

int gmf_status_copy_async(gmf_handle* h, void* host_dst, void* stream) {
  if (!h || !host_dst) { set_error("null handle/dst"); return GMF_ERR_STATE; }
  GMF_CUDA(cudaMemcpyAsync(host_dst, h->P.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost,
                           (cudaStream_t)stream));
  return GMF_OK;
}

int gmf_status_decode(const void* raw, gmf_status* out) {
  if (!raw || !out) { set_error("null raw/out"); return GMF_ERR_STATE; }
  Ctrl c;
  memcpy(&c, raw, sizeof(Ctrl));
  out->t = c.t;
  out->trace_len = c.trace_len;
  out->snapshot_trace_len = c.snapshot_trace_len;
  out->nb_shape = c.nb_shape;
  out->phi = c.phi;
  out->last_objective = c.last_obj;
  out->converged = c.converged;
  out->diverged = c.diverged;
  out->diverged_init = c.diverged_init;
  out->stopped = c.stopped;
  return GMF_OK;
}

int gmf_time_grad(gmf_handle* h, int64_t row_block, int32_t iters, double* avg_ms, void* stream) {
  if (h && (h->desc.flags & GMF_DESC_EVAL_ONLY)) { set_error("evaluation-only handle (GMF_DESC_EVAL_ONLY): no fit, gradient or deviance calls"); return GMF_ERR_STATE; }
  if (!h || !avg_ms || iters < 1) { set_error("gmf_time_grad: bad arguments"); return GMF_ERR_CONFIG; }
  if (row_block < 0 || row_block >= h->P.R) { set_error("row block out of range"); return GMF_ERR_CONFIG; }
  GMF_CUDA(cudaSetDevice(h->desc.device));
  cudaStream_t st = (cudaStream_t)stream;
  gmf_status s;
  int rc = gmf_status_read(h, &s, stream);
  if (rc) return rc;
  const double alpha = s.nb_shape > 0 ? s.nb_shape : 1.0;
  cudaEvent_t a, b;
  GMF_CUDA(cudaEventCreate(&a));
  GMF_CUDA(cudaEventCreate(&b));
  rc = launch_grad(h->P, h->desc.dtype, h->NK, st, row_block, 0, alpha);   // warm
  if (rc) return rc;
  h->launches += 1 + iters;
  GMF_CUDA(cudaEventRecord(a, st));
  for (int i = 0; i < iters && rc == GMF_OK; ++i)
    rc = launch_grad(h->P, h->desc.dtype, h->NK, st, row_block, 0, alpha);
  GMF_CUDA(cudaEventRecord(b, st));
  GMF_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  GMF_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *avg_ms = ms / iters;
  return rc;
}

int gmf_trace_read(gmf_handle* h, double* obj, double* nb, int64_t n, void* stream) {
  if (!h) { set_error("null handle"); return GMF_ERR_STATE; }
  if (n <= 0) return GMF_OK;
  if (n > h->cfg.max_epochs + 1) n = h->cfg.max_epochs + 1;
  cudaStream_t st = (cudaStream_t)stream;
  if (obj) GMF_CUDA(cudaMemcpyAsync(obj, h->P.trace_obj, n * 8, cudaMemcpyDeviceToHost, st));
  if (nb) GMF_CUDA(cudaMemcpyAsync(nb, h->P.trace_nb, n * 8, cudaMemcpyDeviceToHost, st));
  GMF_CUDA(cudaStreamSynchronize(st));
  return GMF_OK;
}

int gmf_trace_phi_read(gmf_handle* h, double* phi, int64_t n, void* stream) {
  if (!h || !phi) { set_error("null handle/out"); return GMF_ERR_STATE; }
  if (n <= 0) return GMF_OK;
  if (n > h->cfg.max_epochs + 1) n = h->cfg.max_epochs + 1;
  cudaStream_t st = (cudaStream_t)stream;
  GMF_CUDA(cudaMemcpyAsync(phi, h->P.trace_phi, n * 8, cudaMemcpyDeviceToHost, st));
  GMF_CUDA(cudaStreamSynchronize(st));
  return GMF_OK;
}

int gmf_objective_full(gmf_handle* h, double* dev_sum, void* stream) {
  if (h && (h->desc.flags & GMF_DESC_EVAL_ONLY)) { set_error("evaluation-only handle (GMF_DESC_EVAL_ONLY): no fit, gradient or deviance calls"); return GMF_ERR_STATE; }
  if (!h || !dev_sum) { set_error("null handle/out"); return GMF_ERR_STATE; }
  gmf_status s;
  int rc = gmf_status_read(h, &s, stream);
  if (rc) return rc;
  h->launches += 1;
  return launch_objfull(h->P, h->desc.dtype, s.nb_shape, 0, h->full_part, h->full_ticket, dev_sum,
                        (cudaStream_t)stream);
}

int gmf_loglik_full(gmf_handle* h, double* out2, void* stream) {
  if (h && (h->desc.flags & GMF_DESC_EVAL_ONLY)) { set_error("evaluation-only handle (GMF_DESC_EVAL_ONLY): no fit, gradient or deviance calls"); return GMF_ERR_STATE; }
  if (!h || !out2) { set_error("null handle/out"); return GMF_ERR_STATE; }
  gmf_status s;
  int rc = gmf_status_read(h, &s, stream);
  if (rc) return rc;
  const int nb = h->desc.family == GMF_NEG_BINOMIAL && !h->P.gen;   // general mode: caller adds c(phi)
  cudaStream_t st = (cudaStream_t)stream;
  if (!nb) GMF_CUDA(cudaMemsetAsync(out2 + 1, 0, sizeof(double), st));
  h->launches += 1;
  return launch_objfull(h->P, h->desc.dtype, s.nb_shape, nb, h->full_part, h->full_ticket, out2,
                        st);
}

int gmf_entries_eval(gmf_handle* h, const int64_t* rows, const int32_t* cols, const double* y,
                     int64_t n, double ybar, double* mu_out, double* sums4, void* stream) {
  if (!h) { set_error("null handle"); return GMF_ERR_STATE; }
  if (n < 0 || (n > 0 && (!rows || !cols))) { set_error("entries: null rows/cols"); return GMF_ERR_CONFIG; }
  if (sums4 && !y) { set_error("entries: sums need y"); return GMF_ERR_CONFIG; }
  gmf_status s;
  int rc = gmf_status_read(h, &s, stream);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) {
    if (sums4) GMF_CUDA(cudaMemsetAsync(sums4, 0, 4 * sizeof(double), st));
    return GMF_OK;
  }
  h->launches += 1;
  return launch_entries(h->P, h->desc.dtype, s.nb_shape, rows, cols, y, n, ybar, mu_out,
                        h->full_part, h->full_ticket, sums4, st);
}

void* gmf_stream_ready_ptr(gmf_handle* h) { return h ? (void*)h->P.ready : nullptr; }

int gmf_run_stream(gmf_handle* h, int64_t n_steps, void* host_status, void* stream) {
  if (h && (h->desc.flags & GMF_DESC_EVAL_ONLY)) { set_error("evaluation-only handle (GMF_DESC_EVAL_ONLY): no fit, gradient or deviance calls"); return GMF_ERR_STATE; }
  if (!h || !h->reset_done) { set_error("gmf_run_stream before gmf_reset"); return GMF_ERR_STATE; }
  if (h->desc.world_size != 1) { set_error("gmf_run_stream is single-rank"); return GMF_ERR_STATE; }
  if (h->fit_grid <= 0) { set_error("gmf_run_stream needs the persistent fit kernel"); return GMF_ERR_UNSUPPORTED; }
  if (n_steps <= 0) return GMF_OK;
  GMF_CUDA(cudaSetDevice(h->desc.device));
  Params P = h->P;
  P.RS = h->fit_rs;
  P.stream_mode = 1;
  P.host_status = host_status;
  h->launches += 1;
  return launch_fit(P, h->desc.dtype, h->NK, h->fit_grid, n_steps, (cudaStream_t)stream);
}

int gmf_stream_signal(gmf_handle* h, int64_t value, void* stream) {
  if (!h) { set_error("null handle"); return GMF_ERR_STATE; }
  const int64_t ms = h->bufs.max_steps;
  if (value < 0 || value > ms) { set_error("stream signal %lld outside [0, %lld]", (long long)value, (long long)ms); return GMF_ERR_CONFIG; }
  if (!h->ready_vals) {
    GMF_CUDA(cudaMallocHost(&h->ready_vals, (ms + 1) * sizeof(unsigned long long)));
    for (int64_t t = 0; t <= ms; ++t) h->ready_vals[t] = (unsigned long long)t;
    h->n_ready_vals = ms + 1;
  }
  GMF_CUDA(cudaMemcpyAsync((void*)h->P.ready, h->ready_vals + value, sizeof(unsigned long long),
                           cudaMemcpyHostToDevice, (cudaStream_t)stream));
  return GMF_OK;
}

int gmf_k1_impl(gmf_handle* h) { return h ? (h->P.tcm ? GMF_K1_TENSOR : GMF_K1_CUDA_CORES) : -1; }

int gmf_k1_version(gmf_handle* h) { return h ? h->P.tcm : -1; }

int64_t gmf_launch_count(gmf_handle* h) { return h ? h->launches : -1; }

}  // extern "C"
