// Device-side state and launch parameters of the aSGD fit engine.
#pragma once
#include "gmf_common.cuh"

namespace gmf {

constexpr int TC = 64;                    // columns per CTA tile (K1)
constexpr int TR = 32;                    // rows per chunk (K1)
constexpr int NG = kThreads / TC;         // row groups in phase 1 (4)
constexpr int NQ = kThreads / (2 * TR);   // column quarters in phase 2 (4)
constexpr int REC_HDR = 8;                // doubles in the rank-record header
constexpr int kSnapCtas = 32;

// rank record header slots (doubles)
enum { R_DEV = 0, R_NGAM = 1, R_NU = 2, R_NB = 3, R_NV = 4, R_NBNUM = 5, R_NBDEN = 6 };

// Mutable fit control block, device resident.  Read by every kernel of a
// step; written only by the last CTA of k_apply (ticket), so its value is
// immutable while any kernel of the step reads it.
struct Ctrl {
  long long t;                  // steps applied
  long long trace_len;          // objective_trace entries
  long long last_snap_t;        // step index of the last snapshot (-1: none)
  long long snapshot_trace_len;
  double nb_shape;
  double phi;
  double last_obj;
  int streak, converged, diverged, diverged_init, stopped;
};

struct Params {
  int64_t n, m;
  int p, q, d, KA, Kr, Kc;
  int fam, yfmt, has_w, has_off;
  const int32_t* y;
  const int64_t* rp;
  const int32_t* ci;
  const int32_t* cv;
  const void* w;
  const void* x;
  const void* z;
  const void* off;
  void* th_row;
  void* th_col;
  void* gb_row;
  void* hb_row;
  void* gb_col;
  void* hb_col;
  void* sn_row;
  void* sn_col;
  const int64_t* rbp;
  const double* rbscale;
  int64_t R;
  const int32_t* cidx;
  const int64_t* cbp;
  const int32_t* cpos;
  const int32_t* cbof;
  int64_t S;
  int col_identity;   // S == 1 and col_idx == arange(m)
  const int32_t* bseq;
  int64_t max_steps;
  const int64_t* erow;
  const int32_t* ecol;
  int64_t E;
  // config
  double a1, a2, damp, tol;
  double lam_b, lam_g, lam_u, lam_v;
  double nbfloor, nbceil, escale, phi;
  int est_alpha, snap_stride, world;
  const double* rho_tab;     // learning_rate(t)        (optim.py:130-134)
  const double* alpt_tab;    // bias_correction(t + 1)  (optim.py:142-148)
  // workspace
  Ctrl* ctrl;
  double* trace_obj;
  double* trace_nb;
  void* rowpart;       // [CT][nstar_max][2 Kr]          T
  void* colpart;       // [CT][RS][TC][2 Kc]            T
  double* nbpart;      // [CT * RS][2]
  unsigned int* tickets;   // [CT] col tiles, [CT] grad-global, [CT+1] obj, [CT+2] apply
  double* rec;         // rank record: REC_HDR doubles + [jmax][2 Kc] T
  int64_t rec_stride;  // bytes between gathered records
  double* objpart;     // [n_obj_ctas]
  double* rnpart;      // [n_row_ctas][2]
  double* blocksum;    // [R][2] (gamma, u) squared norms per row block
  long long* last_mod; // [R]
  int RS, CT;
  int64_t nstar_max, jmax;
  int n_obj_ctas, n_row_ctas, n_col_ctas;
};

template <typename T>
GMF_D T* tptr(void* p) { return reinterpret_cast<T*>(p); }
template <typename T>
GMF_D const T* tptr(const void* p) { return reinterpret_cast<const T*>(p); }

}  // namespace gmf
