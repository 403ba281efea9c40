// Native launch sequence of one single-column GD+k iteration (the body the
// solver captures as a CUDA graph, eigensolver.py:563-700 on device):
//
//   expansion   svdsb_cgs_fused   select the candidate residual by its device
//                                 index, Jacobi division, +k copy, DGKS CGS
//                                 against V[:, :g], normalise into V[:, g]
//   operator    svdsb_apply_normal  W[:, g] = A^T A V[:, g]  (two CSR SpMVs)
//   projection  svdsb_gram   H column g = V[:, :g+1]^T W[:, g], written into H
//                            (column and row) by the kernel's last CTA
//   extraction  svdsb_syev_update  warm Rayleigh-Ritz update of the spectrum
//   candidates  svdsb_ritz_residual  R = W Y - V Y Lambda for p candidates;
//                                   its last CTA writes the status record (Ritz
//                                   values, residual norms, DGKS state)
//                                   straight into pinned host memory
//
// One C call instead of seven ctypes calls from the host loop: capturing a
// new iteration graph (a new basis size, or a new matrix) costs the graph
// instantiation only.
#include "common.cuh"

extern "C" int svdsb_gdk_iteration(svdsb_ctx *ctx, const svdsb_gdk_iter_args *a, void *stream) {
  SVDSB_CHECK_ARG(ctx != nullptr && a != nullptr && a->csr != nullptr, "svdsb_gdk_iteration: NULL argument");
  SVDSB_CHECK_ARG(a->g >= 1 && a->p >= 1 && a->p <= a->g + 1, "svdsb_gdk_iteration: bad basis / candidate count");
  const int g = a->g, gn = g + 1;
  double *vnew = a->v + (int64_t)g * a->ldv;
  double *wnew = a->w + (int64_t)g * a->ldw;
  const double *vcols[1] = {a->v};
  const int64_t vld[1] = {a->ldv};
  int ncol[1] = {g};
  int rc = svdsb_cgs_fused(ctx, a->n, 1, vcols, vld, ncol, a->rsrc, a->ldr, a->ci, a->d, vnew, a->yin, a->ldyin, g,
                           a->kk, a->prev, a->ldprev, a->passes, a->dgks, stream);
  if (rc) return rc;
  rc = svdsb_apply_normal(ctx, a->csr, a->side, vnew, a->ldv, wnew, a->ldw, 1, a->tmp, a->ldtmp, stream);
  if (rc) return rc;
  ncol[0] = gn;
  // H column (and row) g written by the Gram's last CTA (svdsb_h_insert's job)
  // (svdsb_tune_set key 4 = 1: the separate h_insert / status_pack launches)
  const bool fuse = svdsb::g_tune[4] != 1;
  svdsb::HInsert hi;
  if (fuse) {
    hi.h = a->h;
    hi.ldh = a->ldh;
    hi.g = g;
  }
  rc = svdsb::gram_impl(ctx, a->n, 1, vcols, vld, ncol, wnew, a->ldw, 1, a->hc, a->ldhc, nullptr, stream, hi);
  if (rc) return rc;
  if (!fuse && (rc = svdsb_h_insert(g, 1, a->hc, a->ldhc, a->h, a->ldh, stream))) return rc;
  rc = svdsb_syev_update(a->g0, gn - a->g0, a->h, a->ldh, a->y0, a->ldy0, a->l0, a->order, a->shift, a->lout,
                         a->yout, a->ldyout, stream);
  if (rc) return rc;
  // status record copied to pinned host memory by the Ritz kernel's last
  // CTA (svdsb_status_pack's job) when the candidates fit its wide path
  svdsb::StatusOut so;
  if (fuse && a->p <= 32) {
    so.lams = a->lout;
    so.gn = gn;
    so.st = a->dgks;
    so.host = a->status_host;
  }
  rc = svdsb::ritz_impl(ctx, a->n, a->v, a->ldv, a->w, a->ldw, gn, a->yout, a->ldyout, a->lout, a->p, a->rout,
                        a->ldrout, nullptr, 1, nullptr, 1, a->rn2, stream, so);
  if (rc) return rc;
  if (so.host != nullptr) return SVDSB_OK;
  return svdsb_status_pack(a->lout, gn, a->rn2, a->p, a->dgks, a->status_host, stream);
}
