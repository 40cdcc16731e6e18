// C ABI entry points (include/wf4dvar.h).  Argument checking, context
// lifetime, profiling bookkeeping; every compute step is a kernel launched
// from saddle.cu / model.cu / gemm.cu / trsm.cu / vec.cu / krylov.cu.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"

struct wf4dvar_ctx_s {
  wf::Ctx c;
};

static std::string g_create_error;

namespace wf {

void Ctx::prof_begin(int cls, double flops_, double bytes_, cudaEvent_t *ev) {
  *ev = nullptr;
  if (!prof.on) return;
  prof.launches[cls]++;
  prof.flops[cls] += flops_;
  prof.bytes[cls] += bytes_;
  cudaEvent_t a;
  if (!prof.pool.empty()) { a = prof.pool.back(); prof.pool.pop_back(); }
  else cudaEventCreate(&a);
  cudaEventRecord(a, st);
  *ev = a;
}

void Ctx::prof_end(int cls, cudaEvent_t a) {
  if (!a) return;
  cudaEvent_t b;
  if (!prof.pool.empty()) { b = prof.pool.back(); prof.pool.pop_back(); }
  else cudaEventCreate(&b);
  cudaEventRecord(b, st);
  prof.pending.push_back({a, b, cls});
}

}  // namespace wf

using wf::Ctx;
using wf::Error;

// copy the preconditioner description, including the caller's pvec array
static void set_pc(Ctx &c, const wf4dvar_precond &pc) {
  c.pc = pc;
  c.pvec_store.clear();
  if (pc.pvec) {
    WF_REQUIRE(pc.npvec >= 1 && pc.npvec <= 512, WF4DVAR_EINVAL, "R_block: 1 <= npvec <= 512");
    for (int j = 0; j < pc.npvec; ++j) {
      WF_REQUIRE(pc.pvec[j] >= 1, WF4DVAR_EINVAL, "R_block: pvec entries must be >= 1");
      c.pvec_store.push_back(pc.pvec[j]);
    }
    c.pc.pvec = c.pvec_store.data();
  }
}

template <class F>
static wf4dvar_status guarded(wf4dvar_ctx ctx, F &&f) {
  if (!ctx) return WF4DVAR_EINVAL;
  try {
    cudaSetDevice(ctx->c.device);
    f(ctx->c);
    ctx->c.last_error.clear();
    return WF4DVAR_OK;
  } catch (const Error &e) {
    ctx->c.last_error = e.msg;
    return e.st;
  } catch (const std::exception &e) {
    ctx->c.last_error = e.what();
    return WF4DVAR_ECUDA;
  }
}

extern "C" {

const char *wf4dvar_version(void) {
  return "wf4dvar 0.1 (sm_100a, FP64 DMMA + cp.async; arXiv 2105.06975 hot path)";
}

wf4dvar_status wf4dvar_create(const wf4dvar_problem *prob, const wf4dvar_precond *pc,
                              const wf4dvar_dist *dist, wf4dvar_ctx *out) {
  if (!out) { g_create_error = "out is NULL"; return WF4DVAR_EINVAL; }
  *out = nullptr;
  wf4dvar_ctx h = new wf4dvar_ctx_s();
  Ctx &c = h->c;
  try {
    WF_REQUIRE(prob && pc, WF4DVAR_EINVAL, "prob/pc is NULL");
    const wf4dvar_problem &p = *prob;
    WF_REQUIRE(p.s >= 1 && p.p >= 1 && p.N >= 0 && p.m >= 1, WF4DVAR_EINVAL, "bad s/p/N/m");
    WF_REQUIRE(p.p <= p.s, WF4DVAR_EINVAL, "p must be <= s");
    WF_REQUIRE(p.B && p.Q && p.R && (p.H_idx || p.H_rowptr), WF4DVAR_EINVAL,
               "B/Q/R and H_idx or H_rowptr must be non-NULL");
    if (p.H_rowptr) {
      WF_REQUIRE(p.H_col && p.H_val && p.H_rowptr[0] == 0, WF4DVAR_EINVAL, "bad CSR H");
      for (int j = 0; j < p.p; ++j)
        WF_REQUIRE(p.H_rowptr[j + 1] >= p.H_rowptr[j], WF4DVAR_EINVAL, "CSR H rowptr not monotone");
      for (int k = 0; k < p.H_rowptr[p.p]; ++k)
        WF_REQUIRE(p.H_col[k] >= 0 && p.H_col[k] < p.s, WF4DVAR_EINVAL, "CSR H column out of range");
    } else {
      for (int j = 0; j < p.p; ++j) {
        WF_REQUIRE(p.H_idx[j] >= 0 && p.H_idx[j] < p.s, WF4DVAR_EINVAL, "H_idx out of range");
        if (j) WF_REQUIRE(p.H_idx[j] > p.H_idx[j - 1], WF4DVAR_EINVAL, "H_idx not strictly increasing");
      }
    }
    WF_REQUIRE(p.model == WF4DVAR_M_DENSE || p.model == WF4DVAR_M_HEAT || p.model == WF4DVAR_M_L96 ||
               p.model == WF4DVAR_M_HEAT_EXPLICIT, WF4DVAR_EINVAL, "unknown model");
    int rank = 0, world = 1;
    if (dist) {
      world = dist->world <= 0 ? 1 : dist->world;
      rank = dist->rank;
      WF_REQUIRE(rank >= 0 && rank < world, WF4DVAR_EINVAL, "dist: need 0 <= rank < world");
      WF_REQUIRE(world <= p.N + 1, WF4DVAR_EINVAL, "dist: world must be <= N+1 (windows)");
      c.device = dist->device;
      c.st = (cudaStream_t)dist->stream;
    }
    WF_CUDA(cudaSetDevice(c.device));
    if (const char *e = getenv("WF4DVAR_AUX_PRIORITY")) c.aux_priority = atoi(e) != 0;
    if (const char *e = getenv("WF4DVAR_FORK")) c.fork_on = atoi(e) != 0;
    for (int i = 0; i < 2; ++i) {
      // the aux streams carry the latency-bound triangular solves (D_hat^{-1},
      // R_hat^{-1}): highest priority, so their CTAs take SM slots as soon as
      // co-running GEMM CTAs retire and the GEMMs fill the idle tensor pipes
      int lo_pri = 0, hi_pri = 0;
      WF_CUDA(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
      WF_CUDA(cudaStreamCreateWithPriority(&c.aux[i], cudaStreamNonBlocking,
                                           c.aux_priority ? hi_pri : 0));
      WF_CUDA(cudaEventCreateWithFlags(&c.ev_join[i], cudaEventDisableTiming));
    }
    WF_CUDA(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
    {
      int lo_pri = 0, hi_pri = 0;
      WF_CUDA(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
      WF_CUDA(cudaStreamCreateWithPriority(&c.aux2, cudaStreamNonBlocking, c.aux_priority ? hi_pri : 0));
      WF_CUDA(cudaStreamCreateWithFlags(&c.kside, cudaStreamNonBlocking));
      WF_CUDA(cudaEventCreateWithFlags(&c.ev_kfork, cudaEventDisableTiming));
      WF_CUDA(cudaEventCreateWithFlags(&c.ev_kjoin, cudaEventDisableTiming));
      for (auto &e : c.ev_split) WF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    WF_CUDA(cudaEventCreateWithFlags(&c.ev_halo, cudaEventDisableTiming));
    WF_CUDA(cudaStreamCreateWithFlags(&c.cpy, cudaStreamNonBlocking));
    for (auto &e : c.ev_in) WF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto &e : c.ev_chunk) WF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.s = p.s; c.p = p.p; c.N = p.N; c.WG = p.N + 1; c.m = p.m; c.model = p.model;
    int wb = 0, we = c.WG;
    wf::partition(c.WG, world, rank, &wb, &we);
    c.w0 = wb;
    c.W = we - wb;
    c.ncol = (int64_t)c.W * c.m;
    if (world > 1 || (dist && dist->transport != WF4DVAR_TRANSPORT_NONE)) {
      c.comm = wf::make_comm(*dist);
      const size_t sm = (size_t)c.s * c.m;
      c.halo_lo = c.alloc<double>(sm);
      c.halo_hi = c.alloc<double>(sm);
      c.pack_lo = c.alloc<double>(sm);
      c.pack_hi = c.alloc<double>(sm);
      c.gath = c.alloc<double>(sm * world);
      WF_CUDA(cudaMemsetAsync(c.halo_lo, 0, sm * 8, c.st));
      WF_CUDA(cudaMemsetAsync(c.halo_hi, 0, sm * 8, c.st));
    }
    c.n = (int64_t)(2 * c.s + c.p) * c.ncol;
    c.B = c.alloc<double>((size_t)c.s * c.s);
    c.Q = c.alloc<double>((size_t)c.s * c.s);
    c.R = c.alloc<double>((size_t)c.p * c.p);
    WF_CUDA(memcpy_sync(c, c.B, p.B, (size_t)c.s * c.s * 8, cudaMemcpyHostToDevice));
    WF_CUDA(memcpy_sync(c, c.Q, p.Q, (size_t)c.s * c.s * 8, cudaMemcpyHostToDevice));
    WF_CUDA(memcpy_sync(c, c.R, p.R, (size_t)c.p * c.p * 8, cudaMemcpyHostToDevice));
    // compact-support covariances: column ranges of their non-zero tiles
    register_tile_ranges(c, c.B, c.s, c.s, c.s);
    register_tile_ranges(c, c.Q, c.s, c.s, c.s);
    register_tile_ranges(c, c.R, c.p, c.p, c.p);
    if (p.H_rowptr) {
      // general H_i: CSR and its transpose (built here, host side)
      c.H_general = true;
      const int nnz = p.H_rowptr[c.p];
      std::vector<int> trp(c.s + 1, 0), tcol(nnz);
      std::vector<double> tval(nnz);
      for (int k = 0; k < nnz; ++k) trp[p.H_col[k] + 1]++;
      for (int i = 0; i < c.s; ++i) trp[i + 1] += trp[i];
      std::vector<int> fill(trp.begin(), trp.end() - 1);
      for (int j = 0; j < c.p; ++j)
        for (int k = p.H_rowptr[j]; k < p.H_rowptr[j + 1]; ++k) {
          int dst = fill[p.H_col[k]]++;
          tcol[dst] = j;
          tval[dst] = p.H_val[k];
        }
      c.Hrp = c.alloc<int>(c.p + 1); c.Hcol = c.alloc<int>(nnz); c.Hval = c.alloc<double>(nnz);
      c.HTrp = c.alloc<int>(c.s + 1); c.HTcol = c.alloc<int>(nnz); c.HTval = c.alloc<double>(nnz);
      WF_CUDA(memcpy_sync(c, c.Hrp, p.H_rowptr, (c.p + 1) * 4, cudaMemcpyHostToDevice));
      if (nnz) {
        WF_CUDA(memcpy_sync(c, c.Hcol, p.H_col, nnz * 4, cudaMemcpyHostToDevice));
        WF_CUDA(memcpy_sync(c, c.Hval, p.H_val, nnz * 8, cudaMemcpyHostToDevice));
        WF_CUDA(memcpy_sync(c, c.HTcol, tcol.data(), nnz * 4, cudaMemcpyHostToDevice));
        WF_CUDA(memcpy_sync(c, c.HTval, tval.data(), nnz * 8, cudaMemcpyHostToDevice));
      }
      WF_CUDA(memcpy_sync(c, c.HTrp, trp.data(), (c.s + 1) * 4, cudaMemcpyHostToDevice));
    } else {
      c.H_idx = c.alloc<int>(c.p);
      c.H_inv = c.alloc<int>(c.s);
      std::vector<int> inv(c.s, -1);
      for (int j = 0; j < c.p; ++j) inv[p.H_idx[j]] = j;
      WF_CUDA(memcpy_sync(c, c.H_idx, p.H_idx, c.p * 4, cudaMemcpyHostToDevice));
      WF_CUDA(memcpy_sync(c, c.H_inv, inv.data(), c.s * 4, cudaMemcpyHostToDevice));
    }
    wf::setup_model(c, p);
    // CUDA graphs for launch-bound sizes (per-iteration GPU work well under the
    // ~50 launches' overhead); WF4DVAR_GRAPHS=0/1 forces
    c.use_graphs = c.n <= (int64_t)8 << 20;
    if (const char *e = getenv("WF4DVAR_GRAPHS")) c.use_graphs = atoi(e) != 0;
    c.ws_seg = c.alloc<double>((size_t)c.s * c.ncol);
    // dot partials: gy <= 2*148 blocks x up to 4 dots x m
    c.dot_part_cap = 8 * 148 * 4 * std::max(c.m, 256) + 4096;
    c.dot_part = c.alloc<double>(c.dot_part_cap);
    WF_CUDA(cudaMallocHost((void **)&c.hpin, 16 * sizeof(int)));
    set_pc(c, *pc);
    wf::setup_precond(c);
    WF_CUDA(cudaStreamSynchronize(c.st));
  } catch (const Error &e) {
    g_create_error = e.msg;
    wf4dvar_destroy(h);
    return e.st;
  } catch (const std::exception &e) {
    g_create_error = e.what();
    wf4dvar_destroy(h);
    return WF4DVAR_ECUDA;
  }
  *out = h;
  return WF4DVAR_OK;
}

wf4dvar_status wf4dvar_set_precond(wf4dvar_ctx ctx, const wf4dvar_precond *pc) {
  return guarded(ctx, [&](Ctx &c) {
    WF_REQUIRE(pc, WF4DVAR_EINVAL, "pc is NULL");
    WF_CUDA(cudaStreamSynchronize(c.st));
    set_pc(c, *pc);
    wf::setup_precond(c);
  });
}

wf4dvar_status wf4dvar_destroy(wf4dvar_ctx ctx) {
  if (!ctx) return WF4DVAR_EINVAL;
  Ctx &c = ctx->c;
  cudaSetDevice(c.device);
  if (c.st) cudaStreamSynchronize(c.st); else cudaDeviceSynchronize();
  for (int i = 0; i < 2; ++i) {
    if (c.aux[i]) { cudaStreamSynchronize(c.aux[i]); cudaStreamDestroy(c.aux[i]); }
    if (c.ev_join[i]) cudaEventDestroy(c.ev_join[i]);
  }
  if (c.ev_fork) cudaEventDestroy(c.ev_fork);
  if (c.aux2) { cudaStreamSynchronize(c.aux2); cudaStreamDestroy(c.aux2); }
  if (c.kside) { cudaStreamSynchronize(c.kside); cudaStreamDestroy(c.kside); }
  if (c.ev_kfork) cudaEventDestroy(c.ev_kfork);
  if (c.ev_kjoin) cudaEventDestroy(c.ev_kjoin);
  for (auto &e : c.ev_split) if (e) cudaEventDestroy(e);
  if (c.ev_halo) cudaEventDestroy(c.ev_halo);
  if (c.cpy) { cudaStreamSynchronize(c.cpy); cudaStreamDestroy(c.cpy); }
  for (auto &e : c.ev_in) if (e) cudaEventDestroy(e);
  for (auto &e : c.ev_chunk) if (e) cudaEventDestroy(e);
  c.drop_graphs();
  if (c.own_st) { cudaStreamSynchronize(c.own_st); cudaStreamDestroy(c.own_st); }
  delete c.comm;
  c.comm = nullptr;
  for (auto &e : c.sk_states) {
    if (e.ws) cudaFree(e.ws);
    if (e.flags) cudaFree(e.flags);
    if (e.splitk) cudaFree(e.splitk);
    if (e.df_flags) cudaFree(e.df_flags);
    if (e.df_ep) cudaFree(e.df_ep);
  }
  for (void *p : c.retired) cudaFree(p);
  for (void *p : c.allocs) cudaFree(p);
  for (auto &pe : c.prof.pending) { cudaEventDestroy(pe.a); cudaEventDestroy(pe.b); }
  for (auto e : c.prof.pool) cudaEventDestroy(e);
  if (c.hostbuf) cudaFreeHost(c.hostbuf);
  if (c.hpin) cudaFreeHost(c.hpin);
  if (c.kws) cudaFree(c.kws);
  for (auto e : c.iter_events) cudaEventDestroy(e);
  if (c.ev_init) cudaEventDestroy(c.ev_init);
  delete ctx;
  return WF4DVAR_OK;
}

wf4dvar_status wf4dvar_local_windows(wf4dvar_ctx ctx, int32_t *w_begin, int32_t *w_end) {
  return guarded(ctx, [&](Ctx &c) {
    WF_REQUIRE(w_begin && w_end, WF4DVAR_EINVAL, "NULL output");
    *w_begin = c.w0;
    *w_end = c.w0 + c.W;
  });
}

wf4dvar_status wf4dvar_vector_len(wf4dvar_ctx ctx, int64_t *n_local) {
  return guarded(ctx, [&](Ctx &c) {
    WF_REQUIRE(n_local, WF4DVAR_EINVAL, "NULL output");
    *n_local = c.n;
  });
}

wf4dvar_status wf4dvar_apply_A(wf4dvar_ctx ctx, const double *x, double *y) {
  return guarded(ctx, [&](Ctx &c) {
    WF_REQUIRE(x && y && x != y, WF4DVAR_EINVAL, "apply_A: bad pointers");
    wf::apply_A(c, x, y);
  });
}

wf4dvar_status wf4dvar_apply_P(wf4dvar_ctx ctx, const double *x, double *y) {
  return guarded(ctx, [&](Ctx &c) {
    WF_REQUIRE(x && y && x != y, WF4DVAR_EINVAL, "apply_P: bad pointers");
    wf::apply_P(c, x, y);
  });
}

wf4dvar_status wf4dvar_apply_AP(wf4dvar_ctx ctx, const double *x, double *t, double *y) {
  return guarded(ctx, [&](Ctx &c) {
    WF_REQUIRE(x && t && y && x != t && t != y && x != y, WF4DVAR_EINVAL, "apply_AP: bad pointers");
    wf::apply_P(c, x, t);
    wf::apply_A(c, t, y);
  });
}

wf4dvar_status wf4dvar_apply_AP_host(wf4dvar_ctx ctx, const double *x_host, double *y_host) {
  return guarded(ctx, [&](Ctx &c) {
    WF_REQUIRE(x_host && y_host, WF4DVAR_EINVAL, "apply_AP_host: bad pointers");
    if (!c.dev_io_x) {
      c.dev_io_x = c.alloc<double>(c.n);
      c.dev_io_t = c.alloc<double>(c.n);
      c.dev_io_y = c.alloc<double>(c.n);
    }
    // block-wise copies overlapped with the blocks' solves / products (see apply_P /
    // apply_A): the input blocks land in the order the streams consume them, each
    // output block leaves as soon as it is computed
    wf::apply_P(c, c.dev_io_x, c.dev_io_t, x_host);
    wf::apply_A(c, c.dev_io_t, c.dev_io_y, y_host);
    WF_CUDA(cudaStreamSynchronize(c.st));
  });
}

wf4dvar_status wf4dvar_solve(wf4dvar_ctx ctx, const double *rhs, double *x,
                             const wf4dvar_solve_opts *opts, wf4dvar_report *rep) {
  return guarded(ctx, [&](Ctx &c) {
    WF_REQUIRE(rhs && x && opts && rhs != x, WF4DVAR_EINVAL, "solve: bad pointers");
    wf::solve(c, rhs, x, *opts, rep);
  });
}

wf4dvar_status wf4dvar_solve_host(wf4dvar_ctx ctx, const double *rhs_host, double *x_host,
                                  const wf4dvar_solve_opts *opts, wf4dvar_report *rep) {
  return guarded(ctx, [&](Ctx &c) {
    WF_REQUIRE(rhs_host && x_host && opts, WF4DVAR_EINVAL, "solve_host: bad pointers");
    if (!c.dev_io_x) {
      c.dev_io_x = c.alloc<double>(c.n);
      c.dev_io_t = c.alloc<double>(c.n);
      c.dev_io_y = c.alloc<double>(c.n);
    }
    WF_CUDA(cudaMemcpyAsync(c.dev_io_x, rhs_host, c.n * 8, cudaMemcpyHostToDevice, c.st));
    wf4dvar_status st = WF4DVAR_OK;
    try {
      wf::solve(c, c.dev_io_x, c.dev_io_y, *opts, rep);
    } catch (const Error &e) {
      if (e.st != WF4DVAR_ENOCONV) throw;
      st = e.st;
      c.last_error = e.msg;
    }
    WF_CUDA(cudaMemcpyAsync(x_host, c.dev_io_y, c.n * 8, cudaMemcpyDeviceToHost, c.st));
    WF_CUDA(cudaStreamSynchronize(c.st));
    if (st != WF4DVAR_OK) throw Error{st, c.last_error};
  });
}

wf4dvar_status wf4dvar_outer_loop(wf4dvar_ctx ctx, const double *xb, const double *y, double *x,
                                  int32_t n_outer, const wf4dvar_solve_opts *inner,
                                  int32_t *inner_iters, double *dx_norm2, double *res_norm2) {
  return guarded(ctx, [&](Ctx &c) {
    WF_REQUIRE(y && x && inner, WF4DVAR_EINVAL, "outer_loop: bad pointers");
    WF_REQUIRE(xb || c.w0 > 0, WF4DVAR_EINVAL, "outer_loop: xb is NULL on the rank owning window 0");
    wf::outer_loop(c, xb, y, x, n_outer, *inner, inner_iters, dx_norm2, res_norm2);
  });
}

wf4dvar_status wf4dvar_lanczos(wf4dvar_ctx ctx, int32_t op, const double *v0, int32_t steps,
                               double *ritz_min, double *ritz_max, double *alpha, double *beta) {
  return guarded(ctx, [&](Ctx &c) {
    WF_REQUIRE(v0, WF4DVAR_EINVAL, "lanczos: v0 is NULL");
    wf::lanczos(c, op, v0, steps, ritz_min, ritz_max, alpha, beta);
  });
}

wf4dvar_status wf4dvar_profile_enable(wf4dvar_ctx ctx, int32_t enable) {
  return guarded(ctx, [&](Ctx &c) {
    WF_CUDA(cudaStreamSynchronize(c.st));
    for (auto &pe : c.prof.pending) { c.prof.pool.push_back(pe.a); c.prof.pool.push_back(pe.b); }
    c.prof.pending.clear();
    for (int k = 0; k < wf::K_NCLASS; ++k) {
      c.prof.launches[k] = 0; c.prof.flops[k] = 0; c.prof.bytes[k] = 0; c.prof.ms[k] = 0;
    }
    c.prof.on = enable != 0;
  });
}

wf4dvar_status wf4dvar_profile_read(wf4dvar_ctx ctx, wf4dvar_kstat *out, int32_t max_n,
                                    int32_t *n_out) {
  return guarded(ctx, [&](Ctx &c) {
    WF_CUDA(cudaStreamSynchronize(c.st));
    for (auto &pe : c.prof.pending) {
      float ms = 0;
      cudaEventElapsedTime(&ms, pe.a, pe.b);
      c.prof.ms[pe.cls] += ms;
      c.prof.pool.push_back(pe.a);
      c.prof.pool.push_back(pe.b);
    }
    c.prof.pending.clear();
    int n = std::min<int>(max_n, wf::K_NCLASS);
    for (int k = 0; k < n; ++k) {
      memset(out[k].name, 0, sizeof(out[k].name));
      strncpy(out[k].name, wf::kClassName[k], sizeof(out[k].name) - 1);
      out[k].launches = c.prof.launches[k];
      out[k].ms = c.prof.ms[k];
      out[k].flops = c.prof.flops[k];
      out[k].bytes = c.prof.bytes[k];
    }
    if (n_out) *n_out = n;
  });
}

int64_t wf4dvar_launch_count(wf4dvar_ctx ctx) { return ctx ? ctx->c.launches : -1; }

wf4dvar_status wf4dvar_partition(int32_t W, int32_t world, int32_t rank, int32_t *w_begin,
                                 int32_t *w_end) {
  if (!w_begin || !w_end || W < 1 || world < 1 || world > W || rank < 0 || rank >= world)
    return WF4DVAR_EINVAL;
  int b, e;
  wf::partition(W, world, rank, &b, &e);
  *w_begin = b;
  *w_end = e;
  return WF4DVAR_OK;
}

wf4dvar_status wf4dvar_chain_plan(int32_t W, int32_t k, int32_t w_begin, int32_t w_end,
                                  int32_t transpose, wf4dvar_chain_step *out, int32_t max_steps,
                                  int32_t *n_steps) {
  if (W < 1 || k < 1 || k > W || w_begin < 0 || w_end <= w_begin || w_end > W || !n_steps)
    return WF4DVAR_EINVAL;
  std::vector<wf::ChainStep> plan = wf::chain_plan(W, k, w_begin, w_end, transpose != 0);
  *n_steps = (int32_t)plan.size();
  for (int i = 0; i < (int)plan.size() && i < max_steps && out; ++i) {
    const wf::ChainStep &s = plan[i];
    out[i].j = s.j; out[i].recv = s.recv; out[i].send = s.send; out[i].nl = s.nl;
    for (int l = 0; l < 2; ++l) {
      out[i].first[l] = s.first[l]; out[i].stride[l] = s.stride[l]; out[i].count[l] = s.count[l];
    }
  }
  return WF4DVAR_OK;
}

wf4dvar_status wf4dvar_rblock_plan(const double *R, int32_t p, const int32_t *pvec, int32_t npvec,
                                   double block_tol, int32_t maxsize, int32_t numproc,
                                   int32_t *starts_out, int32_t max_out, int32_t *n_out) {
  if (!R || p < 1 || !pvec || npvec < 1 || !n_out) return WF4DVAR_EINVAL;
  try {
    std::vector<double> Rh(R, R + (size_t)p * p);
    std::vector<int> pv(pvec, pvec + npvec);
    std::vector<int> st = wf::algorithm1_blocks(Rh, p, pv, block_tol, maxsize, numproc);
    *n_out = (int32_t)st.size();
    for (int i = 0; i < (int)st.size() && i < max_out && starts_out; ++i) starts_out[i] = st[i];
  } catch (const Error &e) {
    g_create_error = e.msg;
    return e.st;
  }
  return WF4DVAR_OK;
}

wf4dvar_status wf4dvar_nccl_unique_id(void *out128) {
  if (!out128) return WF4DVAR_EINVAL;
  try {
    wf::nccl_unique_id(out128);
  } catch (const Error &e) {
    g_create_error = e.msg;
    return e.st;
  }
  return WF4DVAR_OK;
}

wf4dvar_status wf4dvar_local_group_create(int32_t world, void **out) {
  if (!out || world < 1 || world > 64) return WF4DVAR_EINVAL;
  *out = wf::local_group_create(world);
  return WF4DVAR_OK;
}

wf4dvar_status wf4dvar_local_group_destroy(void *group) {
  if (!group) return WF4DVAR_EINVAL;
  wf::local_group_destroy((wf::LocalGroup *)group);
  return WF4DVAR_OK;
}

const char *wf4dvar_last_error(wf4dvar_ctx ctx) {
  if (!ctx) return g_create_error.c_str();
  return ctx->c.last_error.c_str();
}

}  // extern "C"

// ---------------------------------------------------------------- test hooks
#include "../../include/wf4dvar_testing.h"

extern "C" int wf4dvar_test_gemm(int M, int N, int K, double alpha, const double *A, int64_t lda,
                                 const double *X, int64_t ldx, double beta, const double *Z,
                                 int64_t ldz, double *Y, int64_t ldy, void *stream) {
  if (M < 0 || N < 0 || K < 0 || !A || !X || !Y) return WF4DVAR_EINVAL;
  try {
    static thread_local Ctx c;   // persistent: keeps the stream-K workspace across calls
    c.st = (cudaStream_t)stream;
    wf::GemmProb g{};
    g.A = A; g.lda = lda; g.X = X; g.ldx = ldx; g.Y = Y; g.ldy = ldy; g.Z = Z; g.ldz = ldz;
    g.M = M; g.N = N; g.K = K; g.alpha = alpha; g.beta = Z ? beta : 0.0;
    wf::launch_gemm(c, &g, 1, 1);
  } catch (const Error &e) {
    return e.st;
  }
  return 0;
}

extern "C" int wf4dvar_test_trsm(int n, int ncols, int upper, int blk, const double *G,
                                 const double *X, double *Y, void *stream) {
  if (n <= 0 || ncols <= 0 || !G || !X || !Y || blk < 0) return WF4DVAR_EINVAL;
  try {
    static thread_local Ctx c;
    c.st = (cudaStream_t)stream;
    wf::TrsmProb p{G, n, X, ncols, Y, ncols, n, ncols, blk};
    // the production path uses setup-time diagonal-tile packs: rebuild one on the same
    // stream for every call (an address-keyed cache could go stale when the caller
    // reuses memory), into a per-thread buffer grown on demand
    static thread_local double *pk = nullptr;
    static thread_local size_t pk_cap = 0;
    const size_t need = wf::diag_pack_doubles(n);
    if (need > pk_cap) {
      if (pk) cudaFree(pk);
      WF_CUDA(cudaMalloc(&pk, need * 8));
      pk_cap = need;
    }
    wf::fill_diag_pack(c, G, n, upper != 0, pk);
    p.dpack = pk;
    wf::launch_trsm(c, &p, 1, upper != 0);
  } catch (const Error &e) {
    return e.st;
  }
  return 0;
}
