// fls_comm.cu -- the multi-rank half of the C ABI: communicator (fls_comm_*) and the TSQR
// least-squares solve behind fls_solve / fls_solve_mu when a communicator is attached.
//
// Product code.  Paper = PAPER.md (arxiv 2602.10541), cited P:L<line>.
//
// Alg. 1 line 5 ("beta* = argmin ||A beta - b||^2 via QR") over row-sharded [A | b]
// (SURVEY §8(e)), with the Tikhonov term of P:L156-160 (reading A16: sqrt(mu) = tau ||A||_F,
// ||A||_F^2 summed over the ranks):
//
//   local:  [A_r | b_r] = Q_r [R_r | c_r]                     (geqrf on each GPU)
//   gather: R_0 .. R_{P-1} -> root                            (transport below)
//   root:   [R_0 | c_0; ...; R_{P-1} | c_{P-1}; sqrt(mu) I | 0] = Q R  (structured stacked QR)
//           beta = R^-1 (Q^T b)[0:F],  residual |R(F, F)|
//   bcast:  beta and the residual to every rank
//
// Transports of the R factors (the one data exchange):
//   P2P  -- the root allocates the stacking buffer and exports it by CUDA IPC; every rank maps it
//           and its R-extraction kernel stores the upper trapezoid of its factor straight into
//           the root's memory over NVLink / NVSwitch (the kernel's stores ARE the transfer, no
//           staging copy); beta comes back through the same mapping.
//   NCCL -- grouped ncclSend / ncclRecv of each rank's zero-padded factor into the root's
//           block-contiguous stack, ncclBroadcast of beta.
// AUTO (default) tries P2P and falls back to NCCL when any rank cannot map the buffer.
//
// Control plane (small host-semantics allgathers that agree on sizes, norms and per-rank
// status before every step that could otherwise leave a peer waiting): the NCCL communicator
// (fls_comm_init, ncclUniqueId passed by the caller), or caller-supplied host callbacks
// (fls_comm_init_host; e.g. torch.distributed / MPI / gloo), which also lets several processes
// share one GPU in tests (NCCL refuses two ranks on one device).  NCCL is loaded at run time
// (dlopen "libnccl.so.2", FLS_NCCL_LIB overrides), so libfls loads where NCCL is absent and
// fls_comm_init then returns FLS_ENCCL.
#include <dlfcn.h>
#include <nccl.h>  // types and enums only; every function is resolved by dlsym

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "fls_ctx.h"

namespace fls {

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

template <class T>
bool sym(void *h, const char *name, T &fn) {
  fn = reinterpret_cast<T>(dlsym(h, name));
  return fn != nullptr;
}

NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *path = getenv("FLS_NCCL_LIB");
    // a process that already loaded NCCL (e.g. torch) gets that copy back: dlopen matches the
    // soname of loaded libraries first
    void *h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      const char *e = dlerror();
      api.err = std::string("cannot load NCCL: ") + (e ? e : "dlopen failed");
      return;
    }
    bool ok = sym(h, "ncclGetUniqueId", api.GetUniqueId) && sym(h, "ncclCommInitRank", api.CommInitRank) &&
              sym(h, "ncclCommDestroy", api.CommDestroy) && sym(h, "ncclAllGather", api.AllGather) &&
              sym(h, "ncclBroadcast", api.Broadcast) && sym(h, "ncclSend", api.Send) &&
              sym(h, "ncclRecv", api.Recv) && sym(h, "ncclGroupStart", api.GroupStart) &&
              sym(h, "ncclGroupEnd", api.GroupEnd) && sym(h, "ncclGetErrorString", api.GetErrorString);
    if (!ok) {
      api.err = "NCCL library lacks a required symbol";
      return;
    }
    api.ok = true;
  });
  return api;
}

fls_status nccl_fail(ncclResult_t r, const char *where) {
  return fail(FLS_ENCCL, "%s: %s", where, nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
}

#define FLS_NCCL(call)                                   \
  do {                                                   \
    ncclResult_t r_ = (call);                            \
    if (r_ != ncclSuccess) return nccl_fail(r_, #call);  \
  } while (0)

}  // namespace

enum : int32_t { kTransportNone = 0 };

struct Comm {
  int32_t nranks = 1, rank = 0;
  bool is_nccl = false;
  ncclComm_t nc = nullptr;
  fls_host_coll host = {nullptr, nullptr};
  int32_t transport = FLS_TSQR_AUTO;
  int32_t force_tsqr = 0;
  int32_t last_transport = kTransportNone;
  char *dstage = nullptr;  // device staging of the NCCL control plane (grow-only)
  size_t dstage_bytes = 0;
  double *sendbuf = nullptr;  // NCCL transport: this rank's zero-padded factor (grow-only)
  size_t send_bytes = 0;
  double *gat = nullptr;  // NCCL transport, root: the block-contiguous stack (grow-only)
  size_t gat_bytes = 0;
};

namespace {

fls_status grow(void *&p, size_t &cap, size_t bytes, cudaStream_t st, const char *what) {
  if (bytes <= cap) return FLS_OK;
  cudaStreamSynchronize(st);
  cudaFree(p);
  p = nullptr;
  cap = 0;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(FLS_ENOMEM, "%s: %zu bytes", what, bytes);
  }
  cap = bytes;
  return FLS_OK;
}

// every rank contributes `bytes` from send; recv (nranks * bytes, host) gets rank r's at r*bytes
fls_status allgather(fls_ctx *ctx, const void *send, void *recv, size_t bytes) {
  Comm *c = ctx->comm;
  if (!c->is_nccl) {
    if (c->host.allgather(c->host.user, send, recv, (int64_t)bytes) != 0)
      return fail(FLS_ENCCL, "host allgather callback failed (%zu bytes)", bytes);
    return FLS_OK;
  }
  const size_t slot = (bytes + 255) & ~size_t(255);
  void *p = c->dstage;
  if (fls_status s = grow(p, c->dstage_bytes, slot * (c->nranks + 1), ctx->stream, "NCCL staging"))
    return s;
  c->dstage = static_cast<char *>(p);
  FLS_CUDA(cudaMemcpyAsync(c->dstage, send, bytes, cudaMemcpyHostToDevice, ctx->stream));
  // recv slots are `bytes` apart (NCCL allgather layout), after the send slot
  FLS_NCCL(nccl().AllGather(c->dstage, c->dstage + slot, bytes, ncclUint8, c->nc, ctx->stream));
  FLS_CUDA(cudaMemcpyAsync(recv, c->dstage + slot, bytes * c->nranks, cudaMemcpyDeviceToHost,
                           ctx->stream));
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  return FLS_OK;
}

// agreement step: every rank publishes its status; returns the first failing rank's status
// (its own message is kept on that rank; the others report which rank failed)
fls_status agree(fls_ctx *ctx, fls_status mine, const char *step) {
  Comm *c = ctx->comm;
  std::string keep = mine ? fls_last_error() : "";
  std::vector<int32_t> all(c->nranks);
  const int32_t m = (int32_t)mine;
  if (fls_status s = allgather(ctx, &m, all.data(), sizeof m)) return s;
  for (int r = 0; r < c->nranks; ++r) {
    if (all[r] == FLS_OK) continue;
    if (r == c->rank) return fail(mine, "%s (rank %d): %s", step, r, keep.c_str());
    return fail((fls_status)all[r], "%s failed on rank %d (%s there)", step, r,
                fls_status_string((fls_status)all[r]));
  }
  return FLS_OK;
}

struct Plan {
  int32_t P = 1, root = 0;
  int64_t F = 0, nc = 0, k = 0, kmax = 0;
  double sqrt_mu = 0.0;
};

// P2P transport.  *fell_back = true (and FLS_OK) when some rank could not map the root's
// buffer: nothing has been exchanged yet and the caller switches to NCCL.
fls_status tsqr_p2p(fls_ctx *ctx, const Plan &pl, double *Ab, int64_t lda, fls_status qr_status,
                    double *beta, double *resid_norm, bool *fell_back) {
  Comm *c = ctx->comm;
  *fell_back = false;
  const bool root = c->rank == pl.root;
  const size_t stack = (size_t)pl.P * pl.kmax * pl.nc;       // doubles of the factor stack
  const size_t total = stack + (size_t)pl.nc;                // + tail: beta (F), residual
  double *S = nullptr;       // root: its allocation
  double *base = nullptr;    // every rank: where the stack starts in this process
  struct {
    uint8_t h[FLS_IPC_HANDLE_BYTES];
    int32_t status;
    int32_t pad;
  } mine = {}, *hs = nullptr;
  std::vector<uint8_t> hbuf;
  fls_status st = FLS_OK;
  if (root) {
    if (cudaMalloc((void **)&S, total * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      st = fail(FLS_ENOMEM, "TSQR stack of %zu bytes", total * sizeof(double));
    } else {
      cudaError_t e = cudaMemsetAsync(S, 0, total * sizeof(double), ctx->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
      cudaIpcMemHandle_t h;
      if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, S);
      // test hook: FLS_TEST_NO_IPC=1 makes the export fail (e.g. a VMM allocator), =2 makes
      // the other ranks' mapping fail (no peer access), so the fallback paths run on a machine
      // where IPC works
      const char *no_ipc = getenv("FLS_TEST_NO_IPC");
      if (e == cudaSuccess && no_ipc && *no_ipc == '1') e = cudaErrorNotSupported;
      if (e != cudaSuccess) {
        cudaGetLastError();
        mine.status = -1;  // cannot export (e.g. allocator without IPC): fall back
      } else {
        std::memcpy(mine.h, &h, sizeof h);
      }
      base = S;
    }
  }
  mine.status = st != FLS_OK ? (int32_t)st : mine.status;
  hbuf.resize(sizeof mine * pl.P);
  if (fls_status s = allgather(ctx, &mine, hbuf.data(), sizeof mine)) {
    cudaFree(S);
    return s;
  }
  hs = reinterpret_cast<decltype(hs)>(hbuf.data());
  const int32_t root_status = hs[pl.root].status;
  if (root_status > 0) {  // root allocation failed: every rank returns that error
    cudaFree(S);
    return root ? st : fail((fls_status)root_status, "TSQR: root allocation failed");
  }
  int32_t ipc_ok = root_status == 0 ? 1 : 0;
  if (!root && ipc_ok) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hs[pl.root].h, sizeof h);
    void *p = nullptr;
    const char *no_ipc = getenv("FLS_TEST_NO_IPC");
    if ((no_ipc && *no_ipc == '2') ||
        cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ipc_ok = 0;
    } else {
      base = static_cast<double *>(p);
    }
  }
  // agree: mapped everywhere, and every local QR succeeded
  struct {
    int32_t ipc_ok, qr;
  } flags = {ipc_ok, (int32_t)qr_status};
  std::vector<decltype(flags)> all(pl.P);
  auto cleanup = [&]() {
    if (!root && base) cudaIpcCloseMemHandle(base);
    if (root) cudaFree(S);
  };
  std::string keep = qr_status ? fls_last_error() : "";
  if (fls_status s = allgather(ctx, &flags, all.data(), sizeof flags)) {
    cleanup();
    return s;
  }
  for (int r = 0; r < pl.P; ++r)
    if (all[r].qr != FLS_OK) {
      cleanup();
      if (r == c->rank) return fail(qr_status, "local QR (rank %d): %s", r, keep.c_str());
      return fail((fls_status)all[r].qr, "local QR failed on rank %d", r);
    }
  for (int r = 0; r < pl.P; ++r)
    if (!all[r].ipc_ok) {
      cleanup();
      *fell_back = true;
      return FLS_OK;
    }
  // the exchange: this rank's R-extraction kernel writes its trapezoid into the root's stack
  st = FLS_OK;
  if (pl.k > 0) {
    cudaError_t e = launch_copy_upper(Ab, lda, pl.k, pl.nc, base + (size_t)c->rank * pl.kmax * pl.nc,
                                      pl.kmax, ctx->stream, pl.kmax, /*upper_only=*/true);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) st = cuda_fail(e, "TSQR peer store");
  }
  if (fls_status s = agree(ctx, st, "TSQR peer store")) {
    cleanup();
    return s;
  }
  // root: structured QR of the stack + trsv; beta and the residual into the tail
  double res = 0.0;
  if (root) {
    st = solve_stacked_impl(ctx, S, pl.P, pl.kmax, pl.kmax * pl.nc, pl.kmax, pl.F, pl.sqrt_mu,
                            beta, &res);
    if (st == FLS_OK) {
      cudaError_t e = cudaMemcpyAsync(S + stack, beta, pl.F * sizeof(double),
                                      cudaMemcpyDeviceToDevice, ctx->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
      if (e != cudaSuccess) st = cuda_fail(e, "TSQR beta publish");
    }
  }
  struct {
    int32_t status, pad;
    double res;
  } rs = {(int32_t)st, 0, res};
  std::vector<decltype(rs)> rall(pl.P);
  std::string rkeep = st ? fls_last_error() : "";
  if (fls_status s = allgather(ctx, &rs, rall.data(), sizeof rs)) {
    cleanup();
    return s;
  }
  if (rall[pl.root].status != FLS_OK) {
    cleanup();
    if (root) return fail(st, "TSQR root solve: %s", rkeep.c_str());
    return fail((fls_status)rall[pl.root].status, "TSQR root solve failed on rank %d (%s there)",
                pl.root, fls_status_string((fls_status)rall[pl.root].status));
  }
  st = FLS_OK;
  if (!root) {  // beta back over the same mapping (peer read)
    cudaError_t e = cudaMemcpyAsync(beta, base + stack, pl.F * sizeof(double), cudaMemcpyDefault,
                                    ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) st = cuda_fail(e, "TSQR beta read");
  }
  fls_status fin = agree(ctx, st, "TSQR beta read");  // nobody unmaps / frees before all read
  cleanup();
  if (fin) return fin;
  if (resid_norm) *resid_norm = rall[pl.root].res;
  c->last_transport = FLS_TSQR_P2P;
  return FLS_OK;
}

fls_status tsqr_nccl(fls_ctx *ctx, const Plan &pl, double *Ab, int64_t lda, fls_status qr_status,
                     double *beta, double *resid_norm) {
  Comm *c = ctx->comm;
  const bool root = c->rank == pl.root;
  const size_t blk = (size_t)pl.kmax * pl.nc;
  fls_status st = qr_status;
  if (st == FLS_OK) {
    void *p = c->sendbuf;
    // also the broadcast buffer of a non-root rank: [beta (F), residual, root status]
    st = grow(p, c->send_bytes, std::max(blk, (size_t)pl.nc + 1) * sizeof(double), ctx->stream,
              "TSQR send buffer");
    c->sendbuf = static_cast<double *>(p);
  }
  if (st == FLS_OK && root) {
    void *p = c->gat;
    st = grow(p, c->gat_bytes, (blk * pl.P + pl.nc + 1) * sizeof(double), ctx->stream,
              "TSQR stack");
    c->gat = static_cast<double *>(p);
  }
  if (st == FLS_OK) {
    cudaError_t e = pl.k > 0 ? launch_copy_upper(Ab, lda, pl.k, pl.nc, c->sendbuf, pl.kmax,
                                                 ctx->stream, pl.kmax, false)
                             : cudaMemsetAsync(c->sendbuf, 0, blk * sizeof(double), ctx->stream);
    if (e != cudaSuccess) st = cuda_fail(e, "TSQR factor extraction");
  }
  if (fls_status s = agree(ctx, st, "TSQR local factor")) return s;
  FLS_NCCL(nccl().GroupStart());
  if (root)
    for (int r = 0; r < pl.P; ++r)
      FLS_NCCL(nccl().Recv(c->gat + (size_t)r * blk, blk, ncclFloat64, r, c->nc, ctx->stream));
  FLS_NCCL(nccl().Send(c->sendbuf, blk, ncclFloat64, pl.root, c->nc, ctx->stream));
  FLS_NCCL(nccl().GroupEnd());
  // the broadcast buffer: [beta (F), residual, root status]; a non-root rank reuses its send
  // buffer (stream order: the send has completed before the broadcast writes it)
  double *bb = root ? c->gat + blk * pl.P : c->sendbuf;
  std::string rkeep;
  if (root) {
    double res = 0.0;
    st = solve_stacked_impl(ctx, c->gat, pl.P, pl.kmax, blk, pl.kmax, pl.F, pl.sqrt_mu, bb, &res);
    if (st) rkeep = fls_last_error();
    double tail[2] = {res, (double)(int32_t)st};
    FLS_CUDA(cudaMemcpyAsync(bb + pl.F, tail, sizeof tail, cudaMemcpyHostToDevice, ctx->stream));
  } else {
    FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  FLS_NCCL(nccl().Broadcast(bb, bb, pl.nc + 1, ncclFloat64, pl.root, c->nc, ctx->stream));
  double tail[2] = {0.0, 0.0};
  FLS_CUDA(cudaMemcpyAsync(tail, bb + pl.F, sizeof tail, cudaMemcpyDeviceToHost, ctx->stream));
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  const int32_t rst = (int32_t)tail[1];
  if (rst != FLS_OK) {
    if (root) return fail(st, "TSQR root solve: %s", rkeep.c_str());
    return fail((fls_status)rst, "TSQR root solve failed on rank %d (%s there)", pl.root,
                fls_status_string((fls_status)rst));
  }
  if (bb != beta)
    FLS_CUDA(cudaMemcpyAsync(beta, bb, pl.F * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (resid_norm) *resid_norm = tail[0];
  c->last_transport = FLS_TSQR_NCCL;
  return FLS_OK;
}

}  // namespace

void comm_destroy(fls_ctx *ctx) {
  Comm *c = ctx->comm;
  if (!c) return;
  if (c->is_nccl && c->nc && nccl().ok) nccl().CommDestroy(c->nc);
  cudaFree(c->dstage);
  cudaFree(c->sendbuf);
  cudaFree(c->gat);
  delete c;
  ctx->comm = nullptr;
}

fls_status comm_solve(fls_ctx *ctx, double *Ab, int64_t n_local, int64_t lda, int64_t F,
                      double ridge_rel, double sqrt_mu_abs, double *beta, double *resid_norm,
                      bool *handled, fls_status pending) {
  Comm *c = ctx->comm;
  *handled = false;
  if (!c || (c->nranks == 1 && !c->force_tsqr)) return FLS_OK;
  *handled = true;
  NvtxRange nvtx_("fls_solve TSQR");
  const bool relative = sqrt_mu_abs < 0.0;
  Plan pl;
  pl.P = c->nranks;
  pl.F = F;
  pl.nc = F + 1;
  pl.k = std::min<int64_t>(n_local, pl.nc);
  // step 0: local argument check and the local ||A_r||_F^2, then agree on sizes and the ridge
  fls_status st = pending;  // (its message is already in fls_last_error)
  if (st == FLS_OK && lda < n_local)
    st = fail(FLS_EINVAL, "lda %lld < n_local %lld", (long long)lda, (long long)n_local);
  double fro2 = 0.0;
  if (st == FLS_OK && relative && ridge_rel > 0.0 && n_local > 0)
    st = frob2_host(ctx, Ab, n_local, lda, F, &fro2);
  struct Hdr {
    int32_t status, pad;
    int64_t F, k;
    double fro2, ridge;
  } h = {(int32_t)st, 0, F, pl.k, fro2, relative ? ridge_rel : sqrt_mu_abs};
  std::string keep = st ? fls_last_error() : "";
  std::vector<Hdr> all(pl.P);
  if (fls_status s = allgather(ctx, &h, all.data(), sizeof h)) return s;
  for (int r = 0; r < pl.P; ++r) {
    if (all[r].status != FLS_OK) {
      if (r == c->rank) return fail(st, "%s", keep.c_str());
      return fail((fls_status)all[r].status, "fls_solve failed on rank %d (%s there)", r,
                  fls_status_string((fls_status)all[r].status));
    }
    if (all[r].F != F || all[r].ridge != h.ridge)
      return fail(FLS_EINVAL, "fls_solve: n_features / ridge differ between ranks (rank %d)", r);
  }
  double tot = 0.0;  // rank order: every rank sums the same values in the same order
  for (int r = 0; r < pl.P; ++r) {
    tot += all[r].fro2;
    pl.kmax = std::max(pl.kmax, all[r].k);
  }
  if (pl.kmax == 0) return fail(FLS_EINVAL, "fls_solve: no rows on any rank");
  pl.sqrt_mu = relative ? ridge_rel * std::sqrt(tot) : sqrt_mu_abs;
  // step 1: local Householder QR (R in the upper trapezoid of Ab)
  fls_status qr = FLS_OK;
  if (pl.k > 0) {
    qr = ensure_handles(ctx);
    if (qr == FLS_OK) qr = geqrf_inplace(ctx, Ab, n_local, lda, pl.nc);
  }
  // step 2: exchange + root solve + broadcast
  int32_t mode = c->transport;
  if (mode != FLS_TSQR_NCCL) {
    bool fell_back = false;
    fls_status s = tsqr_p2p(ctx, pl, Ab, lda, qr, beta, resid_norm, &fell_back);
    if (!fell_back) return s;
    if (mode == FLS_TSQR_P2P)
      return fail(FLS_EUNSUPPORTED, "TSQR: peer-memory transport unavailable (CUDA IPC mapping failed)");
  }
  if (!c->is_nccl)
    return fail(FLS_EUNSUPPORTED, "TSQR: peer-memory transport unavailable and no NCCL communicator");
  return tsqr_nccl(ctx, pl, Ab, lda, qr, beta, resid_norm);
}

}  // namespace fls

using namespace fls;

extern "C" {

fls_status fls_comm_unique_id(void *id) {
  if (!id) return fail(FLS_EINVAL, "id is NULL");
  NcclApi &api = nccl();
  if (!api.ok) return fail(FLS_ENCCL, "%s", api.err.c_str());
  static_assert(sizeof(ncclUniqueId) == FLS_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId u;
  FLS_NCCL(api.GetUniqueId(&u));
  std::memcpy(id, &u, sizeof u);
  return FLS_OK;
}

fls_status fls_comm_init(fls_ctx *ctx, const void *nccl_unique_id, int32_t nranks, int32_t rank) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (!nccl_unique_id) return fail(FLS_EINVAL, "nccl_unique_id is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(FLS_EINVAL, "rank %d not in [0, %d)", rank, nranks);
  if (ctx->comm) return fail(FLS_EINVAL, "ctx already has a communicator (fls_comm_destroy first)");
  NcclApi &api = nccl();
  if (!api.ok) return fail(FLS_ENCCL, "%s", api.err.c_str());
  DeviceGuard g(ctx->device);
  ncclUniqueId u;
  std::memcpy(&u, nccl_unique_id, sizeof u);
  ncclComm_t nc = nullptr;
  FLS_NCCL(api.CommInitRank(&nc, nranks, u, rank));
  Comm *c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  c->is_nccl = true;
  c->nc = nc;
  ctx->comm = c;
  return FLS_OK;
}

fls_status fls_comm_init_host(fls_ctx *ctx, int32_t nranks, int32_t rank, const fls_host_coll *coll) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (!coll || !coll->allgather) return fail(FLS_EINVAL, "coll or coll->allgather is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(FLS_EINVAL, "rank %d not in [0, %d)", rank, nranks);
  if (ctx->comm) return fail(FLS_EINVAL, "ctx already has a communicator (fls_comm_destroy first)");
  Comm *c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  c->host = *coll;
  ctx->comm = c;
  return FLS_OK;
}

fls_status fls_comm_destroy(fls_ctx *ctx) {
  if (fls_status s = check_ctx(ctx)) return s;
  DeviceGuard g(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  comm_destroy(ctx);
  return FLS_OK;
}

fls_status fls_comm_config(fls_ctx *ctx, int32_t transport, int32_t force_tsqr) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (!ctx->comm) return fail(FLS_EINVAL, "ctx has no communicator");
  if (transport < FLS_TSQR_AUTO || transport > FLS_TSQR_NCCL)
    return fail(FLS_EINVAL, "transport %d not one of FLS_TSQR_AUTO/P2P/NCCL", transport);
  if (transport == FLS_TSQR_NCCL && !ctx->comm->is_nccl)
    return fail(FLS_EINVAL, "FLS_TSQR_NCCL needs an NCCL communicator (fls_comm_init)");
  ctx->comm->transport = transport;
  ctx->comm->force_tsqr = force_tsqr != 0;
  return FLS_OK;
}

fls_status fls_comm_info(fls_ctx *ctx, int32_t *nranks, int32_t *rank, int32_t *last_transport) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (!nranks || !rank || !last_transport) return fail(FLS_EINVAL, "NULL output");
  const Comm *c = ctx->comm;
  *nranks = c ? c->nranks : 0;
  *rank = c ? c->rank : 0;
  *last_transport = c ? c->last_transport : 0;
  return FLS_OK;
}

}  // extern "C"
