// comm.cu -- the NCCL communicator of librc (rc_comm, row a8 of SURVEY.md
// §8(a)): the tile exchange sends every partial segment record to the rank
// that owns its image tile ("non-blocking send ... to
// each receiver", PAPER.md:1112-1127 receives at the writers).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: the instance torch
// already loaded when there is one, else the system library), so librc
// carries no link-time NCCL dependency and loads on machines without it;
// rc_comm_create fails with RC_ERR_NCCL when NCCL is not available.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <string.h>

#include <mutex>

#include "rc_internal.cuh"

namespace rc {

namespace {
// the subset of nccl.h librc uses (ABI-stable since NCCL 2.0)
typedef struct ncclComm* ncclComm_t;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclInt8 = 0, ncclUint8 = 1, ncclInt64 = 4 } ncclDataType_t;
typedef struct {
  char internal[128];
} ncclUniqueId;

struct NcclApi {
  bool ok = false;
  void* handle = nullptr;
  int (*GetUniqueId)(ncclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*CommAbort)(ncclComm_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

bool load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.ok) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy torch loaded, if any
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  NcclApi a;
  a.handle = h;
#define SYM(field, name)                                      \
  *reinterpret_cast<void**>(&a.field) = dlsym(h, name);      \
  if (!a.field) return false;
  SYM(GetUniqueId, "ncclGetUniqueId")
  SYM(CommInitRank, "ncclCommInitRank")
  SYM(CommDestroy, "ncclCommDestroy")
  SYM(CommAbort, "ncclCommAbort")
  SYM(Send, "ncclSend")
  SYM(Recv, "ncclRecv")
  SYM(GroupStart, "ncclGroupStart")
  SYM(GroupEnd, "ncclGroupEnd")
  SYM(GetErrorString, "ncclGetErrorString")
#undef SYM
  a.ok = true;
  g_nccl = a;
  return true;
}
}  // namespace

const char* nccl_error_string(int r) { return g_nccl.ok ? g_nccl.GetErrorString(r) : "NCCL not loaded"; }

// Grouped exchange of variable-size byte blocks: send[p] bytes from sbuf+soff[p]
// to every peer p != rank, receive rcnt[p] bytes into rbuf+roff[p]; the block
// to itself is a device copy.  All on stream s.
int nccl_exchange(rc_comm* c, const char* sbuf, const int64_t* soff, const int64_t* scnt, char* rbuf,
                  const int64_t* roff, const int64_t* rcnt, cudaStream_t s) {
  int r = g_nccl.GroupStart();
  if (r) return r;
  for (int p = 0; p < c->nranks; ++p) {
    if (p == c->rank) continue;
    if (scnt[p] > 0 && (r = g_nccl.Send(sbuf + soff[p], (size_t)scnt[p], ncclUint8, p, (ncclComm_t)c->nccl, s)))
      break;
    if (rcnt[p] > 0 && (r = g_nccl.Recv(rbuf + roff[p], (size_t)rcnt[p], ncclUint8, p, (ncclComm_t)c->nccl, s)))
      break;
  }
  const int r2 = g_nccl.GroupEnd();
  if (r) return r;
  if (r2) return r2;
  if (scnt[c->rank] > 0 &&
      cudaMemcpyAsync(rbuf + roff[c->rank], sbuf + soff[c->rank], (size_t)scnt[c->rank], cudaMemcpyDeviceToDevice,
                      s) != cudaSuccess)
    return -1;
  return 0;
}

// One int64 to / from every peer (the count all-to-all of the tile exchange).
int nccl_alltoall_i64(rc_comm* c, const int64_t* d_send, int64_t* d_recv, cudaStream_t s) {
  int r = g_nccl.GroupStart();
  if (r) return r;
  for (int p = 0; p < c->nranks; ++p) {
    if (p == c->rank) continue;
    if ((r = g_nccl.Send(d_send + p, 1, ncclInt64, p, (ncclComm_t)c->nccl, s))) break;
    if ((r = g_nccl.Recv(d_recv + p, 1, ncclInt64, p, (ncclComm_t)c->nccl, s))) break;
  }
  const int r2 = g_nccl.GroupEnd();
  if (r) return r;
  if (r2) return r2;
  if (cudaMemcpyAsync(d_recv + c->rank, d_send + c->rank, sizeof(int64_t), cudaMemcpyDeviceToDevice, s) !=
      cudaSuccess)
    return -1;
  return 0;
}

// One int64 to every discovered receiver, one from every discovered sender
// (rc_comm_set_partners); entries of other peers are left untouched.
int nccl_partner_i64(rc_comm* c, const int64_t* d_send, int64_t* d_recv, cudaStream_t s) {
  int r = g_nccl.GroupStart();
  if (r) return r;
  for (int p = 0; p < c->nranks; ++p) {
    if (p == c->rank) continue;
    if (c->send_to[p] && (r = g_nccl.Send(d_send + p, 1, ncclInt64, p, (ncclComm_t)c->nccl, s))) break;
    if (c->recv_from[p] && (r = g_nccl.Recv(d_recv + p, 1, ncclInt64, p, (ncclComm_t)c->nccl, s))) break;
  }
  const int r2 = g_nccl.GroupEnd();
  if (r) return r;
  if (r2) return r2;
  if (cudaMemcpyAsync(d_recv + c->rank, d_send + c->rank, sizeof(int64_t), cudaMemcpyDeviceToDevice, s) !=
      cudaSuccess)
    return -1;
  return 0;
}

}  // namespace rc

using namespace rc;

extern "C" rc_status rc_comm_set_partners(rc_comm* c, const uint8_t* h_send_to, const uint8_t* h_recv_from) {
  if (!c) return rc_fail(RC_ERR_INVALID_ARG, "rc_comm_set_partners: null communicator");
  if (!h_send_to != !h_recv_from) return rc_fail(RC_ERR_INVALID_ARG, "rc_comm_set_partners: give both lists or neither");
  c->partners = h_send_to != nullptr;
  for (int p = 0; p < c->nranks; ++p) {
    c->send_to[p] = c->partners ? (h_send_to[p] != 0) : 0;
    c->recv_from[p] = c->partners ? (h_recv_from[p] != 0) : 0;
  }
  return RC_OK;
}

extern "C" rc_status rc_comm_unique_id(uint8_t id[128]) {
  if (!id) return rc_fail(RC_ERR_INVALID_ARG, "rc_comm_unique_id: null argument");
  if (!load_nccl()) return rc_fail(RC_ERR_NCCL, "rc_comm_unique_id: libnccl.so.2 not found");
  ncclUniqueId u;
  const int r = g_nccl.GetUniqueId(&u);
  if (r) return rc_fail(RC_ERR_NCCL, "ncclGetUniqueId: %s", g_nccl.GetErrorString(r));
  memcpy(id, u.internal, 128);
  return RC_OK;
}

extern "C" rc_status rc_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, void* stream,
                                    rc_comm** out) {
  (void)stream;
  if (!id || !out) return rc_fail(RC_ERR_INVALID_ARG, "rc_comm_create: null argument");
  *out = nullptr;
  if (nranks < 1 || nranks > RC_MAX_RANKS || rank < 0 || rank >= nranks)
    return rc_fail(RC_ERR_INVALID_ARG, "rc_comm_create: bad nranks/rank (%d/%d)", nranks, rank);
  if (!load_nccl()) return rc_fail(RC_ERR_NCCL, "rc_comm_create: libnccl.so.2 not found");
  ncclUniqueId u;
  memcpy(u.internal, id, 128);
  ncclComm_t comm = nullptr;
  const int r = g_nccl.CommInitRank(&comm, nranks, u, rank);
  if (r) return rc_fail(RC_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
  rc_comm* c = new rc_comm();
  c->nccl = comm;
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->device);
  *out = c;
  return RC_OK;
}

extern "C" rc_status rc_comm_destroy(rc_comm* c) {
  if (!c) return RC_OK;
  int r = 0;
  if (c->nccl && g_nccl.ok) r = g_nccl.CommDestroy((ncclComm_t)c->nccl);
  delete c;
  if (r) return rc_fail(RC_ERR_NCCL, "ncclCommDestroy: %s", g_nccl.GetErrorString(r));
  return RC_OK;
}
