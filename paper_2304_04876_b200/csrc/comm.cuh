// Peer-memory collectives for the sharded solve (one process per GPU).
//
// Every rank exports one device "mailbox" through CUDA IPC; every rank maps
// every peer's mailbox (NVLink / NVSwitch peer stores on one node; the same
// device for the 2-processes-on-1-GPU tests). A collective is one kernel:
// the sending CTAs store the payload straight into the destination rank's
// mailbox slot, then publish a sequence number with a system-scope release
// store into that rank's flag; the receiving CTA spins on its own flag with
// system-scope acquire loads, then consumes. No NCCL, no host round trip.
//
// Sequence numbers live on the device (one counter per channel): every
// collective kernel reads its channel's counter, uses counter + 1, and the
// last CTA to finish stores it back. So a captured CUDA graph that contains
// collectives replays with fresh sequence numbers every time -- the sharded
// GMRES passes and applies are graphed like the single-GPU ones.
//
// Slots are double buffered by sequence parity. Every exchange is
// symmetric (all participants send to each other every call), so a rank
// can only start writing parity p of call k+2 after it observed the peer's
// flag of call k+1, which the peer publishes only after consuming call k:
// the slot being overwritten is always consumed.
//
// Reductions are all-gather + fixed rank-order sums: every rank computes
// the identical, run-to-run reproducible result.
#pragma once
#include "common.cuh"

namespace gdsw {

constexpr int COMM_MAX_RANKS = 16;
constexpr int COMM_MAX_NBR = 8;

// CH_RED: GMRES block / norms; CH_CRS: the coarse right-hand side (issued on
// the apply's side stream, so it has its own counter and slots)
enum CommChannel : int { CH_RED = 0, CH_FWD = 1, CH_REV = 2, CH_CRS = 3, CH_COUNT = 4 };

struct MailboxLayout {
  int nranks = 1;
  int64_t red_max = 0;   // doubles per reduction contribution
  int64_t halo_max = 0;  // doubles per halo message
  // byte offsets inside a mailbox
  size_t flags = 0;      // [CH_COUNT][COMM_MAX_RANKS] uint64
  size_t red = 0;        // [2][nranks][red_max] double
  size_t crs = 0;        // [2][nranks][red_max] double (coarse rhs channel)
  size_t fwd = 0;        // [2][COMM_MAX_RANKS][halo_max] double (slot = sender rank)
  size_t rev = 0;        // [2][COMM_MAX_RANKS][halo_max] double
  size_t bytes = 0;
  void init(int n, int64_t rmax, int64_t hmax) {
    nranks = n;
    red_max = rmax;
    halo_max = hmax;
    flags = 0;
    red = 256 + (size_t)CH_COUNT * COMM_MAX_RANKS * 8;
    red = (red + 255) & ~size_t(255);
    crs = red + (size_t)2 * n * rmax * 8;
    crs = (crs + 255) & ~size_t(255);
    fwd = crs + (size_t)2 * n * rmax * 8;
    fwd = (fwd + 255) & ~size_t(255);
    rev = fwd + (size_t)2 * COMM_MAX_RANKS * hmax * 8;
    rev = (rev + 255) & ~size_t(255);
    bytes = rev + (size_t)2 * COMM_MAX_RANKS * hmax * 8;
  }
};

struct PeerTable {
  char* box[COMM_MAX_RANKS];  // mapped mailboxes (box[rank] = own)
};

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until(const uint64_t* flag, uint64_t seq) {
  while (ld_acquire_sys(flag) < seq) __nanosleep(64);
}

// device sequence counter of one channel: every CTA reads it at start;
// the last CTA to finish publishes seq (stream order serialises launches)
struct SeqCounter {
  uint64_t* seq;     // [CH_COUNT]
  unsigned* done;    // [CH_COUNT] CTA tickets (self-resetting)
};
__device__ __forceinline__ uint64_t seq_begin(const SeqCounter& C, int ch) {
  return *reinterpret_cast<volatile uint64_t*>(C.seq + ch) + 1;
}
__device__ __forceinline__ void seq_end(const SeqCounter& C, int ch, uint64_t seq) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(C.done + ch, 1u) == gridDim.x - 1) {
      C.done[ch] = 0;
      C.seq[ch] = seq;
      __threadfence();
    }
  }
}

// all-gather-sum of m doubles: out[k] = sum over ranks q (ascending) of in_q[k]
// one CTA; channel CH_RED or CH_CRS (own counter and slots)
__global__ void k_comm_allreduce(PeerTable T, MailboxLayout L, int rank, SeqCounter SC, int ch,
                                 const double* __restrict__ in, double* __restrict__ out,
                                 int64_t m) {
  const uint64_t seq = seq_begin(SC, ch);
  const int par = (int)(seq & 1);
  const size_t area = ch == CH_CRS ? L.crs : L.red;
  // 1) my contribution into slot [par][rank] of every mailbox
  for (int q = 0; q < L.nranks; ++q) {
    double* dst = reinterpret_cast<double*>(T.box[q] + area) + ((size_t)par * L.nranks + rank) * L.red_max;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) dst[k] = in[k];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < L.nranks; ++q) {
      uint64_t* f = reinterpret_cast<uint64_t*>(T.box[q] + L.flags) + ch * COMM_MAX_RANKS + rank;
      st_release_sys(f, seq);
    }
    // 2) wait for everyone's contribution in my mailbox
    const uint64_t* mine = reinterpret_cast<const uint64_t*>(T.box[rank] + L.flags) + ch * COMM_MAX_RANKS;
    for (int q = 0; q < L.nranks; ++q) spin_until(mine + q, seq);
  }
  __syncthreads();
  const double* src = reinterpret_cast<const double*>(T.box[rank] + area) + (size_t)par * L.nranks * L.red_max;
  for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < L.nranks; ++q) s += __ldcv(src + (size_t)q * L.red_max + k);
    out[k] = s;
  }
  seq_end(SC, ch, seq);
}

struct HaloSpec {
  int nn = 0;                       // neighbours
  int rank[COMM_MAX_NBR];           // their ranks (ascending)
  int64_t send_lo[COMM_MAX_NBR];    // forward: my owned rows they need (ext-local)
  int64_t send_hi[COMM_MAX_NBR];
  int64_t recv_lo[COMM_MAX_NBR];    // forward: their owned rows in my halo (ext-local)
  int64_t recv_hi[COMM_MAX_NBR];
};

// forward halo: x[recv ranges] <- owners' values. grid = 2 * nn CTAs:
// CTA i < nn sends to neighbour i, CTA nn + i receives from neighbour i.
__global__ void k_comm_halo_fwd(PeerTable T, MailboxLayout L, HaloSpec H, int rank, SeqCounter SC,
                                double* __restrict__ x) {
  const uint64_t seq = seq_begin(SC, CH_FWD);
  const int par = (int)(seq & 1);
  const int i = blockIdx.x % H.nn;
  const int q = H.rank[i];
  if ((int)blockIdx.x < H.nn) {
    double* dst = reinterpret_cast<double*>(T.box[q] + L.fwd) + ((size_t)par * COMM_MAX_RANKS + rank) * L.halo_max;
    const int64_t lo = H.send_lo[i], len = H.send_hi[i] - lo;
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x) dst[k] = x[lo + k];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0)
      st_release_sys(reinterpret_cast<uint64_t*>(T.box[q] + L.flags) + CH_FWD * COMM_MAX_RANKS + rank, seq);
  } else {
    if (threadIdx.x == 0)
      spin_until(reinterpret_cast<const uint64_t*>(T.box[rank] + L.flags) + CH_FWD * COMM_MAX_RANKS + q, seq);
    __syncthreads();
    const double* src = reinterpret_cast<const double*>(T.box[rank] + L.fwd) + ((size_t)par * COMM_MAX_RANKS + q) * L.halo_max;
    const int64_t lo = H.recv_lo[i], len = H.recv_hi[i] - lo;
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x) x[lo + k] = __ldcv(src + k);
  }
  seq_end(SC, CH_FWD, seq);
}

// reverse halo: my partial sums over my halo rows go to their owners; the
// owner receives neighbour partials into `recv` (laid out like my own send
// ranges, ext-local) for the final ordered combination.
__global__ void k_comm_halo_rev(PeerTable T, MailboxLayout L, HaloSpec H, int rank, SeqCounter SC,
                                const double* __restrict__ part, double* __restrict__ recv) {
  const uint64_t seq = seq_begin(SC, CH_REV);
  const int par = (int)(seq & 1);
  const int i = blockIdx.x % H.nn;
  const int q = H.rank[i];
  if ((int)blockIdx.x < H.nn) {
    double* dst = reinterpret_cast<double*>(T.box[q] + L.rev) + ((size_t)par * COMM_MAX_RANKS + rank) * L.halo_max;
    const int64_t lo = H.recv_lo[i], len = H.recv_hi[i] - lo;  // my halo rows = their owned rows
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x) dst[k] = part[lo + k];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0)
      st_release_sys(reinterpret_cast<uint64_t*>(T.box[q] + L.flags) + CH_REV * COMM_MAX_RANKS + rank, seq);
  } else {
    if (threadIdx.x == 0)
      spin_until(reinterpret_cast<const uint64_t*>(T.box[rank] + L.flags) + CH_REV * COMM_MAX_RANKS + q, seq);
    __syncthreads();
    const double* src = reinterpret_cast<const double*>(T.box[rank] + L.rev) + ((size_t)par * COMM_MAX_RANKS + q) * L.halo_max;
    const int64_t lo = H.send_lo[i], len = H.send_hi[i] - lo;  // their halo rows = my owned rows
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x) recv[lo + k] = __ldcv(src + k);
  }
  seq_end(SC, CH_REV, seq);
}

}  // namespace gdsw
