// Sharded layout of one rank (one process per GPU): the rank owns a
// contiguous global row range and a contiguous range of subdomains; its
// vectors live in an "extended" local index space [ext_lo, ext_hi) that
// adds the halo rows its operator rows and overlapped subdomains touch.
// Owned rows sit at [own_off, own_off + n_own) of the extended vector.
#pragma once
#include <vector>

#include "comm.cuh"
#include "common.cuh"

struct gdsw_dist {
  int rank = 0, nranks = 1;
  int64_t n_ext = 0, own_off = 0, n_own = 0;
  gdsw::HaloSpec halo;
  // remote partial combination ranges (ext-local): rows owned by me that
  // receive partial sums from lower ranks (start value) / higher (tail)
  int64_t pre_lo = 0, pre_hi = 0, post_lo = 0, post_hi = 0;
  gdsw::MailboxLayout layout;
  gdsw::DBuf<char> box;
  gdsw::PeerTable peers{};
  std::vector<char*> opened;
  // per-channel sequence counters + CTA tickets on the device (graph-safe)
  gdsw::DBuf<uint64_t> dseq;
  gdsw::DBuf<unsigned> ddone;
  bool ready = false;
  gdsw::SeqCounter counters() const { return gdsw::SeqCounter{dseq.p, ddone.p}; }
  gdsw::DBuf<double> red_in, red_out;  // scratch for reductions
  ~gdsw_dist() {
    for (size_t q = 0; q < opened.size(); ++q)
      if (opened[q] && (int)q != rank) cudaIpcCloseMemHandle(opened[q]);
  }

  void allreduce(const double* d_in, double* d_out, int64_t m, cudaStream_t s, int ch = gdsw::CH_RED) {
    gdsw::require(ready, "distributed layout has no opened peers");
    gdsw::require(m <= layout.red_max, "reduction larger than the mailbox slot");
    if (nranks == 1) {
      if (d_in != d_out) CK(cudaMemcpyAsync(d_out, d_in, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
      return;
    }
    gdsw::k_comm_allreduce<<<1, 256, 0, s>>>(peers, layout, rank, counters(), ch, d_in, d_out, m);
    CK_LAUNCH();
  }
  void halo_fwd(double* x_ext, cudaStream_t s) {
    if (nranks == 1 || halo.nn == 0) return;
    gdsw::k_comm_halo_fwd<<<2 * halo.nn, 1024, 0, s>>>(peers, layout, halo, rank, counters(), x_ext);
    CK_LAUNCH();
  }
  void halo_rev(const double* part_ext, double* recv_ext, cudaStream_t s) {
    if (nranks == 1 || halo.nn == 0) return;
    gdsw::k_comm_halo_rev<<<2 * halo.nn, 1024, 0, s>>>(peers, layout, halo, rank, counters(), part_ext,
                                                         recv_ext);
    CK_LAUNCH();
  }
};
