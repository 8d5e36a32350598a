// Host-staged x-slab transport (TOPO_DIST_HOST): one process per slab, the
// halo planes, scalar allreduces, level-1 allreduce and moduli all-gather go
// through a POSIX shared-memory segment.  Every exchange is stream-ordered and
// CUDA-graph capturable: device -> pinned staging copy, a host node that
// publishes to this rank's mailbox, waits on a process-shared barrier and reads
// the peers' mailboxes (sums / maxima in rank order: deterministic), then a
// staging -> device copy.  It runs the SAME per-rank control flow as the NCCL
// transport (each process owns one slab and only its planes), so the
// partition, halo and reduction logic of the multi-GPU path is testable with
// several processes on one GPU (tests/test_dist_host.py); it is a test and
// fallback transport, not the fast path (NCCL over NVLink is).
#pragma once
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <deque>
#include <string>

namespace topo {

struct HostShmHeader {
  std::atomic<int> arrive;
  std::atomic<int> sense;
  std::atomic<int> error;     // set by any rank on a timeout: every waiter gives up
  std::atomic<int> attached;
  int world;
  long long mbox_bytes;
};

class HostTransport {
 public:
  int rank = 0, world = 1;
  long long mbox = 0;
  double timeout_s = 120.0;
  std::atomic<int> failed{0};   // this process saw a timeout / peer error
  double* hsend = nullptr;      // pinned staging (device <-> host), mbox bytes each
  double* hrecv = nullptr;

  // name: NUL-terminated, <= 127 chars ("/topo_<hex>"); rank 0 creates the segment
  bool open(const char* name, int rank_, int world_, long long mbox_bytes, std::string& err) {
    rank = rank_;
    world = world_;
    mbox = (mbox_bytes + 63) / 64 * 64;
    name_ = name;
    bytes_ = (long long)sizeof(HostShmHeader) + 64 + (long long)world * mbox;
    int fd = -1;
    const auto t0 = std::chrono::steady_clock::now();
    if (rank == 0) {
      fd = shm_open(name, O_CREAT | O_RDWR, 0600);
      if (fd < 0 || ftruncate(fd, bytes_) != 0) { err = "shm_open/ftruncate failed"; if (fd >= 0) close(fd); return false; }
    } else {
      while (true) {   // wait for rank 0 to create and size the segment
        fd = shm_open(name, O_RDWR, 0600);
        struct stat sb;
        if (fd >= 0 && fstat(fd, &sb) == 0 && sb.st_size == bytes_) break;
        if (fd >= 0) close(fd);
        if (elapsed(t0) > timeout_s) { err = "host transport: segment never appeared"; return false; }
        usleep(1000);
      }
    }
    void* p = mmap(nullptr, (size_t)bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) { err = "mmap failed"; return false; }
    base_ = static_cast<char*>(p);
    hdr_ = reinterpret_cast<HostShmHeader*>(base_);
    if (rank == 0) {   // fresh segment (ftruncate zero-fills): header fields
      hdr_->world = world;
      hdr_->mbox_bytes = mbox;
      hdr_->attached.store(0);
    }
    // every rank attached (rank 0 initialised the header before anyone counts)
    if (rank != 0)
      while (hdr_->world != world && elapsed(t0) < timeout_s) usleep(1000);
    hdr_->attached.fetch_add(1);
    while (hdr_->attached.load() < world) {
      if (elapsed(t0) > timeout_s) { err = "host transport: not every rank attached"; return false; }
      usleep(1000);
    }
    if (hdr_->mbox_bytes != mbox) { err = "host transport: mailbox size differs between ranks"; return false; }
    return true;
  }

  void close_all() {
    if (base_) {
      munmap(base_, (size_t)bytes_);
      if (rank == 0) shm_unlink(name_.c_str());
      base_ = nullptr;
    }
  }

  char* mailbox(int r) { return base_ + sizeof(HostShmHeader) + 64 + (long long)r * mbox; }

  // sense-reversing barrier over the world (process-shared atomics); false on
  // timeout or a peer's error
  bool barrier() {
    if (failed.load()) return false;
    local_sense_ = 1 - local_sense_;
    const auto t0 = std::chrono::steady_clock::now();
    if (hdr_->arrive.fetch_add(1) == world - 1) {
      hdr_->arrive.store(0);
      hdr_->sense.store(local_sense_);
      return true;
    }
    int spins = 0;
    while (hdr_->sense.load() != local_sense_) {
      if (hdr_->error.load()) { failed.store(1); return false; }
      if (++spins > 1024) {
        sched_yield();
        if (elapsed(t0) > timeout_s) {
          hdr_->error.store(1);
          failed.store(1);
          return false;
        }
      }
    }
    return true;
  }

 private:
  static double elapsed(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  std::string name_;
  char* base_ = nullptr;
  HostShmHeader* hdr_ = nullptr;
  long long bytes_ = 0;
  int local_sense_ = 0;
};

// One captured host-side step (the userData of a cudaLaunchHostFunc node; the
// context keeps them alive for the graphs' lifetime).
struct HostOp {
  HostTransport* t = nullptr;
  int kind = 0;                 // 0 halo exchange, 1 allreduce (f64), 2 allreduce (f32), 3 all-gather
  // halo exchange: this rank's send block [nblk][2][len] in hsend (0 = to the left, 1 =
  // to the right); the neighbours' blocks are read into hrecv with the same layout
  // (recv[.][0] from the left neighbour's "to the right" block, [.][1] from the right's "to the left")
  long long len = 0;
  int nblk = 0;
  // allreduce: n values, maxmask (bit k: slot k is a max, for n <= 32)
  long long n = 0;
  unsigned maxmask = 0;
  // all-gather: rank r contributes cnt[r] doubles, placed at off[r] in hrecv
  long long cnt[16] = {}, off[16] = {};
};

inline void host_op_run(HostOp* op) {
  HostTransport& t = *op->t;
  const int r = t.rank, W = t.world;
  char* mine = t.mailbox(r);
  if (op->kind == 0) {
    const size_t blk = sizeof(double) * 2 * op->len;
    memcpy(mine, t.hsend, blk * op->nblk);
    if (!t.barrier()) return;
    for (int b = 0; b < op->nblk; ++b) {
      double* rv = t.hrecv + (long long)b * 2 * op->len;
      if (r > 0)
        memcpy(rv, reinterpret_cast<const double*>(t.mailbox(r - 1) + b * blk) + op->len, sizeof(double) * op->len);
      if (r < W - 1)
        memcpy(rv + op->len, reinterpret_cast<const double*>(t.mailbox(r + 1) + b * blk), sizeof(double) * op->len);
    }
    t.barrier();
  } else if (op->kind == 1 || op->kind == 2) {
    const size_t es = op->kind == 1 ? sizeof(double) : sizeof(float);
    memcpy(mine, t.hsend, es * op->n);
    if (!t.barrier()) return;
    if (op->kind == 1) {
      double* out = t.hrecv;
      for (long long k = 0; k < op->n; ++k) {
        const bool mx = k < 32 && ((op->maxmask >> k) & 1);
        double a = reinterpret_cast<const double*>(t.mailbox(0))[k];
        for (int q = 1; q < W; ++q) {
          const double v = reinterpret_cast<const double*>(t.mailbox(q))[k];
          a = mx ? (v > a ? v : a) : a + v;
        }
        out[k] = a;
      }
    } else {
      float* out = reinterpret_cast<float*>(t.hrecv);
      for (long long k = 0; k < op->n; ++k) {
        float a = reinterpret_cast<const float*>(t.mailbox(0))[k];
        for (int q = 1; q < W; ++q) a += reinterpret_cast<const float*>(t.mailbox(q))[k];
        out[k] = a;
      }
    }
    t.barrier();
  } else {
    memcpy(mine, t.hsend, sizeof(double) * op->cnt[r]);
    if (!t.barrier()) return;
    for (int q = 0; q < W; ++q) memcpy(t.hrecv + op->off[q], t.mailbox(q), sizeof(double) * op->cnt[q]);
    t.barrier();
  }
}

}  // namespace topo
