// ooc_file.cu -- the out-of-core engine of §4 with secondary storage: the X_R
// stream is read from a file, the b stream written to a file, in blocks of problems.
//
//   mode GLS_OOC_SYNC  (Alg. 7, "non-overlapping synchronous I/O"): per block a
//        blocking read, the solve, a blocking write;
//   mode GLS_OOC_ASYNC (Alg. 8, double buffering): two host workspaces
//        (fig:workspaces) swap roles per block; a reader thread performs
//        async_read(next X_blk) (line 7) and a writer thread async_write(current b_blk) (line 15);
//        the orchestrator waits for the current block (line 8) and for the previous write (line 16).
//
// Three-stage pipeline on B200: storage -> pinned host workspace (pread, reader thread) -> HBM
// (the library's own double-buffered copy-engine stream inside gls_solve_block_ex) -> int8/FP64
// kernels -> b back to the pinned host workspace -> storage (pwrite, writer thread).  The waits are
// measured at the algorithm's wait points and returned in a gls_ooc_report.
// Block schedule: an optional warm-up block (§4.3: "initiate the computation with
// a small block size ... and increase it after a few iterations"), then blocks of block_groups.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gls.h"

namespace {

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a, Clock::time_point b) { return std::chrono::duration<double>(b - a).count(); }

// pread/pwrite of exactly `bytes` (retrying short transfers); false on error or EOF.
bool read_full(int fd, void* dst, size_t bytes, off_t off) {
  char* p = (char*)dst;
  while (bytes > 0) {
    const ssize_t r = pread(fd, p, bytes, off);
    if (r <= 0) return false;
    p += r;
    off += r;
    bytes -= (size_t)r;
  }
  return true;
}
bool write_full(int fd, const void* src, size_t bytes, off_t off) {
  const char* p = (const char*)src;
  while (bytes > 0) {
    const ssize_t r = pwrite(fd, p, bytes, off);
    if (r <= 0) return false;
    p += r;
    off += r;
    bytes -= (size_t)r;
  }
  return true;
}

struct Block {
  int64_t g0, cnt;  // first problem, problems
};

std::vector<Block> plan(int64_t m, int64_t k, int64_t warm) {
  std::vector<Block> b;
  int64_t g = 0;
  if (warm > 0 && warm < k && warm < m) {
    b.push_back({0, warm});
    g = warm;
  }
  while (g < m) {
    const int64_t c = (m - g < k) ? m - g : k;
    b.push_back({g, c});
    g += c;
  }
  return b;
}

// One of the two workspaces of fig:workspaces: an X_R block and its b (and status) block, pinned.
struct Workspace {
  void* x = nullptr;
  double* b = nullptr;
  int32_t* st = nullptr;
  // state machine, guarded by the engine mutex: 0 free, 1 loading, 2 loaded, 3 computed, 4 writing
  int state = 0;
  int64_t block = -1;
};

}  // namespace

extern "C" int gls_solve_file(gls_ctx* ctx, const char* xr_path, int64_t xr_offset, int32_t elem_bytes,
                              int64_t m, const char* b_path, const char* status_path, int64_t block_groups,
                              int64_t warmup_groups, int32_t mode, gls_ooc_report* rep) {
  if (!ctx || !xr_path || !b_path || (elem_bytes != 1 && elem_bytes != 8) || xr_offset < 0 ||
      (mode != GLS_OOC_SYNC && mode != GLS_OOC_ASYNC))
    return GLS_ERR_ARG;
  int64_t n = 0;
  int32_t pL = 0, pR = 0;
  int rc0 = gls_get_dims(ctx, &n, &pL, &pR);
  if (rc0) return rc0;
  const int32_t p = pL + pR;
  if (m < 1 || block_groups < 1 || warmup_groups < 0) return GLS_ERR_DIM;
  // X_R is read with O_DIRECT when every block is 4 KiB-aligned in offset and length (no page cache,
  // no kernel readahead: Alg. 7 is then really synchronous and Alg. 8's overlap is all ours), else
  // buffered.  The pinned workspaces are page-aligned.
  const int fx_buf = open(xr_path, O_RDONLY);
  if (fx_buf < 0) return GLS_ERR_ARG;
  int fx_direct = -1;
  const int fb = open(b_path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  const int fs = status_path ? open(status_path, O_WRONLY | O_CREAT | O_TRUNC, 0644) : -1;
  if (fb < 0 || (status_path && fs < 0)) {
    close(fx_buf);
    if (fb >= 0) close(fb);
    if (fs >= 0) close(fs);
    return GLS_ERR_ARG;
  }
  const size_t col_bytes = (size_t)n * elem_bytes;
  const size_t xcap = (size_t)block_groups * pR * col_bytes;
  Workspace ws[2];
  int rc = GLS_OK;
  for (int k = 0; k < 2 && rc == GLS_OK; ++k) {
    if (cudaHostAlloc(&ws[k].x, xcap, cudaHostAllocPortable) != cudaSuccess ||
        cudaHostAlloc((void**)&ws[k].b, (size_t)block_groups * p * sizeof(double), cudaHostAllocPortable) !=
            cudaSuccess ||
        cudaHostAlloc((void**)&ws[k].st, (size_t)block_groups * sizeof(int32_t), cudaHostAllocPortable) !=
            cudaSuccess) {
      cudaGetLastError();
      rc = GLS_ERR_OOM;
    }
  }
  const std::vector<Block> blocks = plan(m, block_groups, warmup_groups);
  {
    bool aligned = xr_offset % 4096 == 0;
    for (const Block& bk : blocks)
      aligned = aligned && ((int64_t)bk.g0 * pR * (int64_t)col_bytes) % 4096 == 0 &&
                (bk.g0 + bk.cnt == m || ((int64_t)bk.cnt * pR * (int64_t)col_bytes) % 4096 == 0);
    if (aligned && xcap % 4096 == 0) fx_direct = open(xr_path, O_RDONLY | O_DIRECT);
  }
  const int fx = fx_direct >= 0 ? fx_direct : fx_buf;
  gls_ooc_report r;
  memset(&r, 0, sizeof r);
  r.blocks = (int64_t)blocks.size();
  auto solve = [&](Workspace& w, const Block& bk) -> int {
    return elem_bytes == 1
               ? gls_solve_block_i8(ctx, (const int8_t*)w.x, n, bk.cnt, w.b, w.st, 0)
               : gls_solve_block_ex(ctx, (const double*)w.x, bk.cnt, w.b, w.st, 0);
  };
  auto do_read = [&](Workspace& w, const Block& bk) -> bool {
    const size_t bytes = (size_t)bk.cnt * pR * col_bytes;
    const off_t off = (off_t)(xr_offset + (int64_t)bk.g0 * pR * (int64_t)col_bytes);
    if (fx != fx_direct || bytes % 4096 == 0) return read_full(fx, w.x, bytes, off);
    // last block under O_DIRECT: read whole 4 KiB units (the file may end inside the last one)
    const size_t up = (bytes + 4095) & ~(size_t)4095;
    if (up > xcap) return read_full(fx_buf, w.x, bytes, off);
    char* p = (char*)w.x;
    size_t got = 0;
    while (got < up) {
      const ssize_t rr = pread(fx, p + got, up - got, off + (off_t)got);
      if (rr <= 0) break;
      got += (size_t)rr;
    }
    return got >= bytes;
  };
  auto do_write = [&](Workspace& w, const Block& bk) -> bool {
    bool ok = write_full(fb, w.b, (size_t)bk.cnt * p * sizeof(double), (off_t)(bk.g0 * p * (int64_t)sizeof(double)));
    if (ok && fs >= 0) ok = write_full(fs, w.st, (size_t)bk.cnt * sizeof(int32_t), (off_t)(bk.g0 * 4));
    return ok;
  };
  const auto t_start = Clock::now();
  if (rc == GLS_OK && mode == GLS_OOC_SYNC) {
    // Alg. 7: read (blocking) -> compute -> write (blocking); every wait is exposed
    for (size_t j = 0; j < blocks.size() && rc == GLS_OK; ++j) {
      const auto t0 = Clock::now();
      if (!do_read(ws[0], blocks[j])) {
        rc = GLS_ERR_ARG;
        break;
      }
      const auto t1 = Clock::now();
      rc = solve(ws[0], blocks[j]);
      const auto t2 = Clock::now();
      if (rc == GLS_OK && !do_write(ws[0], blocks[j])) rc = GLS_ERR_ARG;
      const auto t3 = Clock::now();
      r.read_wait_s += secs(t0, t1);
      r.compute_s += secs(t1, t2);
      r.write_wait_s += secs(t2, t3);
      if (j == 0) r.first_load_s = secs(t0, t1);
      r.bytes_read += (int64_t)blocks[j].cnt * pR * (int64_t)col_bytes;
      r.bytes_written += blocks[j].cnt * p * (int64_t)sizeof(double);
    }
  } else if (rc == GLS_OK) {
    // Alg. 8: reader and writer threads service one transfer of each kind at a time, in order.
    // io_error is sticky: the reader or the writer sets it on a failed transfer and nothing clears
    // it; the orchestrator checks it after every wait and once more at the end, and on any failure
    // it stops the helpers instead of handing the workspace to the writer (so no stale or
    // uninitialised b is ever written, and a failed write cannot be masked by a later read).
    std::mutex mu;
    std::condition_variable cv;
    bool stop = false;
    bool io_error = false;
    std::thread reader([&] {
      for (size_t j = 0; j < blocks.size(); ++j) {
        Workspace& w = ws[j & 1];
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return stop || w.state == 0; });
          if (stop) return;
          w.state = 1;
          w.block = (int64_t)j;
        }
        const bool ok = do_read(w, blocks[j]);
        {
          std::lock_guard<std::mutex> lk(mu);
          if (!ok) io_error = true;
          w.state = 2;
        }
        cv.notify_all();
        if (!ok) return;
      }
    });
    std::thread writer([&] {
      for (size_t j = 0; j < blocks.size(); ++j) {
        Workspace& w = ws[j & 1];
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return stop || (w.state == 3 && w.block == (int64_t)j); });
          if (stop) return;
          w.state = 4;
        }
        const bool ok = do_write(w, blocks[j]);
        {
          std::lock_guard<std::mutex> lk(mu);
          if (!ok) io_error = true;
          w.state = 0;  // free: the reader may load block j + 2 into it
        }
        cv.notify_all();
        if (!ok) return;
      }
    });
    for (size_t j = 0; j < blocks.size() && rc == GLS_OK; ++j) {
      Workspace& w = ws[j & 1];
      const auto t0 = Clock::now();
      {  // line 8: wait(current X_blk)
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return io_error || (w.state == 2 && w.block == (int64_t)j); });
        if (io_error) rc = GLS_ERR_ARG;
      }
      if (rc != GLS_OK) break;
      const auto t1 = Clock::now();
      rc = solve(w, blocks[j]);  // lines 9-14
      if (rc != GLS_OK) break;  // never hand an unsolved workspace to the writer
      const auto t2 = Clock::now();
      {  // line 15: async_write(current b_blk)
        std::lock_guard<std::mutex> lk(mu);
        w.state = 3;
      }
      cv.notify_all();
      // line 16: wait(previous b_blk) -- its workspace must be free before the next load into it
      if (j >= 1) {
        Workspace& pw = ws[(j - 1) & 1];
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return io_error || pw.state == 0 || pw.state == 1 || pw.state == 2; });
        if (io_error) rc = GLS_ERR_ARG;
      }
      const auto t3 = Clock::now();
      r.read_wait_s += secs(t0, t1);
      r.compute_s += secs(t1, t2);
      r.write_wait_s += secs(t2, t3);
      if (j == 0) r.first_load_s = secs(t0, t1);
      r.bytes_read += (int64_t)blocks[j].cnt * pR * (int64_t)col_bytes;
      r.bytes_written += blocks[j].cnt * p * (int64_t)sizeof(double);
    }
    {
      // the last write: wait for it, or stop the helpers on failure
      std::unique_lock<std::mutex> lk(mu);
      if (rc == GLS_OK) {
        Workspace& lw = ws[(blocks.size() - 1) & 1];
        const auto t0 = Clock::now();
        cv.wait(lk, [&] { return io_error || lw.state == 0; });
        r.write_wait_s += secs(t0, Clock::now());
      }
      if (rc == GLS_OK && io_error) rc = GLS_ERR_ARG;
      stop = true;
    }
    cv.notify_all();
    reader.join();
    writer.join();
  }
  r.wall_s = secs(t_start, Clock::now());
  for (int k = 0; k < 2; ++k) {
    if (ws[k].x) cudaFreeHost(ws[k].x);
    if (ws[k].b) cudaFreeHost(ws[k].b);
    if (ws[k].st) cudaFreeHost(ws[k].st);
  }
  close(fx_buf);
  if (fx_direct >= 0) close(fx_direct);
  close(fb);
  if (fs >= 0) close(fs);
  if (rep) *rep = r;
  return rc;
}

// §4.3: time(computation) > time(load) + time(store) per block, two workspaces in
// the memory limit.  Returns the largest block (problems) meeting both, with a 10 % margin on the
// time condition; if none meets the time condition, the largest that fits and
// *io_bound = 1.  Costs are modelled as per-block latency + per-problem linear terms.
extern "C" int64_t gls_select_block_size(int64_t n, int32_t p, int32_t pR, int32_t elem_bytes,
                                         int64_t mem_limit_bytes, double compute_groups_per_s,
                                         double io_bytes_per_s, double io_latency_s, int32_t* io_bound) {
  if (n < 1 || p < 1 || pR < 1 || (elem_bytes != 1 && elem_bytes != 8) || mem_limit_bytes <= 0 ||
      !(compute_groups_per_s > 0) || !(io_bytes_per_s > 0) || io_latency_s < 0)
    return -1;
  const double per_group_bytes = (double)pR * n * elem_bytes + (double)p * 8 + 4;
  const int64_t kmax = (int64_t)((double)mem_limit_bytes / (2.0 * per_group_bytes));
  if (kmax < 1) return -1;
  // compute(k) = k / rc ; io(k) = 2 lat + k bytes / rio ; need compute >= 1.1 io
  const double slope = 1.0 / compute_groups_per_s - 1.1 * per_group_bytes / io_bytes_per_s;
  const bool ok_at_kmax = slope * (double)kmax >= 1.1 * 2.0 * io_latency_s;
  if (io_bound) *io_bound = ok_at_kmax ? 0 : 1;
  return kmax;
}
