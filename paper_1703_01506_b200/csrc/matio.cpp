// matio.cpp -- the reference's `.mat0` binary matrix format on the host side
// of the engine (reference matio.py:23-91): a 44-byte little-endian header
// (8-byte magic "RMXMAT0\0", u32 version 1, u64 rows, cols, n1, n2) and a
// row-major little-endian float64 payload.  The payload is read with
// parallel positional reads straight into the caller's buffer (page-locked
// memory for the upload, hostmem.py) and scanned for non-finite values in
// the same pass; the Python layer (matio.py) formats the reference's error
// messages from the returned fields.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "rmx.h"

namespace {

int mset(rmx_status* st, int code, const char* fmt, ...) {
  if (st) {
    st->code = code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(st->msg, sizeof(st->msg), fmt, ap);
    va_end(ap);
  }
  return code;
}

constexpr int64_t kHeader = 44;

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

// read exactly n bytes at offset off (short only at end of file)
int64_t pread_full(int fd, void* buf, int64_t n, int64_t off) {
  int64_t got = 0;
  char* p = static_cast<char*>(buf);
  while (got < n) {
    const ssize_t r = pread(fd, p + got, (size_t)std::min<int64_t>(n - got, 1 << 30), off + got);
    if (r < 0) {
      if (errno == EINTR) continue;
      return -1;
    }
    if (r == 0) break;
    got += r;
  }
  return got;
}

}  // namespace

extern "C" {

int rmx_mat0_header(const char* path, rmx_mat0_info* info, rmx_status* st) {
  if (st) {
    st->code = 0;
    st->msg[0] = 0;
  }
  if (!path || !info) return mset(st, RMX_E_USAGE, "null argument");
  memset(info, 0, sizeof(*info));
  Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return mset(st, RMX_E_IO, "%s: %s", path, strerror(errno));
  struct stat sb;
  if (fstat(f.fd, &sb) != 0) return mset(st, RMX_E_IO, "%s: %s", path, strerror(errno));
  info->file_bytes = (int64_t)sb.st_size;
  unsigned char h[kHeader];
  const int64_t got = pread_full(f.fd, h, kHeader, 0);
  if (got < 0) return mset(st, RMX_E_IO, "%s: %s", path, strerror(errno));
  info->header_bytes = got;
  if (got < kHeader) return 0;  // truncated: the caller reports it
  memcpy(info->magic, h, 8);
  uint32_t ver;
  uint64_t d[4];
  memcpy(&ver, h + 8, 4);
  memcpy(d, h + 12, 32);
  info->version = ver;
  info->rows = (int64_t)d[0];
  info->cols = (int64_t)d[1];
  info->n1 = (int64_t)d[2];
  info->n2 = (int64_t)d[3];
  return 0;
}

int rmx_mat0_read(const char* path, int64_t rows, int64_t cols, double* out, int32_t threads,
                  int64_t* bad_index, rmx_status* st) {
  if (st) {
    st->code = 0;
    st->msg[0] = 0;
  }
  if (bad_index) *bad_index = -1;
  if (!path || !out || rows < 1 || cols < 1) return mset(st, RMX_E_USAGE, "bad arguments");
  Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return mset(st, RMX_E_IO, "%s: %s", path, strerror(errno));
  const int64_t n = rows * cols;
  const int64_t bytes = n * 8;
  int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  T = std::max(1, std::min(T, 64));
  // whole 1 MiB pieces per thread; each thread scans what it read
  const int64_t piece = 1 << 20;
  const int64_t pieces = (bytes + piece - 1) / piece;
  std::atomic<int64_t> next{0}, first_bad{INT64_MAX}, short_at{INT64_MAX};
  std::atomic<int> io_err{0};
  auto work = [&]() {
    for (;;) {
      const int64_t pc = next.fetch_add(1);
      if (pc >= pieces || io_err.load()) return;
      const int64_t off = pc * piece, len = std::min(piece, bytes - off);
      const int64_t got = pread_full(f.fd, reinterpret_cast<char*>(out) + off, len, kHeader + off);
      if (got < 0) {
        io_err.store(errno ? errno : EIO);
        return;
      }
      if (got < len) {
        int64_t cur = short_at.load();
        while (off + got < cur && !short_at.compare_exchange_weak(cur, off + got)) {
        }
      }
      const int64_t e0 = off / 8, e1 = (off + got) / 8;
      for (int64_t e = e0; e < e1; ++e) {
        if (!std::isfinite(out[e])) {
          int64_t cur = first_bad.load();
          while (e < cur && !first_bad.compare_exchange_weak(cur, e)) {
          }
          break;
        }
      }
    }
  };
  std::vector<std::thread> pool;
  const int nt = (int)std::min<int64_t>(T, pieces);
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  if (io_err.load()) return mset(st, RMX_E_IO, "%s: %s", path, strerror(io_err.load()));
  if (short_at.load() != INT64_MAX) {
    if (bad_index) *bad_index = short_at.load();  // bytes actually present
    return mset(st, RMX_E_FORMAT, "%s: payload shorter than %lld bytes", path, (long long)bytes);
  }
  if (first_bad.load() != INT64_MAX) {
    if (bad_index) *bad_index = first_bad.load();
    return mset(st, RMX_E_FORMAT, "%s: non-finite entry at element %lld", path,
                (long long)first_bad.load());
  }
  return 0;
}

int rmx_mat0_write(const char* path, const double* a, int64_t rows, int64_t cols, int64_t n1,
                   int64_t n2, rmx_status* st) {
  if (st) {
    st->code = 0;
    st->msg[0] = 0;
  }
  if (!path || !a || rows < 0 || cols < 0) return mset(st, RMX_E_USAGE, "bad arguments");
  Fd f;
  f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (f.fd < 0) return mset(st, RMX_E_IO, "%s: %s", path, strerror(errno));
  unsigned char h[kHeader];
  memcpy(h, "RMXMAT0\0", 8);
  const uint32_t ver = 1;
  const uint64_t d[4] = {(uint64_t)rows, (uint64_t)cols, (uint64_t)n1, (uint64_t)n2};
  memcpy(h + 8, &ver, 4);
  memcpy(h + 12, d, 32);
  const char* p = reinterpret_cast<const char*>(h);
  int64_t left = kHeader, off = 0;
  auto put = [&](const char* src, int64_t n, int64_t at) -> bool {
    int64_t done = 0;
    while (done < n) {
      const ssize_t w = pwrite(f.fd, src + done, (size_t)std::min<int64_t>(n - done, 1 << 30),
                               at + done);
      if (w < 0) {
        if (errno == EINTR) continue;
        return false;
      }
      done += w;
    }
    return true;
  };
  if (!put(p, left, off)) return mset(st, RMX_E_IO, "%s: %s", path, strerror(errno));
  if (!put(reinterpret_cast<const char*>(a), rows * cols * 8, kHeader))
    return mset(st, RMX_E_IO, "%s: %s", path, strerror(errno));
  return 0;
}

}  // extern "C"
