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

namespace {

// elements [e0, e0 + count) of the payload -> out, by `threads` parallel
// positional reads of whole 1 MiB pieces, each thread scanning what it read
// for non-finite values.  *bad: first non-finite flat element index (file
// numbering), *short_at: payload bytes present when the file ends early.
int read_elems(int fd, int64_t e0, int64_t count, double* out, int threads, int64_t* bad,
               int64_t* short_at_out, int* err) {
  const int64_t bytes = count * 8;
  int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  T = std::max(1, std::min(T, 64));
  const int64_t piece = 1 << 20;
  const int64_t pieces = (bytes + piece - 1) / piece;
  std::atomic<int64_t> next{0}, first_bad{INT64_MAX}, short_at{INT64_MAX};
  std::atomic<int> io_err{0};
  auto work = [&]() {
    for (;;) {
      const int64_t pc = next.fetch_add(1);
      if (pc >= pieces || io_err.load()) return;
      const int64_t off = pc * piece, len = std::min(piece, bytes - off);
      const int64_t got =
          pread_full(fd, reinterpret_cast<char*>(out) + off, len, kHeader + e0 * 8 + off);
      if (got < 0) {
        io_err.store(errno ? errno : EIO);
        return;
      }
      if (got < len) {
        int64_t cur = short_at.load();
        while (e0 * 8 + off + got < cur &&
               !short_at.compare_exchange_weak(cur, e0 * 8 + off + got)) {
        }
      }
      for (int64_t e = off / 8, e1 = (off + got) / 8; e < e1; ++e) {
        if (!std::isfinite(out[e])) {
          int64_t cur = first_bad.load();
          while (e0 + e < cur && !first_bad.compare_exchange_weak(cur, e0 + e)) {
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
  *err = io_err.load();
  *bad = first_bad.load() == INT64_MAX ? -1 : first_bad.load();
  *short_at_out = short_at.load() == INT64_MAX ? -1 : short_at.load();
  return 0;
}

// write all n bytes at offset `at` (EINTR-safe)
bool pwrite_full(int fd, const char* src, int64_t n, int64_t at) {
  int64_t done = 0;
  while (done < n) {
    const ssize_t w =
        pwrite(fd, src + done, (size_t)std::min<int64_t>(n - done, 1 << 30), at + done);
    if (w < 0) {
      if (errno == EINTR) continue;
      return false;
    }
    done += w;
  }
  return true;
}

}  // namespace

int rmx_mat0_read(const char* path, int64_t rows, int64_t cols, double* out, int32_t threads,
                  int64_t* bad_index, rmx_status* st) {
  return rmx_mat0_read_rows(path, cols, 0, rows, out, threads, bad_index, st);
}

int rmx_mat0_read_rows(const char* path, int64_t cols, int64_t row0, int64_t row1, double* out,
                       int32_t threads, int64_t* bad_index, rmx_status* st) {
  if (st) {
    st->code = 0;
    st->msg[0] = 0;
  }
  if (bad_index) *bad_index = -1;
  if (!path || !out || row0 < 0 || row1 <= row0 || cols < 1)
    return mset(st, RMX_E_USAGE, "bad arguments");
  Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return mset(st, RMX_E_IO, "%s: %s", path, strerror(errno));
  int64_t bad = -1, short_at = -1;
  int err = 0;
  read_elems(f.fd, row0 * cols, (row1 - row0) * cols, out, threads, &bad, &short_at, &err);
  if (err) return mset(st, RMX_E_IO, "%s: %s", path, strerror(err));
  if (short_at >= 0) {
    if (bad_index) *bad_index = short_at;  // payload bytes actually present
    return mset(st, RMX_E_FORMAT, "%s: payload shorter than %lld bytes", path,
                (long long)(row1 * cols * 8));
  }
  if (bad >= 0) {
    if (bad_index) *bad_index = bad;
    return mset(st, RMX_E_FORMAT, "%s: non-finite entry at element %lld", path, (long long)bad);
  }
  return 0;
}

int rmx_mat0_create(const char* path, int64_t rows, int64_t cols, int64_t n1, int64_t n2,
                    rmx_status* st) {
  if (st) {
    st->code = 0;
    st->msg[0] = 0;
  }
  if (!path || rows < 0 || cols < 0) return mset(st, RMX_E_USAGE, "bad arguments");
  Fd f;
  f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (f.fd < 0) return mset(st, RMX_E_IO, "%s: %s", path, strerror(errno));
  unsigned char h[kHeader];
  memcpy(h, "RMXMAT0\0", 8);
  const uint32_t ver = 1;
  const uint64_t d[4] = {(uint64_t)rows, (uint64_t)cols, (uint64_t)n1, (uint64_t)n2};
  memcpy(h + 8, &ver, 4);
  memcpy(h + 12, d, 32);
  if (!pwrite_full(f.fd, reinterpret_cast<const char*>(h), kHeader, 0) ||
      ftruncate(f.fd, kHeader + rows * cols * 8) != 0)
    return mset(st, RMX_E_IO, "%s: %s", path, strerror(errno));
  return 0;
}

int rmx_mat0_write_rows(const char* path, int64_t cols, int64_t row0, int64_t row1,
                        const double* a, int32_t threads, rmx_status* st) {
  if (st) {
    st->code = 0;
    st->msg[0] = 0;
  }
  if (!path || !a || row0 < 0 || row1 < row0 || cols < 0)
    return mset(st, RMX_E_USAGE, "bad arguments");
  Fd f;
  f.fd = open(path, O_WRONLY | O_CLOEXEC);
  if (f.fd < 0) return mset(st, RMX_E_IO, "%s: %s", path, strerror(errno));
  const int64_t bytes = (row1 - row0) * cols * 8, at = kHeader + row0 * cols * 8;
  const int64_t piece = 8 << 20;
  const int64_t pieces = (bytes + piece - 1) / piece;
  int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  T = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(T, 32), pieces));
  std::atomic<int64_t> next{0};
  std::atomic<int> io_err{0};
  auto work = [&]() {
    for (;;) {
      const int64_t pc = next.fetch_add(1);
      if (pc >= pieces || io_err.load()) return;
      const int64_t off = pc * piece, len = std::min(piece, bytes - off);
      if (!pwrite_full(f.fd, reinterpret_cast<const char*>(a) + off, len, at + off))
        io_err.store(errno ? errno : EIO);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  if (io_err.load()) return mset(st, RMX_E_IO, "%s: %s", path, strerror(io_err.load()));
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
