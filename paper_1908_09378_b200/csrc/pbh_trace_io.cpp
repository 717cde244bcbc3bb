// Op-trace files: the reference's text format (trace_format.cpp:34-126) and
// a packed binary form with a streaming chunk reader. See include/pbh_trace_io.h.
#include "../../include/pbh_trace_io.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <charconv>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <string_view>
#include <vector>

#include "../../include/pbh_gpu.h"

struct pbh_trace_buf {
  std::vector<uint8_t> kinds;
  std::vector<uint64_t> offsets{0};
  std::vector<uint32_t> values;
  std::vector<uint64_t> prios;
};

struct pbh_trace_reader {
  FILE* f = nullptr;
  uint64_t n_ops = 0, n_elems = 0;
  uint64_t off_kinds = 0, off_offsets = 0, off_values = 0, off_prios = 0;
};

namespace {

thread_local std::string g_err;

int fail(int st, const std::string& m) {
  g_err = m;
  return st;
}

uint64_t pad8(uint64_t x) { return (x + 7) & ~uint64_t(7); }

bool write_all(FILE* f, const void* p, size_t n) { return n == 0 || fwrite(p, 1, n, f) == n; }
bool write_pad(FILE* f, size_t n) {
  static const uint8_t z[8] = {0};
  return n == 0 || fwrite(z, 1, n, f) == n;
}

// ---------------------------------------------------------------- text reader
// The whole file is mapped read-only and scanned once: lines are split with
// memchr, '#' cuts a line, and tokens are maximal runs of non-space bytes.
// Numbers follow the stream-extraction rules the reference relies on
// (`line >> u64`, trace_format.cpp:13-30): leading blanks skipped, an
// optional sign, at least one digit, overflow is a bad number, "-n" wraps
// modulo 2^64, and characters after the digits stay for the next read.

struct MappedFile {
  const char* data = nullptr;
  size_t size = 0;
  std::vector<char> copy;  // fallback when mmap is unavailable (pipes, empty files)
  void* map = nullptr;
  bool open(const char* path) {
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) return false;
    struct stat st {};
    if (fstat(fd, &st) == 0 && S_ISREG(st.st_mode) && st.st_size > 0) {
      map = mmap(nullptr, (size_t)st.st_size, PROT_READ, MAP_PRIVATE, fd, 0);
      if (map != MAP_FAILED) {
        madvise(map, (size_t)st.st_size, MADV_SEQUENTIAL);
        data = static_cast<const char*>(map);
        size = (size_t)st.st_size;
        ::close(fd);
        return true;
      }
      map = nullptr;
    }
    char buf[1 << 16];
    for (ssize_t n; (n = ::read(fd, buf, sizeof buf)) > 0;) copy.insert(copy.end(), buf, buf + n);
    ::close(fd);
    data = copy.data();
    size = copy.size();
    return true;
  }
  ~MappedFile() {
    if (map) munmap(map, size);
  }
};

inline bool is_blank(char ch) {
  return ch == ' ' || ch == '\t' || ch == '\r' || ch == '\v' || ch == '\f';
}

struct LineScanner {
  const char* p;
  const char* end;
  void skip_blanks() {
    while (p < end && is_blank(*p)) ++p;
  }
  // next maximal non-blank run; empty when the line is exhausted
  std::string_view token() {
    skip_blanks();
    const char* b = p;
    while (p < end && !is_blank(*p)) ++p;
    return {b, size_t(p - b)};
  }
  bool at_end() {
    skip_blanks();
    return p == end;
  }
  bool number(uint64_t* out) {
    skip_blanks();
    bool neg = false;
    if (p < end && (*p == '+' || *p == '-')) neg = *p++ == '-';
    uint64_t x = 0;
    const auto r = std::from_chars(p, end, x, 10);
    if (r.ec != std::errc()) return false;  // no digits, or overflow
    p = r.ptr;
    *out = neg ? uint64_t(0) - x : x;
    return true;
  }
};

struct TraceSyntax {
  uint64_t op;
  std::string msg;
};

}  // namespace

extern "C" {

const char* pbh_trace_last_error(void) { return g_err.c_str(); }

int pbh_trace_load_text(const char* path, pbh_trace_buf** out, uint64_t* failed_op) {
  if (!path || !out) return fail(PBH_PRECONDITION, "null argument");
  *out = nullptr;
  if (failed_op) *failed_op = ~0ull;
  MappedFile f;
  if (!f.open(path)) {
    if (failed_op) *failed_op = 0;
    return fail(PBH_TRACE, std::string("cannot open trace file: ") + path);
  }
  std::unique_ptr<pbh_trace_buf> t(new pbh_trace_buf());
  // value / priority ranges of Element (element.hpp:8-9); a batch holds at
  // most 2^24 elements in the text format (trace_format.cpp:60)
  const uint64_t value_max = 0xffffffffull, prio_max = ~0ull, batch_max = 1ull << 24;
  const char* cur = f.data;
  const char* const stop = f.data + f.size;
  uint64_t line = 0;
  try {
    while (cur < stop) {
      const char* nl = static_cast<const char*>(std::memchr(cur, '\n', size_t(stop - cur)));
      const char* eol = nl ? nl : stop;
      ++line;
      const char* hash = static_cast<const char*>(std::memchr(cur, '#', size_t(eol - cur)));
      LineScanner s{cur, hash ? hash : eol};
      cur = nl ? nl + 1 : stop;
      const std::string_view tag = s.token();
      if (tag.empty()) continue;
      const uint64_t op = t->kinds.size();
      const std::string where = "line " + std::to_string(line) + ": ";
      auto num = [&](const char* what, uint64_t max) {
        uint64_t x = 0;
        if (!s.number(&x)) throw TraceSyntax{op, where + "missing or bad " + what};
        if (x > max) throw TraceSyntax{op, where + what + " out of range"};
        return x;
      };
      auto done = [&] {
        if (!s.at_end()) throw TraceSyntax{op, where + "trailing tokens"};
      };
      const char kind = tag.size() == 1 ? tag[0] : '?';
      if (kind == 'U') {
        const uint64_t v = num("value", value_max);
        const uint64_t pr = num("priority", prio_max);
        done();
        t->values.push_back((uint32_t)v);
        t->prios.push_back(pr);
      } else if (kind == 'B') {
        const uint64_t k = num("batch size", batch_max);
        if (!k) throw TraceSyntax{op, where + "empty batch"};
        for (uint64_t j = 0; j < k; ++j) {
          const uint64_t v = num("value", value_max);
          t->values.push_back((uint32_t)v);
          t->prios.push_back(num("priority", prio_max));
        }
        done();
      } else if (kind == 'E') {
        done();
      } else if (kind == 'D') {
        const uint64_t v = num("value", value_max);
        done();
        t->values.push_back((uint32_t)v);
        t->prios.push_back(0);
      } else {
        throw TraceSyntax{op, where + "unknown op '" + std::string(tag) + "'"};
      }
      t->kinds.push_back((uint8_t)kind);
      t->offsets.push_back(t->values.size());
    }
  } catch (const TraceSyntax& e) {
    if (failed_op) *failed_op = e.op;
    return fail(PBH_TRACE, "op " + std::to_string(e.op) + ": " + e.msg);
  }
  *out = t.release();
  return PBH_OK;
}

void pbh_trace_buf_sizes(const pbh_trace_buf* t, uint64_t* n_ops, uint64_t* n_elems) {
  if (n_ops) *n_ops = t ? t->kinds.size() : 0;
  if (n_elems) *n_elems = t ? t->values.size() : 0;
}

void pbh_trace_buf_export(const pbh_trace_buf* t, uint8_t* kinds, uint64_t* offsets,
                          uint32_t* values, uint64_t* priorities) {
  if (!t) return;
  if (kinds && !t->kinds.empty()) std::memcpy(kinds, t->kinds.data(), t->kinds.size());
  if (offsets) std::memcpy(offsets, t->offsets.data(), t->offsets.size() * 8);
  if (values && !t->values.empty()) std::memcpy(values, t->values.data(), t->values.size() * 4);
  if (priorities && !t->prios.empty()) std::memcpy(priorities, t->prios.data(), t->prios.size() * 8);
}

void pbh_trace_buf_free(pbh_trace_buf* t) { delete t; }

int pbh_trace_save_text(const char* path, uint64_t n_ops, const uint8_t* kinds,
                        const uint64_t* offsets, const uint32_t* values,
                        const uint64_t* priorities) {
  if (!path || (n_ops && (!kinds || !offsets))) return fail(PBH_PRECONDITION, "null argument");
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(PBH_TRACE, std::string("cannot open trace file for writing: ") + path);
  // one line per op in the reference's text syntax (trace_format.hpp:16-33),
  // formatted with to_chars into a 1 MiB block that is flushed when full
  std::vector<char> blk(1 << 20);
  size_t at = 0;
  bool ok = true;
  auto flush = [&] {
    ok = ok && write_all(f, blk.data(), at);
    at = 0;
  };
  auto room = [&](size_t n) {
    if (at + n > blk.size()) flush();
  };
  auto put_u = [&](uint64_t x) {
    room(24);
    at = size_t(std::to_chars(blk.data() + at, blk.data() + blk.size(), x).ptr - blk.data());
  };
  auto put_c = [&](char ch) {
    room(1);
    blk[at++] = ch;
  };
  for (uint64_t i = 0; i < n_ops && ok; ++i) {
    const uint64_t b = offsets[i], e = offsets[i + 1];
    const uint8_t k = kinds[i];
    if (k != 'U' && k != 'B' && k != 'E' && k != 'D') {
      std::fclose(f);
      return fail(PBH_TRACE, "op " + std::to_string(i) + ": unknown op kind");
    }
    put_c((char)k);
    if (k == 'B') {
      put_c(' ');
      put_u(e - b);
    }
    if (k != 'E') {
      // U: one (value, priority); B: the batch; D: the value only
      const uint64_t last = k == 'B' ? e : b + 1;
      for (uint64_t j = b; j < last; ++j) {
        put_c(' ');
        put_u(values[j]);
        if (k != 'D') {
          put_c(' ');
          put_u(priorities[j]);
        }
      }
    }
    put_c('\n');
  }
  flush();
  ok = (std::fclose(f) == 0) && ok;
  return ok ? PBH_OK : fail(PBH_TRACE, "write failed");
}

int pbh_trace_save_binary(const char* path, uint64_t n_ops, const uint8_t* kinds,
                          const uint64_t* offsets, const uint32_t* values,
                          const uint64_t* priorities) {
  if (!path || (n_ops && (!kinds || !offsets))) return fail(PBH_PRECONDITION, "null argument");
  const uint64_t n_el = n_ops ? offsets[n_ops] : 0;
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(PBH_TRACE, std::string("cannot open trace file for writing: ") + path);
  const char magic[4] = {'P', 'B', 'H', 'T'};
  const uint32_t version = 1;
  const uint64_t zero = 0;
  bool ok = write_all(f, magic, 4) && write_all(f, &version, 4) && write_all(f, &n_ops, 8) &&
            write_all(f, &n_el, 8) && write_all(f, kinds, n_ops) &&
            write_pad(f, pad8(n_ops) - n_ops) &&
            (n_ops ? write_all(f, offsets, (n_ops + 1) * 8) : write_all(f, &zero, 8)) &&
            write_all(f, values, n_el * 4) && write_pad(f, pad8(n_el * 4) - n_el * 4) &&
            write_all(f, priorities, n_el * 8);
  ok = (std::fclose(f) == 0) && ok;
  return ok ? PBH_OK : fail(PBH_TRACE, "write failed");
}

int pbh_trace_open_binary(const char* path, pbh_trace_reader** out, uint64_t* n_ops,
                          uint64_t* n_elems) {
  if (!path || !out) return fail(PBH_PRECONDITION, "null argument");
  *out = nullptr;
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(PBH_TRACE, std::string("cannot open trace file: ") + path);
  char magic[4];
  uint32_t version = 0;
  uint64_t no = 0, ne = 0;
  if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "PBHT", 4) != 0 ||
      std::fread(&version, 4, 1, f) != 1 || version != 1 || std::fread(&no, 8, 1, f) != 1 ||
      std::fread(&ne, 8, 1, f) != 1) {
    std::fclose(f);
    return fail(PBH_TRACE, std::string("not a pbh binary trace (v1): ") + path);
  }
  auto* r = new pbh_trace_reader();
  r->f = f;
  r->n_ops = no;
  r->n_elems = ne;
  r->off_kinds = 24;
  r->off_offsets = r->off_kinds + pad8(no);
  r->off_values = r->off_offsets + (no + 1) * 8;
  r->off_prios = r->off_values + pad8(ne * 4);
  // the stored element count must agree with the last offset
  uint64_t last = 0;
  if (std::fseek(f, (long)(r->off_offsets + no * 8), SEEK_SET) != 0 ||
      std::fread(&last, 8, 1, f) != 1 || last != ne) {
    pbh_trace_close(r);
    return fail(PBH_TRACE, "corrupt binary trace: offsets do not match the element count");
  }
  if (n_ops) *n_ops = no;
  if (n_elems) *n_elems = ne;
  *out = r;
  return PBH_OK;
}

int pbh_trace_chunk_elems(pbh_trace_reader* r, uint64_t op0, uint64_t n, uint64_t* n_elems) {
  if (!r || !n_elems || op0 + n > r->n_ops) return fail(PBH_PRECONDITION, "op range out of bounds");
  uint64_t ab[2] = {0, 0};
  if (std::fseek(r->f, (long)(r->off_offsets + op0 * 8), SEEK_SET) != 0 ||
      std::fread(&ab[0], 8, 1, r->f) != 1 ||
      std::fseek(r->f, (long)(r->off_offsets + (op0 + n) * 8), SEEK_SET) != 0 ||
      std::fread(&ab[1], 8, 1, r->f) != 1)
    return fail(PBH_TRACE, "read failed");
  *n_elems = ab[1] - ab[0];
  return PBH_OK;
}

int pbh_trace_read_chunk(pbh_trace_reader* r, uint64_t op0, uint64_t n, uint8_t* kinds,
                         uint64_t* offsets, uint32_t* values, uint64_t* priorities) {
  if (!r || op0 + n > r->n_ops || !kinds || !offsets)
    return fail(PBH_PRECONDITION, "op range out of bounds");
  FILE* f = r->f;
  if (std::fseek(f, (long)(r->off_kinds + op0), SEEK_SET) != 0 ||
      (n && std::fread(kinds, 1, n, f) != n) ||
      std::fseek(f, (long)(r->off_offsets + op0 * 8), SEEK_SET) != 0 ||
      std::fread(offsets, 8, n + 1, f) != n + 1)
    return fail(PBH_TRACE, "read failed");
  const uint64_t e0 = offsets[0], ne = offsets[n] - e0;
  for (uint64_t i = 0; i <= n; ++i) offsets[i] -= e0;
  if (ne) {
    if (!values || !priorities) return fail(PBH_PRECONDITION, "null element arrays");
    if (std::fseek(f, (long)(r->off_values + e0 * 4), SEEK_SET) != 0 ||
        std::fread(values, 4, ne, f) != ne ||
        std::fseek(f, (long)(r->off_prios + e0 * 8), SEEK_SET) != 0 ||
        std::fread(priorities, 8, ne, f) != ne)
      return fail(PBH_TRACE, "read failed");
  }
  return PBH_OK;
}

void pbh_trace_close(pbh_trace_reader* r) {
  if (!r) return;
  if (r->f) std::fclose(r->f);
  delete r;
}

}  // extern "C"
