// Op-trace files: the reference's text format (trace_format.cpp:34-126) and
// a packed binary form with a streaming chunk reader. See include/pbh_trace_io.h.
#include "../../include/pbh_trace_io.h"

#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
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

struct ParseError {
  uint64_t op;
  std::string msg;
};

// trace_format.cpp:13-23
uint64_t parse_number(std::istringstream& line, uint64_t op, uint64_t line_no, const char* what,
                      uint64_t max) {
  uint64_t x = 0;
  if (!(line >> x))
    throw ParseError{op, "line " + std::to_string(line_no) + ": missing or bad " + what};
  if (x > max) throw ParseError{op, "line " + std::to_string(line_no) + ": " + what + " out of range"};
  return x;
}

void require_line_end(std::istringstream& line, uint64_t op, uint64_t line_no) {
  std::string rest;
  if (line >> rest) throw ParseError{op, "line " + std::to_string(line_no) + ": trailing tokens"};
}

bool write_all(FILE* f, const void* p, size_t n) { return n == 0 || fwrite(p, 1, n, f) == n; }
bool write_pad(FILE* f, size_t n) {
  static const uint8_t z[8] = {0};
  return n == 0 || fwrite(z, 1, n, f) == n;
}

}  // namespace

extern "C" {

const char* pbh_trace_last_error(void) { return g_err.c_str(); }

int pbh_trace_load_text(const char* path, pbh_trace_buf** out, uint64_t* failed_op) {
  if (!path || !out) return fail(PBH_PRECONDITION, "null argument");
  *out = nullptr;
  if (failed_op) *failed_op = ~0ull;
  std::ifstream in(path);
  if (!in) {
    if (failed_op) *failed_op = 0;
    return fail(PBH_TRACE, std::string("cannot open trace file: ") + path);
  }
  auto* t = new pbh_trace_buf();
  constexpr uint64_t kMaxValue = std::numeric_limits<uint32_t>::max();
  constexpr uint64_t kMaxPrio = std::numeric_limits<uint64_t>::max();
  std::string raw;
  uint64_t line_no = 0;
  try {
    while (std::getline(in, raw)) {
      ++line_no;
      const auto hash = raw.find('#');
      if (hash != std::string::npos) raw.erase(hash);
      std::istringstream line(raw);
      std::string tag;
      if (!(line >> tag)) continue;  // blank or comment-only line
      const uint64_t op = t->kinds.size();
      if (tag.size() != 1)
        throw ParseError{op, "line " + std::to_string(line_no) + ": unknown op '" + tag + "'"};
      switch (tag[0]) {
        case 'U': {
          const uint64_t v = parse_number(line, op, line_no, "value", kMaxValue);
          const uint64_t p = parse_number(line, op, line_no, "priority", kMaxPrio);
          require_line_end(line, op, line_no);
          t->values.push_back((uint32_t)v);
          t->prios.push_back(p);
          break;
        }
        case 'B': {
          const uint64_t k = parse_number(line, op, line_no, "batch size", 1u << 24);
          if (k == 0) throw ParseError{op, "line " + std::to_string(line_no) + ": empty batch"};
          for (uint64_t j = 0; j < k; ++j) {
            t->values.push_back((uint32_t)parse_number(line, op, line_no, "value", kMaxValue));
            t->prios.push_back(parse_number(line, op, line_no, "priority", kMaxPrio));
          }
          require_line_end(line, op, line_no);
          break;
        }
        case 'E':
          require_line_end(line, op, line_no);
          break;
        case 'D': {
          const uint64_t v = parse_number(line, op, line_no, "value", kMaxValue);
          require_line_end(line, op, line_no);
          t->values.push_back((uint32_t)v);
          t->prios.push_back(0);
          break;
        }
        default:
          throw ParseError{op, "line " + std::to_string(line_no) + ": unknown op '" + tag + "'"};
      }
      t->kinds.push_back((uint8_t)tag[0]);
      t->offsets.push_back(t->values.size());
    }
  } catch (const ParseError& e) {
    delete t;
    if (failed_op) *failed_op = e.op;
    return fail(PBH_TRACE, "op " + std::to_string(e.op) + ": " + e.msg);
  }
  *out = t;
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
  std::ofstream out(path);
  if (!out) return fail(PBH_TRACE, std::string("cannot open trace file for writing: ") + path);
  for (uint64_t i = 0; i < n_ops; ++i) {
    const uint64_t b = offsets[i], e = offsets[i + 1];
    switch (kinds[i]) {
      case 'U':
        out << "U " << values[b] << ' ' << priorities[b] << '\n';
        break;
      case 'B':
        out << "B " << (e - b);
        for (uint64_t j = b; j < e; ++j) out << ' ' << values[j] << ' ' << priorities[j];
        out << '\n';
        break;
      case 'E':
        out << "E\n";
        break;
      case 'D':
        out << "D " << values[b] << '\n';
        break;
      default:
        return fail(PBH_TRACE, "op " + std::to_string(i) + ": unknown op kind");
    }
  }
  return out ? PBH_OK : fail(PBH_TRACE, "write failed");
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
