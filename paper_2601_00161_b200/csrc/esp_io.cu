// esp_io.cu — native reader/writer of the reference's particle-file format
// (host code).
//
// Reference: prolate_ewald/cli.py:57-112 (read_particles, _parse_floats,
// write_particles).  Format: '#' starts a comment; blank lines are skipped;
// the first content line is the header 'cell Lx Ly Lz' or 'cell3' followed
// by the 9 entries of h in column order (cell vectors a, b, c); every other
// content line is 'x y z q m'.  Numbers are written with "%.17g".
// Diagnostics carry path:line[:column] like the reference's InputError.
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "esp_internal.cuh"

using esp::set_error;

struct esp_particles {
  int triclinic = 0;
  double h[9] = {0};  // row-major, columns = cell vectors
  std::vector<double> rows;  // n x 5
};

namespace {

// Python's str.splitlines() boundaries after read_text()'s universal-newline
// translation: \n, \r, \r\n, \v, \f, \x1c-\x1e and the UTF-8 encodings of
// U+0085, U+2028, U+2029.  Returns the byte length of the break at i (0: none).
size_t line_break(const std::string& t, size_t i) {
  const unsigned char c = (unsigned char)t[i];
  if (c == '\r') return (i + 1 < t.size() && t[i + 1] == '\n') ? 2 : 1;
  if (c == '\n' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e)) return 1;
  if (c == 0xC2 && i + 1 < t.size() && (unsigned char)t[i + 1] == 0x85) return 2;
  if (c == 0xE2 && i + 2 < t.size() && (unsigned char)t[i + 1] == 0x80 &&
      ((unsigned char)t[i + 2] == 0xA8 || (unsigned char)t[i + 2] == 0xA9))
    return 3;
  return 0;
}

// Python's str.split() / strip() whitespace (str.isspace) inside a line:
// ASCII \t \n \v \f \r space \x1c-\x1f, and the UTF-8 encodings of U+0085,
// U+00A0, U+1680, U+2000-U+200A, U+2028, U+2029, U+202F, U+205F, U+3000.
// Returns the byte length of the whitespace character at i (0: none).
size_t space_len(const std::string& t, size_t i) {
  const unsigned char c = (unsigned char)t[i];
  if (c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f)) return 1;
  auto b = [&](size_t k) { return i + k < t.size() ? (unsigned char)t[i + k] : 0u; };
  if (c == 0xC2 && (b(1) == 0x85 || b(1) == 0xA0)) return 2;
  if (c == 0xE1 && b(1) == 0x9A && b(2) == 0x80) return 3;
  if (c == 0xE2 && b(1) == 0x80 && ((b(2) >= 0x80 && b(2) <= 0x8A) || b(2) == 0xA8 ||
                                    b(2) == 0xA9 || b(2) == 0xAF))
    return 3;
  if (c == 0xE2 && b(1) == 0x81 && b(2) == 0x9F) return 3;
  if (c == 0xE3 && b(1) == 0x80 && b(2) == 0x80) return 3;
  return 0;
}

bool is_digit(char c) { return c >= '0' && c <= '9'; }

// One token as a Python float(): the whole token must parse.  Underscores
// are accepted only between two digits (PEP 515) and removed; hex forms and
// 'nan(...)', which strtod accepts and float() does not, are rejected.
bool parse_double(const std::string& raw, double* out) {
  if (raw.empty()) return false;
  std::string tok;
  tok.reserve(raw.size());
  for (size_t i = 0; i < raw.size(); ++i) {
    const char c = raw[i];
    if (c == 'x' || c == 'X' || c == 'p' || c == 'P' || c == '(') return false;
    if (c == '_') {
      if (i == 0 || i + 1 >= raw.size() || !is_digit(raw[i - 1]) || !is_digit(raw[i + 1]))
        return false;
      continue;
    }
    tok.push_back(c);
  }
  const char* s = tok.c_str();
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(s, &end);
  if (end == s || *end != '\0') return false;
  *out = v;  // overflow gives +-inf like float('1e999')
  return true;
}

std::string where(const char* path, long long ln) {
  return std::string(path) + ":" + std::to_string(ln);
}

}  // namespace

extern "C" {

int esp_particles_read(const char* path, esp_particles** out) {
  if (!path || !out) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  *out = nullptr;
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    set_error(std::string(path) + ": cannot open: " + std::strerror(errno));
    return ESP_ERR_INPUT;
  }
  std::string text;
  {
    char buf[1 << 16];
    size_t k;
    while ((k = std::fread(buf, 1, sizeof(buf), f)) > 0) text.append(buf, k);
    std::fclose(f);
  }
  esp_particles* p = new esp_particles();
  bool have_cell = false;
  long long ln = 0;
  size_t pos = 0;
  std::vector<std::string> cols;
  std::vector<double> vals;
  auto fail = [&](const std::string& msg) {
    set_error(msg);
    delete p;
    return ESP_ERR_INPUT;
  };
  while (pos < text.size()) {
    size_t eol = pos, brk = 0;
    while (eol < text.size() && (brk = line_break(text, eol)) == 0) ++eol;
    ++ln;
    size_t stop = text.find('#', pos);
    if (stop == std::string::npos || stop > eol) stop = eol;
    cols.clear();
    size_t a = pos;
    while (a < stop) {
      size_t w;
      while (a < stop && (w = space_len(text, a)) > 0) a += w;
      size_t b = a;
      while (b < stop && space_len(text, b) == 0) ++b;
      if (b > a) cols.emplace_back(text, a, b - a);
      a = b;
    }
    pos = eol + (brk ? brk : 1);
    if (cols.empty()) continue;
    if (!have_cell) {
      const bool ortho = cols[0] == "cell", tri = cols[0] == "cell3";
      if (!ortho && !tri)
        return fail(where(path, ln) + ": expected 'cell' or 'cell3' header, got '" + cols[0] +
                    "'");
      const size_t need = ortho ? 4 : 10;
      if (cols.size() != need)
        return fail(where(path, ln) + ": '" + cols[0] + "' header needs " +
                    (ortho ? "3 lengths" : "9 entries") + ", got " +
                    std::to_string(cols.size() - 1));
      vals.assign(need - 1, 0.0);
      for (size_t c = 1; c < need; ++c)
        if (!parse_double(cols[c], &vals[c - 1]))
          return fail(where(path, ln) + ":" + std::to_string(c + 1) + ": not a number: '" +
                      cols[c] + "'");
      if (ortho) {
        for (int d = 0; d < 3; ++d) p->h[4 * d] = vals[d];
      } else {
        // column order: entry 3*c + r is h[r][c]
        for (int c = 0; c < 3; ++c)
          for (int r = 0; r < 3; ++r) p->h[3 * r + c] = vals[3 * c + r];
        p->triclinic = 1;
      }
      have_cell = true;
      continue;
    }
    if (cols.size() != 5)
      return fail(where(path, ln) + ": expected 5 columns (x y z q m), got " +
                  std::to_string(cols.size()));
    for (size_t c = 0; c < 5; ++c) {
      double v;
      if (!parse_double(cols[c], &v))
        return fail(where(path, ln) + ":" + std::to_string(c + 1) + ": not a number: '" +
                    cols[c] + "'");
      p->rows.push_back(v);
    }
  }
  if (!have_cell) return fail(std::string(path) + ": missing 'cell' header line");
  if (p->rows.empty()) return fail(std::string(path) + ": no particle lines");
  *out = p;
  return ESP_OK;
}

int esp_particles_info(const esp_particles* p, int64_t* n, int32_t* triclinic, double* h9) {
  if (!p || !n || !triclinic || !h9) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  *n = (int64_t)(p->rows.size() / 5);
  *triclinic = p->triclinic;
  for (int k = 0; k < 9; ++k) h9[k] = p->h[k];
  return ESP_OK;
}

int esp_particles_copy(const esp_particles* p, double* pos, double* q, double* m) {
  if (!p || !pos || !q || !m) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  const size_t n = p->rows.size() / 5;
  for (size_t i = 0; i < n; ++i) {
    const double* r = &p->rows[5 * i];
    pos[3 * i] = r[0];
    pos[3 * i + 1] = r[1];
    pos[3 * i + 2] = r[2];
    q[i] = r[3];
    m[i] = r[4];
  }
  return ESP_OK;
}

int esp_particles_free(esp_particles* p) {
  delete p;
  return ESP_OK;
}

int esp_particles_write(const char* path, int64_t n, const double* h9, int32_t triclinic,
                        const double* pos, const double* q, const double* m) {
  if (!path || !h9 || n < 0 || (n > 0 && (!pos || !q || !m))) {
    set_error("null argument");
    return ESP_ERR_PARAM;
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    set_error(std::string(path) + ": cannot open for writing: " + std::strerror(errno));
    return ESP_ERR_INPUT;
  }
  std::string line;
  char num[40];
  auto put = [&](double v) {
    std::snprintf(num, sizeof(num), "%.17g", v);
    if (!line.empty() && line.back() != '\n') line.push_back(' ');
    line.append(num);
  };
  line = triclinic ? "cell3" : "cell";
  if (triclinic) {
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) put(h9[3 * r + c]);
  } else {
    for (int d = 0; d < 3; ++d) put(h9[4 * d]);
  }
  line.push_back('\n');
  bool ok = std::fwrite(line.data(), 1, line.size(), f) == line.size();
  std::string buf;
  buf.reserve(1 << 20);
  for (int64_t i = 0; i < n && ok; ++i) {
    line.clear();
    put(pos[3 * i]);
    put(pos[3 * i + 1]);
    put(pos[3 * i + 2]);
    put(q[i]);
    put(m[i]);
    line.push_back('\n');
    buf += line;
    if (buf.size() > (1 << 20)) {
      ok = std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
      buf.clear();
    }
  }
  if (ok && !buf.empty()) ok = std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) {
    set_error(std::string(path) + ": write failed");
    return ESP_ERR_INPUT;
  }
  return ESP_OK;
}

}  // extern "C"
