// sgns_io.cpp -- word2vec vector files, host C++: writer and reader.
//
// Byte-identical to the reference's save_model (sgns/model.py:118-139):
//   header "V D\n"; text: "token v1 v2 ... vD\n" with each value formatted "%.6g"
//   (Python's f"{v:.6g}" of the row's own value: float32 promoted to double, or the
//   float64 value of a float64 model); binary: token, b" ", D little-endian float32
//   (a float64 row is cast, as np.ascontiguousarray(rows, dtype="<f4")), b"\n".
// Rows may live in device memory: they are streamed device->host through a pinned
// staging buffer in slabs, so a 1.2 GB M_in never needs a second host copy.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/sgns_b200.h"
#include "sgns_text.hpp"

extern "C" int sgns_write_vectors(const char *path, const char *tokens_blob, const int64_t *token_offsets,
                                  int64_t vocab, int32_t dim, const void *rows, int64_t ld,
                                  int32_t binary, int32_t rows_on_device, int32_t dtype) {
  if (!path || !tokens_blob || !token_offsets || !rows || vocab < 1 || dim < 1 || ld < dim ||
      (dtype != SGNS_F32 && dtype != SGNS_F64))
    return SGNS_E_ARG;
  const int64_t esz = dtype == SGNS_F64 ? 8 : 4;
  FILE *f = std::fopen(path, "wb");
  if (!f) return SGNS_E_IO;
  std::vector<char> buf;
  buf.reserve(1 << 22);
  auto flush = [&]() {
    if (!buf.empty()) std::fwrite(buf.data(), 1, buf.size(), f);
    buf.clear();
  };
  char tmp[64];
  int n = std::snprintf(tmp, sizeof(tmp), "%lld %d\n", (long long)vocab, dim);
  buf.insert(buf.end(), tmp, tmp + n);
  const int64_t slab = rows_on_device ? std::max<int64_t>(1, (int64_t(64) << 20) / (ld * esz)) : vocab;
  unsigned char *stage = nullptr;
  if (rows_on_device && cudaMallocHost(&stage, (size_t)(slab * ld * esz)) != cudaSuccess) {
    std::fclose(f);
    return SGNS_E_ARG;
  }
  int rc = SGNS_OK;
  for (int64_t r0 = 0; r0 < vocab && rc == SGNS_OK; r0 += slab) {
    const int64_t nr = std::min(slab, vocab - r0);
    const unsigned char *src = static_cast<const unsigned char *>(rows) + r0 * ld * esz;
    if (rows_on_device) {
      const cudaError_t e = cudaMemcpy(stage, src, (size_t)(nr * ld * esz), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) { rc = (int)e; break; }
      src = stage;
    }
    for (int64_t i = 0; i < nr; ++i) {
      const int64_t w = r0 + i;
      buf.insert(buf.end(), tokens_blob + token_offsets[w], tokens_blob + token_offsets[w + 1]);
      buf.push_back(' ');
      const unsigned char *row = src + i * ld * esz;
      auto value = [&](int j) -> double {
        if (esz == 8) {
          double v;
          std::memcpy(&v, row + 8 * j, 8);
          return v;
        }
        float v;
        std::memcpy(&v, row + 4 * j, 4);
        return (double)v;
      };
      if (binary) {
        for (int j = 0; j < dim; ++j) {
          const float v = (float)value(j);  // little-endian host
          const char *b = reinterpret_cast<const char *>(&v);
          buf.insert(buf.end(), b, b + 4);
        }
      } else {
        for (int j = 0; j < dim; ++j) {
          const int k = std::snprintf(tmp, sizeof(tmp), j ? " %.6g" : "%.6g", value(j));
          buf.insert(buf.end(), tmp, tmp + k);
        }
      }
      buf.push_back('\n');
      if (buf.size() > (size_t(1) << 22)) flush();
    }
  }
  flush();
  if (stage) cudaFreeHost(stage);
  if (std::fclose(f) != 0 && rc == SGNS_OK) rc = SGNS_E_IO;
  return rc;
}

// ------------------------------------------------------------------ reader ----
// The reference's load_model / detect_format (sgns/model.py:140-225) with the file mapped
// once: header "V D", a format sniff on the first row, then every row.  Anything the
// fast path cannot decide with certainty -- a text line that is not "token v1 .. vD" with
// plain ASCII numbers, a binary token that is not valid UTF-8 -- is handed back to the
// caller (status 1 with the row and its byte offset), which applies Python's own rules to
// that one row (raising exactly what the reference raises) and resumes here.
namespace {

struct FileBytes {
  std::vector<unsigned char> data;
  bool load(const char *path) {
    FILE *f = std::fopen(path, "rb");
    if (!f) return false;
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    data.resize(n > 0 ? (size_t)n : 0);
    const bool ok = data.empty() || std::fread(data.data(), 1, data.size(), f) == data.size();
    std::fclose(f);
    return ok;
  }
};

// ASCII integer with Python int() syntax (sign, digits, single underscores); false: not
// decidable here
bool parse_int(const unsigned char *p, const unsigned char *e, int64_t *v) {
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p == e || *p < '0' || *p > '9') return false;
  int64_t x = 0;
  while (p < e) {
    if (*p >= '0' && *p <= '9') {
      x = x * 10 + (*p++ - '0');
      if (x > (int64_t(1) << 50)) return false;
    } else if (*p == '_' && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
      ++p;
    } else {
      return false;
    }
  }
  *v = neg ? -x : x;
  return true;
}

}  // namespace

extern "C" int sgns_vectors_header(const char *path, int64_t *vocab, int32_t *dim, int64_t *header_bytes) {
  if (!path || !vocab || !dim || !header_bytes) return SGNS_E_ARG;
  FILE *f = std::fopen(path, "rb");
  if (!f) return SGNS_E_IO;
  std::vector<unsigned char> line;
  int c;
  while ((c = std::fgetc(f)) != EOF) {
    line.push_back((unsigned char)c);
    if (c == '\n') break;
  }
  std::fclose(f);
  *header_bytes = (int64_t)line.size();
  const unsigned char *p = line.data(), *e = p + line.size();
  if (!sgns_text::utf8_valid(p, e)) return 1;
  const unsigned char *f0[3], *f1[3];
  int nf = 0;
  while (p < e) {
    int w;
    while (p < e && (w = sgns_text::ws_len(p, e)) > 0) p += w;
    if (p == e) break;
    if (nf == 2) return 1;  // a third field: malformed
    f0[nf] = p;
    while (p < e && sgns_text::ws_len(p, e) == 0) ++p;
    f1[nf++] = p;
  }
  int64_t v, d;
  if (nf != 2 || !parse_int(f0[0], f1[0], &v) || !parse_int(f0[1], f1[1], &d)) return 1;
  if (v < 1 || d < 1 || d > (int64_t(1) << 30)) return 1;
  *vocab = v;
  *dim = (int32_t)d;
  return SGNS_OK;
}

// *binary <- 1 / 0 as detect_format decides; status 1: a probe field needs Python's float()
extern "C" int sgns_vectors_sniff(const char *path, int64_t header_bytes, int32_t dim, int32_t *binary) {
  if (!path || !binary || dim < 1) return SGNS_E_ARG;
  FILE *f = std::fopen(path, "rb");
  if (!f) return SGNS_E_IO;
  std::vector<unsigned char> probe((size_t)dim * 16 + 64);
  std::fseek(f, (long)header_bytes, SEEK_SET);
  probe.resize(std::fread(probe.data(), 1, probe.size(), f));
  std::fclose(f);
  const unsigned char *p = probe.data(), *e = p + probe.size();
  if (!sgns_text::utf8_valid(p, e)) {
    *binary = 1;
    return SGNS_OK;
  }
  int nf = 0;
  bool unsure = false;
  while (p < e && nf < dim + 1) {
    int w;
    while (p < e && (w = sgns_text::ws_len(p, e)) > 0) p += w;
    if (p == e) break;
    const unsigned char *s0 = p;
    while (p < e && sgns_text::ws_len(p, e) == 0) ++p;
    if (nf++ == 0) continue;  // the token
    double x;
    const sgns_text::Num r = sgns_text::parse_float(s0, p, &x);
    if (r == sgns_text::Num::invalid) {
      *binary = 1;
      return SGNS_OK;
    }
    unsure |= r == sgns_text::Num::unsure;
  }
  if (nf < dim + 1) {
    *binary = probe.empty() ? 0 : 1;
    return SGNS_OK;
  }
  if (unsure) return 1;
  *binary = 0;
  return SGNS_OK;
}

// Rows [*row, vocab) from byte *offset on.  vectors: vocab x dim float32; tokens are
// returned as byte spans [tok_start, tok_end) of the file.  Status: SGNS_OK (done), 1 (row
// *row at *offset needs the caller), SGNS_E_TRUNC (the file ends inside row *row).
extern "C" int sgns_parse_vectors(const char *path, int32_t binary, int64_t vocab, int32_t dim,
                                  float *vectors, int64_t *tok_start, int64_t *tok_end, int64_t *row,
                                  int64_t *offset) {
  if (!path || !vectors || !tok_start || !tok_end || !row || !offset || vocab < 1 || dim < 1)
    return SGNS_E_ARG;
  FileBytes fb;
  if (!fb.load(path)) return SGNS_E_IO;
  const unsigned char *base = fb.data.data(), *end = base + fb.data.size();
  const unsigned char *p = base + *offset;
  int64_t i = *row;
  for (; i < vocab; ++i) {
    *row = i;
    *offset = p - base;
    float *out = vectors + i * (int64_t)dim;
    if (binary) {
      const unsigned char *t0 = p;
      while (p < end && *p != ' ') ++p;
      if (p == end) return SGNS_E_TRUNC;
      const unsigned char *t1 = p++;
      if (end - p < (int64_t)dim * 4) return SGNS_E_TRUNC;
      if (!sgns_text::utf8_valid(t0, t1)) return 1;
      while (t0 < t1 && *t0 == '\n') ++t0;  // .lstrip("\n") of the decoded token
      tok_start[i] = t0 - base;
      tok_end[i] = t1 - base;
      std::memcpy(out, p, (size_t)dim * 4);  // little-endian host, as "<f4"
      p += (size_t)dim * 4;
      if (p < end && *p == '\n') ++p;
      continue;
    }
    // text: one line as Python's text mode yields it (universal newlines), split on ' '
    if (p == end) return SGNS_E_TRUNC;
    const unsigned char *l0 = p;
    while (p < end && *p != '\n' && *p != '\r') ++p;
    const unsigned char *l1 = p;
    if (p < end) p += (*p == '\r' && p + 1 < end && p[1] == '\n') ? 2 : 1;
    if (!sgns_text::utf8_valid(l0, l1)) return 1;
    const unsigned char *q = l0;
    while (q < l1 && *q != ' ') ++q;
    tok_start[i] = l0 - base;
    tok_end[i] = q - base;
    int j = 0;
    while (q < l1) {
      const unsigned char *f0 = ++q;  // past the separating space
      while (q < l1 && *q != ' ') ++q;
      double x;
      if (j == dim || sgns_text::parse_float(f0, q, &x) != sgns_text::Num::ok) return 1;
      out[j++] = (float)x;
    }
    if (j != dim) return 1;
  }
  *row = vocab;
  *offset = p - base;
  return SGNS_OK;
}
