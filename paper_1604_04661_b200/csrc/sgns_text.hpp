// sgns_text.hpp -- Python text semantics shared by the host-side readers (ingestion,
// vector files): str.split() whitespace and float() number syntax, on UTF-8 bytes.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>

namespace sgns_text {

// length of the whitespace code point starting at p (0: not whitespace), as str.split()
// sees it: ASCII \t\n\v\f\r, space, \x1c-\x1f and the Unicode spaces U+0085, U+00A0,
// U+1680, U+2000-U+200A, U+2028, U+2029, U+202F, U+205F, U+3000
inline int ws_len(const unsigned char *p, const unsigned char *end) {
  const unsigned char c = p[0];
  if (c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f)) return 1;
  if (c < 0xc2) return 0;
  if (c == 0xc2 && p + 1 < end && (p[1] == 0x85 || p[1] == 0xa0)) return 2;
  if (c == 0xe1 && p + 2 < end && p[1] == 0x9a && p[2] == 0x80) return 3;
  if (c == 0xe2 && p + 2 < end) {
    if (p[1] == 0x80 && ((p[2] >= 0x80 && p[2] <= 0x8a) || p[2] == 0xa8 || p[2] == 0xa9 || p[2] == 0xaf))
      return 3;
    if (p[1] == 0x81 && p[2] == 0x9f) return 3;
  }
  if (c == 0xe3 && p + 2 < end && p[1] == 0x80 && p[2] == 0x80) return 3;
  return 0;
}

// strict UTF-8 validity of [p, end) (what bytes.decode("utf-8") accepts)
inline bool utf8_valid(const unsigned char *p, const unsigned char *end) {
  while (p < end) {
    const unsigned char c = *p;
    int n;
    uint32_t cp;
    if (c < 0x80) { ++p; continue; }
    if (c >= 0xc2 && c <= 0xdf) { n = 1; cp = c & 0x1f; }
    else if (c >= 0xe0 && c <= 0xef) { n = 2; cp = c & 0x0f; }
    else if (c >= 0xf0 && c <= 0xf4) { n = 3; cp = c & 0x07; }
    else return false;
    if (end - p <= n) return false;
    for (int i = 1; i <= n; ++i) {
      if ((p[i] & 0xc0) != 0x80) return false;
      cp = (cp << 6) | (p[i] & 0x3f);
    }
    if ((n == 2 && (cp < 0x800 || (cp >= 0xd800 && cp <= 0xdfff))) || (n == 3 && (cp < 0x10000 || cp > 0x10ffff)))
      return false;
    p += n + 1;
  }
  return true;
}

enum class Num { ok, invalid, unsure };

// float(s) for a field without surrounding whitespace: ok (value in *out, the double
// Python computes), invalid (float() raises), or unsure (non-ASCII bytes: Python's own
// float() must decide -- it also accepts other Unicode decimal digits)
inline Num parse_float(const unsigned char *p, const unsigned char *end, double *out) {
  if (p == end) return Num::invalid;
  std::string clean;
  clean.reserve(end - p);
  const unsigned char *q = p;
  if (*q == '+' || *q == '-') clean.push_back((char)*q++);
  auto word = [&](const char *w) {
    const size_t n = std::strlen(w);
    if ((size_t)(end - q) != n) return false;
    for (size_t i = 0; i < n; ++i)
      if ((q[i] | 0x20) != (unsigned char)w[i]) return false;
    return true;
  };
  for (const unsigned char *r = p; r < end; ++r)
    if (*r >= 0x80) return Num::unsure;
  if (word("inf") || word("infinity") || word("nan")) {
    clean.append(reinterpret_cast<const char *>(q), end - q);
    *out = std::strtod(clean.c_str(), nullptr);
    return Num::ok;
  }
  // digitpart: digit ("_"? digit)*
  auto digits = [&](bool required) {
    const unsigned char *s0 = q;
    if (q < end && *q >= '0' && *q <= '9') {
      clean.push_back((char)*q++);
      while (q < end) {
        if (*q >= '0' && *q <= '9') clean.push_back((char)*q++);
        else if (*q == '_' && q + 1 < end && q[1] >= '0' && q[1] <= '9') ++q;
        else break;
      }
    }
    return q > s0 || !required;
  };
  const bool int_part = q < end && *q >= '0' && *q <= '9';
  digits(false);
  bool frac_part = false;
  if (q < end && *q == '.') {
    clean.push_back('.');
    ++q;
    frac_part = q < end && *q >= '0' && *q <= '9';
    digits(false);
  }
  if (!int_part && !frac_part) return Num::invalid;
  if (q < end && (*q == 'e' || *q == 'E')) {
    clean.push_back('e');
    ++q;
    if (q < end && (*q == '+' || *q == '-')) clean.push_back((char)*q++);
    if (!digits(true)) return Num::invalid;
  }
  if (q != end) return Num::invalid;
  *out = std::strtod(clean.c_str(), nullptr);
  return Num::ok;
}

}  // namespace sgns_text
