// sgns_ingest.cpp -- host-side corpus ingestion, multithreaded C++.
//
// Produces exactly what the reference's build_vocab(read_tokens(path), min_count)
// (sgns/corpus.py:86-105, :268-272) and encode_corpus(path, vocab)
// (sgns/corpus.py:275-311) produce:
//  * lines as Python's text mode iterates them (universal newlines: \n, \r\n, \r);
//  * tokens as str.split() finds them: runs of non-whitespace, whitespace being
//    ASCII \t\n\v\f\r, space, \x1c-\x1f and the Unicode spaces U+0085, U+00A0,
//    U+1680, U+2000-U+200A, U+2028, U+2029, U+202F, U+205F, U+3000 (UTF-8 input);
//  * vocabulary: count >= min_count, ordered by count descending, ties by first
//    occurrence;
//  * encoding: out-of-vocabulary tokens dropped, a sentence emitted every
//    max_sentence in-vocabulary ids and at line end if non-empty, sentence bytes =
//    sum of (UTF-8 length + 1) of every token since the previous emission.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "../../include/sgns_b200.h"
#include "sgns_text.hpp"

namespace {

using sgns_text::ws_len;

struct Mapped {
  const unsigned char *data = nullptr;
  size_t size = 0;
  int fd = -1;
  bool open(const char *path) {
    fd = ::open(path, O_RDONLY);
    if (fd < 0) return false;
    struct stat st;
    if (fstat(fd, &st) != 0) return false;
    size = (size_t)st.st_size;
    if (size == 0) return true;
    void *m = mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
    if (m == MAP_FAILED) return false;
    madvise(m, size, MADV_SEQUENTIAL);
    data = static_cast<const unsigned char *>(m);
    return true;
  }
  ~Mapped() {
    if (data) munmap(const_cast<unsigned char *>(data), size);
    if (fd >= 0) ::close(fd);
  }
};

// Split [0, size) into ranges that start at line starts (after a \n, or after a \r not
// followed by \n).
std::vector<size_t> line_aligned_cuts(const unsigned char *d, size_t size, int parts) {
  std::vector<size_t> cuts{0};
  for (int k = 1; k < parts; ++k) {
    size_t pos = std::max(cuts.back(), size * (size_t)k / (size_t)parts);
    while (pos < size) {
      if (d[pos] == '\n') { ++pos; break; }
      if (d[pos] == '\r') {
        ++pos;
        if (pos < size && d[pos] == '\n') ++pos;
        break;
      }
      ++pos;
    }
    if (pos > cuts.back() && pos < size) cuts.push_back(pos);
  }
  cuts.push_back(size);
  return cuts;
}

// Calls fn(token_view) for every token and eol() at each line end of [lo, hi).
template <typename F, typename E>
void scan(const unsigned char *d, size_t lo, size_t hi, F &&fn, E &&eol) {
  size_t i = lo;
  size_t tok = SIZE_MAX;
  const unsigned char *end = d + hi;
  while (i < hi) {
    const unsigned char c = d[i];
    if (c == '\n' || c == '\r') {
      if (tok != SIZE_MAX) {
        fn(std::string_view(reinterpret_cast<const char *>(d + tok), i - tok));
        tok = SIZE_MAX;
      }
      eol();
      i += (c == '\r' && i + 1 < hi && d[i + 1] == '\n') ? 2 : 1;
      continue;
    }
    const int w = ws_len(d + i, end);
    if (w) {
      if (tok != SIZE_MAX) {
        fn(std::string_view(reinterpret_cast<const char *>(d + tok), i - tok));
        tok = SIZE_MAX;
      }
      i += w;
      continue;
    }
    if (tok == SIZE_MAX) tok = i;
    ++i;
  }
  if (tok != SIZE_MAX) fn(std::string_view(reinterpret_cast<const char *>(d + tok), hi - tok));
  if (hi > lo && d[hi - 1] != '\n' && d[hi - 1] != '\r') eol();  // unterminated last line
}

struct Entry {
  int64_t count;
  int64_t first;  // global token ordinal of the first occurrence
};

inline uint64_t hash_bytes(const char *p, size_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;  // FNV-1a, then a final avalanche
  for (size_t i = 0; i < n; ++i) h = (h ^ (unsigned char)p[i]) * 0x100000001b3ULL;
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdULL;
  h ^= h >> 33;
  return h;
}

// Open-addressing table keyed by byte strings that outlive it (mmap or owned strings).
struct FlatMap {
  struct Slot {
    uint64_t h;
    const char *p;
    uint32_t len;  // 0 with p == nullptr: empty
    int64_t a, b;  // (count, first) while counting; (id, -) for the vocabulary index
  };
  std::vector<Slot> slots;
  size_t mask = 0, n = 0;
  explicit FlatMap(size_t cap = 1 << 12) { reset(cap); }
  void reset(size_t cap) {
    size_t c = 16;
    while (c < cap) c <<= 1;
    slots.assign(c, Slot{0, nullptr, 0, 0, 0});
    mask = c - 1;
    n = 0;
  }
  void grow() {
    std::vector<Slot> old;
    old.swap(slots);
    slots.assign(old.size() * 2, Slot{0, nullptr, 0, 0, 0});
    mask = slots.size() - 1;
    for (auto &s : old)
      if (s.p) {
        size_t i = s.h & mask;
        while (slots[i].p) i = (i + 1) & mask;
        slots[i] = s;
      }
  }
  // returns the slot; inserted == true when the key was new (a, b left zero)
  Slot *upsert(std::string_view k, uint64_t h, bool &inserted) {
    if ((n + 1) * 2 > slots.size()) grow();
    size_t i = h & mask;
    while (true) {
      Slot &s = slots[i];
      if (!s.p) {
        s.h = h;
        s.p = k.data();
        s.len = (uint32_t)k.size();
        ++n;
        inserted = true;
        return &s;
      }
      if (s.h == h && s.len == k.size() && std::memcmp(s.p, k.data(), k.size()) == 0) {
        inserted = false;
        return &s;
      }
      i = (i + 1) & mask;
    }
  }
  const Slot *find(std::string_view k, uint64_t h) const {
    size_t i = h & mask;
    while (true) {
      const Slot &s = slots[i];
      if (!s.p) return nullptr;
      if (s.h == h && s.len == k.size() && std::memcmp(s.p, k.data(), k.size()) == 0) return &s;
      i = (i + 1) & mask;
    }
  }
};

}  // namespace

struct sgns_vocab {
  std::vector<std::string> tokens;
  std::vector<int64_t> counts;
  FlatMap index;
  int64_t total_tokens = 0;
  int64_t tokens_bytes = 0;
  void build_index() {
    index.reset(tokens.size() * 2 + 16);
    tokens_bytes = 0;
    for (size_t i = 0; i < tokens.size(); ++i) {
      std::string_view k(tokens[i]);
      bool ins;
      auto *sl = index.upsert(k, hash_bytes(k.data(), k.size()), ins);
      if (ins) sl->a = (int64_t)i;  // first id wins if a vocabulary repeats a token
      tokens_bytes += (int64_t)tokens[i].size();
    }
  }
  int32_t lookup(std::string_view k) const {
    const auto *sl = index.find(k, hash_bytes(k.data(), k.size()));
    return sl ? (int32_t)sl->a : -1;
  }
};

struct sgns_encoded {
  std::vector<int32_t> ids;
  std::vector<int64_t> offsets;
  std::vector<int64_t> sentence_bytes;
};

extern "C" {

int sgns_vocab_build(const char *path, int32_t min_count, int32_t threads, sgns_vocab **out,
                     int64_t *vocab_size, int64_t *tokens_bytes) {
  if (!path || !out || !vocab_size || !tokens_bytes || min_count < 1) return SGNS_E_ARG;
  Mapped mf;
  if (!mf.open(path)) return SGNS_E_IO;
  const int T = std::max(1, threads);
  const auto cuts = line_aligned_cuts(mf.data, mf.size, T);
  const int parts = (int)cuts.size() - 1;
  std::vector<FlatMap> maps(parts);
  std::vector<int64_t> ntok(parts, 0);
  std::vector<std::thread> pool;
  for (int t = 0; t < parts; ++t)
    pool.emplace_back([&, t] {
      auto &m = maps[t];
      m.reset(1 << 16);
      int64_t k = 0;
      scan(mf.data, cuts[t], cuts[t + 1],
           [&](std::string_view tok) {
             bool ins;
             auto *sl = m.upsert(tok, hash_bytes(tok.data(), tok.size()), ins);
             if (ins) sl->b = k;
             sl->a += 1;
             ++k;
           },
           [] {});
      ntok[t] = k;
    });
  for (auto &th : pool) th.join();
  std::vector<int64_t> base(parts, 0);
  for (int t = 1; t < parts; ++t) base[t] = base[t - 1] + ntok[t - 1];
  size_t guess = 0;
  for (auto &m : maps) guess = std::max(guess, m.n);
  FlatMap all(guess * 2 + 16);
  for (int t = 0; t < parts; ++t)  // parts in file order: the first insert is the first occurrence
    for (auto &sl : maps[t].slots)
      if (sl.p) {
        bool ins;
        auto *d = all.upsert(std::string_view(sl.p, sl.len), sl.h, ins);
        if (ins) d->b = sl.b + base[t];
        d->a += sl.a;
      }
  std::vector<std::pair<std::string_view, Entry>> kept;
  kept.reserve(all.n);
  for (auto &sl : all.slots)
    if (sl.p && sl.a >= min_count) kept.emplace_back(std::string_view(sl.p, sl.len), Entry{sl.a, sl.b});
  if (kept.empty()) return SGNS_E_EMPTY;
  std::sort(kept.begin(), kept.end(), [](const auto &a, const auto &b) {
    if (a.second.count != b.second.count) return a.second.count > b.second.count;
    return a.second.first < b.second.first;
  });
  auto *v = new sgns_vocab();
  v->tokens.reserve(kept.size());
  v->counts.reserve(kept.size());
  for (auto &kv : kept) {
    v->tokens.emplace_back(kv.first);
    v->counts.push_back(kv.second.count);
    v->total_tokens += kv.second.count;
  }
  v->build_index();
  *out = v;
  *vocab_size = (int64_t)v->tokens.size();
  *tokens_bytes = v->tokens_bytes;
  return SGNS_OK;
}

int sgns_vocab_from_tokens(const char *blob, const int64_t *token_offsets, const int64_t *counts,
                           int64_t n, sgns_vocab **out) {
  if (!blob || !token_offsets || !out || n < 1) return SGNS_E_ARG;
  auto *v = new sgns_vocab();
  v->tokens.reserve(n);
  for (int64_t i = 0; i < n; ++i) {
    v->tokens.emplace_back(blob + token_offsets[i], (size_t)(token_offsets[i + 1] - token_offsets[i]));
    const int64_t c = counts ? counts[i] : 1;
    v->counts.push_back(c);
    v->total_tokens += c;
  }
  v->build_index();
  *out = v;
  return SGNS_OK;
}

int sgns_vocab_export(const sgns_vocab *v, char *blob, int64_t *token_offsets, int64_t *counts) {
  if (!v || !blob || !token_offsets || !counts) return SGNS_E_ARG;
  int64_t pos = 0;
  for (size_t i = 0; i < v->tokens.size(); ++i) {
    token_offsets[i] = pos;
    std::memcpy(blob + pos, v->tokens[i].data(), v->tokens[i].size());
    pos += (int64_t)v->tokens[i].size();
    counts[i] = v->counts[i];
  }
  token_offsets[v->tokens.size()] = pos;
  return SGNS_OK;
}

void sgns_vocab_free(sgns_vocab *v) { delete v; }

int sgns_encode(const sgns_vocab *v, const char *path, int32_t max_sentence, int32_t threads,
                sgns_encoded **out, int64_t *n_tokens, int64_t *n_sentences) {
  if (!v || !path || !out || !n_tokens || !n_sentences || max_sentence < 1) return SGNS_E_ARG;
  Mapped mf;
  if (!mf.open(path)) return SGNS_E_IO;
  const int T = std::max(1, threads);
  const auto cuts = line_aligned_cuts(mf.data, mf.size, T);
  const int parts = (int)cuts.size() - 1;
  std::vector<sgns_encoded> piece(parts);
  std::vector<std::thread> pool;
  for (int t = 0; t < parts; ++t)
    pool.emplace_back([&, t] {
      auto &e = piece[t];
      int64_t cur = 0, bytes = 0;  // ids in the open sentence, its byte footprint
      scan(mf.data, cuts[t], cuts[t + 1],
           [&](std::string_view tok) {
             bytes += (int64_t)tok.size() + 1;
             const int32_t id = v->lookup(tok);
             if (id < 0) return;
             e.ids.push_back(id);
             if (++cur >= max_sentence) {
               e.offsets.push_back(cur);
               e.sentence_bytes.push_back(bytes);
               cur = 0;
               bytes = 0;
             }
           },
           [&] {
             if (cur > 0) {
               e.offsets.push_back(cur);
               e.sentence_bytes.push_back(bytes);
             }
             cur = 0;
             bytes = 0;
           });
    });
  for (auto &th : pool) th.join();
  auto *r = new sgns_encoded();
  size_t nid = 0, ns = 0;
  for (auto &e : piece) {
    nid += e.ids.size();
    ns += e.offsets.size();
  }
  r->ids.reserve(nid);
  r->offsets.reserve(ns + 1);
  r->sentence_bytes.reserve(ns);
  r->offsets.push_back(0);
  for (auto &e : piece) {
    r->ids.insert(r->ids.end(), e.ids.begin(), e.ids.end());
    for (size_t s = 0; s < e.offsets.size(); ++s) {
      r->offsets.push_back(r->offsets.back() + e.offsets[s]);
      r->sentence_bytes.push_back(e.sentence_bytes[s]);
    }
  }
  *out = r;
  *n_tokens = (int64_t)r->ids.size();
  *n_sentences = (int64_t)r->sentence_bytes.size();
  return SGNS_OK;
}

int sgns_encoded_export(const sgns_encoded *e, int32_t *ids, int64_t *offsets, int64_t *sentence_bytes) {
  if (!e || !ids || !offsets || !sentence_bytes) return SGNS_E_ARG;
  if (!e->ids.empty()) std::memcpy(ids, e->ids.data(), e->ids.size() * sizeof(int32_t));
  std::memcpy(offsets, e->offsets.data(), e->offsets.size() * sizeof(int64_t));
  if (!e->sentence_bytes.empty())
    std::memcpy(sentence_bytes, e->sentence_bytes.data(), e->sentence_bytes.size() * sizeof(int64_t));
  return SGNS_OK;
}

void sgns_encoded_free(sgns_encoded *e) { delete e; }

}  // extern "C"
