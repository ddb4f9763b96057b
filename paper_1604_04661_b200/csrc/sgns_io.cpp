// sgns_io.cpp -- word2vec vector-file writer, host C++.
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
