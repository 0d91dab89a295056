// tbik_io.cu -- the reference's TBIK matrix file (matrix.hpp:86-87,
// matrix.cpp:185-284): "TBIK" magic, u16 format version 1, u16 dtype (0 = f32,
// 1 = bf16), u64 rows, u64 cols, then the row-major payload, all little-endian.
// Host-only; the same errors as the reference (Io, Truncated, BadMagic,
// UnknownDtype for an unknown version or dtype code).  Goldens written by the
// reference library and by this one are byte-identical (tests/test_io.py).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "tbik_common.cuh"
#include "tbik_internal.h"

namespace tbik_b200 {
namespace {

constexpr char kMagic[4] = {'T', 'B', 'I', 'K'};
constexpr uint16_t kFormatVersion = 1;

void put_u16(std::vector<unsigned char>& b, uint16_t v) {
  b.push_back(static_cast<unsigned char>(v & 0xFF));
  b.push_back(static_cast<unsigned char>(v >> 8));
}
void put_u64(std::vector<unsigned char>& b, uint64_t v) {
  for (int i = 0; i < 8; ++i) b.push_back(static_cast<unsigned char>((v >> (8 * i)) & 0xFF));
}
uint16_t get_u16(const unsigned char* p) { return static_cast<uint16_t>(p[0] | (p[1] << 8)); }
uint64_t get_u64(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

// Reads the whole file (matrix.cpp:236-243) and validates the header
// (matrix.cpp:245-266).
tbik_status load(const char* path, std::vector<unsigned char>* buf, int* dtype, int64_t* rows, int64_t* cols) {
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return set_error(TBIK_IO, std::string("cannot open for reading: ") + path);
  unsigned char chunk[65536];
  size_t n;
  while ((n = std::fread(chunk, 1, sizeof(chunk), f)) > 0) buf->insert(buf->end(), chunk, chunk + n);
  std::fclose(f);
  const unsigned char* p = buf->data();
  if (buf->size() < 24) return set_error(TBIK_TRUNCATED, std::string("truncated header: ") + path);
  if (std::memcmp(p, kMagic, 4) != 0) return set_error(TBIK_BAD_MAGIC, std::string("bad magic in ") + path);
  const uint16_t version = get_u16(p + 4);
  if (version != kFormatVersion)
    return set_error(TBIK_UNKNOWN_DTYPE, "unsupported format version " + std::to_string(version) + " in " + path);
  const uint16_t code = get_u16(p + 6);
  if (code > 1)
    return set_error(TBIK_UNKNOWN_DTYPE, "unknown dtype code " + std::to_string(code) + " in " + path);
  const uint64_t r = get_u64(p + 8), c = get_u64(p + 16);
  const uint64_t esz = code == 0 ? 4 : 2;
  if (c != 0 && r > UINT64_MAX / c) return set_error(TBIK_TRUNCATED, std::string("truncated payload in ") + path);
  const uint64_t elems = r * c;
  if (elems > (UINT64_MAX - 24) / esz || buf->size() != 24 + elems * esz)
    return set_error(TBIK_TRUNCATED, std::string("truncated payload in ") + path);
  // a Matrix needs rows, cols >= 1 (Matrix::from_f32 / from_bf16 -> BadDimension)
  if (r == 0 || c == 0 || r > INT64_MAX || c > INT64_MAX)
    return set_error(TBIK_BAD_DIMENSION, std::string("matrix dimensions must be >= 1 in ") + path);
  *dtype = code == 0 ? TBIK_F32 : TBIK_BF16;
  *rows = static_cast<int64_t>(r);
  *cols = static_cast<int64_t>(c);
  return TBIK_OK;
}

}  // namespace
}  // namespace tbik_b200

using namespace tbik_b200;

extern "C" {

tbik_status tbik_matrix_write(const char* path, const void* data, int dtype, int64_t rows, int64_t cols) {
  if (!path || (!data && rows * cols > 0)) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  if (dtype != TBIK_F32 && dtype != TBIK_BF16) return set_error(TBIK_UNKNOWN_DTYPE, "unknown dtype");
  if (rows < 1 || cols < 1) return set_error(TBIK_BAD_DIMENSION, "matrix dimensions must be >= 1");
  const size_t esz = dtype == TBIK_F32 ? 4 : 2;
  const size_t elems = static_cast<size_t>(rows) * static_cast<size_t>(cols);
  std::vector<unsigned char> buf;
  buf.reserve(24 + elems * esz);
  buf.insert(buf.end(), kMagic, kMagic + 4);
  put_u16(buf, kFormatVersion);
  put_u16(buf, static_cast<uint16_t>(dtype == TBIK_F32 ? 0 : 1));
  put_u64(buf, static_cast<uint64_t>(rows));
  put_u64(buf, static_cast<uint64_t>(cols));
  // explicit little-endian payload (matrix.cpp:218-227)
  const unsigned char* src = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < elems; ++i) {
    if (esz == 4) {
      uint32_t u;
      std::memcpy(&u, src + 4 * i, 4);
      for (int b = 0; b < 4; ++b) buf.push_back(static_cast<unsigned char>((u >> (8 * b)) & 0xFF));
    } else {
      uint16_t u;
      std::memcpy(&u, src + 2 * i, 2);
      put_u16(buf, u);
    }
  }
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return set_error(TBIK_IO, std::string("cannot open for writing: ") + path);
  const size_t written = std::fwrite(buf.data(), 1, buf.size(), f);
  std::fclose(f);
  if (written != buf.size()) return set_error(TBIK_IO, std::string("short write: ") + path);
  return TBIK_OK;
}

tbik_status tbik_matrix_read_header(const char* path, int* dtype, int64_t* rows, int64_t* cols) {
  if (!path || !dtype || !rows || !cols) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  std::vector<unsigned char> buf;
  return load(path, &buf, dtype, rows, cols);
}

tbik_status tbik_matrix_read(const char* path, void* out, int64_t capacity_bytes) {
  if (!path || !out) return set_error(TBIK_BAD_ARGUMENT, "null argument");
  std::vector<unsigned char> buf;
  int dt = 0;
  int64_t r = 0, c = 0;
  TBIK_TRY(load(path, &buf, &dt, &r, &c));
  const size_t esz = dt == TBIK_F32 ? 4 : 2;
  const size_t elems = static_cast<size_t>(r) * static_cast<size_t>(c);
  if (capacity_bytes < 0 || static_cast<size_t>(capacity_bytes) < elems * esz)
    return set_error(TBIK_BAD_ARGUMENT, "output buffer smaller than the payload");
  unsigned char* dst = static_cast<unsigned char*>(out);
  const unsigned char* p = buf.data() + 24;
  for (size_t i = 0; i < elems; ++i) {
    if (esz == 4) {
      uint32_t u = 0;
      for (int b = 3; b >= 0; --b) u = (u << 8) | p[4 * i + b];
      std::memcpy(dst + 4 * i, &u, 4);
    } else {
      const uint16_t u = get_u16(p + 2 * i);
      std::memcpy(dst + 2 * i, &u, 2);
    }
  }
  return TBIK_OK;
}

}  // extern "C"
