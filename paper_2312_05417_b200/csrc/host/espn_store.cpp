// espn_store.cpp -- the on-disk embedding store (include/espn_store.h):
// build_store / load_manifest (proj/include/espn/store.hpp:37-54,
// SPEC.md:195-251) and a bulk reader that turns a store into the CSR code
// table espn_gpu_table_open takes.  Pure host C++ (no CUDA): the file format
// is the input side of the re-rank path, not part of the device hot loop.
#include "espn_store.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

constexpr char kMagic[8] = {'E', 'S', 'P', 'N', 'S', 'T', 'R', '1'};
constexpr uint32_t kVersion = 1;
constexpr size_t kHeaderBytes = 40;

uint16_t f32_to_f16(float x) {  // IEEE binary16, round to nearest even (subnormals included)
  const _Float16 h = static_cast<_Float16>(x);
  uint16_t c;
  std::memcpy(&c, &h, 2);
  return c;
}
float f16_to_f32(uint16_t c) {
  _Float16 h;
  std::memcpy(&h, &c, 2);
  return static_cast<float>(h);
}
uint16_t f32_to_bf16(float x) {  // round to nearest even; NaN stays NaN
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return static_cast<uint16_t>((u >> 16) | 0x40u);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

struct File {  // RAII fd
  int fd = -1;
  ~File() {
    if (fd >= 0) ::close(fd);
  }
};

std::string path_of(const char* base, const char* ext) { return std::string(base) + ext; }

int write_all(FILE* f, const void* p, size_t n, const std::string& what) {
  if (n && std::fwrite(p, 1, n, f) != n) return fail(ESPN_E_IO, "write failed: " + what);
  return ESPN_OK;
}

// Reads and validates <base>.manifest.
int load_manifest(const char* base, espn_store_header* h, std::vector<espn_manifest_record>* recs) {
  if (!base || !h) return fail(ESPN_E_INVALID_INPUT, "null argument");
  const std::string mp = path_of(base, ".manifest");
  FILE* f = std::fopen(mp.c_str(), "rb");
  if (!f) return fail(ESPN_E_IO, "cannot open " + mp);
  unsigned char hdr[kHeaderBytes];
  const size_t got = std::fread(hdr, 1, kHeaderBytes, f);
  if (got != kHeaderBytes) {
    std::fclose(f);
    return fail(ESPN_E_FORMAT, "manifest shorter than its header: " + mp);
  }
  if (std::memcmp(hdr, kMagic, 8) != 0) {
    std::fclose(f);
    return fail(ESPN_E_FORMAT, "bad manifest magic (expected ESPNSTR1): " + mp);
  }
  uint32_t u[6];
  std::memcpy(u, hdr + 8, 24);
  uint64_t count;
  std::memcpy(&count, hdr + 32, 8);
  h->version = u[0];
  h->d = u[1];
  h->d_cls = u[2];
  h->value_width = u[3];
  h->alignment = u[4];
  h->count = count;
  if (h->version != kVersion || h->d == 0 || (h->value_width != 2 && h->value_width != 4) ||
      (h->alignment != 1 && h->alignment != 512 && h->alignment != 4096)) {
    std::fclose(f);
    return fail(ESPN_E_FORMAT, "unsupported manifest header (version / d / value_width / alignment): " + mp);
  }
  if (recs) {
    // the untrusted count must match the file size before anything is sized by it
    if (std::fseek(f, 0, SEEK_END) != 0) {
      std::fclose(f);
      return fail(ESPN_E_IO, "cannot seek " + mp);
    }
    const long fsz = std::ftell(f);
    if (fsz < 0 || (uint64_t)fsz < kHeaderBytes || count != ((uint64_t)fsz - kHeaderBytes) / sizeof(espn_manifest_record) ||
        ((uint64_t)fsz - kHeaderBytes) % sizeof(espn_manifest_record) != 0) {
      std::fclose(f);
      return fail(ESPN_E_FORMAT, "manifest record count does not match its file size: " + mp);
    }
    std::fseek(f, (long)kHeaderBytes, SEEK_SET);
    try {
      recs->resize(count);
    } catch (const std::exception&) {
      std::fclose(f);
      return fail(ESPN_E_FORMAT, "manifest record count too large: " + mp);
    }
    if (count && std::fread(recs->data(), sizeof(espn_manifest_record), count, f) != count) {
      std::fclose(f);
      return fail(ESPN_E_FORMAT, "manifest truncated: " + mp);
    }
    uint64_t end = 0;
    for (uint64_t i = 0; i < count; ++i) {
      const espn_manifest_record& r = (*recs)[i];
      const uint64_t want = (uint64_t(h->d_cls) + uint64_t(r.token_count) * h->d) * h->value_width;
      if (r.token_count == 0 || r.byte_length != want || (r.byte_offset % h->alignment) != 0 || r.byte_offset < end) {
        std::fclose(f);
        return fail(ESPN_E_FORMAT, "manifest record " + std::to_string(i) +
                                       " inconsistent (token_count >= 1, byte_length == record_bytes, aligned,"
                                       " non-overlapping)");
      }
      end = r.byte_offset + r.byte_length;
    }
  }
  std::fclose(f);
  return ESPN_OK;
}

}  // namespace

extern "C" {

const char* espn_store_last_error(void) { return g_err.c_str(); }

int espn_store_build(const char* base, uint64_t n_docs, uint32_t d, uint32_t d_cls, uint32_t value_width,
                     uint32_t alignment, const uint64_t* row_ptr, const float* rows, const float* cls) {
  if (!base || (n_docs && (!row_ptr || !rows))) return fail(ESPN_E_INVALID_INPUT, "null argument");
  if (d == 0) return fail(ESPN_E_INVALID_INPUT, "d must be positive");
  if (value_width != 2 && value_width != 4) return fail(ESPN_E_INVALID_CONFIG, "value_width must be 2 or 4");
  if (alignment != 1 && alignment != 512 && alignment != 4096)
    return fail(ESPN_E_INVALID_CONFIG, "alignment must be 1, 512 or 4096");
  if (n_docs && row_ptr[0] != 0) return fail(ESPN_E_INVALID_INPUT, "row_ptr[0] must be 0");
  // validate before touching the file system (types.hpp:64-68: t >= 1, finite values)
  for (uint64_t i = 0; i < n_docs; ++i) {
    if (row_ptr[i + 1] <= row_ptr[i]) return fail(ESPN_E_INVALID_INPUT, "doc " + std::to_string(i) + " has no tokens");
    const uint64_t t = row_ptr[i + 1] - row_ptr[i];
    if (t > 0xFFFFFFFFull / d) return fail(ESPN_E_INVALID_INPUT, "doc too long for a u32 record");
  }
  const uint64_t nv = n_docs ? row_ptr[n_docs] * d : 0;
  for (uint64_t i = 0; i < nv; ++i)
    if (!std::isfinite(rows[i])) return fail(ESPN_E_INVALID_INPUT, "non-finite BOW value");
  if (cls)
    for (uint64_t i = 0; i < n_docs * d_cls; ++i)
      if (!std::isfinite(cls[i])) return fail(ESPN_E_INVALID_INPUT, "non-finite CLS value");

  const std::string dp = path_of(base, ".espn");
  FILE* f = std::fopen(dp.c_str(), "wb");
  if (!f) return fail(ESPN_E_IO, "cannot create " + dp);
  std::vector<char> fbuf(1 << 22);
  std::setvbuf(f, fbuf.data(), _IOFBF, fbuf.size());
  std::vector<espn_manifest_record> recs(n_docs);
  std::vector<unsigned char> rec;
  std::vector<unsigned char> zeros(alignment, 0);
  uint64_t cursor = 0;
  int st = ESPN_OK;
  for (uint64_t i = 0; i < n_docs && st == ESPN_OK; ++i) {
    const uint64_t t = row_ptr[i + 1] - row_ptr[i];
    const uint64_t off = (cursor + alignment - 1) / alignment * alignment;
    st = write_all(f, zeros.data(), off - cursor, dp);  // pad to the record start
    const uint64_t nval = d_cls + t * d;
    rec.resize(nval * value_width);
    for (uint64_t j = 0; j < nval; ++j) {
      const float x = j < d_cls ? (cls ? cls[i * d_cls + j] : 0.0f) : rows[row_ptr[i] * d + (j - d_cls)];
      if (value_width == 2) {
        const uint16_t c = f32_to_f16(x);
        std::memcpy(&rec[j * 2], &c, 2);
      } else {
        std::memcpy(&rec[j * 4], &x, 4);
      }
    }
    if (st == ESPN_OK) st = write_all(f, rec.data(), rec.size(), dp);
    recs[i] = espn_manifest_record{off, static_cast<uint32_t>(rec.size()), static_cast<uint32_t>(t)};
    cursor = off + rec.size();
  }
  // the last record also fills whole blocks, so block-granular (direct) reads stay in-file
  if (st == ESPN_OK) st = write_all(f, zeros.data(), (cursor + alignment - 1) / alignment * alignment - cursor, dp);
  if (std::fclose(f) != 0 && st == ESPN_OK) st = fail(ESPN_E_IO, "close failed: " + dp);
  if (st != ESPN_OK) return st;

  const std::string mp = path_of(base, ".manifest");
  FILE* m = std::fopen(mp.c_str(), "wb");
  if (!m) return fail(ESPN_E_IO, "cannot create " + mp);
  unsigned char hdr[kHeaderBytes] = {};
  std::memcpy(hdr, kMagic, 8);
  const uint32_t u[6] = {kVersion, d, d_cls, value_width, alignment, 0};
  std::memcpy(hdr + 8, u, 24);
  std::memcpy(hdr + 32, &n_docs, 8);
  st = write_all(m, hdr, kHeaderBytes, mp);
  if (st == ESPN_OK) st = write_all(m, recs.data(), recs.size() * sizeof(espn_manifest_record), mp);
  if (std::fclose(m) != 0 && st == ESPN_OK) st = fail(ESPN_E_IO, "close failed: " + mp);
  if (st != ESPN_OK) return st;

  const std::string jp = path_of(base, ".manifest.json");
  FILE* j = std::fopen(jp.c_str(), "wb");
  if (!j) return fail(ESPN_E_IO, "cannot create " + jp);
  std::fprintf(j, "{\"magic\": \"ESPNSTR1\", \"version\": %u, \"d\": %u, \"d_cls\": %u, \"value_width\": %u, "
                  "\"alignment\": %u, \"count\": %llu, \"records\": [",
               kVersion, d, d_cls, value_width, alignment, static_cast<unsigned long long>(n_docs));
  for (uint64_t i = 0; i < n_docs; ++i)
    std::fprintf(j, "%s[%llu, %u, %u]", i ? ", " : "", static_cast<unsigned long long>(recs[i].byte_offset),
                 recs[i].byte_length, recs[i].token_count);
  std::fprintf(j, "]}\n");
  if (std::fclose(j) != 0) return fail(ESPN_E_IO, "close failed: " + jp);
  return ESPN_OK;
}

int espn_store_load_manifest(const char* base, espn_store_header* header, espn_manifest_record* records) {
  std::vector<espn_manifest_record> recs;
  const int st = load_manifest(base, header, records ? &recs : nullptr);
  if (st != ESPN_OK) return st;
  if (records && !recs.empty()) std::memcpy(records, recs.data(), recs.size() * sizeof(espn_manifest_record));
  return ESPN_OK;
}

int espn_store_read_table(const char* base, uint32_t dtype, uint64_t* row_ptr_out, uint16_t* codes_out,
                          float* cls_out) {
  if (dtype != ESPN_DTYPE_F16 && dtype != ESPN_DTYPE_BF16) return fail(ESPN_E_INVALID_INPUT, "dtype must be f16 or bf16");
  espn_store_header h{};
  std::vector<espn_manifest_record> recs;
  int st = load_manifest(base, &h, &recs);
  if (st != ESPN_OK) return st;
  if (!row_ptr_out || (h.count && !codes_out)) return fail(ESPN_E_INVALID_INPUT, "null output");
  const std::string dp = path_of(base, ".espn");
  File fd;
  fd.fd = ::open(dp.c_str(), O_RDONLY);
  if (fd.fd < 0) return fail(ESPN_E_IO, "cannot open " + dp);
  struct stat sb {};
  if (::fstat(fd.fd, &sb) != 0) return fail(ESPN_E_IO, "cannot stat " + dp);
  const uint64_t size = static_cast<uint64_t>(sb.st_size);
  const uint64_t need = recs.empty() ? 0 : recs.back().byte_offset + recs.back().byte_length;
  if (size < need) return fail(ESPN_E_IO, "short data file (truncated store): " + dp);
  const unsigned char* data = nullptr;
  if (size) {
    void* m = ::mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd.fd, 0);
    if (m == MAP_FAILED) return fail(ESPN_E_IO, "mmap failed: " + dp);
    ::madvise(m, size, MADV_SEQUENTIAL);
    data = static_cast<const unsigned char*>(m);
  }
  row_ptr_out[0] = 0;
  const uint32_t w = h.value_width;
  for (uint64_t i = 0; i < h.count; ++i) {
    const espn_manifest_record& r = recs[i];
    const uint64_t t = r.token_count;
    row_ptr_out[i + 1] = row_ptr_out[i] + t;
    const unsigned char* p = data + r.byte_offset;
    if (cls_out) {
      for (uint32_t j = 0; j < h.d_cls; ++j) {
        if (w == 2) {
          uint16_t c;
          std::memcpy(&c, p + 2 * j, 2);
          cls_out[i * h.d_cls + j] = f16_to_f32(c);
        } else {
          std::memcpy(&cls_out[i * h.d_cls + j], p + 4 * j, 4);
        }
      }
    }
    const unsigned char* b = p + uint64_t(h.d_cls) * w;
    uint16_t* out = codes_out + row_ptr_out[i] * h.d;
    const uint64_t nv = t * h.d;
    if (w == 2 && dtype == ESPN_DTYPE_F16) {
      std::memcpy(out, b, nv * 2);  // bit-exact: the store's own fp16 codes
    } else {
      for (uint64_t j = 0; j < nv; ++j) {
        float x;
        if (w == 2) {
          uint16_t c;
          std::memcpy(&c, b + 2 * j, 2);
          x = f16_to_f32(c);
        } else {
          std::memcpy(&x, b + 4 * j, 4);
        }
        out[j] = dtype == ESPN_DTYPE_F16 ? f32_to_f16(x) : f32_to_bf16(x);
      }
    }
  }
  if (data) ::munmap(const_cast<unsigned char*>(data), size);
  (void)st;
  return ESPN_OK;
}

}  // extern "C"
