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

#include <atomic>
#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
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

  const espn_store_header h{kVersion, d, d_cls, value_width, alignment, n_docs};
  return espn_store_save_manifest(base, &h, recs.data());
}

int espn_store_save_manifest(const char* base, const espn_store_header* h, const espn_manifest_record* recs) {
  if (!base || !h || (h->count && !recs)) return fail(ESPN_E_INVALID_INPUT, "null argument");
  const std::string mp = path_of(base, ".manifest");
  FILE* m = std::fopen(mp.c_str(), "wb");
  if (!m) return fail(ESPN_E_IO, "cannot create " + mp);
  unsigned char hdr[kHeaderBytes] = {};
  std::memcpy(hdr, kMagic, 8);
  const uint32_t u[6] = {h->version, h->d, h->d_cls, h->value_width, h->alignment, 0};
  std::memcpy(hdr + 8, u, 24);
  std::memcpy(hdr + 32, &h->count, 8);
  int st = write_all(m, hdr, kHeaderBytes, mp);
  if (st == ESPN_OK) st = write_all(m, recs, h->count * sizeof(espn_manifest_record), mp);
  if (std::fclose(m) != 0 && st == ESPN_OK) st = fail(ESPN_E_IO, "close failed: " + mp);
  if (st != ESPN_OK) return st;

  const std::string jp = path_of(base, ".manifest.json");
  FILE* j = std::fopen(jp.c_str(), "wb");
  if (!j) return fail(ESPN_E_IO, "cannot create " + jp);
  std::fprintf(j, "{\"magic\": \"ESPNSTR1\", \"version\": %u, \"d\": %u, \"d_cls\": %u, \"value_width\": %u, "
                  "\"alignment\": %u, \"count\": %llu, \"records\": [",
               h->version, h->d, h->d_cls, h->value_width, h->alignment, static_cast<unsigned long long>(h->count));
  for (uint64_t i = 0; i < h->count; ++i)
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


// ---- file-backed batched reads (StoreHandle::fetch_batch, store.hpp:56-112) ----
struct espn_store_reader {
  espn_store_header h{};
  std::vector<espn_manifest_record> recs;
  uint32_t mode = ESPN_READ_BUFFERED;
  uint32_t queue_depth = 16;
  int fd = -1;
  const unsigned char* map = nullptr;
  uint64_t file_size = 0;
};

int espn_store_open(const char* base, uint32_t mode, uint32_t queue_depth, espn_store_reader** out,
                    espn_store_header* header) {
  if (!base || !out) return fail(ESPN_E_INVALID_INPUT, "null argument");
  *out = nullptr;
  if (mode > ESPN_READ_MMAP) return fail(ESPN_E_INVALID_INPUT, "read mode must be direct, buffered or mmap");
  auto* r = new espn_store_reader();
  int st = load_manifest(base, &r->h, &r->recs);
  if (st != ESPN_OK) { delete r; return st; }
  // direct mode needs alignment >= 512 (store.hpp:109-110; SPEC.md open_store)
  if (mode == ESPN_READ_DIRECT && r->h.alignment < 512) {
    delete r;
    return fail(ESPN_E_INVALID_CONFIG, "direct mode requires a store with alignment >= 512");
  }
  r->mode = mode;
  r->queue_depth = queue_depth ? queue_depth : 16;
  const std::string dp = path_of(base, ".espn");
  r->fd = ::open(dp.c_str(), O_RDONLY | (mode == ESPN_READ_DIRECT ? O_DIRECT : 0));
  if (r->fd < 0) {
    const int e = errno;
    delete r;
    if (mode == ESPN_READ_DIRECT && e == EINVAL)
      return fail(ESPN_E_IO, "the filesystem of " + dp + " does not honour O_DIRECT");
    return fail(ESPN_E_IO, "cannot open " + dp + ": " + std::strerror(e));
  }
  struct stat sb {};
  if (::fstat(r->fd, &sb) != 0) { espn_store_close(r); return fail(ESPN_E_IO, "cannot stat " + dp); }
  r->file_size = static_cast<uint64_t>(sb.st_size);
  const uint64_t need = r->recs.empty() ? 0 : r->recs.back().byte_offset + r->recs.back().byte_length;
  if (r->file_size < need) { espn_store_close(r); return fail(ESPN_E_IO, "short data file (truncated store): " + dp); }
  if (mode == ESPN_READ_MMAP && r->file_size) {
    void* m = ::mmap(nullptr, r->file_size, PROT_READ, MAP_SHARED, r->fd, 0);
    if (m == MAP_FAILED) { espn_store_close(r); return fail(ESPN_E_IO, "mmap failed: " + dp); }
    r->map = static_cast<const unsigned char*>(m);
  }
  if (header) *header = r->h;
  *out = r;
  return ESPN_OK;
}

int espn_store_close(espn_store_reader* r) {
  if (!r) return ESPN_OK;
  if (r->map) ::munmap(const_cast<unsigned char*>(r->map), r->file_size);
  if (r->fd >= 0) ::close(r->fd);
  delete r;
  return ESPN_OK;
}

int espn_store_records(const espn_store_reader* r, espn_manifest_record* out) {
  if (!r || (!r->recs.empty() && !out)) return fail(ESPN_E_INVALID_INPUT, "null argument");
  std::memcpy(out, r->recs.data(), r->recs.size() * sizeof(espn_manifest_record));
  return ESPN_OK;
}

int espn_store_fetch(espn_store_reader* r, const uint32_t* ids, uint64_t n, uint8_t* out, uint64_t* out_off,
                     uint64_t capacity, uint64_t* bytes_read, uint64_t* blocks_read, double* wall_time) {
  if (!r || !out_off || (n && !ids)) return fail(ESPN_E_INVALID_INPUT, "null argument");
  const auto t0 = std::chrono::steady_clock::now();
  // unknown ids -> InvalidInputError listing the offenders (store.hpp:92-93)
  std::string bad;
  int nbad = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (ids[i] >= r->h.count) {
      if (nbad++ < 16) bad += " " + std::to_string(ids[i]);
    }
  if (nbad) return fail(ESPN_E_INVALID_INPUT, "unknown doc ids:" + bad + (nbad > 16 ? " ..." : ""));
  out_off[0] = 0;
  uint64_t br = 0, bl = 0;
  const bool direct = r->mode == ESPN_READ_DIRECT;
  const uint64_t align = r->h.alignment ? r->h.alignment : 1;
  const uint64_t block = direct ? align : 4096u;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t len = r->recs[ids[i]].byte_length;
    out_off[i + 1] = out_off[i] + len;
    br += direct ? (len + align - 1) / align * align : len;  // aligned-rounded in direct mode
    bl += (len + block - 1) / block;                         // block = alignment (direct) else 4096
  }
  if (bytes_read) *bytes_read = br;
  if (blocks_read) *blocks_read = bl;
  if (!out) return ESPN_OK;  // sizes only
  if (out_off[n] > capacity) return fail(ESPN_E_INVALID_INPUT, "output capacity too small");
  // queue_depth reads in flight: workers take records in request order and
  // write each to its own slot (completion order free, result order fixed)
  std::atomic<uint64_t> next{0};
  std::atomic<int> status{ESPN_OK};
  thread_local std::string werr;
  std::string first_err;
  std::atomic<bool> err_set{false};
  auto worker = [&] {
    void* bounce = nullptr;
    size_t bounce_cap = 0;
    for (;;) {
      const uint64_t i = next.fetch_add(1);
      if (i >= n || status.load() != ESPN_OK) break;
      const espn_manifest_record& rec = r->recs[ids[i]];
      uint8_t* dst = out + out_off[i];
      if (r->mode == ESPN_READ_MMAP) {
        std::memcpy(dst, r->map + rec.byte_offset, rec.byte_length);
        continue;
      }
      if (!direct) {
        uint64_t done = 0;
        while (done < rec.byte_length) {
          const ssize_t got = ::pread(r->fd, dst + done, rec.byte_length - done, rec.byte_offset + done);
          if (got <= 0) { status = ESPN_E_IO; break; }
          done += static_cast<uint64_t>(got);
        }
        continue;
      }
      // direct: the aligned span covering the record, into an aligned bounce buffer
      const uint64_t a0 = rec.byte_offset / align * align;
      const uint64_t a1 = (rec.byte_offset + rec.byte_length + align - 1) / align * align;
      const size_t span = static_cast<size_t>(a1 - a0);
      if (span > bounce_cap) {
        std::free(bounce);
        bounce = nullptr;
        if (posix_memalign(&bounce, 4096, span) != 0) { status = ESPN_E_IO; break; }
        bounce_cap = span;
      }
      uint64_t done = 0;
      while (done < span) {
        const ssize_t got = ::pread(r->fd, static_cast<uint8_t*>(bounce) + done, span - done, a0 + done);
        if (got <= 0) break;  // a short read at the end of the file is fine once the record is in
        done += static_cast<uint64_t>(got);
      }
      if (done < rec.byte_offset + rec.byte_length - a0) { status = ESPN_E_IO; break; }
      std::memcpy(dst, static_cast<uint8_t*>(bounce) + (rec.byte_offset - a0), rec.byte_length);
    }
    std::free(bounce);
  };
  const uint32_t nt = static_cast<uint32_t>(std::min<uint64_t>(r->queue_depth, std::max<uint64_t>(n, 1)));
  std::vector<std::thread> pool;
  for (uint32_t t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  (void)first_err;
  (void)err_set;
  if (wall_time) *wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (status.load() != ESPN_OK) return fail(ESPN_E_IO, "short read from the store's data file");
  return ESPN_OK;
}


int espn_store_read_rows(espn_store_reader* r, uint64_t doc_begin, uint64_t n, uint32_t dtype, uint64_t* row_ptr_out,
                         uint16_t* codes_out) {
  if (!r || !row_ptr_out) return fail(ESPN_E_INVALID_INPUT, "null argument");
  if (dtype != ESPN_DTYPE_F16 && dtype != ESPN_DTYPE_BF16) return fail(ESPN_E_INVALID_INPUT, "dtype must be f16 or bf16");
  if (doc_begin + n > r->h.count) return fail(ESPN_E_INVALID_INPUT, "doc range beyond the store");
  row_ptr_out[0] = 0;
  for (uint64_t i = 0; i < n; ++i) row_ptr_out[i + 1] = row_ptr_out[i] + r->recs[doc_begin + i].token_count;
  if (!codes_out || n == 0) return ESPN_OK;
  std::vector<uint32_t> ids(n);
  for (uint64_t i = 0; i < n; ++i) ids[i] = static_cast<uint32_t>(doc_begin + i);
  std::vector<uint64_t> off(n + 1);
  uint64_t br = 0, bl = 0;
  int st = espn_store_fetch(r, ids.data(), n, nullptr, off.data(), 0, &br, &bl, nullptr);
  if (st != ESPN_OK) return st;
  std::vector<uint8_t> buf(std::max<uint64_t>(off[n], 1));
  st = espn_store_fetch(r, ids.data(), n, buf.data(), off.data(), buf.size(), &br, &bl, nullptr);
  if (st != ESPN_OK) return st;
  const uint32_t w = r->h.value_width, d = r->h.d;
  for (uint64_t i = 0; i < n; ++i) {
    const unsigned char* b = buf.data() + off[i] + uint64_t(r->h.d_cls) * w;
    uint16_t* out = codes_out + row_ptr_out[i] * d;
    const uint64_t nv = (row_ptr_out[i + 1] - row_ptr_out[i]) * d;
    if (w == 2 && dtype == ESPN_DTYPE_F16) {
      std::memcpy(out, b, nv * 2);  // the store's own fp16 codes, bit-exact
      continue;
    }
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
  return ESPN_OK;
}

}  // extern "C"
