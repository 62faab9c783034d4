// Host-side ingestion (dataset.py:68-118 of the reference): binary PGM ("P5")
// decode straight into float32 planes, in parallel, into a caller buffer
// (normally pinned host memory that train_network uploads chunk by chunk).
// Same parsing rules as load_pgm: '#' comments up to end of line inside the
// header, whitespace-separated width / height / maxval, one whitespace byte
// before the payload, 8-bit samples or big-endian 16-bit when maxval > 255,
// values / maxval. Errors map to DDCCA_ESHAPE (I/O, parse) with the message in
// ddcca_last_error().
#include <algorithm>
#include <atomic>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace ddcca {

struct PgmHeader {
  int width = 0, height = 0, maxval = 0;
  size_t payload = 0;  // byte offset of the samples
};

static bool read_file(const char* path, std::vector<unsigned char>* buf, std::string* err) {
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    *err = std::string("cannot read ") + path;
    return false;
  }
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  buf->resize(n > 0 ? (size_t)n : 0);
  const size_t got = n > 0 ? std::fread(buf->data(), 1, (size_t)n, f) : 0;
  std::fclose(f);
  if ((long)got != n) {
    *err = std::string("cannot read ") + path;
    return false;
  }
  return true;
}

static bool parse_header(const std::vector<unsigned char>& raw, const char* path, PgmHeader* h, std::string* err) {
  size_t pos = 0;
  auto token = [&](std::string* out) -> bool {
    while (pos < raw.size()) {
      const unsigned char c = raw[pos];
      if (c == '#') {
        while (pos < raw.size() && raw[pos] != '\n' && raw[pos] != '\r') ++pos;
      } else if (std::isspace(c)) {
        ++pos;
      } else {
        break;
      }
    }
    const size_t start = pos;
    while (pos < raw.size() && !std::isspace(raw[pos])) ++pos;
    if (start == pos) {
      *err = std::string(path) + ": truncated PGM header";
      return false;
    }
    out->assign(reinterpret_cast<const char*>(raw.data()) + start, pos - start);
    return true;
  };
  std::string magic, w, hh, mv;
  if (!token(&magic)) return false;
  if (magic != "P5") {
    *err = std::string(path) + ": not a binary PGM (only P5 supported)";
    return false;
  }
  if (!token(&w) || !token(&hh) || !token(&mv)) return false;
  auto to_int = [&](const std::string& s, int* v) -> bool {
    if (s.empty() || s.size() > 9) return false;
    int x = 0;
    for (char c : s) {
      if (c < '0' || c > '9') return false;
      x = x * 10 + (c - '0');
    }
    *v = x;
    return true;
  };
  if (!to_int(w, &h->width) || !to_int(hh, &h->height) || !to_int(mv, &h->maxval)) {
    *err = std::string(path) + ": malformed PGM header";
    return false;
  }
  if (h->width < 1 || h->height < 1) {
    *err = std::string(path) + ": invalid PGM dimensions";
    return false;
  }
  if (h->maxval < 1 || h->maxval > 65535) {
    *err = std::string(path) + ": PGM maxval out of range";
    return false;
  }
  h->payload = pos + 1;  // single whitespace byte separates header from payload
  return true;
}

static bool decode(const std::vector<unsigned char>& raw, const PgmHeader& h, const char* path, float* out,
                   std::string* err) {
  const int item = h.maxval > 255 ? 2 : 1;
  const size_t n = (size_t)h.width * h.height;
  if (h.payload > raw.size() || raw.size() - h.payload < n * item) {
    *err = std::string(path) + ": truncated PGM payload";
    return false;
  }
  const unsigned char* p = raw.data() + h.payload;
  const double inv = (double)h.maxval;
  if (item == 1) {
    for (size_t i = 0; i < n; ++i) out[i] = (float)((double)p[i] / inv);
  } else {
    for (size_t i = 0; i < n; ++i) out[i] = (float)((double)((p[2 * i] << 8) | p[2 * i + 1]) / inv);
  }
  return true;
}

}  // namespace ddcca

using namespace ddcca;

extern "C" {

int ddcca_pgm_info(const char* path, int* width, int* height, int* maxval, int64_t* payload_offset) {
  std::vector<unsigned char> raw;
  std::string err;
  PgmHeader h;
  if (!read_file(path, &raw, &err) || !parse_header(raw, path, &h, &err)) return fail(DDCCA_ESHAPE, "%s", err.c_str());
  *width = h.width;
  *height = h.height;
  *maxval = h.maxval;
  if (payload_offset) *payload_offset = (int64_t)h.payload;
  return DDCCA_OK;
}

int ddcca_pgm_load_many(const char* const* paths, int64_t n, int height, int width, float* out, int threads) {
  if (n < 0 || height < 1 || width < 1) return fail(DDCCA_ESHAPE, "pgm: bad request");
  if (n == 0) return DDCCA_OK;
  const int nt = std::max(1, std::min<int>(threads, (int)std::min<int64_t>(n, 256)));
  std::atomic<int64_t> next(0);
  std::atomic<int64_t> bad(-1);
  std::vector<std::string> errs(nt);
  auto work = [&](int tid) {
    std::vector<unsigned char> raw;
    for (;;) {
      const int64_t i = next.fetch_add(1);
      if (i >= n || bad.load() >= 0) return;
      PgmHeader h;
      std::string err;
      bool ok = read_file(paths[i], &raw, &err) && parse_header(raw, paths[i], &h, &err);
      if (ok && (h.height != height || h.width != width)) {
        err = std::string(paths[i]) + ": sample size differs from the corpus";
        ok = false;
      }
      ok = ok && decode(raw, h, paths[i], out + i * (int64_t)height * width, &err);
      if (!ok) {
        int64_t expect = -1;
        if (bad.compare_exchange_strong(expect, i)) errs[tid] = err;
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  if (bad.load() >= 0) {
    for (const auto& e : errs)
      if (!e.empty()) return fail(DDCCA_ESHAPE, "%s", e.c_str());
    return fail(DDCCA_ESHAPE, "pgm: load failed");
  }
  return DDCCA_OK;
}

}  // extern "C"

// ----------------------------------------------------------------------------
// Feature CSV writer (run_extract, pipeline.py:143-166): one line per sample,
// "index,v0,v1,..." with every value formatted by the caller as Python's
// format(v, ".17g"). The values are IQ features of block counts, so the caller
// passes the formatted string of each LUT entry (count 0 .. bpc) once and the
// writer only copies strings: rows are formatted by `threads` workers in blocks
// and written in order. Counts: kind 0 u8, 1 saturating u8 (255 = the block
// remainder), 2 u16; bins per block = `bins`, `bpc` pixels per block.
// ----------------------------------------------------------------------------
namespace ddcca {

static inline unsigned count_at(const void* counts, int kind, int64_t row, int64_t col, int64_t cols, int bins,
                                int bpc) {
  if (kind == 2) return static_cast<const uint16_t*>(counts)[row * cols + col];
  const uint8_t* r = static_cast<const uint8_t*>(counts) + row * cols;
  unsigned c = r[col];
  if (kind == 1 && c == 255) {
    const int64_t b0 = col / bins * bins;
    unsigned s = 0;
    for (int k = 0; k < bins; ++k) s += r[b0 + k];
    c = 255 + (unsigned)(bpc - (int)s);
  }
  return c;
}

}  // namespace ddcca

extern "C" int ddcca_write_feature_csv(const void* counts, int count_kind, int64_t rows, int64_t cols, int bins,
                                       int bpc, const char* const* lut_str, const int* lut_len, int64_t first_index,
                                       const char* path, int threads) {
  if (rows < 0 || cols < 1 || bins < 1 || bpc < 1 || count_kind < 0 || count_kind > 2)
    return fail(DDCCA_ESHAPE, "feature csv: bad shape");
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(DDCCA_ESHAPE, "cannot write %s", path);
  const int nt = std::max(1, std::min(threads, 64));
  const int64_t block = 16;  // rows per work item
  const int64_t nblocks = (rows + block - 1) / block;
  std::vector<std::string> out(nt);
  bool ok = true;
  for (int64_t b0 = 0; b0 < nblocks && ok; b0 += nt) {
    std::vector<std::thread> pool;
    auto fmt = [&](int t) {
      const int64_t b = b0 + t;
      std::string& s = out[t];
      s.clear();
      if (b >= nblocks) return;
      for (int64_t r = b * block; r < std::min(rows, (b + 1) * block); ++r) {
        s += std::to_string(first_index + r);
        for (int64_t c = 0; c < cols; ++c) {
          const unsigned k = count_at(counts, count_kind, r, c, cols, bins, bpc);
          s += ',';
          if (k <= (unsigned)bpc) s.append(lut_str[k], (size_t)lut_len[k]);
          else s += "nan";
        }
        s += '\n';
      }
    };
    for (int t = 1; t < nt; ++t) pool.emplace_back(fmt, t);
    fmt(0);
    for (auto& th : pool) th.join();
    for (int t = 0; t < nt && ok; ++t)
      if (!out[t].empty() && std::fwrite(out[t].data(), 1, out[t].size(), f) != out[t].size()) ok = false;
  }
  if (std::fclose(f) != 0) ok = false;
  if (!ok) return fail(DDCCA_ESHAPE, "cannot write %s", path);
  return DDCCA_OK;
}
