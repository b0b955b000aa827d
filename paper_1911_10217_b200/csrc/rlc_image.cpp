// rlc_image.cpp -- image I/O and error metrics of the reference's image
// module (proj/include/rlcuts/image.hpp:65-78, proj/src/image.cpp:43-136)
// behind the C-ABI: PFM (float32 RGB, little-endian, bottom row first), the
// gamma-2.2 PPM preview, mse and relative_mse.  Host code: these are file
// formats and whole-image reductions in the reference's sequential order,
// so results (bytes written, doubles returned) are identical to it.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <string>
#include <vector>

#include "rlc_build.h"
#include "rlcuts_b200.h"

namespace rlc {

ImageIoError::ImageIoError(int code, const std::string& msg)
    : std::runtime_error(msg), code_(code) {}

namespace {

void require_image(const double* px, int32_t w, int32_t h, const char* what) {
  if (px == nullptr || w <= 0 || h <= 0) throw InvalidArgument(std::string(what) + ": bad image");
}

// Host little-endian float32 bytes of one value (the format's byte order).
void put_f32le(std::vector<char>& out, size_t at, float v) {
  uint32_t bits;
  std::memcpy(&bits, &v, 4);
  for (int k = 0; k < 4; ++k) out[at + size_t(k)] = char((bits >> (8 * k)) & 0xffu);
}

float get_f32(const char* p, bool little) {
  uint32_t bits = 0;
  for (int k = 0; k < 4; ++k) {
    const uint32_t b = uint8_t(p[little ? k : 3 - k]);
    bits |= b << (8 * k);
  }
  float v;
  std::memcpy(&v, &bits, 4);
  return v;
}

// image.cpp:27-31: clamp to [0, 1], gamma 1/2.2, lround(x * 255)
uint8_t srgb_byte(double c) {
  const double clamped = std::clamp(c, 0.0, 1.0);
  return uint8_t(std::lround(std::pow(clamped, 1.0 / 2.2) * 255.0));
}

}  // namespace

// write_pfm, image.cpp:43-60
void write_pfm(const double* px, int32_t w, int32_t h, const std::string& path) {
  require_image(px, w, h, "write_pfm");
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ImageIoError(RLC_ERR_IO, "cannot open for writing: " + path);
  out << "PF\n" << w << " " << h << "\n-1.0\n";
  std::vector<char> row(size_t(w) * 12);
  for (int32_t y = h - 1; y >= 0; --y) {
    const double* r = px + size_t(y) * size_t(w) * 3;
    for (size_t i = 0; i < size_t(w) * 3; ++i) put_f32le(row, 4 * i, float(r[i]));
    out.write(row.data(), std::streamsize(row.size()));
  }
  if (!out) throw ImageIoError(RLC_ERR_IO, "write failed: " + path);
}

// read_pfm, image.cpp:62-94.  px == nullptr (or too small) only reports the
// size.
void read_pfm(const std::string& path, double* px, uint64_t cap_pixels, int32_t* w_out,
              int32_t* h_out) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ImageIoError(RLC_ERR_IO, "cannot open for reading: " + path);
  std::string magic;
  int w = 0, h = 0;
  double scale = 0;
  in >> magic >> w >> h >> scale;
  if (!in || magic != "PF") throw ImageIoError(RLC_ERR_PARSE, "not a color PFM file: " + path);
  if (w <= 0 || h <= 0 || scale == 0) throw ImageIoError(RLC_ERR_PARSE, "bad PFM header: " + path);
  in.get();  // the single whitespace byte after the scale
  *w_out = w;
  *h_out = h;
  const uint64_t npix = uint64_t(w) * uint64_t(h);
  if (px == nullptr || cap_pixels < npix) return;
  const bool little = scale < 0;
  const double mag = std::fabs(scale);
  std::vector<char> row(size_t(w) * 12);
  for (int y = h - 1; y >= 0; --y) {
    in.read(row.data(), std::streamsize(row.size()));
    if (!in) throw ImageIoError(RLC_ERR_PARSE, "truncated PFM data: " + path);
    double* r = px + size_t(y) * size_t(w) * 3;
    for (size_t i = 0; i < size_t(w) * 3; ++i) r[i] = double(get_f32(row.data() + 4 * i, little));
  }
  if (mag != 1.0)
    for (uint64_t i = 0; i < 3 * npix; ++i) px[i] = px[i] * mag;
}

// write_ppm, image.cpp:96-112
void write_ppm(const double* px, int32_t w, int32_t h, const std::string& path) {
  require_image(px, w, h, "write_ppm");
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ImageIoError(RLC_ERR_IO, "cannot open for writing: " + path);
  out << "P6\n" << w << " " << h << "\n255\n";
  std::vector<char> row(size_t(w) * 3);
  for (int32_t y = 0; y < h; ++y) {
    const double* r = px + size_t(y) * size_t(w) * 3;
    for (size_t i = 0; i < size_t(w) * 3; ++i) row[i] = char(srgb_byte(r[i]));
    out.write(row.data(), std::streamsize(row.size()));
  }
  if (!out) throw ImageIoError(RLC_ERR_IO, "write failed: " + path);
}

// The sequential sum of mse (image.cpp:114-124) over per-pixel terms
// e_i = dx*dx + dy*dy + dz*dz, in pixel order.
double sum_terms(const double* e, uint64_t n) {
  double total = 0;
  for (uint64_t i = 0; i < n; ++i) total += e[i];
  return total;
}

double mse(const double* a, const double* b, uint64_t npix) {
  double total = 0;
  for (uint64_t i = 0; i < npix; ++i) {
    const double dx = a[3 * i] - b[3 * i], dy = a[3 * i + 1] - b[3 * i + 1],
                 dz = a[3 * i + 2] - b[3 * i + 2];
    total += dx * dx + dy * dy + dz * dz;
  }
  return total / (3.0 * double(npix));
}

// relative_mse, image.cpp:126-136
double relative_mse(const double* a, const double* b, uint64_t npix) {
  const double err = mse(a, b, npix);
  double ref = 0;
  for (uint64_t i = 0; i < npix; ++i)
    ref += b[3 * i] * b[3 * i] + b[3 * i + 1] * b[3 * i + 1] + b[3 * i + 2] * b[3 * i + 2];
  ref /= 3.0 * double(npix);
  if (ref == 0) return err == 0 ? 0 : std::numeric_limits<double>::infinity();
  return err / ref;
}

}  // namespace rlc
