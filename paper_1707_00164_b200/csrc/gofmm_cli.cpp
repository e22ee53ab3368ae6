// gofmm_b200_cli — the reference command-line driver's compress / bench subcommands
// (proj/tools/gfmm_cli.cpp:113-212) over the B200 C-ABI (include/gofmm_b200.h): compress on the
// host + GPU (gofmm_compress), evaluation, error_eps2 and the dense comparison product on the GPU.
//
// Same flags, same key=value report in the same order (golden-tested by the reference at
// tests/test_cli.cpp:61-80), same CSV for bench, same exit codes (2 invalid argument, 3 I/O,
// 4 numeric). Values print through std::ostream's default 6-significant-digit format, as the
// reference's do. Sources: --gen gaussian | laplace | poly | exponential (a generated Gaussian
// cloud, PointCloud::random_gaussian, or --points FILE in the GPTS format, io.hpp:85-110).
// Stored-matrix sources (--matrix, randspd, invsqlap, cosine) are not part of the GPU build
// (their blocks cannot be regenerated on the device) and exit 2 with a message.
// Extensions: --entries host|device (host = the reference compress bit for bit; device = ANN and
// sampled blocks on the GPU, the default), --device N.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/gofmm_b200.h"

namespace {

struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check(int rc, const char* what, const char* (*msg)() = gofmm_last_error) {
  if (rc != GOFMM_OK) throw Failure(rc, std::string(what) + ": " + msg());
}

struct Flags {
  std::string sub;
  // SourceFlags (gfmm_cli.cpp:16-29)
  std::string gen, matrix_path, points_path;
  int n = 4096, d = 6;
  double bandwidth = 1.0, delta = -1.0, shift = 1.0, ridge = 1e-8, lambda = 1.0;
  int degree = 2;
  uint64_t seed = 0;
  // RunConfig (compress.hpp:12-22) + the CLI's own
  gofmm_compress_config cfg{};
  int r = 1;
  std::string dist = "kernel", mode = "tasks", entries = "device";
  bool f32 = false;
  std::string n_list = "2048,4096", r_list = "64";
};

int to_int(const std::string& k, const std::string& v) {
  try {
    size_t pos = 0;
    long long x = std::stoll(v, &pos);
    if (pos != v.size()) throw std::invalid_argument(v);
    return int(x);
  } catch (const std::exception&) {
    throw Failure(GOFMM_ERR_INVALID, "bad integer for " + k + ": " + v);
  }
}

double to_double(const std::string& k, const std::string& v) {
  try {
    size_t pos = 0;
    double x = std::stod(v, &pos);
    if (pos != v.size()) throw std::invalid_argument(v);
    return x;
  } catch (const std::exception&) {
    throw Failure(GOFMM_ERR_INVALID, "bad number for " + k + ": " + v);
  }
}

uint64_t to_u64(const std::string& k, const std::string& v) {
  try {
    size_t pos = 0;
    if (!v.empty() && v[0] == '-') throw std::invalid_argument(v);
    const unsigned long long x = std::stoull(v, &pos);
    if (pos != v.size()) throw std::invalid_argument(v);
    return uint64_t(x);
  } catch (const std::exception&) {
    throw Failure(GOFMM_ERR_INVALID, "bad seed for " + k + ": " + v);
  }
}

std::vector<int> int_list(const std::string& s) {  // parse_int_list (gfmm_cli.cpp:98-105)
  std::vector<int> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ',')) out.push_back(to_int("list", item));
  if (out.empty()) throw Failure(GOFMM_ERR_INVALID, "empty list: " + s);
  return out;
}

Flags parse(int argc, char** argv) {
  Flags f;
  gofmm_compress_default_config(&f.cfg);
  f.cfg.threads = 1;  // RunConfig::threads default (compress.hpp:22)
  if (argc < 2) throw Failure(GOFMM_ERR_INVALID, "a subcommand is required: compress | bench");
  f.sub = argv[1];
  if (f.sub != "compress" && f.sub != "bench") {
    if (f.sub == "gen" || f.sub == "ann")
      throw Failure(GOFMM_ERR_INVALID, "subcommand '" + f.sub + "' is not part of the GPU build (compress, bench)");
    throw Failure(GOFMM_ERR_INVALID, "unknown subcommand: " + f.sub);
  }
  const bool is_compress = f.sub == "compress";
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k == "--f32" && is_compress) {
      f.f32 = true;
      continue;
    }
    if (i + 1 >= argc) throw Failure(GOFMM_ERR_INVALID, "missing value for " + k);
    std::string v = argv[++i];
    if (k == "--gen") f.gen = v;
    else if (k == "--matrix") f.matrix_path = v;
    else if (k == "--points") f.points_path = v;
    else if (k == "--n") f.n = to_int(k, v);
    else if (k == "--d") f.d = to_int(k, v);
    else if (k == "--h") f.bandwidth = to_double(k, v);
    else if (k == "--delta") f.delta = to_double(k, v);
    else if (k == "--shift") f.shift = to_double(k, v);
    else if (k == "--degree") f.degree = to_int(k, v);
    else if (k == "--ridge") f.ridge = to_double(k, v);
    else if (k == "--lambda") f.lambda = to_double(k, v);
    else if (k == "--seed") f.seed = to_u64(k, v);
    else if (k == "--m") f.cfg.m = to_int(k, v);
    else if (k == "--s") f.cfg.s = to_int(k, v);
    else if (k == "--tau") f.cfg.tau = to_double(k, v);
    else if (k == "--k") f.cfg.kappa = to_int(k, v);
    else if (k == "--budget") f.cfg.budget = to_double(k, v);
    else if (k == "--dist") f.dist = v;
    else if (k == "--threads") f.cfg.threads = to_int(k, v);
    else if (k == "--iters") f.cfg.ann_iterations = to_int(k, v);
    else if (k == "--entries") f.entries = v;
    else if (k == "--device") f.cfg.device = to_int(k, v);
    else if (k == "--r" && is_compress) f.r = to_int(k, v);
    else if (k == "--mode" && is_compress) f.mode = v;
    else if (k == "--n-list" && !is_compress) f.n_list = v;
    else if (k == "--r-list" && !is_compress) f.r_list = v;
    else throw Failure(GOFMM_ERR_INVALID, "unknown option: " + k);
  }
  f.cfg.seed = f.seed;  // gfmm_cli.cpp:271
  if (f.dist == "geom") f.cfg.distance = GOFMM_DIST_GEOMETRIC;
  else if (f.dist == "kernel") f.cfg.distance = GOFMM_DIST_KERNEL;
  else if (f.dist == "angle") f.cfg.distance = GOFMM_DIST_ANGLE;
  else throw Failure(GOFMM_ERR_INVALID, "unknown distance kind: " + f.dist);
  if (f.mode != "levels" && f.mode != "tasks") throw Failure(GOFMM_ERR_INVALID, "unknown traversal mode: " + f.mode);
  if (f.entries == "host") f.cfg.entries = GOFMM_ENTRIES_HOST;
  else if (f.entries == "device") f.cfg.entries = GOFMM_ENTRIES_DEVICE;
  else throw Failure(GOFMM_ERR_INVALID, "--entries must be host or device");
  // RunConfig::validate's r check (compress.hpp:29); the rest is gofmm_compress's
  if (f.r < 1) throw Failure(GOFMM_ERR_INVALID, "r must be >= 1");
  return f;
}

// read_points_file (io.hpp:97-110): "GPTS" | u32 version 1 | u64 n | u64 d | n*d f64 point-major
std::vector<double> read_points(const std::string& path, int& n, int& d) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Failure(GOFMM_ERR_IO, "cannot open " + path);
  auto rd = [&](void* p, size_t b, const char* what) {
    in.read(static_cast<char*>(p), std::streamsize(b));
    if (!in) throw Failure(GOFMM_ERR_IO, std::string("truncated ") + what + " in " + path);
  };
  char magic[4];
  rd(magic, 4, "magic");
  if (std::memcmp(magic, "GPTS", 4) != 0) throw Failure(GOFMM_ERR_IO, "bad magic in " + path + " (expected GPTS)");
  uint32_t version = 0;
  rd(&version, 4, "version");
  if (version != 1) throw Failure(GOFMM_ERR_IO, "unsupported format version in " + path);
  uint64_t nn = 0, dd = 0;
  rd(&nn, 8, "n");
  rd(&dd, 8, "d");
  if (nn == 0 || dd == 0 || nn > 100000000ULL / dd) throw Failure(GOFMM_ERR_IO, "point count out of range in " + path);
  std::vector<double> x(nn * dd);
  rd(x.data(), sizeof(double) * x.size(), "coordinates");
  for (double v : x)
    if (!std::isfinite(v)) throw Failure(GOFMM_ERR_IO, "non-finite coordinates in " + path);
  n = int(nn);
  d = int(dd);
  return x;
}

// make_source (gfmm_cli.cpp:55-92) for the kernel generators the device regenerates
struct Source {
  int kernel = -1, n = 0, d = 0;
  double kparam[4] = {0, 0, 0, 0};
  std::vector<double> coords;  // d x n
};

Source make_source(const Flags& f) {
  if (!f.matrix_path.empty()) {
    // file_oracle -> read_matrix_file (io.hpp:65-78): unreadable or malformed files are I/O errors
    // (exit 3) as in the reference; a well-formed dense matrix is a stored source (exit 2)
    std::ifstream in(f.matrix_path, std::ios::binary);
    if (!in) throw Failure(GOFMM_ERR_IO, "cannot open " + f.matrix_path);
    char magic[4] = {0, 0, 0, 0};
    uint32_t version = 0;
    in.read(magic, 4);
    in.read(reinterpret_cast<char*>(&version), 4);
    if (!in || std::memcmp(magic, "GFMM", 4) != 0 || version != 1)
      throw Failure(GOFMM_ERR_IO, "bad magic or version in " + f.matrix_path + " (expected GFMM v1)");
    throw Failure(GOFMM_ERR_INVALID, "--matrix (stored dense source) is not part of the GPU build");
  }
  if (f.gen.empty()) throw Failure(GOFMM_ERR_INVALID, "either --gen or --matrix is required");
  if (f.gen == "randspd" || f.gen == "invsqlap" || f.gen == "cosine")
    throw Failure(GOFMM_ERR_INVALID, "generator '" + f.gen + "' (stored blocks) is not part of the GPU build");
  Source s;
  if (f.gen == "gaussian") s.kernel = GOFMM_KERNEL_GAUSSIAN;
  else if (f.gen == "laplace") s.kernel = GOFMM_KERNEL_LAPLACE;
  else if (f.gen == "poly") s.kernel = GOFMM_KERNEL_POLYNOMIAL;
  else if (f.gen == "exponential") s.kernel = GOFMM_KERNEL_EXPONENTIAL;
  else throw Failure(GOFMM_ERR_INVALID, "unknown generator: " + f.gen);
  if (f.points_path.empty()) {
    if (f.n < 1 || f.d < 1) throw Failure(GOFMM_ERR_INVALID, "--n and --d must be >= 1");
    s.n = f.n;
    s.d = f.d;
    s.coords.resize(size_t(s.n) * s.d);
    check(gofmm_points_gaussian(s.n, s.d, f.seed, s.coords.data()), "points");
  } else {
    s.coords = read_points(f.points_path, s.n, s.d);
  }
  switch (s.kernel) {
    case GOFMM_KERNEL_GAUSSIAN:
    case GOFMM_KERNEL_EXPONENTIAL:
      s.kparam[0] = f.bandwidth;
      break;
    case GOFMM_KERNEL_LAPLACE:
      if (f.delta >= 0) s.kparam[0] = f.delta;
      else check(gofmm_default_laplace_floor(s.d, s.n, s.coords.data(), f.seed, &s.kparam[0]), "laplace floor");
      break;
    case GOFMM_KERNEL_POLYNOMIAL:
      if (f.degree < 1) throw Failure(GOFMM_ERR_INVALID, "polynomial degree must be >= 1");
      s.kparam[0] = f.shift;
      s.kparam[1] = double(f.degree);
      break;
  }
  return s;
}

struct Compressed {
  gofmm_compressed* c = nullptr;
  ~Compressed() {
    if (c) gofmm_compressed_free(c);
  }
};

struct Handle {
  gofmm_handle* h = nullptr;
  ~Handle() {
    if (h) gofmm_destroy(h);
  }
};

void compress(const Flags& f, const Source& s, Compressed& out, gofmm_compress_stats& st) {
  check(gofmm_compress(s.kernel, s.kparam, s.d, s.n, s.coords.data(), &f.cfg, &out.c), "compress",
        gofmm_compress_last_error);
  check(gofmm_compressed_stats(out.c, &st), "compress stats", gofmm_compress_last_error);
}

void create(const Flags& f, const Compressed& c, Handle& h) {
  gofmm_tree_desc desc;
  check(gofmm_compressed_desc(c.c, &desc), "compressed desc", gofmm_compress_last_error);
  gofmm_options opts{};  // matrix-free blocks, FP64
  opts.device = f.cfg.device;
  check(gofmm_create(&desc, &opts, &h.h), "create");
}

double report_value(double v, bool f32) { return f32 ? double(float(v)) : v; }  // gfmm_cli.cpp:107-111

// cmd_compress (gfmm_cli.cpp:113-137)
int cmd_compress(const Flags& f) {
  const Source s = make_source(f);
  Compressed c;
  gofmm_compress_stats st{};
  compress(f, s, c, st);
  for (int i = 0; i < st.ann_iterations_done; ++i)
    std::cout << "ann_recall_iter_" << (i + 1) << "=" << st.ann_recall[i] << "\n";
  std::cout << "tree_seconds=" << st.tree_seconds << "\n";
  // print_compress_stats (compress.hpp:437-444)
  std::cout << "entries_evaluated=" << st.entries_evaluated << '\n'
            << "compress_flops=" << st.compress_flops << '\n'
            << "compress_seconds=" << st.compress_seconds << '\n'
            << "near_field_entries=" << st.near_field_entries << '\n'
            << "max_skeleton=" << st.max_skeleton << '\n'
            << "mean_skeleton=" << st.mean_skeleton << '\n';
  Handle h;
  create(f, c, h);
  gofmm_eps2_report rep{};
  check(gofmm_error_eps2(h.h, f.r, std::min(100, s.n), f.seed, &rep, nullptr), "error_eps2");
  // print_eval_stats (evaluate.hpp:375-384)
  std::cout << "eval_flops=" << rep.eval_flops << '\n'
            << "eval_seconds=" << rep.eval_seconds << '\n'
            << "eps2=" << report_value(rep.eps2, f.f32) << '\n';
  std::cout << "eps2_first10=";
  for (int i = 0; i < rep.num_per_entry; ++i) std::cout << (i ? "," : "") << report_value(rep.per_entry[i], f.f32);
  std::cout << '\n';
  std::cout << "eps2_mean100=" << report_value(rep.mean_sample, f.f32) << '\n';
  return 0;
}

// cmd_bench (gfmm_cli.cpp:173-212): dense K W vs compress + evaluate. The dense product runs on
// the GPU too — all N exact rows of K W generated matrix-free (gofmm_exact_rows) — so the speedup
// column compares the two device paths, not the GPU against the CPU.
int cmd_bench(const Flags& f0) {
  const std::vector<int> ns = int_list(f0.n_list), rs = int_list(f0.r_list);
  std::cout << "N,r,dense_seconds,compress_seconds,eval_seconds,speedup\n";
  for (int n : ns) {
    if (n > 16384) throw Failure(GOFMM_ERR_IO, "bench N exceeds desk-scale cap");  // kDeskScaleCap
    Flags f = f0;
    f.n = n;
    const Source s = make_source(f);
    Compressed c;
    gofmm_compress_stats st{};
    compress(f, s, c, st);
    Handle h;
    create(f, c, h);
    std::vector<int32_t> all(n);
    for (int i = 0; i < n; ++i) all[i] = i;
    for (int r : rs) {
      if (r < 1) throw Failure(GOFMM_ERR_INVALID, "r must be >= 1");
      // Rng(cfg.seed, 0xbe7c), gauss, column-major (gfmm_cli.cpp:195-198)
      std::vector<double> w(size_t(n) * r), u(size_t(n) * r);
      check(gofmm_rng_gauss_stream(f.seed, 0xbe7c, n, r, w.data(), n), "rhs");
      double* d_w = nullptr;
      double* d_k = nullptr;
      if (cudaMalloc(&d_w, w.size() * 8) != cudaSuccess || cudaMalloc(&d_k, w.size() * 8) != cudaSuccess)
        throw Failure(GOFMM_ERR_CUDA, "device allocation failed");
      cudaMemcpy(d_w, w.data(), w.size() * 8, cudaMemcpyHostToDevice);
      cudaDeviceSynchronize();
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, nullptr);
      int rc = gofmm_exact_rows(h.h, all.data(), n, d_w, n, r, d_k, n, nullptr);
      cudaEventRecord(e1, nullptr);
      cudaDeviceSynchronize();
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      cudaFree(d_w);
      cudaFree(d_k);
      check(rc, "dense product");
      const double dense_s = ms * 1e-3;
      gofmm_eval_stats es{};
      check(gofmm_evaluate(h.h, w.data(), n, r, u.data(), n, &es), "evaluate");
      std::printf("%d,%d,%.6f,%.6f,%.6f,%.3f\n", n, r, dense_s, st.compress_seconds, es.seconds,
                  dense_s / es.seconds);
      std::fflush(stdout);
    }
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    Flags f = parse(argc, argv);
    return f.sub == "compress" ? cmd_compress(f) : cmd_bench(f);
  } catch (const Failure& e) {
    std::cerr << "error: " << e.what() << "\n";
    // gfmm_cli.cpp:289-305: invalid_argument 2, io_error 3, numeric_error 4, anything else 3
    if (e.code == GOFMM_ERR_INVALID) return 2;
    if (e.code == GOFMM_ERR_NUMERIC) return 4;
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  }
}
