// C++ tests of the drop-in API (include/ecc/*.hpp) against the oracle's C
// restatement, written like the reference's own unit tests
// (proj/tests/test_streaming.cpp, test_kernel.cpp, acceptance.cpp).
//
//   test_api cpu   -- host-only cases (planning, validation, types)
//   test_api gpu   -- GPU cases through libecc_b200.so (bit-exact parity)
//
// Built by tests/test_native_cpu.py / paper_2203_09087_b200/build.py.
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "ecc.hpp"

extern "C" {
// oracle/ecc_oracle.c (test infrastructure)
int ecc_oracle_vcec_u8(const uint8_t*, uint64_t, uint64_t, uint64_t, int64_t*, int64_t*);
int ecc_oracle_vcec_u16(const uint16_t*, uint64_t, uint64_t, uint64_t, int64_t*, int64_t*);
int64_t ecc_oracle_vcec_f32(const float*, uint64_t, uint64_t, uint64_t, float*, int64_t*);
void ecc_oracle_fill_u8(uint8_t*, uint64_t, uint64_t, uint64_t);
int ecc_oracle_changes_u16_as_f32(const uint16_t*, uint64_t, uint64_t, uint64_t, int8_t*);
int ecc_oracle_changes_u8(const uint8_t*, uint64_t, uint64_t, uint64_t, int8_t*);
void ecc_oracle_uniform_noise(float*, uint64_t, uint64_t);
int ecc_oracle_gaussian_smooth(const float*, float*, uint64_t, uint64_t, uint64_t, double, int);
}

using namespace ecc;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                   \
  do {                                                                             \
    ++g_checks;                                                                    \
    if (!(c)) {                                                                    \
      ++g_fail;                                                                    \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);           \
    }                                                                              \
  } while (0)
#define CHECK_THROWS_WITH(expr, needle)                                            \
  do {                                                                             \
    ++g_checks;                                                                    \
    bool thrown_ = false;                                                          \
    try {                                                                          \
      (void)(expr);                                                                \
    } catch (const ecc::error& e_) {                                               \
      thrown_ = std::string(e_.what()).find(needle) != std::string::npos;          \
      if (!thrown_) std::printf("  message was: %s\n", e_.what());                  \
    }                                                                              \
    if (!thrown_) {                                                                \
      ++g_fail;                                                                    \
      std::printf("  CHECK_THROWS failed %s:%d: %s\n", __FILE__, __LINE__, #expr); \
    }                                                                              \
  } while (0)

struct Case {
  const char* name;
  bool gpu;
  std::function<void()> fn;
};
static std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, bool g, std::function<void()> f) { registry().push_back({n, g, f}); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CPU(name) static Reg CAT(reg_, __LINE__)(name, false, []()
#define TEST_GPU(name) static Reg CAT(reg_, __LINE__)(name, true, []()
#define END_TEST );

template <class T>
static Image<T> image_2d(std::vector<std::vector<T>> rows) {
  Image<T> img;
  img.dims = {rows.size(), rows[0].size(), 1};
  for (auto& r : rows) img.values.insert(img.values.end(), r.begin(), r.end());
  return img;
}

template <class T>
static GlobalVcec<T> run_engine(const Image<T>& img, std::uint64_t chunks = 1) {
  return process_image(img, plan_chunks<T>(img.dims, ChunkTarget::count(chunks)));
}

template <class T>
static GlobalVcec<T> oracle_vcec(const Image<T>& img) {
  GlobalVcec<T> out;
  const Dims& d = img.dims;
  if constexpr (std::is_same_v<T, float>) {
    std::vector<float> v(img.values.size());
    std::vector<int64_t> c(img.values.size());
    const int64_t m = ecc_oracle_vcec_f32(img.values.data(), d.w0, d.w1, d.w2, v.data(), c.data());
    v.resize(m);
    c.resize(m);
    out.values = v;
    out.changes = c;
  } else {
    const int nb = std::is_same_v<T, uint8_t> ? 256 : 65536;
    std::vector<int64_t> h(nb), n(nb);
    if constexpr (std::is_same_v<T, uint8_t>)
      ecc_oracle_vcec_u8(img.values.data(), d.w0, d.w1, d.w2, h.data(), n.data());
    else
      ecc_oracle_vcec_u16(img.values.data(), d.w0, d.w1, d.w2, h.data(), n.data());
    for (int b = 0; b < nb; ++b)
      if (n[b]) {
        out.values.push_back(static_cast<T>(b));
        out.changes.push_back(h[b]);
      }
  }
  return out;
}

template <class T>
static bool same(const GlobalVcec<T>& a, const GlobalVcec<T>& b) {
  if (a.values.size() != b.values.size() || a.changes != b.changes) return false;
  return std::memcmp(a.values.data(), b.values.data(), a.values.size() * sizeof(T)) == 0;
}

// ------------------------------------------------------------------ host only
TEST_CPU("plan_chunks splits with ceiling lengths") {  // test_streaming.cpp:13-19
  const auto plan = plan_chunks<float>({10, 1, 1}, ChunkTarget::count(3));
  CHECK(plan.ranges.size() == 3);
  CHECK((plan.ranges[0] == ChunkRange{0, 4}));
  CHECK((plan.ranges[1] == ChunkRange{4, 8}));
  CHECK((plan.ranges[2] == ChunkRange{8, 10}));
} END_TEST

TEST_CPU("plan invariants hold for many (w0, c) pairs") {  // test_streaming.cpp:27-45
  for (std::uint64_t w0 : {1, 2, 3, 7, 10, 64, 100})
    for (std::uint64_t c : {1, 2, 3, 5, 8, 200}) {
      const auto plan = plan_chunks<float>({w0, 4, 4}, ChunkTarget::count(c));
      const std::uint64_t eff = std::min<std::uint64_t>(c, w0);
      const std::uint64_t max_len = (w0 + eff - 1) / eff;
      std::uint64_t b = 0;
      for (const auto& r : plan.ranges) {
        CHECK(r.begin == b);
        CHECK(r.end > r.begin);
        CHECK(r.len() <= max_len);
        b = r.end;
      }
      CHECK(b == w0);
    }
} END_TEST

TEST_CPU("budget-based planning keeps each padded chunk within budget") {
  const Dims dims{4096, 512, 512};
  const std::uint64_t budget = 64ull << 20;
  const auto plan = plan_chunks<float>(dims, ChunkTarget::memory_budget(budget));
  std::uint64_t max_len = 0;
  for (const auto& r : plan.ranges) max_len = std::max(max_len, r.len());
  CHECK(padded_chunk_bytes<float>(dims, max_len) <= budget);
} END_TEST

TEST_CPU("an infeasible budget names the minimum") {  // test_streaming.cpp:56-66
  const Dims dims{8, 1024, 1024};
  CHECK_THROWS_WITH(plan_chunks<float>(dims, ChunkTarget::memory_budget(1024)),
                    std::to_string(2 * padded_chunk_bytes<float>(dims, 1)));
} END_TEST

TEST_CPU("linear_index names out-of-range coordinates") {
  CHECK_THROWS_WITH(linear_index({3, 0, 0}, Dims{3, 2, 2}), "out of range for dims 3x2x2");
  CHECK(linear_index({1, 1, 1}, Dims{3, 2, 2}) == 7);
} END_TEST

TEST_CPU("vcec_to_ecc prefix-sums and rejects an empty VCEC") {
  GlobalVcec<float> v{{1, 2, 3}, {3, -1, -1}};
  const auto c = vcec_to_ecc(v);
  CHECK((c.chi == std::vector<std::int64_t>{3, 2, 1}));
  CHECK_THROWS_WITH(vcec_to_ecc(GlobalVcec<float>{}), "empty VCEC");
} END_TEST

// ------------------------------------------------------------------ GPU
TEST_GPU("staircase with two chunks gives {1:1, 2:0, 3:0, 4:0}") {  // test_streaming.cpp:84-89
  const auto img = image_2d<float>({{1, 2}, {3, 4}});
  const auto v = run_engine(img, 2);
  CHECK((v.values == std::vector<float>{1, 2, 3, 4}));
  CHECK((v.changes == std::vector<std::int64_t>{1, 0, 0, 0}));
} END_TEST

TEST_GPU("u8 merge keeps values that occur with zero net change") {  // :115-120
  const auto img = image_2d<std::uint8_t>({{0, 0, 0}, {0, 9, 0}, {0, 0, 0}});
  const auto v = run_engine(img, 1);
  CHECK((v.values == std::vector<std::uint8_t>{0, 9}));
  CHECK((v.changes == std::vector<std::int64_t>{0, 1}));
} END_TEST

TEST_GPU("ring curve (acceptance.cpp:182-198)") {
  const auto img = image_2d<float>({{0, 0, 0}, {0, 9, 0}, {0, 0, 0}});
  const auto c = vcec_to_ecc(run_engine(img));
  CHECK((c.thresholds == std::vector<float>{0, 9}));
  CHECK((c.chi == std::vector<std::int64_t>{0, 1}));
} END_TEST

TEST_GPU("random images: every type, every chunking == oracle") {
  std::mt19937 rng(1);
  for (int t = 0; t < 240; ++t) {
    const Dims d = (t % 2) ? Dims{1 + rng() % 7, 1 + rng() % 7, 1 + rng() % 7}
                           : Dims{1 + rng() % 9, 1 + rng() % 9, 1};
    const auto n = d.voxel_count();
    const int kind = t % 3;
    for (std::uint64_t c : {std::uint64_t{1}, std::uint64_t{2}, std::uint64_t{3}, d.w0}) {
      if (kind == 0) {
        Image<std::uint8_t> img{d, {}};
        for (std::uint64_t i = 0; i < n; ++i) img.values.push_back(rng() % 6);
        CHECK(same(run_engine(img, c), oracle_vcec(img)));
      } else if (kind == 1) {
        Image<float> img{d, {}};
        for (std::uint64_t i = 0; i < n; ++i) img.values.push_back(0.25f * (rng() % 5) - 0.5f);
        CHECK(same(run_engine(img, c), oracle_vcec(img)));
      } else {
        Image<std::uint16_t> img{d, {}};
        for (std::uint64_t i = 0; i < n; ++i) img.values.push_back(rng() % 5 * 9000);
        CHECK(same(run_engine(img, c), oracle_vcec(img)));
      }
    }
  }
} END_TEST

TEST_GPU("u8 and f32 paths agree on the same values (test_streaming.cpp:138-153)") {
  std::mt19937 rng(7);
  Image<std::uint8_t> u{{9, 13, 17}, {}};
  Image<float> f{{9, 13, 17}, {}};
  for (std::uint64_t i = 0; i < u.dims.voxel_count(); ++i) {
    u.values.push_back(rng() % 256);
    f.values.push_back(u.values.back());
  }
  const auto a = run_engine(u, 3);
  const auto b = run_engine(f, 2);
  CHECK(a.changes == b.changes);
  CHECK(a.values.size() == b.values.size());
  for (std::size_t i = 0; i < a.values.size(); ++i) CHECK(float(a.values[i]) == b.values[i]);
} END_TEST

TEST_GPU("a failing source names the chunk and the cause (test_streaming.cpp:164-198)") {
  struct Flaky final : ChunkSource<float> {
    Image<float> img;
    Dims dims() const override { return img.dims; }
    void read_rows(std::uint64_t r0, std::uint64_t r1, float* dst) override {
      if (r1 > 5) throw std::runtime_error("simulated device failure");
      std::memcpy(dst, img.values.data() + r0 * 9, (r1 - r0) * 9 * sizeof(float));
    }
  } src;
  src.img.dims = {8, 3, 3};
  src.img.values.assign(72, 1.0f);
  const auto plan = plan_chunks<float>(src.img.dims, ChunkTarget::count(4));
  CHECK_THROWS_WITH(process_image<float>(src, plan), "simulated device failure");
  CHECK_THROWS_WITH(process_image<float>(src, plan), "chunk");
} END_TEST

TEST_GPU("invalid plans are rejected (streaming.hpp:186-195)") {
  Image<float> img{{4, 1, 1}, {1, 2, 3, 4}};
  CHECK_THROWS_WITH(process_image(img, ChunkPlan{}), "empty chunk plan");
  CHECK_THROWS_WITH(process_image(img, ChunkPlan{{{0, 2}, {3, 4}}}), "contiguously");
  CHECK_THROWS_WITH(process_image(img, ChunkPlan{{{0, 2}, {2, 3}}}), "w0 = 4");
} END_TEST

TEST_GPU("C1 synthetic 256x256 u8 (SURVEY.md Appendix B)") {
  Image<std::uint8_t> img{{256, 256, 1}, std::vector<std::uint8_t>(65536)};
  ecc_oracle_fill_u8(img.values.data(), 65536, 1, 0);
  const auto c = device::curve(img.values.data(), img.dims);
  CHECK(c.size() == 256);
  CHECK(c.thresholds[0] == 0 && c.chi[0] == 238);
  CHECK(c.chi.back() == 1);
  CHECK(*std::min_element(c.chi.begin(), c.chi.end()) == -8214);
  CHECK(*std::max_element(c.chi.begin(), c.chi.end()) == 4833);
  CHECK(c == vcec_to_ecc(run_engine(img, 8)));
} END_TEST

TEST_GPU("3D u8 volumes through the fused fast path == oracle") {
  std::mt19937 rng(3);
  for (Dims d : {Dims{40, 35, 48}, Dims{7, 61, 64}, Dims{64, 64, 64}, Dims{2, 1, 16}}) {
    Image<std::uint8_t> img{d, {}};
    for (std::uint64_t i = 0; i < d.voxel_count(); ++i) img.values.push_back(rng() % 256);
    const auto v = device::vcec(img.values.data(), d);
    CHECK(same(v, oracle_vcec(img)));
  }
} END_TEST

TEST_GPU("quantised f32 with the affine bin map (config 4 shape)") {
  std::mt19937 rng(5);
  Image<float> img{{20, 21, 22}, {}};
  for (std::uint64_t i = 0; i < img.dims.voxel_count(); ++i)
    img.values.push_back(float(rng() % 65536) * (1.0f / 65536.0f));
  const BinMap bm = BinMap::affine(65536, 0.0f, 1.0f / 65536.0f);
  CHECK(same(device::vcec(img.values.data(), img.dims, &bm), oracle_vcec(img)));
  EngineOptions opt;
  opt.bins = bm;
  CHECK(same(process_image(img, plan_chunks<float>(img.dims, ChunkTarget::count(3)), opt),
             oracle_vcec(img)));
  img.values[5] = 0.3f;  // off the grid
  CHECK_THROWS_WITH(device::vcec(img.values.data(), img.dims, &bm), "affine bin grid");
} END_TEST

TEST_GPU("batched 2D rows == per-image process_image") {
  std::mt19937 rng(9);
  const std::uint64_t count = 5, h = 33, w = 47;
  std::vector<std::uint16_t> imgs(count * h * w);
  for (auto& x : imgs) x = rng() % 700;
  std::vector<std::int32_t> chi;
  std::vector<std::uint32_t> pres;
  device::batch2d(imgs.data(), count, h, w, chi, pres);
  for (std::uint64_t b = 0; b < count; ++b) {
    Image<std::uint16_t> one{{h, w, 1}, {imgs.begin() + b * h * w, imgs.begin() + (b + 1) * h * w}};
    const auto want = vcec_to_ecc(run_engine(one, 2));
    const auto got = device::batch_row_curve<std::uint16_t>(chi.data() + b * 65536,
                                                            pres.data() + b * 2048, 65536);
    CHECK(got.thresholds == want.thresholds);
    CHECK(got.chi == want.chi);
  }
} END_TEST

TEST_GPU("engine report has one timing per chunk") {
  Image<std::uint8_t> img{{64, 32, 32}, std::vector<std::uint8_t>(64 * 32 * 32)};
  ecc_oracle_fill_u8(img.values.data(), img.values.size(), 1, 0);
  EngineReport rep;
  const auto v = process_image(img, plan_chunks<std::uint8_t>(img.dims, ChunkTarget::count(4)),
                               {}, &rep);
  CHECK(v.total() == 1);
  CHECK(rep.chunks.size() == 4);
  for (const auto& t : rep.chunks) CHECK(t.kernel_end >= t.kernel_begin);
} END_TEST

TEST_GPU("FileSource: raw f32 little / big endian, NaN and size errors (chunk.hpp:154-189)") {
  std::mt19937 rng(21);
  const Dims d{9, 7, 5};
  std::vector<float> v(d.voxel_count());
  for (auto& x : v) x = float(rng() % 7) * 0.5f;
  Image<float> img{d, v};
  const std::string le = "/tmp/ecc_test_le.raw", be = "/tmp/ecc_test_be.raw";
  {
    std::FILE* f = std::fopen(le.c_str(), "wb");
    std::fwrite(v.data(), 4, v.size(), f);
    std::fclose(f);
    f = std::fopen(be.c_str(), "wb");
    for (float x : v) {
      uint32_t u;
      std::memcpy(&u, &x, 4);
      u = __builtin_bswap32(u);
      std::fwrite(&u, 4, 1, f);
    }
    std::fclose(f);
  }
  const auto plan = plan_chunks<float>(d, ChunkTarget::count(3));
  FileSource<float> a(le, d), b(be, d, RawOptions{true});
  CHECK(same(process_image(a, plan), oracle_vcec(img)));
  CHECK(same(process_image(b, plan), oracle_vcec(img)));
  // the constructor checks the file size, as the reference's does (chunk.hpp:157-169)
  CHECK_THROWS_WITH(FileSource<float>(le, Dims{9, 7, 4}), "size mismatch");
  v[(5 * 7 + 1) * 5 + 2] = std::numeric_limits<float>::quiet_NaN();
  {
    std::FILE* f = std::fopen(le.c_str(), "wb");
    std::fwrite(v.data(), 4, v.size(), f);
    std::fclose(f);
  }
  FileSource<float> nan(le, d);
  CHECK_THROWS_WITH(process_image(nan, plan), "NaN value at linear index 182");
  std::remove(le.c_str());
  std::remove(be.c_str());
} END_TEST

TEST_GPU("PaddedChunk API on the device: u16 / u8 chunks, 2D and 3D, faces vs changes") {
  std::mt19937 rng(123);
  for (const Dims d : {Dims{7, 9, 11}, Dims{8, 13, 1}, Dims{5, 4, 33}}) {
    // u16: compute_changes of a middle chunk == the oracle's changes of those rows
    Image<std::uint16_t> im{d, std::vector<std::uint16_t>(d.voxel_count())};
    for (auto& v : im.values) v = (std::uint16_t)(rng() % 5 + (rng() % 3) * 40000);
    std::vector<std::int8_t> want(d.voxel_count());
    ecc_oracle_changes_u16_as_f32(im.values.data(), d.w0, d.w1, d.w2, want.data());
    const std::uint64_t b = 2, e = d.w0 - 1, row = d.w1 * d.w2;
    const auto ch = extract_padded_chunk(im, b, e);
    std::vector<std::int8_t> got(ch.owned_voxels());
    compute_changes(ch, 0, ch.owned_len(), got);
    CHECK(std::equal(got.begin(), got.end(), want.begin() + b * row));
    // every owned voxel: the signed count of the faces introduced() reports
    // (each face's dimension d - nnz) equals voxel_contribution()
    const int dd = d.is_2d() ? 2 : 3;
    for (std::uint64_t i = b; i < e; i += 2)
      for (std::uint64_t j = 0; j < d.w1; j += 3)
        for (std::uint64_t k = 0; k < d.w2; k += 5) {
          int sum = dd == 2 ? 1 : -1;
          for (int a0 = -1; a0 <= 1; ++a0)
            for (int a1 = -1; a1 <= 1; ++a1)
              for (int a2 = (dd == 2 ? 0 : -1); a2 <= (dd == 2 ? 0 : 1); ++a2) {
                if (!a0 && !a1 && !a2) continue;
                if (introduced(ch, {i, j, k}, {a0, a1, a2}))
                  sum += ((dd - (a0 != 0) - (a1 != 0) - (a2 != 0)) % 2 == 0) ? 1 : -1;
              }
          CHECK(sum == voxel_contribution(ch, {i, j, k}));
          CHECK(sum == want[(i * d.w1 + j) * d.w2 + k]);
        }
    // u8: accumulate_dense_u8 over row pieces == the per-value sums of the changes
    Image<std::uint8_t> i8{d, std::vector<std::uint8_t>(d.voxel_count())};
    for (auto& v : i8.values) v = (std::uint8_t)(rng() % 6);
    std::vector<std::int8_t> w8(d.voxel_count());
    ecc_oracle_changes_u8(i8.values.data(), d.w0, d.w1, d.w2, w8.data());
    const auto c8 = extract_padded_chunk(i8, 0, d.w0);
    std::vector<std::int64_t> acc(256, 0), ref(256, 0);
    for (std::uint64_t r = 0; r < d.w0; ++r) accumulate_dense_u8<std::int64_t>(c8, r, r + 1, acc);
    for (std::uint64_t v = 0; v < d.voxel_count(); ++v) ref[i8.values[v]] += w8[v];
    CHECK(acc == ref);
  }
} END_TEST

TEST_GPU("device curve text == write_curve (curve.hpp:87-121), f32 thresholds") {
  std::mt19937 rng(77);
  EccCurve<float> c;
  for (int i = 0; i < 3000; ++i) {
    float v;
    do {
      uint32_t u = rng();
      std::memcpy(&v, &u, 4);
    } while (!std::isfinite(v));
    c.thresholds.push_back(v);
    c.chi.push_back((int64_t)rng() - (int64_t)rng());
  }
  for (auto fmtk : {CurveFormat::csv, CurveFormat::json}) {
    std::ostringstream os;
    write_curve(c, fmtk, os);
    CHECK(device::format_curve(c, fmtk) == os.str());
  }
} END_TEST

TEST_GPU("bench_run pipeline (pipeline.hpp:236-291) == oracle smoothing + ECC") {
  const Dims d{20, 24, 28};
  const auto rep = bench_run(d, 2, 1, 2.0, 13);
  std::vector<float> x(d.voxel_count()), y(d.voxel_count());
  ecc_oracle_uniform_noise(x.data(), x.size(), 1);
  for (int it = 0; it < 2; ++it) {
    CHECK(ecc_oracle_gaussian_smooth(x.data(), y.data(), d.w0, d.w1, d.w2, 2.0, 13) == 0);
    x.swap(y);
  }
  Image<float> img{d, x};
  const auto want = vcec_to_ecc(oracle_vcec(img));
  CHECK(rep.iterations == 2 && rep.voxels == d.voxel_count());
  CHECK(rep.last_points == want.size());
  CHECK(rep.last_chi_first == want.chi.front() && rep.last_chi_last == want.chi.back());
  CHECK(rep.to_string().find("ECC GVox/s:") != std::string::npos);
  CHECK_THROWS_WITH(bench_run(d, 0), "at least one iteration");
  CHECK_THROWS_WITH(bench_run(d, 1, 1, 2.0, 4), "odd and >= 1");
} END_TEST

// `test_api csv <file>`: file = u64 n, n float32 thresholds, n int64 chi;
// writes the curve CSV (tests/test_native.py compares it with the
// reference's own writer).
static int csv_mode(const char* path) {
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return 2;
  std::uint64_t n = 0;
  if (std::fread(&n, 8, 1, f) != 1) return 2;
  EccCurve<float> c;
  c.thresholds.resize(n);
  c.chi.resize(n);
  if (std::fread(c.thresholds.data(), 4, n, f) != n || std::fread(c.chi.data(), 8, n, f) != n) return 2;
  std::fclose(f);
  std::ostringstream os;
  write_curve(c, CurveFormat::csv, os);
  std::fwrite(os.str().data(), 1, os.str().size(), stdout);
  return 0;
}

TEST_CPU("curve writers: CSV / JSON / VCEC layouts and round trip") {
  EccCurve<float> c{{0.0f, 1.5258789e-05f, 0.5f, 1e10f}, {3, -2, 0, 1}};
  std::ostringstream csv, json, vc;
  write_curve(c, CurveFormat::csv, csv);
  write_curve(c, CurveFormat::json, json);
  CHECK(csv.str() == "threshold,euler_characteristic\n0,3\n1.5258789e-05,-2\n0.5,0\n1e+10,1\n");
  CHECK(json.str() == "[{\"t\":0,\"chi\":3},{\"t\":1.5258789e-05,\"chi\":-2},{\"t\":0.5,\"chi\":0},"
                      "{\"t\":1e+10,\"chi\":1}]\n");
  std::istringstream in(csv.str());
  CHECK(read_curve_csv<float>(in) == c);
  write_vcec(GlobalVcec<std::uint8_t>{{0, 9}, {0, 1}}, vc);
  CHECK(vc.str() == "value,change\n0,0\n9,1\n");
  std::istringstream bad("threshold,chi\n");
  CHECK_THROWS_WITH(read_curve_csv<float>(bad), "bad curve CSV header");
} END_TEST

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  if (mode == "csv" && argc > 2) return csv_mode(argv[2]);
  int ran = 0;
  for (auto& c : registry()) {
    if (c.gpu != (mode == "gpu")) continue;
    const int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  exception: %s\n", e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", c.name);
    ++ran;
  }
  std::printf("%d cases, %d checks, %d failures\n", ran, g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
