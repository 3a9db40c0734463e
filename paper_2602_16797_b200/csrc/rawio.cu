// Raw binary interchange for A.
//
// The reference moves dense matrices as Matrix Market text (io.cpp:174-184,
// write_matrix_market_array: 17 significant digits per entry), ~24 GB at
// C2; parsing it dominates set-up.  This format is the same data as raw
// little-endian fp64, row-major (the device layout), behind a 32-byte header:
//
//   bytes 0-7   magic "MSVDRAW1"
//   bytes 8-15  int64 rows m
//   bytes 16-23 int64 cols n
//   bytes 24-27 int32 layout (0 = row-major)
//   bytes 28-31 int32 reserved (0)
//   then m * n doubles, row r at offset 32 + 8 r n
//
// Exact round trips like the reference's writers (io.hpp:27-31), and a
// row range [row0, row0 + rows) is one contiguous byte range, so a rank of a
// row-sharded run reads only its own rows.  msvd_raw_load_device streams
// them straight to HBM through pinned staging buffers on the context's copy
// stream (two buffers: the disk read of chunk i+1 overlaps the H2D of i).
// Failures are IoError (errors.hpp:21-24) with the reference's message style.
#include <cstdio>
#include <cstring>
#include <string>

#include "msvd_internal.h"

namespace msvd {
namespace {

constexpr char kMagic[8] = {'M', 'S', 'V', 'D', 'R', 'A', 'W', '1'};
constexpr int64_t kHeader = 32;

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

void read_header(FILE* f, const std::string& path, int64_t* m, int64_t* n) {
    unsigned char h[kHeader];
    if (std::fread(h, 1, kHeader, f) != static_cast<size_t>(kHeader))
        fail(MSVD_ERR_IO, path + ": truncated raw header");
    if (std::memcmp(h, kMagic, 8) != 0) fail(MSVD_ERR_IO, path + ": not an MSVDRAW1 file");
    int32_t layout = 0;
    std::memcpy(m, h + 8, 8);
    std::memcpy(n, h + 16, 8);
    std::memcpy(&layout, h + 24, 4);
    if (layout != 0) fail(MSVD_ERR_IO, path + ": unsupported raw layout " + std::to_string(layout));
    if (*m < 0 || *n < 0) fail(MSVD_ERR_IO, path + ": negative dimension in raw header");
    if (std::fseek(f, 0, SEEK_END) != 0) fail(MSVD_ERR_IO, path + ": cannot seek");
    const long long size = std::ftell(f);
    if (size < kHeader + 8LL * (*m) * (*n)) fail(MSVD_ERR_IO, path + ": truncated raw data");
}

FILE* open_read(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) fail(MSVD_ERR_IO, path + ": cannot open for reading");
    return f;
}

void seek_row(FILE* f, const std::string& path, int64_t row, int64_t n) {
    if (std::fseek(f, static_cast<long>(kHeader + 8 * row * n), SEEK_SET) != 0) fail(MSVD_ERR_IO, path + ": cannot seek");
}

}  // namespace

void raw_write(const char* path, const double* hA, int64_t m, int64_t n, int64_t ld) {
    const std::string p = path;
    if (m < 0 || n < 0) fail(MSVD_ERR_DIMENSION, "DenseMatrix: negative dimension");
    if (ld < n) fail(MSVD_ERR_DIMENSION, "msvd: leading dimension below column count");
    File fh;
    fh.f = std::fopen(path, "wb");
    if (!fh.f) fail(MSVD_ERR_IO, p + ": cannot open for writing");
    unsigned char h[kHeader] = {};
    std::memcpy(h, kMagic, 8);
    std::memcpy(h + 8, &m, 8);
    std::memcpy(h + 16, &n, 8);
    bool ok = std::fwrite(h, 1, kHeader, fh.f) == static_cast<size_t>(kHeader);
    if (ld == n) {
        ok = ok && std::fwrite(hA, sizeof(double), static_cast<size_t>(m * n), fh.f) == static_cast<size_t>(m * n);
    } else {
        for (int64_t r = 0; r < m && ok; ++r)
            ok = std::fwrite(hA + r * ld, sizeof(double), static_cast<size_t>(n), fh.f) == static_cast<size_t>(n);
    }
    ok = ok && std::fflush(fh.f) == 0;
    if (!ok) fail(MSVD_ERR_IO, p + ": write failed");
}

void raw_info(const char* path, int64_t* m, int64_t* n) {
    File fh;
    fh.f = open_read(path);
    read_header(fh.f, path, m, n);
}

void raw_read_rows(const char* path, int64_t row0, int64_t rows, double* hA, int64_t ld) {
    const std::string p = path;
    File fh;
    fh.f = open_read(p);
    int64_t m = 0, n = 0;
    read_header(fh.f, p, &m, &n);
    if (row0 < 0 || rows < 0 || row0 + rows > m) fail(MSVD_ERR_DIMENSION, "msvd: raw row range outside the matrix");
    if (ld < n) fail(MSVD_ERR_DIMENSION, "msvd: leading dimension below column count");
    seek_row(fh.f, p, row0, n);
    if (ld == n) {
        if (std::fread(hA, sizeof(double), static_cast<size_t>(rows * n), fh.f) != static_cast<size_t>(rows * n))
            fail(MSVD_ERR_IO, p + ": read failed");
        return;
    }
    for (int64_t r = 0; r < rows; ++r)
        if (std::fread(hA + r * ld, sizeof(double), static_cast<size_t>(n), fh.f) != static_cast<size_t>(n))
            fail(MSVD_ERR_IO, p + ": read failed");
}

void raw_load_device(Ctx& c, const char* path, int64_t row0, int64_t rows, double* dA, int64_t ld) {
    const std::string p = path;
    File fh;
    fh.f = open_read(p);
    int64_t m = 0, n = 0;
    read_header(fh.f, p, &m, &n);
    if (row0 < 0 || rows < 0 || row0 + rows > m) fail(MSVD_ERR_DIMENSION, "msvd: raw row range outside the matrix");
    if (ld < n) fail(MSVD_ERR_DIMENSION, "msvd: leading dimension below column count");
    if (rows == 0 || n == 0) return;
    seek_row(fh.f, p, row0, n);
    if (!c.copy_stream) MSVD_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    const int64_t chunk = std::max<int64_t>(1, (64LL << 20) / (8 * n));  // ~64 MB of rows per buffer
    const size_t bytes = sizeof(double) * static_cast<size_t>(chunk * n);
    double* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    auto release = [&] {
        for (int i = 0; i < 2; ++i) {
            if (done[i]) cudaEventSynchronize(done[i]), cudaEventDestroy(done[i]);
            if (stage[i]) cudaFreeHost(stage[i]);
        }
    };
    try {
        for (int i = 0; i < 2; ++i) {
            MSVD_CUDA(cudaMallocHost(&stage[i], bytes));
            MSVD_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
        }
        int cur = 0;
        for (int64_t r = 0; r < rows; r += chunk, cur ^= 1) {
            const int64_t cnt = std::min(chunk, rows - r);
            MSVD_CUDA(cudaEventSynchronize(done[cur]));  // the buffer's previous copy has drained
            if (std::fread(stage[cur], sizeof(double), static_cast<size_t>(cnt * n), fh.f) !=
                static_cast<size_t>(cnt * n))
                fail(MSVD_ERR_IO, p + ": read failed");
            if (ld == n)  // contiguous rows: one linear DMA
                MSVD_CUDA(cudaMemcpyAsync(dA + r * n, stage[cur], sizeof(double) * n * cnt, cudaMemcpyHostToDevice,
                                          c.copy_stream));
            else
                MSVD_CUDA(cudaMemcpy2DAsync(dA + r * ld, sizeof(double) * ld, stage[cur], sizeof(double) * n,
                                            sizeof(double) * n, cnt, cudaMemcpyHostToDevice, c.copy_stream));
            MSVD_CUDA(cudaEventRecord(done[cur], c.copy_stream));
        }
        MSVD_CUDA(cudaStreamSynchronize(c.copy_stream));
    } catch (...) {
        release();
        throw;
    }
    release();
}

}  // namespace msvd
