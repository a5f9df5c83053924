// OCTF snapshot I/O (snapshot.hpp:10-14, snapshot.cpp:65-121): the reference's binary particle
// format, little-endian: "OCTF", u32 version 1, u64 n, f64 time, f64 G, f64 eps, f64 mass[n],
// f64 pos[3n] (xyz interleaved), f64 vel[3n].  The arrays are exactly the C-ABI layout, so a
// snapshot streams straight into (pinned) host buffers and on to the device without conversion.
// Errors mirror the reference's data_error messages, byte offsets included.
#include "snapshot.hpp"

#include <cstdio>
#include <cstring>
#include <string>

namespace g2 {
namespace {

constexpr char kMagic[4] = {'O', 'C', 'T', 'F'};
constexpr uint32_t kVersion = 1;
constexpr size_t kHeader = 4 + 4 + 8 + 3 * 8;

struct File {
    FILE* f = nullptr;
    explicit File(FILE* p) : f(p) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

// little-endian loads/stores independent of the host byte order
uint64_t le64(const unsigned char* b) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(b[i]) << (8 * i);
    return v;
}
void put64(unsigned char* b, uint64_t v) {
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
}
double asf64(uint64_t u) {
    double d;
    std::memcpy(&d, &u, 8);
    return d;
}
uint64_t asu64(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
}

[[noreturn]] void truncated(const std::string& path, const char* what, size_t offset) {
    throw SnapshotError(path + ": truncated " + what + " at byte " + std::to_string(offset));
}

}  // namespace

SnapshotHeader read_snapshot_header(const std::string& path) {
    File in(std::fopen(path.c_str(), "rb"));
    if (!in.f) throw SnapshotError(path + ": cannot open");
    unsigned char h[kHeader];
    const size_t got = std::fread(h, 1, kHeader, in.f);
    for (int i = 0; i < 4; ++i) {
        if (size_t(i) >= got) truncated(path, "magic", size_t(i));
        if (char(h[i]) != kMagic[i]) throw SnapshotError(path + ": bad magic at byte " + std::to_string(i));
    }
    if (got < 8) truncated(path, "version", 4);
    const uint32_t version = uint32_t(h[4]) | uint32_t(h[5]) << 8 | uint32_t(h[6]) << 16 | uint32_t(h[7]) << 24;
    if (version != kVersion)
        throw SnapshotError(path + ": unsupported version " + std::to_string(version) + " at byte 4");
    if (got < 16) truncated(path, "particle count", 8);
    SnapshotHeader s;
    s.n = le64(h + 8);
    if (s.n == 0) throw SnapshotError(path + ": zero particle count at byte 8");
    if (got < 24) truncated(path, "time", 16);
    s.time = asf64(le64(h + 16));
    if (got < 32) truncated(path, "G", 24);
    s.G = asf64(le64(h + 24));
    if (got < 40) truncated(path, "eps", 32);
    s.eps = asf64(le64(h + 32));
    return s;
}

void check_snapshot_size(const std::string& path, const SnapshotHeader& s) {
    // an untrusted count: 40 + 56 n must not wrap, and the file must hold the three arrays (the
    // error is the one read_snapshot would raise, same byte offset, without allocating n first)
    if (s.n > (uint64_t(SIZE_MAX) - kHeader) / 56) throw SnapshotError(path + ": particle count too large at byte 8");
    File in(std::fopen(path.c_str(), "rb"));
    if (!in.f) throw SnapshotError(path + ": cannot open");
    if (std::fseek(in.f, 0, SEEK_END) != 0) throw SnapshotError(path + ": cannot seek");
    const long end = std::ftell(in.f);
    if (end < 0) throw SnapshotError(path + ": cannot seek");
    const uint64_t size = uint64_t(end), n = s.n;
    const uint64_t ends[3] = {kHeader + 8 * n, kHeader + 32 * n, kHeader + 56 * n};
    const char* what[3] = {"mass array", "position array", "velocity array"};
    uint64_t start = kHeader;
    for (int k = 0; k < 3; ++k) {
        if (size < ends[k]) truncated(path, what[k], size_t(start + (size > start ? (size - start) / 8 * 8 : 0)));
        start = ends[k];
    }
}

SnapshotHeader read_snapshot(const std::string& path, double* mass, double* pos, double* vel, size_t cap) {
    const SnapshotHeader s = read_snapshot_header(path);
    check_snapshot_size(path, s);
    if (s.n > cap) throw SnapshotError(path + ": particle count exceeds the caller's buffers");
    File in(std::fopen(path.c_str(), "rb"));
    if (!in.f) throw SnapshotError(path + ": cannot open");
    std::fseek(in.f, long(kHeader), SEEK_SET);
    size_t offset = kHeader;
    // the reference's Reader reports the offset of the first value that does not fit
    auto block = [&](double* dst, size_t count, const char* what) {
        const size_t got = std::fread(dst, 8, count, in.f);
        if (got < count) truncated(path, what, offset + got * 8);
        offset += count * 8;
#if __BYTE_ORDER__ != __ORDER_LITTLE_ENDIAN__
        for (size_t i = 0; i < count; ++i) {
            unsigned char b[8];
            std::memcpy(b, dst + i, 8);
            dst[i] = asf64(le64(b));
        }
#endif
    };
    block(mass, s.n, "mass array");
    block(pos, 3 * s.n, "position array");
    block(vel, 3 * s.n, "velocity array");
    return s;
}

void write_snapshot(const std::string& path, size_t n, const double* mass, const double* pos, const double* vel,
                    double time, double G, double eps) {
    if (n == 0) throw SnapshotError("write_snapshot: empty system");
    const std::string tmp = path + ".tmp";  // atomic: temp file + rename (csv.cpp write_text_atomic)
    {
        File out(std::fopen(tmp.c_str(), "wb"));
        if (!out.f) throw SnapshotError(tmp + ": cannot open for writing");
        unsigned char h[kHeader];
        std::memcpy(h, kMagic, 4);
        h[4] = kVersion & 0xff, h[5] = h[6] = h[7] = 0;
        put64(h + 8, n);
        put64(h + 16, asu64(time));
        put64(h + 24, asu64(G));
        put64(h + 32, asu64(eps));
        bool ok = std::fwrite(h, 1, kHeader, out.f) == kHeader;
        auto block = [&](const double* src, size_t count) {
#if __BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__
            ok = ok && std::fwrite(src, 8, count, out.f) == count;
#else
            for (size_t i = 0; i < count && ok; ++i) {
                unsigned char b[8];
                put64(b, asu64(src[i]));
                ok = std::fwrite(b, 1, 8, out.f) == 8;
            }
#endif
        };
        block(mass, n);
        block(pos, 3 * n);
        block(vel, 3 * n);
        ok = ok && std::fflush(out.f) == 0;
        if (!ok) {
            std::remove(tmp.c_str());
            throw SnapshotError(tmp + ": write failed");
        }
    }
    if (std::rename(tmp.c_str(), path.c_str()) != 0) {
        std::remove(tmp.c_str());
        throw SnapshotError(path + ": rename failed");
    }
}

}  // namespace g2
