// OCTF snapshot I/O (host code; see snapshot.cpp).
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace g2 {

struct SnapshotError : std::runtime_error {  // the reference's data_error (status 3)
    using std::runtime_error::runtime_error;
};

struct SnapshotHeader {
    uint64_t n = 0;
    double time = 0.0, G = 1.0, eps = 0.0;
};

SnapshotHeader read_snapshot_header(const std::string& path);
// throws unless 40 + 56 n fits size_t and the file holds all three arrays (untrusted n)
void check_snapshot_size(const std::string& path, const SnapshotHeader& h);
// mass[n], pos[3n], vel[3n] into the caller's buffers (cap = their particle capacity)
SnapshotHeader read_snapshot(const std::string& path, double* mass, double* pos, double* vel, size_t cap);
void write_snapshot(const std::string& path, size_t n, const double* mass, const double* pos, const double* vel,
                    double time, double G, double eps);

}  // namespace g2
