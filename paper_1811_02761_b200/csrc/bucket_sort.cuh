// Bucket sort of a rebuild's nearly sorted Morton keys (see bucket_sort.cu).
#pragma once

#include "kernels.cuh"

namespace g2 {

constexpr uint32_t kBucketCap = 8192;      // keys a bucket's region (and the large local sort) holds
constexpr uint32_t kBucketTarget = 2048;   // mean keys per bucket: 2x headroom for a nearly sorted input
constexpr uint32_t kBucketMaxB = 4096;     // splitters: 4 x 4096 samples ranked in 128 KB of shared memory
constexpr size_t kBucketMinN = 1u << 15;
constexpr size_t kBucketMaxN = size_t(kBucketMaxB) * kBucketTarget;  // 2^23

struct BucketScratch {
    DBuf<uint64_t> samples;  // [nb * oversampling] sampled keys, sorted per chunk
    DBuf<uint64_t> split;   // [nb] sorted splitter keys
    DBuf<uint32_t> cursor;  // [nb] keys claimed per bucket
    DBuf<uint32_t> offset;  // [nb] output offset per bucket
    DBuf<uint32_t> big;     // [1 + kMaxBig] count, then the buckets above the mid-size local sort's capacity
    DBuf<uint32_t> mid;     // [1 + nb] count, then the buckets above the small local sort's capacity
    DBuf<int> gate;         // 1: some bucket overflowed (the output is the identity order)
    DBuf<uint64_t> rkeys;   // [nb * kBucketCap] bucket regions
    DBuf<uint32_t> rvals;
    // the three local-sort instances run concurrently (forked from the caller's stream and joined)
    cudaStream_t side[2] = {nullptr, nullptr};
    cudaEvent_t fork = nullptr, join[2] = {nullptr, nullptr};
    BucketScratch() = default;
    BucketScratch(const BucketScratch&) = delete;
    BucketScratch& operator=(const BucketScratch&) = delete;
    ~BucketScratch() {
        for (auto& x : side)
            if (x) cudaStreamDestroy(x);
        for (auto& e : join)
            if (e) cudaEventDestroy(e);
        if (fork) cudaEventDestroy(fork);
    }
};

// number of buckets for n keys (a power of two), 0 when n is outside the supported range
uint32_t bucket_count(size_t n);
// keys of the particles stored in xyzm (storage order) sorted by key into keys_out, their storage
// positions into vals_out (equal keys in any order).  Returns false (nothing launched) when n is out of
// range.  Otherwise sc.gate.p is a device word set iff a bucket overflowed, in which case vals_out is
// the identity permutation (keys_out zero) and the caller must sort by other means.
bool launch_bucket_sort(const double4* xyzm, size_t n, const Cube* cube, BucketScratch& sc, uint64_t* keys_out,
                        uint32_t* vals_out, DevFlags* flags, cudaStream_t s);

}  // namespace g2
