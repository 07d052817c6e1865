// Launch interface of the sm_100a bitset-sort kernels (K2 scatter, K3 scan)
// and the per-sort control block they share. Host orchestration lives in
// capi.cpp; nothing here is exported from libbitsort.so.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace bws_gpu {

// Per-sort device control block. Zeroed (cudaMemsetAsync) before every sort
// together with the scan's tile-status array, which directly follows it.
struct alignas(64) Ctrl {
    unsigned int max_key;          // atomicMax over every in-range key (K2)
    unsigned int bad_keys;         // keys >= key_range (K2); never scattered
    unsigned int ticket;           // K3 dynamic tile ticket
    unsigned int pad0;
    unsigned long long total;      // set bits over the whole scan (K3, last tile)
    unsigned long long pad1[5];
};
static_assert(sizeof(Ctrl) == 64, "Ctrl is one 64-byte line");

// K3 geometry: a tile is SCAN_ROUNDS rounds of SCAN_THREADS consecutive words.
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ROUNDS = 8;
constexpr int SCAN_TILE_WORDS = SCAN_THREADS * SCAN_ROUNDS;  // 2048 words = 65536 keys

// K2 geometry: a tile is SCATTER_VEC uint4 loads per thread.
constexpr int SCATTER_THREADS = 256;
constexpr int SCATTER_VEC = 4;
constexpr int SCATTER_TILE_KEYS = SCATTER_THREADS * SCATTER_VEC * 4;  // 4096 keys
constexpr int SCATTER_SMEM_WORDS = 8192;  // staged bitset window: 32 KB = 262144 keys

enum ScatterMode : int { kAuto = 0, kPlain = 1, kWarpAgg = 2, kSmem = 3 };

inline std::size_t scan_tiles(std::uint64_t n_words) {
    return static_cast<std::size_t>((n_words + SCAN_TILE_WORDS - 1) / SCAN_TILE_WORDS);
}

struct LaunchGeometry {
    int scatter_blocks = 0;
    int scan_blocks = 0;
    int fill_blocks = 0;
};

// Computes persistent-grid sizes (SM count x resident blocks) for `device`.
cudaError_t query_geometry(int device, LaunchGeometry* geo);

// K2: bits[x>>5] |= 1<<(x&31) for every key x < key_range (key_range in
// [1, 2^32]); keys >= key_range are counted in ctrl->bad_keys. Also folds the
// max in-range key into ctrl->max_key.
cudaError_t launch_scatter(const std::uint32_t* keys, std::size_t n, std::uint32_t* bits,
                           std::uint64_t key_range, Ctrl* ctrl, int mode,
                           const LaunchGeometry& geo, cudaStream_t stream);

// K3: single-pass decoupled-lookback scan of n_words words (n_words == 0:
// (ctrl->max_key >> 5) + 1, i.e. derived from K2). Writes key_base + bit index
// of every set bit, ascending, to out[0, out_capacity). Writes the number of
// set bits to ctrl->total and, if non-null, *d_total. With clear != 0 every
// nonzero word is zeroed after it is read (keeps a cached bitset all-zero
// between sorts). `status` holds scan_tiles(n_words) zeroed 64-bit words.
cudaError_t launch_scan(const std::uint32_t* bits, std::uint64_t n_words, std::uint32_t key_base,
                        std::uint32_t* out, std::uint64_t out_capacity, Ctrl* ctrl,
                        unsigned long long* status, unsigned long long* d_total, int clear,
                        const LaunchGeometry& geo, cudaStream_t stream);

}  // namespace bws_gpu
