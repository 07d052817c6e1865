// Golden-vector generator: runs the UNMODIFIED reference (its own C ABI,
// oracle/_ref/libbitsort_ref.so built from /root/reference/proj/src) and writes
// fixtures that the CPU-only tests and the GPU parity tests compare against.
// Only this generator touches the reference; the fixtures it writes are
// committed so nothing at test time needs /root/reference.
//
// Build + run:  make -C oracle ref && oracle/_ref/gen_golden tests/golden
//
// Fixtures
//   acceptance_u32.bin  acceptance criterion 2 inputs for uint32
//                       (proj/tests/acceptance.cpp:65-95: generate_input<uint32_t>
//                       (n, uniform_full_range, seed 1337, trial), n in
//                       {1,2,100,1000}), first 16 trials per n, with the
//                       reference bws_sort(...,32,1,BWS_ALG_BITWISE) output
//   edge_u32.bin        hand-picked distinct-key edge cases, same treatment
//   repeats_u32.bin     inputs with repeated keys from the reference's own
//                       generator (generator.hpp:91-130: uniform_small_range
//                       with spans 16 and 1024, constant), n in {100, 1000,
//                       3000}, trials 0-1, seed 1337, with the reference output
//   widths.bin          every other (width, signedness) bws_sort arm: the
//                       reference generator's five distributions
//                       (generator.hpp:91-130; small range with span 100)
//                       for int8/uint8/int16/uint16/int32/int64/uint64,
//                       n in {17, 1000}, seed 1337, with the reference output
//                       (format: "BWSW" u32 version=1 u32 count, then per
//                       record u32 width, is_unsigned, n, distribution index,
//                       then n keys in, n keys out, little endian)
//   anchors.json        C1-C5 synthetic-input anchors:
//                       C1/C2/C4 generated with the reference's splitmix64,
//                       C3 (Feistel permutation) and C5 (clustered Zipf) with
//                       csrc/datagen.c; every one sorted by the reference
//                       bws_sort(...,32,1,BWS_ALG_BITWISE) and hashed (FNV-1a 64
//                       over the little-endian bytes). C3 takes ~5 min and C5
//                       ~1 min of single-threaded reference sort.
//
// Record format (little endian): "BWSG" u32 version=1 u32 count, then per
// record: u32 n, u32 trial, u32 distinct(0/1), u32 pad, n x u32 input,
// n x u32 reference output.
#include <bitsort/bitsort.h>

#include <algorithm>
#include <cinttypes>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <unordered_set>
#include <vector>

#include "generator.hpp"  // bws::splitmix64, bws::generate_input (reference headers)

// C3/C5 inputs come from this repo's seeded generator (csrc/datagen.c, linked
// into this program by oracle/Makefile): the same bytes the tests and the bench
// generate, so the reference's sorted output of them pins the GPU output.
extern "C" int bws_gen_permutation(uint32_t* out, uint64_t n, uint64_t seed);
extern "C" int bws_gen_clustered(uint32_t* out, uint64_t n, uint32_t clusters, double zipf_s,
                                 uint64_t half_window, uint64_t seed, uint32_t* centres_out);

namespace {

struct record {
    uint32_t n, trial, distinct;
    std::vector<uint32_t> input, output;
};

uint64_t fnv1a64(const std::vector<uint32_t>& v) {
    uint64_t h = 0xcbf29ce484222325ull;
    const auto* p = reinterpret_cast<const unsigned char*>(v.data());
    for (size_t i = 0; i < v.size() * sizeof(uint32_t); ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

std::vector<uint32_t> ref_sort(std::vector<uint32_t> v) {
    if (bws_sort(v.data(), v.size(), 32, 1, BWS_ALG_BITWISE) != BWS_OK) {
        std::fprintf(stderr, "reference bws_sort failed: %s\n", bws_last_error());
        std::exit(1);
    }
    return v;
}

bool all_distinct(const std::vector<uint32_t>& v) {
    std::unordered_set<uint32_t> s(v.begin(), v.end());
    return s.size() == v.size();
}

void write_records(const std::string& path, const std::vector<record>& recs) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) {
        std::perror(path.c_str());
        std::exit(1);
    }
    const uint32_t hdr[3] = {0x47535742u /* "BWSG" */, 1u, static_cast<uint32_t>(recs.size())};
    std::fwrite(hdr, sizeof hdr, 1, f);
    for (const record& r : recs) {
        const uint32_t h[4] = {r.n, r.trial, r.distinct, 0};
        std::fwrite(h, sizeof h, 1, f);
        std::fwrite(r.input.data(), sizeof(uint32_t), r.n, f);
        std::fwrite(r.output.data(), sizeof(uint32_t), r.n, f);
    }
    std::fclose(f);
}

record make_record(std::vector<uint32_t> in, uint32_t trial) {
    record r;
    r.n = static_cast<uint32_t>(in.size());
    r.trial = trial;
    r.distinct = all_distinct(in) ? 1u : 0u;
    r.output = ref_sort(in);
    r.input = std::move(in);
    return r;
}

// forward Fisher-Yates prefix of [0, M) with
// splitmix64{seed}: j = i + next() % (M - i), swap(p[i], p[j]), keys = p[0, n).
std::vector<uint32_t> shuffle_prefix(uint64_t n, uint64_t M, uint64_t seed) {
    std::vector<uint32_t> p(M);
    for (uint64_t i = 0; i < M; ++i) p[i] = static_cast<uint32_t>(i);
    bws::splitmix64 rng{seed};
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t j = i + rng.next() % (M - i);
        std::swap(p[i], p[j]);
    }
    p.resize(n);
    return p;
}

// splitmix64{seed} draws truncated to uint32, keeping
// first occurrences, until n distinct keys are accepted (draw order kept).
std::vector<uint32_t> dedup_draws(uint64_t n, uint64_t seed) {
    std::vector<uint64_t> seen((1ull << 32) / 64, 0);
    std::vector<uint32_t> out;
    out.reserve(n);
    bws::splitmix64 rng{seed};
    while (out.size() < n) {
        const uint32_t x = static_cast<uint32_t>(rng.next());
        uint64_t& w = seen[x >> 6];
        const uint64_t bit = 1ull << (x & 63);
        if (w & bit) continue;
        w |= bit;
        out.push_back(x);
    }
    return out;
}

void anchor(FILE* f, const char* name, const std::vector<uint32_t>& in, bool last) {
    const std::vector<uint32_t> out = ref_sort(in);
    const auto [mn, mx] = std::minmax_element(in.begin(), in.end());
    std::fprintf(f, "  \"%s\": {\"n\": %zu, \"first8\": [", name, in.size());
    for (size_t i = 0; i < 8 && i < in.size(); ++i) std::fprintf(f, "%s%u", i ? ", " : "", in[i]);
    std::fprintf(f,
                 "], \"fnv1a64_input\": \"%016" PRIx64 "\", \"fnv1a64_sorted\": \"%016" PRIx64
                 "\", \"min\": %u, \"max\": %u}%s\n",
                 fnv1a64(in), fnv1a64(out), *mn, *mx, last ? "" : ",");
}

template <class T>
void width_records(FILE* f, uint32_t& count) {
    constexpr uint32_t width = sizeof(T) * 8;
    const uint32_t is_unsigned = std::is_unsigned_v<T> ? 1u : 0u;
    const char* names[] = {"uniform_full_range", "uniform_small_range:100", "sorted", "reverse_sorted",
                           "constant"};
    for (uint32_t di = 0; di < 5; ++di) {
        const bws::distribution_spec d = bws::distribution_spec::parse(names[di]);
        for (const size_t n : {size_t{17}, size_t{1000}}) {
            std::vector<T> in = bws::generate_input<T>(n, d, 1337, 0);
            std::vector<T> out = in;
            if (bws_sort(out.data(), out.size(), width, static_cast<int>(is_unsigned), BWS_ALG_BITWISE) != BWS_OK) {
                std::fprintf(stderr, "reference bws_sort failed: %s\n", bws_last_error());
                std::exit(1);
            }
            const uint32_t h[4] = {width, is_unsigned, static_cast<uint32_t>(n), di};
            std::fwrite(h, sizeof h, 1, f);
            std::fwrite(in.data(), sizeof(T), n, f);
            std::fwrite(out.data(), sizeof(T), n, f);
            ++count;
        }
    }
}

void write_width_records(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) {
        std::perror(path.c_str());
        std::exit(1);
    }
    uint32_t hdr[3] = {0x57535742u /* "BWSW" */, 1u, 0u};
    std::fwrite(hdr, sizeof hdr, 1, f);
    uint32_t count = 0;
    width_records<int8_t>(f, count);
    width_records<uint8_t>(f, count);
    width_records<int16_t>(f, count);
    width_records<uint16_t>(f, count);
    width_records<int32_t>(f, count);
    width_records<int64_t>(f, count);
    width_records<uint64_t>(f, count);
    hdr[2] = count;
    std::fseek(f, 0, SEEK_SET);
    std::fwrite(hdr, sizeof hdr, 1, f);
    std::fclose(f);
}

}  // namespace

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "tests/golden";

    // acceptance criterion 2, uint32 arm (acceptance.cpp:70-77, :88)
    std::vector<record> acc;
    const bws::distribution_spec dist{};
    for (const size_t n : {size_t{1}, size_t{2}, size_t{100}, size_t{1000}})
        for (uint32_t trial = 0; trial < 16; ++trial)
            acc.push_back(make_record(bws::generate_input<uint32_t>(n, dist, 1337, trial), trial));
    write_records(dir + "/acceptance_u32.bin", acc);

    // repeated keys: the reference generator's duplicate-heavy distributions
    std::vector<record> rep;
    for (const char* name : {"uniform_small_range:16", "uniform_small_range:1024", "constant"}) {
        const bws::distribution_spec d = bws::distribution_spec::parse(name);
        for (const size_t n : {size_t{100}, size_t{1000}, size_t{3000}})
            for (uint32_t trial = 0; trial < 2; ++trial)
                rep.push_back(make_record(bws::generate_input<uint32_t>(n, d, 1337, trial), trial));
    }
    write_records(dir + "/repeats_u32.bin", rep);

    write_width_records(dir + "/widths.bin");

    // distinct-key edge cases at the 32-bit boundaries
    std::vector<std::vector<uint32_t>> edges = {
        {0u},
        {0xffffffffu},
        {0xffffffffu, 0u},
        {200u, 3u, 255u, 0u},  // test_capi.cpp:79-81 vector, widened to uint32
        {31u, 32u, 0u, 63u, 64u, 1u},
        {0x80000000u, 0x7fffffffu, 0xfffffffeu, 0xffffffffu, 1u, 0u},
    };
    {
        std::vector<uint32_t> desc(4099);
        for (size_t i = 0; i < desc.size(); ++i) desc[i] = static_cast<uint32_t>(desc.size() - 1 - i);
        edges.push_back(desc);  // reverse run crossing word and tile boundaries
        std::vector<uint32_t> top(70);
        for (size_t i = 0; i < top.size(); ++i) top[i] = 0xffffffffu - static_cast<uint32_t>(3 * i);
        edges.push_back(top);  // keys in the last bitset words of the 2^32 range
    }
    std::vector<record> edge;
    for (size_t i = 0; i < edges.size(); ++i) edge.push_back(make_record(edges[i], static_cast<uint32_t>(i)));
    write_records(dir + "/edge_u32.bin", edge);

    FILE* f = std::fopen((dir + "/anchors.json").c_str(), "w");
    if (!f) {
        std::perror("anchors.json");
        return 1;
    }
    std::fprintf(f, "{\n");
    std::fprintf(f, "  \"_generator\": \"tests/golden/gen_golden.cpp (reference bws_sort via oracle/_ref/libbitsort_ref.so)\",\n");
    anchor(f, "C1", shuffle_prefix(1000000, 1ull << 24, 42), false);
    anchor(f, "C2", shuffle_prefix(1ull << 26, 1ull << 28, 42), false);
    anchor(f, "C4", dedup_draws(1ull << 24, 42), false);
    {
        // C5: 2^28 keys, 4096 clusters, Zipf(1.2), +-2^18 windows, seed 42 (configs.py)
        std::vector<uint32_t> c5(1ull << 28);
        std::vector<uint32_t> centres(4096);
        if (bws_gen_clustered(c5.data(), c5.size(), 4096, 1.2, 1ull << 18, 42, centres.data()) != 0) {
            std::fprintf(stderr, "bws_gen_clustered failed\n");
            return 1;
        }
        anchor(f, "C5", c5, std::getenv("GOLDEN_SKIP_C3") != nullptr);
    }
    if (!std::getenv("GOLDEN_SKIP_C3")) {
        // C3: Feistel permutation of [0, 2^30), seed 42 (configs.py); sorted = identity
        std::vector<uint32_t> c3(1ull << 30);
        if (bws_gen_permutation(c3.data(), c3.size(), 42) != 0) {
            std::fprintf(stderr, "bws_gen_permutation failed\n");
            return 1;
        }
        anchor(f, "C3", c3, true);
    }
    std::fprintf(f, "}\n");
    std::fclose(f);
    std::printf("golden fixtures written to %s\n", dir.c_str());
    return 0;
}
