// bitsort sort — the reference CLI's `sort` subcommand (proj/tools/main.cpp:
// 97-144 read_integer_file/sort_typed, :206-223 run_sort, :352-356 options)
// over the B200 library, talking to it only through the C ABI (bws_sort).
//
//   bitsort sort <input|-> [--width 8|16|32|64] [--unsigned] [--algorithm bitwise]
//                [--out PATH] [--threads N]
//
// Same input format (one decimal value per line; blank lines and lines
// starting with '#' ignored; a bad line is reported as file:line), same
// default (signed 32-bit), same exit statuses (0 ok, 1 usage/config, 2 data,
// 3 integrity; main.cpp:20-31). Unlike the reference, parsing and printing
// run on all host threads (the file is split at line boundaries), because at
// GPU sort speed a 4 GB text file's parse dominates the run (SURVEY.md
// §8(f) f2). The bits/bench/trace subcommands are not on the sort path.
#include <bitsort/bitsort.h>

#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <iterator>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

namespace {

int exit_for(bws_status status) {
    switch (status) {
        case BWS_OK: return 0;
        case BWS_ERROR_CONFIG: return 1;
        case BWS_ERROR_DATA: return 2;
        case BWS_ERROR_RANGE: return 2;
        case BWS_ERROR_INTEGRITY: return 3;
        case BWS_ERROR_INTERNAL: return 1;
    }
    return 1;
}

int fail(bws_status status) {
    std::cerr << "bitsort: " << bws_last_error() << "\n";
    return exit_for(status);
}

std::string_view trim(std::string_view s) {
    while (!s.empty() && (s.front() == ' ' || s.front() == '\t' || s.front() == '\r')) s.remove_prefix(1);
    while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
    return s;
}

struct Options {
    std::string input;
    uint32_t width = 32;
    bool is_unsigned = false;
    std::string algorithm = "bitwise";
    std::string out_path;
    unsigned threads = 0;
};

int usage(const char* msg) {
    if (msg) std::cerr << "bitsort: " << msg << "\n";
    std::cerr << "usage: bitsort sort <input|-> [--width N] [--unsigned] [--algorithm NAME] "
                 "[--out PATH] [--threads N]\n";
    return 1;
}

// One chunk of the text: parsed two's-complement patterns of the key width,
// its line count, and the first error (chunk-relative line number).
struct Chunk {
    std::vector<uint64_t> values;
    size_t lines = 0;
    size_t error_line = 0;  // 0 = none
    std::string error;
};

// Parses one decimal value into its two's-complement pattern at `width` bits
// (main.cpp:58-93: same range checks and messages).
bool parse_value(std::string_view text, uint32_t width, bool is_unsigned, uint64_t& pattern, std::string& error) {
    const std::string w = std::to_string(width) + "-bit";
    if (is_unsigned) {
        uint64_t v = 0;
        const auto [ptr, ec] = std::from_chars(text.data(), text.data() + text.size(), v);
        if (ec != std::errc{} || ptr != text.data() + text.size()) {
            error = "cannot parse '" + std::string(text) + "' as an unsigned integer";
            return false;
        }
        if (width < 64 && (v >> width) != 0) {
            error = "value " + std::string(text) + " out of range for unsigned " + w;
            return false;
        }
        pattern = v;
    } else {
        int64_t v = 0;
        const auto [ptr, ec] = std::from_chars(text.data(), text.data() + text.size(), v);
        if (ec != std::errc{} || ptr != text.data() + text.size()) {
            error = "cannot parse '" + std::string(text) + "' as an integer";
            return false;
        }
        if (width < 64) {
            const int64_t lim = int64_t{1} << (width - 1);
            if (v < -lim || v >= lim) {
                error = "value " + std::string(text) + " out of range for signed " + w;
                return false;
            }
        }
        pattern = static_cast<uint64_t>(v);
    }
    if (width < 64) pattern &= (uint64_t{1} << width) - 1;
    return true;
}

void parse_chunk(std::string_view text, uint32_t width, bool is_unsigned, Chunk& c) {
    c.values.reserve(text.size() / 8);
    size_t pos = 0;
    while (pos < text.size()) {
        size_t nl = text.find('\n', pos);
        if (nl == std::string_view::npos) nl = text.size();
        ++c.lines;
        const std::string_view line = trim(text.substr(pos, nl - pos));
        pos = nl + 1;
        if (line.empty() || line.front() == '#') continue;
        uint64_t pattern = 0;
        if (!parse_value(line, width, is_unsigned, pattern, c.error)) {
            c.error_line = c.lines;
            return;
        }
        c.values.push_back(pattern);
    }
}

bool read_all(const std::string& path, std::string& text) {
    if (path == "-") {
        text.assign(std::istreambuf_iterator<char>(std::cin), std::istreambuf_iterator<char>());
        return true;
    }
    std::ifstream f(path, std::ios::binary);
    if (!f) {
        std::cerr << "bitsort: cannot open '" << path << "'\n";
        return false;
    }
    f.seekg(0, std::ios::end);
    text.resize(static_cast<size_t>(f.tellg()));
    f.seekg(0);
    f.read(text.data(), static_cast<std::streamsize>(text.size()));
    return static_cast<bool>(f) || f.eof();
}

template <class F>
void parallel_for(unsigned n, F&& f) {
    std::vector<std::thread> pool;
    for (unsigned i = 1; i < n; ++i) pool.emplace_back(f, i);
    f(0u);
    for (auto& t : pool) t.join();
}

int run_sort(const Options& o) {
    bws_algorithm algorithm = BWS_ALG_BITWISE;
    if (const bws_status s = bws_algorithm_from_name(o.algorithm.c_str(), &algorithm); s != BWS_OK) return fail(s);
    if (o.width != 8 && o.width != 16 && o.width != 32 && o.width != 64) {  // bws_sort words the error
        uint64_t probe = 0;
        return fail(bws_sort(&probe, 1, o.width, o.is_unsigned ? 1 : 0, algorithm));
    }
    std::string text;
    if (!read_all(o.input, text)) return 2;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nt = std::max(1u, std::min<unsigned>(o.threads ? o.threads : hw,
                                                        static_cast<unsigned>(text.size() / (1u << 20) + 1)));
    // chunk boundaries just after a newline
    std::vector<size_t> cut(nt + 1, text.size());
    cut[0] = 0;
    for (unsigned i = 1; i < nt; ++i) {
        size_t p = text.size() * i / nt;
        while (p < text.size() && text[p - 1] != '\n') ++p;
        cut[i] = std::max(p, cut[i - 1]);
    }
    std::vector<Chunk> chunks(nt);
    const std::string_view all(text);
    parallel_for(nt, [&](unsigned i) {
        parse_chunk(all.substr(cut[i], cut[i + 1] - cut[i]), o.width, o.is_unsigned, chunks[i]);
    });
    size_t lines_before = 0, n = 0;
    for (const Chunk& c : chunks) {
        if (c.error_line) {
            std::cerr << "bitsort: " << (o.input == "-" ? "<stdin>" : o.input) << ":"
                      << lines_before + c.error_line << ": " << c.error << "\n";
            return 2;
        }
        lines_before += c.lines;
        n += c.values.size();
    }
    // the keys at their width, sorted in place by the library
    const size_t kb = o.width / 8;
    std::vector<unsigned char> data(n * kb + 8);
    {
        size_t off = 0;
        for (Chunk& c : chunks) {
            for (const uint64_t v : c.values) {
                std::memcpy(data.data() + off * kb, &v, kb);  // little-endian low bytes
                ++off;
            }
            std::vector<uint64_t>().swap(c.values);
        }
    }
    const bws_status status = bws_sort(data.data(), n, o.width, o.is_unsigned ? 1 : 0, algorithm);
    if (status != BWS_OK) return fail(status);

    // print in parallel into per-thread buffers, then write them in order
    std::vector<std::string> outs(nt);
    parallel_for(nt, [&](unsigned i) {
        const size_t lo = n * i / nt, hi = n * (i + 1) / nt;
        std::string& s = outs[i];
        s.reserve((hi - lo) * (o.width / 3 + 3));
        char buf[24];
        for (size_t k = lo; k < hi; ++k) {
            uint64_t u = 0;
            std::memcpy(&u, data.data() + k * kb, kb);
            std::to_chars_result r;
            if (o.is_unsigned) {
                r = std::to_chars(buf, buf + sizeof buf, u);
            } else {
                const unsigned sh = 64 - o.width;  // sign-extend the width-bit pattern
                r = std::to_chars(buf, buf + sizeof buf, static_cast<int64_t>(u << sh) >> sh);
            }
            s.append(buf, r.ptr);
            s.push_back('\n');
        }
    });
    std::FILE* out = stdout;
    if (!o.out_path.empty()) {
        out = std::fopen(o.out_path.c_str(), "wb");
        if (!out) {
            std::cerr << "bitsort: cannot write '" << o.out_path << "'\n";
            return 2;
        }
    }
    for (const std::string& s : outs) std::fwrite(s.data(), 1, s.size(), out);
    if (out != stdout) std::fclose(out);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || std::strcmp(argv[1], "sort") != 0)
        return usage(argc >= 2 ? "only the 'sort' subcommand is provided by the B200 build" : nullptr);
    Options o;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto value = [&](const char* name) -> const char* {
            if (i + 1 >= argc) {
                usage((std::string(name) + " needs a value").c_str());
                return nullptr;
            }
            return argv[++i];
        };
        if (a == "--unsigned") {
            o.is_unsigned = true;
        } else if (a == "--width") {
            const char* v = value("--width");
            if (!v) return 1;
            o.width = static_cast<uint32_t>(std::strtoul(v, nullptr, 10));
        } else if (a == "--algorithm") {
            const char* v = value("--algorithm");
            if (!v) return 1;
            o.algorithm = v;
        } else if (a == "--out") {
            const char* v = value("--out");
            if (!v) return 1;
            o.out_path = v;
        } else if (a == "--threads") {
            const char* v = value("--threads");
            if (!v) return 1;
            o.threads = static_cast<unsigned>(std::strtoul(v, nullptr, 10));
        } else if (o.input.empty() && (a == "-" || a.rfind("--", 0) != 0)) {
            o.input = a;
        } else {
            return usage(("unknown argument '" + a + "'").c_str());
        }
    }
    if (o.input.empty()) return usage("input is required");
    return run_sort(o);
}
