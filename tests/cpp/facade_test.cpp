// facade_test.cpp — exercises include/cashash_b200/cashash.hpp (the reference-shaped C++ host API
// over libchgpu.so) against the CPU oracle's C ABI (oracle/chor.h).  Reads like a test of the
// reference's own library: build_hash_family -> set_centering -> compute_codes -> match_pair ->
// save_matches.  `--host` runs only the checks that need no GPU.
//
// Built and run by tests/test_cpp_facade.py:
//   g++ -std=c++20 -I include -I oracle tests/cpp/facade_test.cpp -L... -lchgpu -lchoracle
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>

#include "cashash_b200/cashash.hpp"
#include "chor.h"

namespace ch = cashash_b200;

static int g_checks = 0;
#define CHECK(cond)                                                                     \
    do {                                                                                \
        ++g_checks;                                                                     \
        if (!(cond)) {                                                                  \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
            std::exit(1);                                                               \
        }                                                                               \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// uniform u8 descriptors; the first `twins` points are sigma=8 noisy copies of a shared pool
static ch::FeatureSet make_image(std::uint64_t seed, std::uint32_t n, std::uint32_t twins, const std::string& id) {
    std::mt19937_64 pool_rng(12345), rng(seed);
    std::normal_distribution<double> noise(0.0, 8.0);
    ch::FeatureSet fs;
    fs.image_id = id;
    fs.keypoints.resize(n);
    fs.descriptors.resize(n);
    for (std::uint32_t p = 0; p < n; ++p) {
        fs.keypoints[p] = {float(p % 1000), float(p / 1000), 2.0f, 0.0f};
        for (std::size_t c = 0; c < ch::kDescriptorDim; ++c) {
            if (p < twins) {
                const double base = double(pool_rng() & 0xff);
                const double v = std::min(255.0, std::max(0.0, base + noise(rng)));
                fs.descriptors[p][c] = std::uint8_t(v);
            } else {
                fs.descriptors[p][c] = std::uint8_t(rng() & 0xff);
            }
        }
    }
    return fs;
}

static std::string slurp(const std::filesystem::path& p) {
    std::ifstream in(p, std::ios::binary);
    std::ostringstream os;
    os << in.rdbuf();
    return os.str();
}

static chor_family_params to_chor(const ch::FamilyParams& p) { return {p.short_bits, p.long_bits, p.table_count, p.seed}; }
static chor_match_cfg to_chor(const ch::MatchConfig& c) {
    return {c.top_k, c.hamming_threshold, c.ratio, c.min_candidates_for_ratio, c.reduce_rounds};
}

struct OracleCodes {
    std::vector<std::uint32_t> shorts;
    std::vector<std::uint64_t> longs;
};

static OracleCodes oracle_codes(const ch::HashFamily& fam, const ch::FeatureSet& fs, int rr = 3) {
    OracleCodes oc;
    oc.shorts.resize(fs.size() * fam.params.table_count);
    oc.longs.resize(fs.size() * 2);
    const chor_family_params p = to_chor(fam.params);
    const int rc = chor_compute_codes(&p, fam.short_planes.front().data(), fam.long_planes.front().data(),
                                      fam.centering.data(), rr, fs.descriptors.empty() ? nullptr : fs.descriptors.front().data(),
                                      std::uint32_t(fs.size()), oc.shorts.data(), oc.longs.data());
    CHECK(rc == 0);
    return oc;
}

static std::vector<ch::MatchRecord> oracle_match(const ch::HashFamily& fam, const ch::MatchConfig& cfg, const ch::FeatureSet& a,
                                                 const OracleCodes& ca, const ch::FeatureSet& b, const OracleCodes& cb) {
    std::vector<ch::MatchRecord> rec(a.size() + 1);
    std::uint32_t count = 0;
    const chor_family_params p = to_chor(fam.params);
    const chor_match_cfg c = to_chor(cfg);
    const int rc = chor_match_pair(&p, &c, a.descriptors.front().data(), std::uint32_t(a.size()), ca.shorts.data(), ca.longs.data(),
                                   b.descriptors.front().data(), std::uint32_t(b.size()), cb.shorts.data(), cb.longs.data(),
                                   reinterpret_cast<chor_match_record*>(rec.data()), &count, nullptr, nullptr, nullptr);
    CHECK(rc == 0);
    rec.resize(count);
    return rec;
}

static void host_checks(const std::filesystem::path& tmp) {
    // build_hash_family: bit-identical to the oracle's planes; bad parameters throw invalid_argument
    for (const ch::FamilyParams& p : {ch::FamilyParams{}, ch::FamilyParams{10, 96, 4, 99}}) {
        const ch::HashFamily fam = ch::build_hash_family(p);
        std::vector<double> sp(fam.short_planes.size() * 128), lp(fam.long_planes.size() * 128);
        const chor_family_params cp = to_chor(p);
        CHECK(chor_build_family(&cp, sp.data(), lp.data()) == 0);
        CHECK(std::memcmp(sp.data(), fam.short_planes.front().data(), sp.size() * 8) == 0);
        CHECK(std::memcmp(lp.data(), fam.long_planes.front().data(), lp.size() * 8) == 0);
        CHECK(!fam.centering_set);
    }
    CHECK(throws<std::invalid_argument>([] { ch::build_hash_family({0, 128, 6, 1}); }));
    CHECK(throws<std::invalid_argument>([] { ch::build_hash_family({8, 8, 6, 1}); }));
    CHECK(throws<std::invalid_argument>([] { ch::build_hash_family({8, 129, 6, 1}); }));
    CHECK(throws<std::invalid_argument>([] { ch::build_hash_family({8, 128, 0, 1}); }));

    // CHFT round trip and the reference's fault classes / byte offsets (feature_io.cpp:65-106)
    const ch::FeatureSet fs = make_image(3, 37, 5, "img");
    const auto f = tmp / "a.chft";
    ch::save_features(fs, f);
    CHECK(std::filesystem::file_size(f) == 16 + 37 * 144);
    const ch::FeatureSet back = ch::load_features(f);
    CHECK(back.keypoints == fs.keypoints && back.descriptors == fs.descriptors);
    auto fault_of = [&](const std::filesystem::path& p, ch::FeatureFileFault want, std::uint64_t off) {
        try {
            ch::load_features(p);
        } catch (const ch::FeatureFileError& e) {
            return e.fault() == want && e.byte_offset() == off;
        }
        return false;
    };
    CHECK(fault_of(tmp / "nope.chft", ch::FeatureFileFault::MissingFile, 0));
    std::string blob = slurp(f);
    auto write = [&](const std::string& name, const std::string& bytes) {
        std::ofstream(tmp / name, std::ios::binary).write(bytes.data(), std::streamsize(bytes.size()));
        return tmp / name;
    };
    CHECK(fault_of(write("short_header", blob.substr(0, 9)), ch::FeatureFileFault::Truncated, 9));
    std::string bad = blob;
    bad[0] = 'X';
    CHECK(fault_of(write("bad_magic", bad), ch::FeatureFileFault::BadMagic, 0));
    bad = blob;
    bad[4] = 2;
    CHECK(fault_of(write("bad_version", bad), ch::FeatureFileFault::BadVersion, 4));
    CHECK(fault_of(write("cut", blob.substr(0, 16 + 144 * 10 + 77)), ch::FeatureFileFault::Truncated, 16 + 144 * 10 + 77));
    CHECK(throws<ch::FeatureFileError>([&] { ch::save_features(fs, tmp / "no_such_dir" / "x.chft"); }));

    // save_matches: byte-identical to the oracle's writer; integers print without a decimal point
    std::vector<ch::MatchRecord> rec = {{0, 5, 1250.0}, {3, 1, 0.5}, {9, 2, 8323200.0}, {11, 7, 1e-3}};
    ch::save_matches("imgA", "imgB", rec, tmp / "m_ours.txt");
    CHECK(chor_save_matches("imgA", "imgB", reinterpret_cast<const chor_match_record*>(rec.data()), 4,
                            (tmp / "m_ref.txt").string().c_str()) == 0);
    CHECK(slurp(tmp / "m_ours.txt") == slurp(tmp / "m_ref.txt"));
    CHECK(slurp(tmp / "m_ours.txt").rfind("# imgA imgB 4\n0 5 1250\n", 0) == 0);
    CHECK(ch::pair_file_name(3, 41) == "match_000003_000041.txt");
    CHECK(throws<ch::FeatureFileError>([&] { ch::save_matches("a", "b", rec, tmp / "no_such_dir" / "m.txt"); }));

    // plan_exhaustive: every unordered pair exactly once, a < b
    const auto pairs = ch::plan_exhaustive(23, 4, 3);
    CHECK(pairs.size() == 23 * 22 / 2);
    std::vector<char> seen(23 * 23, 0);
    for (const auto& [a, b] : pairs) {
        CHECK(a < b && b < 23 && !seen[a * 23 + b]);
        seen[a * 23 + b] = 1;
    }
    CHECK(throws<std::invalid_argument>([] { ch::plan_exhaustive(0, 1, 1); }));

    // scheduler.hpp:29-134 through the facade: partition, tasks with their pairs, residency traces, sizing
    {
        const ch::Partition part = ch::make_partition(23, 4, 3);
        CHECK(part.block_count() == 6 && part.group_count() == 2 && part.block_size(5) == 3 && part.block_group_of[4] == 1);
        const ch::PairPlan plan = ch::plan_exhaustive(part);
        CHECK(plan.pair_count() == 23 * 22 / 2);
        std::size_t at = 0;
        for (const ch::PlanTask& t : plan.tasks) {
            CHECK(t.block_a <= t.block_b && t.group_a == part.block_group_of[t.block_a] && t.group_b == part.block_group_of[t.block_b]);
            for (const auto& pr : t.pairs) {
                CHECK(pr == pairs[at] && pr.first / 4 == t.block_a && pr.second / 4 == t.block_b);
                ++at;
            }
        }
        const auto rtasks = ch::residency_tasks(plan);
        const auto trace = ch::simulate_residency(rtasks, ch::ResidencyMode::Matching);
        std::uint64_t want_n = 0;
        CHECK(chor_simulate_residency(23, 4, 3, 1, 0, nullptr, 0, nullptr, 0, &want_n) == 0 && want_n == trace.size());
        std::vector<std::uint32_t> want(want_n * 4);
        CHECK(chor_simulate_residency(23, 4, 3, 1, 0, nullptr, 0, want.data(), want_n, &want_n) == 0);
        for (std::size_t i = 0; i < trace.size(); ++i)
            CHECK(std::uint32_t(trace[i].kind) == want[4 * i] && std::uint32_t(trace[i].level) == want[4 * i + 1] &&
                  trace[i].id == want[4 * i + 2] && std::uint32_t(trace[i].prefetch) == want[4 * i + 3]);
        const auto htrace = ch::simulate_residency(ch::hashing_residency_tasks(part), ch::ResidencyMode::Hashing);
        CHECK(chor_simulate_residency(23, 4, 3, 0, 0, nullptr, 0, nullptr, 0, &want_n) == 0 && want_n == htrace.size());
        CHECK(ch::residency_slot_limit(ch::ResidencyMode::Hashing) == 2 && ch::residency_slot_limit(ch::ResidencyMode::Matching) == 3);
        CHECK(throws<std::logic_error>([&] { ch::simulate_residency(rtasks, ch::ResidencyMode::Matching, 3, 1); }));
        const ch::PairPlan guided = ch::plan_guided(part, {{3, 1}, {1, 3}, {20, 2}, {7, 6}});
        CHECK(guided.tasks.size() == 3 && guided.pair_count() == 3);
        CHECK(throws<std::invalid_argument>([&] { ch::plan_guided(part, {{3, 3}}); }));
        const auto lanes = ch::assign_workers(plan, 4);
        CHECK(lanes.size() == 4 && lanes[1][0] == 1 && lanes[1][1] == 5);
        CHECK(throws<std::invalid_argument>([&] { ch::assign_workers(plan, 0); }));
        std::uint32_t bi = 0, bpg = 0;
        CHECK(chor_auto_partition_sizing(1179664, 64ull << 30, &bi, &bpg) == 0);
        const ch::PartitionSizing sz = ch::auto_partition_sizing(1179664, 64ull << 30);
        CHECK(sz.block_images == bi && sz.blocks_per_group == bpg);
        CHECK(throws<std::invalid_argument>([] { ch::make_partition(0, 1, 1); }));
    }

    // code cache (hashing.hpp:134-157): bytes identical to the oracle's file, round trip, header probe, the
    // reference's error classes
    {
        ch::HashFamily fam = ch::build_hash_family(ch::FamilyParams{7, 70, 5, 11});
        for (int x = 0; x < 128; ++x) fam.centering[x] = 100.0 + 0.25 * x;
        fam.centering_set = true;
        const std::uint64_t fp = ch::centering_fingerprint(fam);
        std::uint64_t want_fp = 0;
        CHECK(chor_centering_fingerprint(fam.centering.data(), &want_fp) == 0 && fp == want_fp);
        ch::ImageCodes codes;
        codes.params = fam.params;
        codes.shorts.short_bits = 7;
        codes.shorts.table_count = 5;
        codes.shorts.point_count = 37;
        codes.longs.long_bits = 70;
        std::vector<std::uint64_t> words;
        for (std::uint32_t p = 0; p < 37; ++p) {
            for (std::uint32_t t = 0; t < 5; ++t) codes.shorts.values.push_back((p * 31 + t * 7) & 127);
            ch::LongCode lc;
            lc.words = {0x9e3779b97f4a7c15ull * (p + 1), (0xbf58476d1ce4e5b9ull * (p + 3)) & 0x3f};
            lc.bits = 70;
            codes.longs.codes.push_back(lc);
            words.push_back(lc.words[0]);
            words.push_back(lc.words[1]);
        }
        ch::save_code_cache(codes, fp, tmp / "c_ours.chcc");
        const chor_family_params cp = to_chor(fam.params);
        CHECK(chor_save_code_cache(&cp, fp, codes.shorts.values.data(), words.data(), 37, (tmp / "c_ref.chcc").string().c_str()) == 0);
        CHECK(slurp(tmp / "c_ours.chcc") == slurp(tmp / "c_ref.chcc"));
        ch::CodeCacheHeader hdr;
        CHECK(ch::read_code_cache_header(tmp / "c_ref.chcc", hdr) && hdr.params == fam.params && hdr.centering_fp == fp &&
              hdr.count == 37);
        CHECK(!ch::read_code_cache_header(tmp / "no_such.chcc", hdr));
        const ch::ImageCodes back = ch::load_code_cache(tmp / "c_ref.chcc", fam.params, fp);
        CHECK(back.shorts.values == codes.shorts.values && back.shorts.point_count == 37 && back.longs.codes.size() == 37);
        for (std::size_t p = 0; p < 37; ++p) CHECK(back.longs.codes[p].words == codes.longs.codes[p].words);
        CHECK(throws<std::runtime_error>([&] { ch::load_code_cache(tmp / "c_ref.chcc", fam.params, fp + 1); }));
        CHECK(throws<std::runtime_error>([&] { ch::load_code_cache(tmp / "c_ref.chcc", ch::FamilyParams{}, fp); }));
        CHECK(throws<ch::FeatureFileError>([&] { ch::load_code_cache(tmp / "no_such.chcc", fam.params, fp); }));
        std::string cut = slurp(tmp / "c_ref.chcc");
        cut.resize(cut.size() - 9);
        std::ofstream(tmp / "c_cut.chcc", std::ios::binary) << cut;
        try {
            ch::load_code_cache(tmp / "c_cut.chcc", fam.params, fp);
            CHECK(false);
        } catch (const ch::FeatureFileError& e) {
            CHECK(e.fault() == ch::FeatureFileFault::Truncated);
        }
        CHECK(throws<ch::FeatureFileError>([&] { ch::save_code_cache(codes, fp, tmp / "no_such_dir" / "c.chcc"); }));
    }

    // plan_guided: the accepted pairs (either order, duplicates collapse) in the exhaustive plan's order == the oracle's
    {
        std::vector<std::pair<std::uint32_t, std::uint32_t>> acc;
        for (std::uint32_t i = 0; i < 23; ++i)
            for (std::uint32_t d = 1; d <= 3 && i + d < 23; ++d) acc.emplace_back(i % 2 ? i + d : i, i % 2 ? i : i + d);
        acc.push_back(acc[5]);
        const auto guided = ch::plan_guided(23, 4, 3, acc);
        std::vector<std::uint32_t> want(acc.size() * 2);
        std::uint64_t n = 0;
        CHECK(chor_plan_guided(23, 4, 3, reinterpret_cast<const std::uint32_t*>(acc.data()), acc.size(), want.data(), &n, nullptr,
                               nullptr) == 0);
        CHECK(guided.size() == n && n == acc.size() - 1);
        for (std::size_t k = 0; k < guided.size(); ++k) CHECK(guided[k].first == want[2 * k] && guided[k].second == want[2 * k + 1]);
        CHECK(throws<std::invalid_argument>([] { ch::plan_guided(23, 4, 3, {{4, 4}}); }));
        CHECK(throws<std::invalid_argument>([] { ch::plan_guided(23, 4, 3, {{4, 23}}); }));
    }
}

static void device_checks(const std::filesystem::path& tmp) {
    ch::HashFamily fam = ch::build_hash_family(ch::FamilyParams{});
    std::vector<ch::FeatureSet> sets;
    for (int i = 0; i < 4; ++i) sets.push_back(make_image(100 + i, i == 3 ? 700 : 1000, 300, "img" + std::to_string(i)));

    // compute_codes before set_centering is a logic error (hashing.cpp:131-132)
    CHECK(throws<std::logic_error>([&] { ch::compute_codes(fam, sets[0]); }));
    CHECK(throws<std::invalid_argument>([&] {
        ch::HashFamily f2 = fam;
        ch::set_centering(f2, std::span<const ch::FeatureSet>{});
    }));

    // set_centering: exact integer sums / count
    ch::set_centering(fam, sets);
    std::uint64_t sums[128] = {0}, count = 0;
    for (const auto& fs : sets) CHECK(chor_centering_accumulate(fs.descriptors.front().data(), fs.size(), sums, &count) == 0);
    double want[128];
    CHECK(chor_centering_apply(sums, count, want) == 0);
    CHECK(fam.centering_set && std::memcmp(want, fam.centering.data(), sizeof(want)) == 0);
    CHECK(throws<std::invalid_argument>([&] { ch::compute_codes(fam, sets[0], 8); }));

    // compute_codes: bit-exact short and long codes, for the default and the extreme reduction orders
    std::vector<ch::ImageCodes> codes;
    std::vector<OracleCodes> ocodes;
    for (const auto& fs : sets) {
        codes.push_back(ch::compute_codes(fam, fs));
        ocodes.push_back(oracle_codes(fam, fs));
        const ch::ImageCodes& c = codes.back();
        CHECK(c.params == fam.params && c.shorts.point_count == fs.size() && c.longs.long_bits == 128);
        CHECK(c.shorts.values == ocodes.back().shorts);
        for (std::size_t p = 0; p < fs.size(); ++p)
            CHECK(c.longs.codes[p].words[0] == ocodes.back().longs[2 * p] && c.longs.codes[p].words[1] == ocodes.back().longs[2 * p + 1] &&
                  c.longs.codes[p].bits == 128);
    }
    for (int rr : {0, 7}) CHECK(ch::compute_codes(fam, sets[1], rr).shorts.values == oracle_codes(fam, sets[1], rr).shorts);

    // build_bucket_index: the reference's CSR over the non-empty codes, ascending ids inside a bucket
    {
        const ch::BucketIndex idx = ch::build_bucket_index(codes[1].shorts);
        const std::uint32_t n = std::uint32_t(sets[1].size());
        std::vector<std::uint32_t> offs(6 * 257), pts(6 * n);
        CHECK(chor_build_bucket_index(8, 6, ocodes[1].shorts.data(), n, offs.data(), pts.data()) == 0);
        CHECK(idx.tables.size() == 6 && idx.point_count == n && idx.short_bits == 8);
        for (std::uint32_t t = 0; t < 6; ++t)
            for (std::uint32_t c = 0; c < 256; ++c) {
                const auto b = idx.bucket(t, c);
                const std::uint32_t lo = offs[t * 257 + c], hi = offs[t * 257 + c + 1];
                CHECK(b.size() == hi - lo);
                for (std::uint32_t k = 0; k < b.size(); ++k) CHECK(b[k] == pts[t * n + lo + k]);
            }
    }

    // match_pair: identical MatchRecords, several configurations incl. the re-rank fallback being off
    ch::MatchConfig strict;
    strict.hamming_threshold = 128;
    ch::MatchConfig loose;
    loose.top_k = 4;
    loose.ratio = 0.9;
    loose.min_candidates_for_ratio = 3;
    for (const ch::MatchConfig& cfg : {ch::MatchConfig{}, strict, loose}) {
        const auto got = ch::match_pair(sets[0], sets[1], codes[0], codes[1], cfg);
        const auto want_rec = oracle_match(fam, cfg, sets[0], ocodes[0], sets[1], ocodes[1]);
        CHECK(!want_rec.empty() && got == want_rec);
    }
    // ragged pair (1000 x 700) both ways, and empty inputs (matcher.cpp:151)
    CHECK(ch::match_pair(sets[2], sets[3], codes[2], codes[3], {}) == oracle_match(fam, {}, sets[2], ocodes[2], sets[3], ocodes[3]));
    CHECK(ch::match_pair(sets[3], sets[2], codes[3], codes[2], {}) == oracle_match(fam, {}, sets[3], ocodes[3], sets[2], ocodes[2]));
    {
        ch::FeatureSet none;
        ch::ImageCodes cnone;
        cnone.params = fam.params;
        cnone.shorts.short_bits = 8;
        cnone.shorts.table_count = 6;
        cnone.longs.long_bits = 128;
        CHECK(ch::match_pair(none, sets[1], cnone, codes[1], {}).empty());
        CHECK(ch::match_pair(sets[1], none, codes[1], cnone, {}).empty());
    }
    // The free functions keep what they upload resident by content (DefaultContext::resident): walking a pair list with
    // match_pair the way the reference's workers do (engine.cpp:686-696) uploads every image once; a changed descriptor
    // under the same address is a different image.
    {
        auto& dc = ch::detail::default_context();
        const std::uint64_t hits0 = dc.cache_hits, miss0 = dc.cache_misses;
        for (int round = 0; round < 2; ++round)
            for (int a = 0; a < 4; ++a)
                for (int b = a + 1; b < 4; ++b)
                    CHECK(ch::match_pair(sets[a], sets[b], codes[a], codes[b], {}) == oracle_match(fam, {}, sets[a], ocodes[a], sets[b], ocodes[b]));
        CHECK(dc.cache_misses - miss0 <= 4);  // (the images of the calls above may be resident already)
        CHECK(dc.cache_hits - hits0 >= 20);
        ch::FeatureSet changed = sets[0];
        changed.descriptors[5][7] ^= 0x55;
        const std::uint64_t miss1 = dc.cache_misses;
        const auto got = ch::match_pair(changed, sets[1], codes[0], codes[1], {});
        CHECK(dc.cache_misses == miss1 + 1);
        CHECK(got == oracle_match(fam, {}, changed, ocodes[0], sets[1], ocodes[1]));
        // more images than the cache holds: the least recently used go, results stay right
        std::vector<ch::FeatureSet> many;
        for (int i = 0; i < 70; ++i) many.push_back(make_image(500 + i, 64, 20, "m" + std::to_string(i)));
        for (int i = 0; i < 70; ++i) {
            const ch::ImageCodes ci = ch::compute_codes(fam, many[i]);
            CHECK(ch::match_pair(many[i], sets[1], ci, codes[1], {}) == oracle_match(fam, {}, many[i], oracle_codes(fam, many[i]), sets[1], ocodes[1]));
        }
        CHECK(dc.cache.size() <= ch::detail::DefaultContext::kCachedImages);
    }
    // argument errors (matcher.cpp:144-148, :9-17)
    {
        ch::ImageCodes other = codes[1];
        other.params.seed = 2;
        CHECK(throws<std::invalid_argument>([&] { ch::match_pair(sets[0], sets[1], codes[0], other, {}); }));
        CHECK(throws<std::invalid_argument>([&] { ch::match_pair(sets[0], sets[3], codes[0], codes[1], {}); }));
        ch::MatchConfig bad;
        bad.top_k = 1;
        CHECK(throws<std::invalid_argument>([&] { ch::match_pair(sets[0], sets[1], codes[0], codes[1], bad); }));
        bad = {};
        bad.ratio = 1.0;
        CHECK(throws<std::invalid_argument>([&] { ch::match_pair(sets[0], sets[1], codes[0], codes[1], bad); }));
        bad = {};
        bad.hamming_threshold = 129;
        CHECK(throws<std::invalid_argument>([&] { ch::match_pair(sets[0], sets[1], codes[0], codes[1], bad); }));
        // beyond the tuned kernels (top_k > 32, short_bits > 12) the same calls take the general path: same records
        ch::MatchConfig wide;
        wide.top_k = ch::kTunedMaxTopK + 1;
        CHECK(ch::match_pair(sets[0], sets[1], codes[0], codes[1], wide) == oracle_match(fam, wide, sets[0], ocodes[0], sets[1], ocodes[1]));
        wide.top_k = 500;
        CHECK(ch::match_pair(sets[0], sets[1], codes[0], codes[1], wide) == oracle_match(fam, wide, sets[0], ocodes[0], sets[1], ocodes[1]));
        {
            ch::FamilyParams fp13;
            fp13.short_bits = ch::kTunedMaxShortBits + 1;
            ch::HashFamily fam13 = ch::build_hash_family(fp13);
            ch::set_centering(fam13, std::span<const ch::FeatureSet>(sets.data(), 2));
            const ch::ImageCodes c0 = ch::compute_codes(fam13, sets[0]), c1 = ch::compute_codes(fam13, sets[1]);
            const OracleCodes o0 = oracle_codes(fam13, sets[0], 3), o1 = oracle_codes(fam13, sets[1], 3);
            CHECK(c0.shorts.values == o0.shorts && c1.shorts.values == o1.shorts);
            const auto want13 = oracle_match(fam13, {}, sets[0], o0, sets[1], o1);
            CHECK(!want13.empty() && ch::match_pair(sets[0], sets[1], c0, c1, {}) == want13);
        }
        // match_pair_filtered (matcher.hpp:102-105) with a host callback that thins, reverses and repeats candidates:
        // the oracle side runs match_pair_filtered with the lists the same callback leaves
        {
            const ch::CandidateFilter filter = [](std::uint32_t q, std::vector<std::uint32_t>& c) {
                if (q % 4 == 0) c.clear();
                else if (q % 4 == 1) std::reverse(c.begin(), c.end());
                else if (q % 4 == 2) c.push_back(c.front());
                return true;
            };
            const auto got = ch::match_pair_filtered(sets[0], sets[1], codes[0], codes[1], {}, filter);
            std::vector<std::uint64_t> lo{0};
            std::vector<std::uint32_t> ids, one(sets[1].size());
            for (std::uint32_t q = 0; q < sets[0].size(); ++q) {
                std::uint32_t cnt = 0;
                CHECK(chor_lookup_candidates(8, 6, ocodes[0].shorts.data() + std::size_t(q) * 6, ocodes[1].shorts.data(),
                                             std::uint32_t(sets[1].size()), one.data(), &cnt) == 0);
                std::vector<std::uint32_t> c(one.begin(), one.begin() + cnt);
                if (!c.empty()) filter(q, c);
                ids.insert(ids.end(), c.begin(), c.end());
                lo.push_back(ids.size());
            }
            std::vector<ch::MatchRecord> want(sets[0].size() + 1);
            std::uint32_t count = 0;
            const chor_family_params p = to_chor(fam.params);
            const chor_match_cfg c = to_chor(ch::MatchConfig{});
            CHECK(chor_match_pair_lists(&p, &c, sets[0].descriptors.front().data(), std::uint32_t(sets[0].size()), ocodes[0].shorts.data(),
                                        ocodes[0].longs.data(), sets[1].descriptors.front().data(), std::uint32_t(sets[1].size()),
                                        ocodes[1].shorts.data(), ocodes[1].longs.data(), lo.data(), ids.data(),
                                        reinterpret_cast<chor_match_record*>(want.data()), &count, nullptr, nullptr, nullptr) == 0);
            want.resize(count);
            CHECK(!want.empty() && got == want);
            CHECK(ch::match_pair_filtered(sets[0], sets[1], codes[0], codes[1], {}, nullptr) ==
                  oracle_match(fam, {}, sets[0], ocodes[0], sets[1], ocodes[1]));
        }
        ch::FamilyParams fp9;
        fp9.table_count = ch::kDeviceMaxTables + 1;
        const ch::HashFamily fam9 = ch::build_hash_family(fp9);
        CHECK(throws<ch::UnsupportedOnDevice>([&] { ch::Matcher m9; m9.set_family(fam9); }));
    }

    // guided_match_pair (geometry.hpp:86-89): the epipolar band between lookup and ranking
    {
        const ch::FundamentalMatrix F = {0.3, -1.2, 210.0, 0.9, 0.4, -350.0, -0.002, 0.001, 1.0};
        for (double band : {1e9, 180.0, 12.0}) {
            const auto got = ch::guided_match_pair(sets[0], sets[1], codes[0], codes[1], F, {}, band);
            std::vector<ch::MatchRecord> want_rec(sets[0].size() + 1);
            std::uint32_t count = 0;
            const chor_family_params p = to_chor(fam.params);
            const chor_match_cfg c = to_chor(ch::MatchConfig{});
            CHECK(chor_guided_match_pair(&p, &c, sets[0].descriptors.front().data(), &sets[0].keypoints.front().x,
                                         std::uint32_t(sets[0].size()), ocodes[0].shorts.data(), ocodes[0].longs.data(),
                                         sets[1].descriptors.front().data(), &sets[1].keypoints.front().x,
                                         std::uint32_t(sets[1].size()), ocodes[1].shorts.data(), ocodes[1].longs.data(), F.data(),
                                         band, reinterpret_cast<chor_match_record*>(want_rec.data()), &count, nullptr, nullptr,
                                         nullptr) == 0);
            want_rec.resize(count);
            CHECK(got == want_rec);
            if (band > 1e8) CHECK(got == ch::match_pair(sets[0], sets[1], codes[0], codes[1], {}));
        }
    }

    // batch interface: upload once, centering + hash on the device, whole pair list in one call,
    // files written with the reference's names and bytes
    {
        ch::Matcher m(0);
        ch::HashFamily fam2 = ch::build_hash_family(ch::FamilyParams{});
        m.set_family(fam2);
        std::vector<std::uint32_t> ids;
        for (std::uint32_t i = 0; i < sets.size(); ++i) {
            if (i % 2 == 0) {
                m.upload(i, sets[i]);
            } else {  // the CHFT path: raw file bytes, split on the device
                ch::save_features(sets[i], tmp / "img.chft");
                const std::string blob = slurp(tmp / "img.chft");
                CHECK(m.upload_chft(i, blob.data(), blob.size()) == sets[i].size());
            }
            ids.push_back(i);
        }
        m.centering_reset();
        for (std::uint32_t i : ids) m.centering_add(i);
        CHECK(m.centering_apply() == fam.centering);
        m.centering_reset();
        m.centering_add(ids);  // the batched form: one launch, the same sums
        CHECK(m.centering_apply() == fam.centering);
        // hash build: fp32 filter + exact fixup (default) and the all-fp64 kernel give the reference's codes
        m.hash(ids);
        CHECK(m.hash_stats().filter_active == 1 && m.hash_stats().overflowed_batches == 0);
        std::vector<ch::ImageCodes> filtered;
        for (std::uint32_t i : ids) filtered.push_back(m.codes(i));
        m.set_exact_hashing(true);
        m.hash(ids);
        for (std::uint32_t i : ids) {
            const ch::ImageCodes c = m.codes(i);
            CHECK(c.shorts.values == filtered[i].shorts.values && c.shorts.values == ocodes[i].shorts);
            for (std::size_t p = 0; p < c.longs.codes.size(); ++p)
                CHECK(c.longs.codes[p].words == filtered[i].longs.codes[p].words &&
                      c.longs.codes[p].words[0] == ocodes[i].longs[2 * p] && c.longs.codes[p].words[1] == ocodes[i].longs[2 * p + 1]);
        }
        m.set_exact_hashing(false);
        m.hash(ids);
        const auto pairs = ch::plan_exhaustive(4, 2, 2);
        ch::MatchStats st{};
        const auto res = m.match_pairs(pairs, {}, &st);
        CHECK(res.size() == 6 && st.pairs == 6);
        std::uint64_t total = 0;
        for (std::size_t k = 0; k < pairs.size(); ++k) {
            const auto [a, b] = pairs[k];
            CHECK(res[k].image_i == a && res[k].image_j == b);
            CHECK(res[k].matches == oracle_match(fam, {}, sets[a], ocodes[a], sets[b], ocodes[b]));
            total += res[k].matches.size();
            const auto f = tmp / ch::pair_file_name(a, b);
            ch::save_matches(sets[a].image_id, sets[b].image_id, res[k].matches, f);
            CHECK(chor_save_matches(sets[a].image_id.c_str(), sets[b].image_id.c_str(),
                                    reinterpret_cast<const chor_match_record*>(res[k].matches.data()),
                                    std::uint32_t(res[k].matches.size()), (tmp / "ref.txt").string().c_str()) == 0);
            CHECK(slurp(f) == slurp(tmp / "ref.txt"));
        }
        CHECK(st.matches == total);
        // a truncated CHFT blob is refused with the reference's fault class and offset
        ch::save_features(sets[0], tmp / "img.chft");
        const std::string blob = slurp(tmp / "img.chft");
        try {
            m.upload_chft(99, blob.data(), blob.size() - 5);
            CHECK(false);
        } catch (const ch::FeatureFileError& e) {
            CHECK(e.fault() == ch::FeatureFileFault::Truncated && e.byte_offset() == blob.size() - 5);
        }
        CHECK(throws<std::out_of_range>([&] { m.codes(12345); }));

        // out-of-core run of the same plan from CHFT files: blocks of one image, three slots (the reference's limit),
        // the next block loading behind the current task — the same records, in plan order
        {
            std::vector<std::filesystem::path> files;
            for (std::uint32_t i = 0; i < sets.size(); ++i) {
                files.push_back(tmp / ("ooc_" + std::to_string(i) + ".chft"));
                ch::save_features(sets[i], files.back());
            }
            ch::Matcher oc(0);
            oc.set_family(fam2);
            std::vector<std::string> failures;
            CHECK(oc.centering_pass_files(files, 2, 2, &failures) == fam.centering && failures.empty());
            const ch::Partition part = ch::make_partition(std::uint32_t(sets.size()), 1, 2);
            std::vector<std::pair<std::uint32_t, std::uint32_t>> seen;
            std::vector<std::vector<ch::MatchRecord>> recs;
            const chgpu_streamed_stats ss = oc.match_plan_streamed(
                files, part, {},
                [&](std::uint32_t, std::span<const std::pair<std::uint32_t, std::uint32_t>> pr, std::span<const std::uint64_t> offs,
                    std::span<const ch::MatchRecord> rec) {
                    for (std::size_t k = 0; k < pr.size(); ++k) {
                        seen.push_back(pr[k]);
                        recs.emplace_back(rec.begin() + offs[k], rec.begin() + offs[k + 1]);
                    }
                },
                nullptr, 0, 0, 2, &failures);
            const auto plan1 = ch::plan_exhaustive(std::uint32_t(sets.size()), 1, 2);
            CHECK(failures.empty() && seen == plan1 && ss.pairs == plan1.size() && ss.max_resident_blocks <= 3);
            CHECK(ss.block_loads > sets.size() - 1 && ss.background_block_loads > 0);
            for (std::size_t k = 0; k < seen.size(); ++k)
                CHECK(recs[k] == oracle_match(fam, {}, sets[seen[k].first], ocodes[seen[k].first], sets[seen[k].second], ocodes[seen[k].second]));
            CHECK(throws<std::out_of_range>([&] { oc.codes(0); }));  // nothing stays resident
            std::filesystem::remove(files[1]);
            failures.clear();
            const chgpu_streamed_stats s2 = oc.match_plan_streamed(files, part, {}, nullptr, nullptr, 0, 0, 2, &failures);
            CHECK(failures.size() >= 1 && s2.pairs_skipped == sets.size() - 1 && s2.pairs == plan1.size() - (sets.size() - 1));
            CHECK(throws<std::invalid_argument>([&] { oc.match_plan_streamed(files, part, {}, nullptr, nullptr, 3, 1); }));
        }

        // several lanes (here: three contexts on the one GPU): replicated working set, sharded pair list,
        // partial centering sums exchanged on the host — the same records in the same order
        const int devs[3] = {0, 0, 0};
        ch::MultiGpuMatcher mg(devs);
        CHECK(mg.lane_count() == 3);
        mg.set_family(fam2);
        for (std::uint32_t i = 0; i < sets.size(); ++i) mg.upload(i, sets[i]);
        CHECK(mg.set_centering(ids) == fam.centering);
        mg.hash(ids);
        ch::MatchStats mst{};
        const auto mres = mg.match_pairs(pairs, {}, &mst);
        CHECK(mres.size() == res.size() && mst.pairs == st.pairs && mst.matches == st.matches &&
              mst.raw_candidates == st.raw_candidates && mst.distances == st.distances);
        for (std::size_t k = 0; k < res.size(); ++k)
            CHECK(mres[k].image_i == res[k].image_i && mres[k].image_j == res[k].image_j && mres[k].matches == res[k].matches);
        CHECK(throws<std::out_of_range>([&] { mg.hash(std::vector<std::uint32_t>{777}); }));  // a lane's error surfaces
    }
}

int main(int argc, char** argv) {
    const bool host_only = argc > 1 && std::string(argv[1]) == "--host";
    const std::filesystem::path tmp = std::filesystem::temp_directory_path() / ("chfacade_" + std::to_string(::getpid()));
    std::filesystem::create_directories(tmp);
    host_checks(tmp);
    if (!host_only) device_checks(tmp);
    std::filesystem::remove_all(tmp);
    std::printf("facade_test ok: %d checks (%s), oracle = %s\n", g_checks, host_only ? "host only" : "host + device", chor_name());
    return 0;
}
