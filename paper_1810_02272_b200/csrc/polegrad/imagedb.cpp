// imagedb.cpp — labelled dataset, weighted sampling and index loading
// (include/polegrad/imagedb.hpp; behaviour of the reference imagedb.cpp:12-215).
#include "polegrad/imagedb.hpp"

#include <algorithm>
#include <bit>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>

#include "polegrad/errors.hpp"

namespace polegrad::imagedb {

void Dataset::add(Entry e) {
  if (entries_.count(e.id)) throw InvalidArgument("dataset: duplicate entry id " + std::to_string(e.id));
  if (!(e.boost >= real(1))) throw InvalidArgument("dataset: boost must be >= 1, got entry id " + std::to_string(e.id));
  const std::int64_t id = e.id;
  const int label = e.label;
  entries_.emplace(id, std::move(e));
  groups_[label].push_back(id);
}

const Entry& Dataset::entry(std::int64_t id) const {
  const auto it = entries_.find(id);
  if (it == entries_.end()) throw NotFound("dataset: no entry with id " + std::to_string(id));
  return it->second;
}

void Dataset::set_boost(std::int64_t id, real boost) {
  if (!(boost >= real(1))) throw InvalidArgument("dataset: boost must be >= 1, got " + std::to_string(boost));
  const auto it = entries_.find(id);
  if (it == entries_.end()) throw NotFound("dataset: no entry with id " + std::to_string(id));
  it->second.boost = boost;
}

namespace {

// floor(u * n) clamped to the last slot (u in [0, 1))
std::size_t uniform_slot(Rng& rng, std::size_t n) {
  return std::min(static_cast<std::size_t>(rng.uniform01() * n), n - 1);
}

// One draw: uniform over `ids`, or proportional to the entries' boosts
// (first id whose running boost sum exceeds u * total).
template <class Ids, class BoostOf>
std::int64_t draw(const Ids& ids, std::size_t n, bool use_boost, Rng& rng, BoostOf boost_of) {
  if (!use_boost) return ids[uniform_slot(rng, n)];
  real total = 0;
  for (std::size_t i = 0; i < n; ++i) total += boost_of(ids[i]);
  const real target = static_cast<real>(rng.uniform01()) * total;
  real run = 0;
  for (std::size_t i = 0; i < n; ++i) {
    run += boost_of(ids[i]);
    if (target < run) return ids[i];
  }
  return ids[n - 1];
}

}  // namespace

const Entry& Dataset::sample(SampleMethod method, bool use_boost, Rng& rng) const {
  if (entries_.empty()) throw InvalidState("dataset: cannot sample from an empty dataset");
  const auto boost_of = [&](std::int64_t id) { return entries_.at(id).boost; };
  if (method == SampleMethod::kUniform) {
    std::vector<std::int64_t> all;
    all.reserve(entries_.size());
    for (const auto& kv : entries_) all.push_back(kv.first);
    return entries_.at(draw(all, all.size(), use_boost, rng, boost_of));
  }
  auto group = groups_.begin();
  std::advance(group, static_cast<std::ptrdiff_t>(uniform_slot(rng, groups_.size())));
  return entries_.at(draw(group->second, group->second.size(), use_boost, rng, boost_of));
}

namespace {

std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r\n");
  if (b == std::string::npos) return {};
  const auto e = s.find_last_not_of(" \t\r\n");
  return s.substr(b, e - b + 1);
}

template <class T>
T parse_number(const std::string& field, int line, const char* what) {
  const std::string t = trim(field);
  try {
    std::size_t used = 0;
    T v;
    if constexpr (std::is_same_v<T, double>) v = std::stod(t, &used);
    else if constexpr (std::is_same_v<T, long long>) v = std::stoll(t, &used);
    else v = std::stoi(t, &used);
    if (used != t.size() || t.empty()) throw std::invalid_argument("trailing");
    return v;
  } catch (const std::exception&) {
    throw LoadError(line, std::string(what) + ": cannot parse '" + t + "'");
  }
}

std::vector<real> read_tensor(const std::filesystem::path& path, std::array<int, 3>& dims) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw InvalidState("cannot open " + path.string());
  const std::vector<unsigned char> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  auto u32 = [&](std::size_t at) {
    std::uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= std::uint32_t(bytes[at + i]) << (8 * i);
    return v;
  };
  if (bytes.size() < 12) throw InvalidState("tensor file " + path.string() + " is truncated");
  std::size_t count = 1;
  for (int i = 0; i < 3; ++i) {
    const std::uint32_t d = u32(std::size_t(i) * 4);
    if (d == 0) throw InvalidState("tensor file " + path.string() + " has a zero dimension");
    dims[i] = int(d);
    count *= d;
  }
  if (bytes.size() != 12 + 4 * count)
    throw InvalidState("tensor file " + path.string() + " holds " + std::to_string((bytes.size() - 12) / 4) +
                       " values, header says " + std::to_string(count));
  std::vector<real> values(count);
  for (std::size_t i = 0; i < count; ++i) values[i] = static_cast<real>(std::bit_cast<float>(u32(12 + 4 * i)));
  return values;
}

}  // namespace

Dataset load(const std::filesystem::path& index_path) {
  std::ifstream in(index_path);
  if (!in) throw LoadError(0, "cannot open index " + index_path.string());
  const std::filesystem::path dir = index_path.parent_path();
  Dataset ds;
  std::string raw;
  int line = 0;
  while (std::getline(in, raw)) {
    ++line;
    const std::string text = trim(raw);
    if (text.empty() || text[0] == '#') continue;
    std::vector<std::string> f;
    std::size_t start = 0;
    for (;;) {
      const auto comma = text.find(',', start);
      f.push_back(text.substr(start, comma == std::string::npos ? std::string::npos : comma - start));
      if (comma == std::string::npos) break;
      start = comma + 1;
    }
    if (f.size() != 4) throw LoadError(line, "expected id,label,boost,relative_path, got " + std::to_string(f.size()) + " fields");
    Entry e;
    e.id = parse_number<long long>(f[0], line, "id");
    e.label = parse_number<int>(f[1], line, "label");
    e.boost = static_cast<real>(parse_number<double>(f[2], line, "boost"));
    if (!(e.boost >= real(1))) throw LoadError(line, "boost must be >= 1");
    const std::string rel = trim(f[3]);
    if (rel.empty()) throw LoadError(line, "empty tensor path");
    try {
      e.tensor = read_tensor(dir / rel, e.dims);
    } catch (const Error& err) {
      throw LoadError(line, err.what());
    }
    try {
      ds.add(std::move(e));
    } catch (const Error& err) {
      throw LoadError(line, err.what());
    }
  }
  return ds;
}

}  // namespace polegrad::imagedb
