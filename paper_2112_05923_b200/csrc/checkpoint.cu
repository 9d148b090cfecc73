// checkpoint.cu -- the PODRCKPT v1 checkpoint format (checkpoint.hpp:16-317) for agents whose
// weights live on the device: the leaderboard's elites are written to / read from disk without a
// host-side AgentArtifact.  Host code (byte-level IO); the device side is one download / upload of
// the flat parameter blob and the Adam moments.
//
// Format (checkpoint.hpp:18-31), integers little-endian:
//   "PODRCKPT" | u32 version = 1 | u32 tensor count |
//   per tensor: u32 name length, name bytes, u32 rank, rank x u64 dims, prod(dims) x f64 |
//   u32 CRC-32 (IEEE, reflected 0xEDB88320) over every preceding byte.
// Tensor table (artifact_to_tensors checkpoint.hpp:212-245): actor/layer{i}/weight [in][out],
// actor/layer{i}/bias, actor/log_std, critic/layer{i}/..., optim/m, optim/v,
// optim/scalars = (t, beta1, beta2, eps, lr), lineage = (parent_pod, seed >> 32, seed & 2^32-1),
// algo_tag (one f64 per byte), optional meta = (wall_seconds, env_steps, score).
// fp32 device values widen to f64 exactly; a reference checkpoint's f64 values round to fp32 once
// on load.
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "prb_internal.h"

using namespace prb;

namespace {

uint32_t crc32_ieee(const uint8_t* data, size_t len) {  // checkpoint.hpp:36-50
  static const auto table = [] {
    std::vector<uint32_t> t(256);
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
      t[i] = c;
    }
    return t;
  }();
  uint32_t crc = 0xFFFFFFFFu;
  for (size_t i = 0; i < len; ++i) crc = table[(crc ^ data[i]) & 0xFFu] ^ (crc >> 8);
  return crc ^ 0xFFFFFFFFu;
}

struct Tensor {
  std::string name;
  std::vector<uint64_t> dims;
  std::vector<double> values;
};

void put_u32(std::vector<uint8_t>& o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back((uint8_t)(v >> (8 * i)));
}
void put_u64(std::vector<uint8_t>& o, uint64_t v) {
  for (int i = 0; i < 8; ++i) o.push_back((uint8_t)(v >> (8 * i)));
}

std::vector<uint8_t> encode(const std::vector<Tensor>& ts) {  // encode_checkpoint checkpoint.hpp:122-143
  std::vector<uint8_t> o = {'P', 'O', 'D', 'R', 'C', 'K', 'P', 'T'};
  put_u32(o, 1);
  put_u32(o, (uint32_t)ts.size());
  for (const Tensor& t : ts) {
    put_u32(o, (uint32_t)t.name.size());
    o.insert(o.end(), t.name.begin(), t.name.end());
    put_u32(o, (uint32_t)t.dims.size());
    uint64_t n = 1;
    for (uint64_t d : t.dims) {
      put_u64(o, d);
      n *= d;
    }
    PRB_REQUIRE(n == t.values.size(), PRB_ERR_USAGE, "encode_checkpoint: tensor '" + t.name + "' dims product " +
                                                         std::to_string(n) + " vs " +
                                                         std::to_string(t.values.size()) + " values");
    for (double v : t.values) {
      uint64_t b;
      std::memcpy(&b, &v, 8);
      put_u64(o, b);
    }
  }
  put_u32(o, crc32_ieee(o.data(), o.size()));
  return o;
}

struct Reader {
  const uint8_t* d;
  size_t n, pos = 0;
  void need(size_t k) const {
    if (pos + k > n) fail(PRB_ERR_CORRUPTION, "checkpoint: truncated record");
  }
  uint32_t u32() {
    need(4);
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= (uint32_t)d[pos + i] << (8 * i);
    pos += 4;
    return v;
  }
  uint64_t u64() {
    need(8);
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)d[pos + i] << (8 * i);
    pos += 8;
    return v;
  }
  std::string bytes(size_t k) {
    need(k);
    std::string s(reinterpret_cast<const char*>(d + pos), k);
    pos += k;
    return s;
  }
};

std::vector<Tensor> decode(const uint8_t* bytes, size_t size) {  // decode_checkpoint checkpoint.hpp:145-196
  PRB_REQUIRE(size >= 8 + 12, PRB_ERR_CORRUPTION, "checkpoint: file too short");
  const size_t body = size - 4;
  uint32_t stored = 0;
  for (int i = 0; i < 4; ++i) stored |= (uint32_t)bytes[body + i] << (8 * i);
  PRB_REQUIRE(crc32_ieee(bytes, body) == stored, PRB_ERR_CORRUPTION, "checkpoint: CRC mismatch");
  Reader r{bytes, body};
  PRB_REQUIRE(r.bytes(8) == "PODRCKPT", PRB_ERR_FORMAT, "checkpoint: bad magic, not a checkpoint file");
  const uint32_t version = r.u32();
  PRB_REQUIRE(version != 0 && version <= 1, PRB_ERR_VERSION,
              "checkpoint: version " + std::to_string(version) + " not supported (max 1)");
  const uint32_t count = r.u32();
  std::vector<Tensor> ts;
  std::map<std::string, bool> seen;
  for (uint32_t i = 0; i < count; ++i) {
    Tensor t;
    t.name = r.bytes(r.u32());
    PRB_REQUIRE(!seen.count(t.name), PRB_ERR_CORRUPTION, "checkpoint: duplicate tensor '" + t.name + "'");
    seen[t.name] = true;
    const uint32_t rank = r.u32();
    uint64_t n = 1;
    for (uint32_t k = 0; k < rank; ++k) {
      t.dims.push_back(r.u64());
      n *= t.dims.back();
    }
    PRB_REQUIRE(n <= (1ULL << 32), PRB_ERR_CORRUPTION, "checkpoint: implausible tensor size");
    r.need(n * 8);
    t.values.resize(n);
    for (uint64_t k = 0; k < n; ++k) {
      const uint64_t b = r.u64();
      std::memcpy(&t.values[k], &b, 8);
    }
    ts.push_back(std::move(t));
  }
  PRB_REQUIRE(r.pos == body, PRB_ERR_CORRUPTION, "checkpoint: trailing bytes after tensor table");
  return ts;
}

struct Shape {
  std::vector<size_t> ad, cd;  // actor / critic dims
};

Shape shape_of(size_t S, size_t A, const size_t* hidden, int nh) {
  Shape sh;
  sh.ad.push_back(S);
  sh.cd.push_back(S);
  for (int i = 0; i < nh; ++i) {
    sh.ad.push_back(hidden[i]);
    sh.cd.push_back(hidden[i]);
  }
  sh.ad.push_back(A);
  sh.cd.push_back(1);
  return sh;
}

size_t param_count(const Shape& sh) {
  size_t P = 0;
  for (size_t i = 0; i + 1 < sh.ad.size(); ++i) P += (sh.ad[i] + 1) * sh.ad[i + 1];
  P += sh.ad.back();
  for (size_t i = 0; i + 1 < sh.cd.size(); ++i) P += (sh.cd[i] + 1) * sh.cd[i + 1];
  return P;
}

// artifact_to_tensors checkpoint.hpp:212-245 over the canonical flat layout
std::vector<Tensor> to_tensors(const Shape& sh, const double* flat, const double* m, const double* v, int64_t t,
                               const double* hyper, int64_t parent, uint64_t mseed, const char* tag,
                               const double* meta) {
  std::vector<Tensor> ts;
  size_t off = 0;
  auto add_mlp = [&](const std::string& prefix, const std::vector<size_t>& d) {
    for (size_t i = 0; i + 1 < d.size(); ++i) {
      const size_t in = d[i], out = d[i + 1];
      ts.push_back({prefix + "/layer" + std::to_string(i) + "/weight", {in, out},
                    std::vector<double>(flat + off, flat + off + in * out)});
      off += in * out;
      ts.push_back({prefix + "/layer" + std::to_string(i) + "/bias", {out}, std::vector<double>(flat + off, flat + off + out)});
      off += out;
    }
  };
  add_mlp("actor", sh.ad);
  const size_t A = sh.ad.back();
  ts.push_back({"actor/log_std", {A}, std::vector<double>(flat + off, flat + off + A)});
  off += A;
  add_mlp("critic", sh.cd);
  const size_t P = off;
  ts.push_back({"optim/m", {P}, std::vector<double>(m, m + P)});
  ts.push_back({"optim/v", {P}, std::vector<double>(v, v + P)});
  ts.push_back({"optim/scalars", {5}, {(double)t, hyper[0], hyper[1], hyper[2], hyper[3]}});
  ts.push_back({"lineage", {3}, {(double)parent, (double)(mseed >> 32), (double)(mseed & 0xFFFFFFFFULL)}});
  std::vector<double> tb;
  for (const char* c = tag ? tag : "ppo"; *c; ++c) tb.push_back((double)(unsigned char)*c);
  ts.push_back({"algo_tag", {tb.size()}, tb});
  if (meta) ts.push_back({"meta", {3}, {meta[0], meta[1], meta[2]}});
  return ts;
}

// artifact_from_tensors checkpoint.hpp:247-303 into the flat layout of `sh` (the receiving agent's
// shapes: a file of other shapes is a DimensionError)
void from_tensors(const std::vector<Tensor>& ts, const Shape& sh, double* flat, double* m, double* v, int64_t* t,
                  double* hyper, int64_t* parent, uint64_t* mseed, std::string* tag, double* meta, int* has_meta) {
  std::map<std::string, const Tensor*> by;
  for (const Tensor& x : ts) by[x.name] = &x;
  auto need = [&](const std::string& name) -> const Tensor& {
    auto it = by.find(name);
    if (it == by.end()) fail(PRB_ERR_CORRUPTION, "checkpoint: missing tensor '" + name + "'");
    return *it->second;
  };
  size_t off = 0;
  auto read_mlp = [&](const std::string& prefix, const std::vector<size_t>& d) {
    size_t nl = 0;
    while (by.count(prefix + "/layer" + std::to_string(nl) + "/weight")) ++nl;
    PRB_REQUIRE(nl > 0, PRB_ERR_CORRUPTION, "checkpoint: no layers under '" + prefix + "'");
    PRB_REQUIRE(nl + 1 == d.size(), PRB_ERR_DIMENSION,
                "checkpoint: '" + prefix + "' has " + std::to_string(nl) + " layers, the agent " +
                    std::to_string(d.size() - 1));
    for (size_t i = 0; i < nl; ++i) {
      const std::string wn = prefix + "/layer" + std::to_string(i) + "/weight";
      const Tensor& w = need(wn);
      const Tensor& b = need(prefix + "/layer" + std::to_string(i) + "/bias");
      PRB_REQUIRE(w.dims.size() == 2 && b.dims.size() == 1 && b.dims[0] == w.dims[1], PRB_ERR_CORRUPTION,
                  "checkpoint: bad shapes for '" + wn + "'");
      PRB_REQUIRE(w.dims[0] == d[i] && w.dims[1] == d[i + 1], PRB_ERR_DIMENSION,
                  "checkpoint: '" + wn + "' is [" + std::to_string(w.dims[0]) + " x " + std::to_string(w.dims[1]) +
                      "], the agent's [" + std::to_string(d[i]) + " x " + std::to_string(d[i + 1]) + "]");
      if (flat) std::memcpy(flat + off, w.values.data(), w.values.size() * 8);
      off += w.values.size();
      if (flat) std::memcpy(flat + off, b.values.data(), b.values.size() * 8);
      off += b.values.size();
    }
  };
  read_mlp("actor", sh.ad);
  const Tensor& ls = need("actor/log_std");
  PRB_REQUIRE(ls.values.size() == sh.ad.back(), PRB_ERR_DIMENSION, "checkpoint: actor/log_std size mismatch");
  if (flat) std::memcpy(flat + off, ls.values.data(), ls.values.size() * 8);
  off += ls.values.size();
  read_mlp("critic", sh.cd);
  const size_t P = off;
  const Tensor& tm = need("optim/m");
  const Tensor& tv = need("optim/v");
  PRB_REQUIRE(tm.values.size() == P && tv.values.size() == P, PRB_ERR_CORRUPTION,
              "checkpoint: optimizer state size mismatch");
  if (m) std::memcpy(m, tm.values.data(), P * 8);
  if (v) std::memcpy(v, tv.values.data(), P * 8);
  const Tensor& sc = need("optim/scalars");
  PRB_REQUIRE(sc.values.size() == 5, PRB_ERR_CORRUPTION, "checkpoint: bad optim/scalars");
  if (t) *t = (int64_t)sc.values[0];
  if (hyper)
    for (int i = 0; i < 4; ++i) hyper[i] = sc.values[1 + i];
  const Tensor& lin = need("lineage");
  PRB_REQUIRE(lin.values.size() == 3, PRB_ERR_CORRUPTION, "checkpoint: bad lineage");
  if (parent) *parent = (int64_t)lin.values[0];
  if (mseed) *mseed = ((uint64_t)lin.values[1] << 32) | (uint64_t)lin.values[2];
  if (tag) {
    tag->clear();
    for (double c : need("algo_tag").values) tag->push_back((char)c);
  }
  if (has_meta) *has_meta = 0;
  if (by.count("meta")) {
    const Tensor& mt = need("meta");
    if (mt.values.size() == 3) {
      if (meta)
        for (int i = 0; i < 3; ++i) meta[i] = mt.values[i];
      if (has_meta) *has_meta = 1;
    }
  }
}

std::vector<uint8_t> read_file(const char* path) {
  FILE* f = fopen(path, "rb");
  PRB_REQUIRE(f, PRB_ERR_USAGE, std::string("load_checkpoint: cannot open '") + path + "'");
  std::vector<uint8_t> b;
  uint8_t buf[65536];
  size_t k;
  while ((k = fread(buf, 1, sizeof(buf), f)) > 0) b.insert(b.end(), buf, buf + k);
  fclose(f);
  return b;
}

void write_file(const char* path, const std::vector<uint8_t>& b) {
  FILE* f = fopen(path, "wb");
  PRB_REQUIRE(f, PRB_ERR_USAGE, std::string("save_checkpoint: cannot open '") + path + "' for writing");
  const size_t k = fwrite(b.data(), 1, b.size(), f);
  const int rc = fclose(f);
  PRB_REQUIRE(k == b.size() && rc == 0, PRB_ERR_USAGE, std::string("save_checkpoint: write failed for '") + path + "'");
}

void copy_tag(const std::string& s, char* out, size_t cap) {
  if (!out || cap == 0) return;
  const size_t n = std::min(s.size(), cap - 1);
  std::memcpy(out, s.data(), n);
  out[n] = 0;
}

// the agent's state on the host, in f64 (the fp32 device values widen exactly)
void agent_state(prb_agent a, std::vector<double>& flat, std::vector<double>& m, std::vector<double>& v,
                 int64_t& t, double* hyper) {
  flat.resize(a->P);
  m.resize(a->P);
  v.resize(a->P);
  int rc = prb_agent_get_host(a, flat.data(), m.data(), v.data(), &t);
  if (rc) fail(rc, prb_last_error());
  hyper[0] = a->beta1;
  hyper[1] = a->beta2;
  hyper[2] = a->eps;
  hyper[3] = a->lr;
}

Shape agent_shape(prb_agent a) {
  Shape sh;
  sh.ad = a->adims;
  sh.cd = a->cdims;
  return sh;
}

void set_agent(prb_agent a, const std::vector<Tensor>& ts, int64_t* parent, uint64_t* mseed, char* tag, size_t tag_cap,
               double* meta, int* has_meta) {
  const Shape sh = agent_shape(a);
  std::vector<double> flat(a->P), m(a->P), v(a->P);
  int64_t t = 0;
  double hyper[4];
  std::string s;
  from_tensors(ts, sh, flat.data(), m.data(), v.data(), &t, hyper, parent, mseed, &s, meta, has_meta);
  int rc = prb_agent_set_host(a, flat.data(), m.data(), v.data(), t, hyper[3]);
  if (rc) fail(rc, prb_last_error());
  a->beta1 = hyper[0];
  a->beta2 = hyper[1];
  a->eps = hyper[2];
  copy_tag(s, tag, tag_cap);
}

}  // namespace

extern "C" {

int prb_checkpoint_encode_host(size_t S, size_t A, const size_t* hidden, int nh, const double* flat, const double* m,
                               const double* v, int64_t t, const double* hyper, int64_t parent_pod,
                               uint64_t mutation_seed, const char* algo_tag, const double* meta, uint8_t* out,
                               size_t capacity, size_t* size) {
  return guard([&] {
    PRB_REQUIRE(flat && m && v && hyper && size && (hidden || nh == 0), PRB_ERR_USAGE,
                "prb_checkpoint_encode_host: NULL argument");
    const std::vector<uint8_t> b = encode(
        to_tensors(shape_of(S, A, hidden, nh), flat, m, v, t, hyper, parent_pod, mutation_seed, algo_tag, meta));
    *size = b.size();
    if (out) {
      PRB_REQUIRE(capacity >= b.size(), PRB_ERR_USAGE, "prb_checkpoint_encode_host: output buffer too small");
      std::memcpy(out, b.data(), b.size());
    }
  });
}

int prb_checkpoint_decode_host(const uint8_t* bytes, size_t size, size_t S, size_t A, const size_t* hidden, int nh,
                               double* flat, double* m, double* v, int64_t* t, double* hyper, int64_t* parent_pod,
                               uint64_t* mutation_seed, char* algo_tag, size_t tag_capacity, double* meta,
                               int* has_meta) {
  return guard([&] {
    PRB_REQUIRE(bytes && (hidden || nh == 0), PRB_ERR_USAGE, "prb_checkpoint_decode_host: NULL argument");
    std::string s;
    from_tensors(decode(bytes, size), shape_of(S, A, hidden, nh), flat, m, v, t, hyper, parent_pod, mutation_seed,
                 &s, meta, has_meta);
    copy_tag(s, algo_tag, tag_capacity);
  });
}

int prb_checkpoint_encode(prb_agent a, int64_t parent_pod, uint64_t mutation_seed, const char* algo_tag,
                          const double* meta, uint8_t* out, size_t capacity, size_t* size) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && size, PRB_ERR_USAGE, "prb_checkpoint_encode: NULL argument");
    std::vector<double> flat, m, v;
    int64_t t = 0;
    double hyper[4];
    agent_state(a, flat, m, v, t, hyper);
    const std::vector<uint8_t> b = encode(to_tensors(agent_shape(a), flat.data(), m.data(), v.data(), t, hyper,
                                                     parent_pod, mutation_seed, algo_tag, meta));
    *size = b.size();
    if (out) {
      PRB_REQUIRE(capacity >= b.size(), PRB_ERR_USAGE, "prb_checkpoint_encode: output buffer too small");
      std::memcpy(out, b.data(), b.size());
    }
  });
}

int prb_checkpoint_decode(prb_agent a, const uint8_t* bytes, size_t size, int64_t* parent_pod, uint64_t* mutation_seed,
                          char* algo_tag, size_t tag_capacity, double* meta, int* has_meta) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && bytes, PRB_ERR_USAGE, "prb_checkpoint_decode: NULL argument");
    set_agent(a, decode(bytes, size), parent_pod, mutation_seed, algo_tag, tag_capacity, meta, has_meta);
  });
}

int prb_checkpoint_save(prb_agent a, const char* path, int64_t parent_pod, uint64_t mutation_seed,
                        const char* algo_tag, const double* meta) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && path, PRB_ERR_USAGE, "save_checkpoint: NULL argument");
    std::vector<double> flat, m, v;
    int64_t t = 0;
    double hyper[4];
    agent_state(a, flat, m, v, t, hyper);
    write_file(path, encode(to_tensors(agent_shape(a), flat.data(), m.data(), v.data(), t, hyper, parent_pod,
                                       mutation_seed, algo_tag, meta)));
  });
}

int prb_checkpoint_load(prb_agent a, const char* path, int64_t* parent_pod, uint64_t* mutation_seed, char* algo_tag,
                        size_t tag_capacity, double* meta, int* has_meta) {
  return guard([&] {
    DeviceScope dev_(a ? a->ctx : nullptr);
    PRB_REQUIRE(a && path, PRB_ERR_USAGE, "load_checkpoint: NULL argument");
    const std::vector<uint8_t> b = read_file(path);
    set_agent(a, decode(b.data(), b.size()), parent_pod, mutation_seed, algo_tag, tag_capacity, meta, has_meta);
  });
}

}  // extern "C"
