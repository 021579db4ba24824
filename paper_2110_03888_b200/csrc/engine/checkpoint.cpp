// Checkpoint container for the Pseudo -> Real hand-off (
// SPEC.md:260-264 [TYPE] Checkpoint, :276-284 [OP] delink, :320 file format).
//
// Layout (all integers little-endian, floats IEEE-754 binary32):
//   bytes 0..7    magic "P2RCKPT\0"
//   bytes 8..11   u32 format version (1)
//   bytes 12..15  u32 manifest length M
//   bytes 16..    UTF-8 manifest (M bytes), then zero padding to a 64-byte boundary
//   payload       fp32 buffers, each 64-byte aligned, at the offsets the manifest lists
// Manifest lines (floats as C hex-floats, so they round-trip exactly):
//   p2r-checkpoint 1
//   config d_model .. d_ff .. n_layers_graph .. n_layers_params .. n_heads .. vocab_size ..
//          seq_len .. n_experts .. n_prototypes .. n_shards .. capacity_factor <hex>
//   ep <world> <rank>
//   stage PSEUDO|REAL / global_step / samples_consumed / wall_time_s <hex> / rng_state / last_eval_step
//   adamw <0|1> <b1> <b2> <eps> <wd> <step_count>
//   buffers <count>
//   buffer <name> f32 <ndim> <dims...> <offset:16 hex digits> <bytes:16 hex digits>
//   end
// Buffer names: param/<reference name>, adam_m/<name>, adam_v/<name>, where the
// reference names are the layer-indexed for_each_param names (model.cpp:188-198).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "p2r/engine.hpp"
#include "offload_state.hpp"

namespace p2r {
namespace {

constexpr char kMagic[8] = {'P', '2', 'R', 'C', 'K', 'P', 'T', '\0'};
constexpr std::uint32_t kVersion = 1;

std::string hexf(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%a", v);
  return b;
}
std::string hex16(std::uint64_t v) {
  char b[32];
  std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(v));
  return b;
}
std::uint64_t align64(std::uint64_t x) { return (x + 63) & ~static_cast<std::uint64_t>(63); }

void put_u32(std::ostream& o, std::uint32_t v) {
  const unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                              static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
  o.write(reinterpret_cast<const char*>(b), 4);
}
std::uint32_t get_u32(const unsigned char* b) {
  return static_cast<std::uint32_t>(b[0]) | (static_cast<std::uint32_t>(b[1]) << 8) |
         (static_cast<std::uint32_t>(b[2]) << 16) | (static_cast<std::uint32_t>(b[3]) << 24);
}
bool host_little_endian() {
  const std::uint32_t one = 1;
  unsigned char c;
  std::memcpy(&c, &one, 1);
  return c == 1;
}

struct BufferEntry {
  std::string name;
  std::vector<int> shape;
  std::uint64_t offset = 0, bytes = 0;
};

struct Manifest {
  ModelConfig cfg;
  int ep_world = 1, ep_rank = 0;
  StageState st;
  bool adamw = false;
  float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f, wd = 0.01f;
  std::int64_t step_count = 0;
  std::vector<BufferEntry> buffers;
};

std::string config_line(const ModelConfig& c) {
  std::ostringstream o;
  o << "config d_model " << c.d_model << " d_ff " << c.d_ff << " n_layers_graph " << c.n_layers_graph
    << " n_layers_params " << c.n_layers_params << " n_heads " << c.n_heads << " vocab_size " << c.vocab_size
    << " seq_len " << c.seq_len << " n_experts " << c.moe.n_experts << " n_prototypes " << c.moe.n_prototypes
    << " n_shards " << c.moe.n_shards << " capacity_factor " << hexf(c.moe.capacity_factor);
  return o.str();
}

Manifest read_manifest(std::ifstream& f, const std::string& path) {
  if (!f) throw std::runtime_error("checkpoint: cannot open " + path);
  unsigned char head[16];
  f.read(reinterpret_cast<char*>(head), 16);
  if (f.gcount() != 16 || std::memcmp(head, kMagic, 8) != 0)
    throw std::runtime_error("checkpoint: not a p2r checkpoint: " + path);
  const std::uint32_t version = get_u32(head + 8), mlen = get_u32(head + 12);
  if (version != kVersion) throw std::runtime_error("checkpoint: unsupported format version " + std::to_string(version));
  std::string text(mlen, '\0');
  f.read(&text[0], mlen);
  if (static_cast<std::uint32_t>(f.gcount()) != mlen) throw std::runtime_error("checkpoint: truncated manifest");
  Manifest m;
  std::istringstream in(text);
  std::string line;
  bool ended = false, magic_line = false;
  while (std::getline(in, line)) {
    std::istringstream l(line);
    std::string key;
    l >> key;
    if (key == "p2r-checkpoint") {
      magic_line = true;
    } else if (key == "config") {
      std::map<std::string, std::string> kv;
      std::string k, v;
      while (l >> k >> v) kv[k] = v;
      auto gi = [&](const char* n) {
        auto it = kv.find(n);
        if (it == kv.end()) throw std::runtime_error(std::string("checkpoint: config lacks ") + n);
        return std::atoi(it->second.c_str());
      };
      m.cfg.d_model = gi("d_model");
      m.cfg.d_ff = gi("d_ff");
      m.cfg.n_layers_graph = gi("n_layers_graph");
      m.cfg.n_layers_params = gi("n_layers_params");
      m.cfg.n_heads = gi("n_heads");
      m.cfg.vocab_size = gi("vocab_size");
      m.cfg.seq_len = gi("seq_len");
      m.cfg.moe.n_experts = gi("n_experts");
      m.cfg.moe.n_prototypes = gi("n_prototypes");
      m.cfg.moe.n_shards = gi("n_shards");
      auto it = kv.find("capacity_factor");
      if (it == kv.end()) throw std::runtime_error("checkpoint: config lacks capacity_factor");
      m.cfg.moe.capacity_factor = static_cast<float>(std::strtod(it->second.c_str(), nullptr));
    } else if (key == "ep") {
      l >> m.ep_world >> m.ep_rank;
    } else if (key == "stage") {
      std::string v;
      l >> v;
      if (v != "PSEUDO" && v != "REAL") throw std::runtime_error("checkpoint: bad stage " + v);
      m.st.stage = v == "REAL" ? 1 : 0;
    } else if (key == "global_step") {
      l >> m.st.global_step;
    } else if (key == "samples_consumed") {
      l >> m.st.samples_consumed;
    } else if (key == "wall_time_s") {
      std::string v;
      l >> v;
      m.st.wall_time_s = std::strtod(v.c_str(), nullptr);
    } else if (key == "rng_state") {
      l >> m.st.rng_state;
    } else if (key == "last_eval_step") {
      l >> m.st.last_eval_step;
    } else if (key == "adamw") {
      int on = 0;
      std::string b1, b2, eps, wd;
      l >> on >> b1 >> b2 >> eps >> wd >> m.step_count;
      m.adamw = on != 0;
      m.b1 = static_cast<float>(std::strtod(b1.c_str(), nullptr));
      m.b2 = static_cast<float>(std::strtod(b2.c_str(), nullptr));
      m.eps = static_cast<float>(std::strtod(eps.c_str(), nullptr));
      m.wd = static_cast<float>(std::strtod(wd.c_str(), nullptr));
    } else if (key == "buffer") {
      BufferEntry e;
      std::string dtype, off, bytes;
      int nd = 0;
      l >> e.name >> dtype >> nd;
      if (dtype != "f32") throw std::runtime_error("checkpoint: unsupported dtype " + dtype);
      e.shape.resize(static_cast<std::size_t>(nd));
      for (int& d : e.shape) l >> d;
      l >> off >> bytes;
      e.offset = std::strtoull(off.c_str(), nullptr, 16);
      e.bytes = std::strtoull(bytes.c_str(), nullptr, 16);
      if (!l) throw std::runtime_error("checkpoint: malformed buffer line");
      m.buffers.push_back(std::move(e));
    } else if (key == "end") {
      ended = true;
    }
  }
  if (!magic_line || !ended) throw std::runtime_error("checkpoint: malformed manifest");
  return m;
}

// Header of a container being written: everything but the buffers.
struct Header {
  ModelConfig cfg;
  int ep_world = 1, ep_rank = 0;
  StageState st;
  bool adamw = false;
  float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f, wd = 0.01f;
  std::int64_t step_count = 0;
};

// Write a container: `fill(b, dst)` produces buffer b's fp32 payload.
template <typename Fill>
void write_container(const std::string& path, const Header& h, std::vector<BufferEntry> bufs, Fill&& fill) {
  if (!host_little_endian()) throw std::runtime_error("checkpoint: big-endian hosts are not supported");
  // fixed-width offsets: the manifest length does not depend on their values
  auto manifest = [&]() {
    std::ostringstream m;
    m << "p2r-checkpoint 1\n" << config_line(h.cfg) << "\n";
    m << "ep " << h.ep_world << " " << h.ep_rank << "\n";
    m << "stage " << (h.st.stage ? "REAL" : "PSEUDO") << "\n";
    m << "global_step " << h.st.global_step << "\n";
    m << "samples_consumed " << h.st.samples_consumed << "\n";
    m << "wall_time_s " << hexf(h.st.wall_time_s) << "\n";
    m << "rng_state " << h.st.rng_state << "\n";
    m << "last_eval_step " << h.st.last_eval_step << "\n";
    m << "adamw " << (h.adamw ? 1 : 0) << " " << hexf(h.b1) << " " << hexf(h.b2) << " " << hexf(h.eps) << " "
      << hexf(h.wd) << " " << h.step_count << "\n";
    m << "buffers " << bufs.size() << "\n";
    for (const BufferEntry& e : bufs) {
      m << "buffer " << e.name << " f32 " << e.shape.size();
      for (int d : e.shape) m << " " << d;
      m << " " << hex16(e.offset) << " " << hex16(e.bytes) << "\n";
    }
    m << "end\n";
    return m.str();
  };
  std::string text = manifest();
  std::uint64_t off = align64(16 + text.size());
  for (BufferEntry& e : bufs) {
    e.offset = off;
    off = align64(off + e.bytes);
  }
  text = manifest();
  // written to a temporary and renamed over the target once complete, so an
  // interrupted save never destroys the previous snapshot
  const std::string tmp = path + ".tmp";
  std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
  if (!f) throw std::runtime_error("checkpoint: cannot create " + path);
  f.write(kMagic, 8);
  put_u32(f, kVersion);
  put_u32(f, static_cast<std::uint32_t>(text.size()));
  f.write(text.data(), static_cast<std::streamsize>(text.size()));
  std::uint64_t pos = 16 + text.size();
  std::vector<float> host;
  static const char zeros[64] = {};
  for (std::size_t b = 0; b < bufs.size(); ++b) {
    f.write(zeros, static_cast<std::streamsize>(bufs[b].offset - pos));
    host.resize(bufs[b].bytes / 4);
    fill(b, host.data());
    f.write(reinterpret_cast<const char*>(host.data()), static_cast<std::streamsize>(bufs[b].bytes));
    pos = bufs[b].offset + bufs[b].bytes;
  }
  f.close();
  if (!f) {
    std::remove(tmp.c_str());
    throw std::runtime_error("checkpoint: write failed: " + path);
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0) {
    std::remove(tmp.c_str());
    throw std::runtime_error("checkpoint: cannot replace " + path);
  }
}

void read_payload(std::ifstream& f, const BufferEntry& e, float* dst) {
  f.seekg(static_cast<std::streamoff>(e.offset));
  f.read(reinterpret_cast<char*>(dst), static_cast<std::streamsize>(e.bytes));
  if (static_cast<std::uint64_t>(f.gcount()) != e.bytes) throw std::runtime_error("checkpoint: truncated buffer " + e.name);
}

// global expert index of "layer.<i>.moe.expert.<e>.<param>" (after the kind prefix), or -1
int expert_of(const std::string& name) {
  const std::string key = ".moe.expert.";
  const std::size_t p = name.find(key);
  if (p == std::string::npos) return -1;
  return std::atoi(name.c_str() + p + key.size());
}

}  // namespace

void Engine::save_checkpoint(const std::string& path, const StageState& st) const {
  // buffer list: every parameter, then AdamW m and v (when attached), for_each order
  std::vector<BufferEntry> bufs;
  std::vector<std::pair<int, int>> src;  // (param index, kind: 0 param, 1 m, 2 v)
  const int kinds = has_opt_ ? 3 : 1;
  static const char* prefix[3] = {"param/", "adam_m/", "adam_v/"};
  for (int kind = 0; kind < kinds; ++kind)
    for (std::size_t i = 0; i < views_.size(); ++i) {
      BufferEntry e;
      e.name = prefix[kind] + views_[i].name;
      e.shape = views_[i].shape;
      e.bytes = static_cast<std::uint64_t>(views_[i].rows) * views_[i].cols * 4;
      bufs.push_back(std::move(e));
      src.emplace_back(static_cast<int>(i), kind);
    }
  Header h;
  h.cfg = cfg_;
  h.ep_world = ep_world_;
  h.ep_rank = ep_rank_;
  h.st = st;
  h.adamw = has_opt_;
  h.b1 = b1_;
  h.b2 = b2_;
  h.eps = eps_;
  h.wd = wd_;
  h.step_count = step_count_;
  write_container(path, h, std::move(bufs), [&](std::size_t b, float* dst) {
    const int i = src[b].first, kind = src[b].second;
    if (kind == 0)
      get_param(i, dst);
    else
      get_moment(i, kind - 1, dst);
  });
}

StageState Engine::load_checkpoint(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  const Manifest m = read_manifest(f, path);
  if (config_line(m.cfg) != config_line(cfg_))
    throw std::invalid_argument("checkpoint: model config does not match the checkpoint (" + config_line(m.cfg) + ")");
  if (m.ep_world != ep_world_ || m.ep_rank != ep_rank_)
    throw std::invalid_argument("checkpoint: expert-parallel shard does not match the checkpoint");
  if (m.adamw) {
    if (!has_opt_) adamw_attach(m.b1, m.b2, m.eps, m.wd);
    b1_ = m.b1;
    b2_ = m.b2;
    eps_ = m.eps;
    wd_ = m.wd;
    step_count_ = m.step_count;
  } else if (has_opt_) {
    // a file without optimizer state restores a fresh optimizer: zero moments and
    // step count, so a revert equals the snapshot bit for bit
    if (off_) offload_sync(*off_);
    for (DevBuf* b : {&emb_m_, &emb_v_, &lay_m_, &lay_v_})
      if (b->p) cuda_check(cudaMemsetAsync(b->p, 0, b->bytes, stream_), "zero moments");
    if (off_ && off_->hm) {
      const std::size_t n = static_cast<std::size_t>(layer_stride_) * off_->slow_list.size();
      std::memset(off_->hm, 0, n * 4);
      std::memset(off_->hv, 0, n * 4);
    }
    step_count_ = 0;
  }
  std::map<std::string, int> index;
  for (std::size_t i = 0; i < views_.size(); ++i) index[views_[i].name] = static_cast<int>(i);
  std::vector<char> seen(views_.size() * 3, 0);
  std::vector<float> host;
  for (const BufferEntry& e : m.buffers) {
    const std::size_t slash = e.name.find('/');
    if (slash == std::string::npos) throw std::runtime_error("checkpoint: bad buffer name " + e.name);
    const std::string kind_s = e.name.substr(0, slash), pname = e.name.substr(slash + 1);
    const int kind = kind_s == "param" ? 0 : kind_s == "adam_m" ? 1 : kind_s == "adam_v" ? 2 : -1;
    auto it = index.find(pname);
    if (kind < 0 || it == index.end()) throw std::runtime_error("checkpoint: unknown buffer " + e.name);
    const ParamView& v = views_[static_cast<std::size_t>(it->second)];
    if (e.shape != v.shape || e.bytes != static_cast<std::uint64_t>(v.rows) * v.cols * 4)
      throw std::runtime_error("checkpoint: shape mismatch for " + e.name);
    if (kind > 0 && !m.adamw) throw std::runtime_error("checkpoint: moment buffer without optimizer state");
    host.resize(e.bytes / 4);
    read_payload(f, e, host.data());
    if (kind == 0)
      set_param(it->second, host.data());
    else
      set_moment(it->second, kind - 1, host.data());
    seen[static_cast<std::size_t>(it->second) * 3 + kind] = 1;
  }
  for (std::size_t i = 0; i < views_.size(); ++i) {
    if (!seen[i * 3]) throw std::runtime_error("checkpoint: missing buffer param/" + views_[i].name);
    if (m.adamw && (!seen[i * 3 + 1] || !seen[i * 3 + 2]))
      throw std::runtime_error("checkpoint: missing moments for " + views_[i].name);
  }
  return m.st;
}

std::unique_ptr<Engine> Engine::from_checkpoint(const std::string& path, StageState* st) {
  Manifest m;
  {
    std::ifstream f(path, std::ios::binary);
    m = read_manifest(f, path);
  }
  std::unique_ptr<Engine> model(new Engine(m.cfg, NoInit{}, m.ep_world, m.ep_rank));
  const StageState s = model->load_checkpoint(path);
  if (st) *st = s;
  return model;
}

StageState delink_checkpoint(const std::string& in_path, const std::string& out_path) {
  StageState st;
  std::unique_ptr<Engine> pseudo = Engine::from_checkpoint(in_path, &st);
  if (st.stage != 0) throw std::logic_error("delink: checkpoint is not in the PSEUDO stage");
  std::unique_ptr<Engine> real = pseudo->delinked();  // weights + moments into every layer
  st.stage = 1;
  real->save_checkpoint(out_path, st);
  return st;
}

int Engine::expert_shard(int expert) const {
  if (!cfg_.moe.enabled()) throw std::logic_error("expert_shard: dense model");
  if (expert < 0 || expert >= cfg_.moe.n_experts) throw std::out_of_range("expert_shard: expert index");
  return expert / (cfg_.moe.n_experts / cfg_.moe.n_shards);
}

std::vector<std::vector<int>> Engine::shard_layout() const {
  if (!cfg_.moe.enabled()) throw std::logic_error("shard_layout: dense model");
  std::vector<std::vector<int>> layout(static_cast<std::size_t>(cfg_.moe.n_shards));
  for (int e = 0; e < cfg_.moe.n_experts; ++e) layout[static_cast<std::size_t>(expert_shard(e))].push_back(e);
  return layout;
}

void Engine::redistribute_experts(int new_n_shards) {
  if (!cfg_.moe.enabled()) throw std::logic_error("redistribute_experts: dense model");
  if (new_n_shards <= 0 || cfg_.moe.n_experts % new_n_shards != 0)
    throw std::invalid_argument("redistribute_experts: n_experts must be divisible by new shard count");
  if (ep_world_ > 1)
    throw std::logic_error("redistribute_experts: an expert-parallel shard re-shards through redistribute_checkpoints");
  cfg_.moe.n_shards = new_n_shards;
}

void redistribute_checkpoints(const std::vector<std::string>& in_paths, const std::vector<std::string>& out_paths) {
  const int W1 = static_cast<int>(in_paths.size()), W2 = static_cast<int>(out_paths.size());
  if (W1 <= 0 || W2 <= 0) throw std::invalid_argument("redistribute_experts: empty shard list");
  std::vector<Manifest> in(static_cast<std::size_t>(W1));
  for (int r = 0; r < W1; ++r) {
    std::ifstream f(in_paths[static_cast<std::size_t>(r)], std::ios::binary);
    in[static_cast<std::size_t>(r)] = read_manifest(f, in_paths[static_cast<std::size_t>(r)]);
    const Manifest& m = in[static_cast<std::size_t>(r)];
    if (m.ep_world != W1 || m.ep_rank != r)
      throw std::invalid_argument("redistribute_experts: input " + std::to_string(r) + " is not shard " +
                                  std::to_string(r) + " of " + std::to_string(W1));
    ModelConfig a = m.cfg, b = in[0].cfg;
    a.moe.n_shards = b.moe.n_shards = 1;
    if (config_line(a) != config_line(b)) throw std::invalid_argument("redistribute_experts: shards disagree on the config");
  }
  const ModelConfig& c0 = in[0].cfg;
  if (!c0.moe.enabled()) throw std::logic_error("redistribute_experts: dense model");
  const int E = c0.moe.n_experts;
  if (E % W2 != 0)  // model.cpp:350-353
    throw std::invalid_argument("redistribute_experts: n_experts must be divisible by new shard count");
  // where each buffer lives: replicated ones in shard 0, expert e in the shard that owns it
  struct Src {
    int shard;
    BufferEntry e;
  };
  std::vector<std::pair<std::string, Src>> replicated;
  std::map<int, std::vector<Src>> experts;  // global expert -> its buffers (all kinds)
  for (int r = 0; r < W1; ++r)
    for (const BufferEntry& e : in[static_cast<std::size_t>(r)].buffers) {
      const int x = expert_of(e.name);
      if (x >= 0)
        experts[x].push_back({r, e});
      else if (r == 0)
        replicated.push_back({e.name, {0, e}});
    }
  if (static_cast<int>(experts.size()) != E) throw std::runtime_error("redistribute_experts: input shards miss experts");
  std::vector<std::ifstream> files;
  for (const std::string& p : in_paths) files.emplace_back(p, std::ios::binary);
  for (int r2 = 0; r2 < W2; ++r2) {
    std::vector<Src> srcs;
    for (const auto& kv : replicated) srcs.push_back(kv.second);
    for (int x = r2 * (E / W2); x < (r2 + 1) * (E / W2); ++x)
      for (const Src& s : experts[x]) srcs.push_back(s);
    Header h;
    h.cfg = c0;
    h.cfg.moe.n_shards = W2;
    h.ep_world = W2;
    h.ep_rank = r2;
    h.st = in[0].st;
    h.adamw = in[0].adamw;
    h.b1 = in[0].b1;
    h.b2 = in[0].b2;
    h.eps = in[0].eps;
    h.wd = in[0].wd;
    h.step_count = in[0].step_count;
    std::vector<BufferEntry> bufs;
    for (const Src& s : srcs) bufs.push_back(s.e);
    write_container(out_paths[static_cast<std::size_t>(r2)], h, std::move(bufs), [&](std::size_t b, float* dst) {
      read_payload(files[static_cast<std::size_t>(srcs[b].shard)], srcs[b].e, dst);
    });
  }
}

}  // namespace p2r
