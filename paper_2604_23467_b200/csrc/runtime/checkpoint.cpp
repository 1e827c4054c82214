// checkpoint.cpp -- safetensors checkpoint loader.
//
// The reference has no checkpoint format: its weights are always drawn from
// one mt19937_64 stream (init_model, model.cpp:30-76).  This loader lets a real
// LLaMA-2 checkpoint (HuggingFace safetensors, one file or a directory of
// shards) or a dump of a graphrt model populate the arena instead.
//
// File format (safetensors): 8-byte little-endian header length N, N bytes of
// JSON {"name": {"dtype": "BF16"|"F16"|"F32", "shape": [..],
// "data_offsets": [begin, end]}, "__metadata__": {...}}, then the raw data
// block (offsets relative to it, row-major, little endian).
//
// Names: graphrt's own logical names ("layers.3.wq", reference [k,n] layout,
// model.hpp:33-45) load as-is; HuggingFace LLaMA names are mapped and their
// nn.Linear [out, in] matrices are read transposed by the device scatter
// (map_copy_kernel), so no host-side transpose pass is needed.  Both q/k
// layouts are rotate-half (HF's convention, the one the oracle and the
// kernels use), so q_proj/k_proj need no permutation beyond the arena's own
// RoPE pair interleave (MapDesc.rope_pair).
#include <cstdint>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <dirent.h>

#include <algorithm>
#include <cstring>

#include "runtime.hpp"

namespace grt {

namespace {

// ---- minimal JSON reader for the safetensors header -------------------------
struct JsonCursor {
  const char* p;
  const char* e;
  [[noreturn]] void fail(const std::string& what) const { raise(GRT_IoError, "safetensors header: " + what); }
  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  bool peek(char c) {
    ws();
    return p < e && *p == c;
  }
  void expect(char c) {
    ws();
    if (p >= e || *p != c) fail(std::string("expected '") + c + "'");
    ++p;
  }
  std::string str() {
    expect('"');
    std::string s;
    while (p < e && *p != '"') {
      if (*p == '\\') {
        ++p;
        if (p >= e) fail("bad escape");
        const char c = *p;
        if (c == 'u') {  // keep the escape verbatim (names are ASCII in practice)
          s += "\\u";
        } else {
          s += c == 'n' ? '\n' : c == 't' ? '\t' : c;
        }
        ++p;
        continue;
      }
      s += *p++;
    }
    if (p >= e) fail("unterminated string");
    ++p;
    return s;
  }
  int64_t integer() {
    ws();
    bool neg = false;
    if (p < e && *p == '-') {
      neg = true;
      ++p;
    }
    if (p >= e || *p < '0' || *p > '9') fail("expected an integer");
    if (neg) fail("negative integer");  // offsets and dims are never negative
    int64_t v = 0;
    while (p < e && *p >= '0' && *p <= '9') {
      const int dgt = *p++ - '0';
      if (v > (INT64_MAX - dgt) / 10) fail("integer overflow");
      v = v * 10 + dgt;
    }
    return v;
  }
  void skip_value() {
    ws();
    if (p >= e) fail("truncated");
    if (*p == '"') {
      str();
    } else if (*p == '{' || *p == '[') {
      const char open = *p, close = open == '{' ? '}' : ']';
      ++p;
      if (peek(close)) {
        ++p;
        return;
      }
      for (;;) {
        if (open == '{') {
          str();
          expect(':');
        }
        skip_value();
        if (peek(',')) {
          ++p;
          continue;
        }
        expect(close);
        return;
      }
    } else {
      while (p < e && *p != ',' && *p != '}' && *p != ']') ++p;
    }
  }
};

int dtype_code(const std::string& s) {
  if (s == "F32") return GRT_F32;
  if (s == "BF16") return GRT_BF16;
  if (s == "F16") return GRT_F16;
  return -1;
}

}  // namespace

SafetensorsFile::SafetensorsFile(const std::string& path) : path_(path) {
  fd_ = ::open(path.c_str(), O_RDONLY);
  if (fd_ < 0) raise(GRT_IoError, "cannot open '" + path + "'");
  struct stat st;
  if (fstat(fd_, &st) != 0) raise(GRT_IoError, "cannot stat '" + path + "'");
  size_ = static_cast<size_t>(st.st_size);
  if (size_ < 8) raise(GRT_IoError, "'" + path + "' is too short for a safetensors file");
  map_ = mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd_, 0);
  if (map_ == MAP_FAILED) {
    map_ = nullptr;
    raise(GRT_IoError, "cannot mmap '" + path + "'");
  }
  const uint8_t* b = static_cast<const uint8_t*>(map_);
  uint64_t n = 0;
  for (int i = 7; i >= 0; --i) n = (n << 8) | b[i];
  if (n > size_ - 8) raise(GRT_IoError, "'" + path + "': header length exceeds the file");
  data_off_ = 8 + n;
  JsonCursor c{reinterpret_cast<const char*>(b + 8), reinterpret_cast<const char*>(b + 8 + n)};
  c.expect('{');
  if (c.peek('}')) return;
  for (;;) {
    const std::string key = c.str();
    c.expect(':');
    if (key == "__metadata__") {
      c.skip_value();
    } else {
      StTensor t;
      t.name = key;
      c.expect('{');
      bool have_off = false;
      for (;;) {
        const std::string f = c.str();
        c.expect(':');
        if (f == "dtype") {
          t.dtype_name = c.str();
          t.dtype = dtype_code(t.dtype_name);
        } else if (f == "shape") {
          c.expect('[');
          if (!c.peek(']')) {
            for (;;) {
              t.shape.push_back(c.integer());
              if (c.peek(',')) {
                ++c.p;
                continue;
              }
              break;
            }
          }
          c.expect(']');
        } else if (f == "data_offsets") {
          c.expect('[');
          t.begin = static_cast<uint64_t>(c.integer());
          c.expect(',');
          t.end = static_cast<uint64_t>(c.integer());
          c.expect(']');
          have_off = true;
        } else {
          c.skip_value();
        }
        if (c.peek(',')) {
          ++c.p;
          continue;
        }
        c.expect('}');
        break;
      }
      if (!have_off || t.end < t.begin || t.end > size_ - data_off_)  // data_off_ <= size_ (checked above)
        raise(GRT_IoError, "'" + path + "': bad data_offsets for '" + key + "'");
      {  // the payload must be exactly numel x element size
        const int64_t es = t.dtype == GRT_F32 ? 4 : 2;
        int64_t numel = 1;
        for (int64_t dim : t.shape) {
          if (dim != 0 && numel > INT64_MAX / dim) raise(GRT_IoError, "'" + path + "': shape overflow for '" + key + "'");
          numel *= dim;
        }
        if (t.dtype >= 0 && (numel > INT64_MAX / es || t.end - t.begin != numel * es))
          raise(GRT_IoError, "'" + path + "': data_offsets of '" + key + "' do not match its shape and dtype");
      }
      tensors_.push_back(std::move(t));
    }
    if (c.peek(',')) {
      ++c.p;
      continue;
    }
    c.expect('}');
    break;
  }
}

SafetensorsFile::~SafetensorsFile() {
  if (map_) munmap(map_, size_);
  if (fd_ >= 0) ::close(fd_);
}

const void* SafetensorsFile::data(const StTensor& t) const {
  return static_cast<const uint8_t*>(map_) + data_off_ + t.begin;
}

// HuggingFace LLaMA name -> graphrt logical name; *out_in = the tensor is an
// nn.Linear weight stored [out, in] (the reference layout is [in, out]).
std::string hf_to_grt_name(const std::string& hf, bool* out_in) {
  *out_in = false;
  if (hf == "model.embed_tokens.weight") return "embedding";
  if (hf == "model.norm.weight") return "lnf_gamma";
  if (hf == "lm_head.weight") {
    *out_in = true;
    return "head";
  }
  static const char* kPrefix = "model.layers.";
  if (hf.compare(0, strlen(kPrefix), kPrefix) != 0) return "";
  const size_t a = strlen(kPrefix), dot = hf.find('.', a);
  if (dot == std::string::npos || dot == a) return "";
  for (size_t i = a; i < dot; ++i)
    if (hf[i] < '0' || hf[i] > '9') return "";
  const std::string layer = "layers." + hf.substr(a, dot - a) + ".";
  const std::string rest = hf.substr(dot + 1);
  static const std::pair<const char*, const char*> kLinear[] = {
      {"self_attn.q_proj.weight", "wq"},    {"self_attn.k_proj.weight", "wk"}, {"self_attn.v_proj.weight", "wv"},
      {"self_attn.o_proj.weight", "wo"},    {"mlp.gate_proj.weight", "w_gate"}, {"mlp.up_proj.weight", "w_up"},
      {"mlp.down_proj.weight", "w_down"}};
  for (const auto& kv : kLinear)
    if (rest == kv.first) {
      *out_in = true;
      return layer + kv.second;
    }
  if (rest == "input_layernorm.weight") return layer + "ln1_gamma";
  if (rest == "post_attention_layernorm.weight") return layer + "ln2_gamma";
  return "";  // e.g. self_attn.rotary_emb.inv_freq: derived, not loaded
}

static std::vector<std::string> checkpoint_files(const std::string& path) {
  struct stat st;
  if (stat(path.c_str(), &st) != 0) raise(GRT_IoError, "no such checkpoint '" + path + "'");
  if (!S_ISDIR(st.st_mode)) return {path};
  std::vector<std::string> files;
  DIR* d = opendir(path.c_str());
  if (!d) raise(GRT_IoError, "cannot list '" + path + "'");
  while (dirent* e = readdir(d)) {
    const std::string n = e->d_name;
    if (n.size() > 12 && n.compare(n.size() - 12, 12, ".safetensors") == 0) files.push_back(path + "/" + n);
  }
  closedir(d);
  std::sort(files.begin(), files.end());
  if (files.empty()) raise(GRT_IoError, "no .safetensors files in '" + path + "'");
  return files;
}

// Loads every recognised tensor; with `strict`, every weight of the model must
// be present exactly once and unknown tensor names are errors.
int load_safetensors(Model& m, const std::string& path, bool strict) {
  std::set<std::string> loaded;
  for (const std::string& f : checkpoint_files(path)) {
    SafetensorsFile st(f);
    for (const StTensor& t : st.tensors()) {
      bool out_in = false;
      std::string name;
      if (m.has_tensor(t.name)) {
        name = t.name;  // graphrt's own naming, reference layout
      } else {
        name = hf_to_grt_name(t.name, &out_in);
        if (name.empty() || !m.has_tensor(name)) {
          if (strict && name.empty() && t.name.find("rotary_emb") == std::string::npos)
            raise(GRT_ShapeMismatch, "checkpoint tensor '" + t.name + "' has no counterpart in this model");
          if (strict && !name.empty()) raise(GRT_ShapeMismatch, "checkpoint tensor '" + t.name + "' (" + name +
                                                                    ") does not exist in this model configuration");
          continue;
        }
      }
      if (t.dtype < 0) raise(GRT_IoError, "tensor '" + t.name + "': unsupported dtype " + t.dtype_name);
      const LogicalTensor& lt = m.tensor(name);
      int64_t r = 1, c = 1;
      if (t.shape.size() == 2) {
        r = t.shape[0];
        c = t.shape[1];
      } else if (t.shape.size() == 1) {
        c = t.shape[0];
      } else {
        raise(GRT_ShapeMismatch, "tensor '" + t.name + "': rank " + std::to_string(t.shape.size()));
      }
      if (out_in) std::swap(r, c);
      if (r != lt.rows || c != lt.cols)
        raise(GRT_ShapeMismatch, "tensor '" + t.name + "': shape [" + std::to_string(t.shape.empty() ? 0 : t.shape[0]) +
                                     (t.shape.size() > 1 ? "," + std::to_string(t.shape[1]) : std::string()) +
                                     "] does not match '" + name + "' [" + std::to_string(lt.rows) + "," +
                                     std::to_string(lt.cols) + "]" + (out_in ? " (transposed)" : ""));
      if (loaded.count(name)) raise(GRT_ShapeMismatch, "tensor '" + name + "' appears twice in the checkpoint");
      m.upload(name, st.data(t), t.end - t.begin, t.dtype, out_in);
      loaded.insert(name);
    }
  }
  if (strict)
    for (const LogicalTensor& lt : m.tensors())
      if (!loaded.count(lt.name)) raise(GRT_ShapeMismatch, "checkpoint has no tensor for '" + lt.name + "'");
  return static_cast<int>(loaded.size());
}

}  // namespace grt
