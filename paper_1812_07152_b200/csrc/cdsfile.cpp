// cdsfile.cpp — zero-copy reader of the reference's on-disk CDS (`hmat.cds`, format CDS1
// version 1: /root/reference/proj/src/serial.cpp:160-211, 271-308), so a CDS written by
// the reference inspector (`hmx inspect`) goes straight to the device: the file is
// memory-mapped, the small structure arrays are decoded, and the generator arrays
// dgen/bgen/vgen are handed to hmxg_upload as pointers into the mapping.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hmxg.h"

struct hmxg_cds_file {
  void* map = MAP_FAILED;
  std::size_t size = 0;
  std::uint64_t n = 0;
  std::uint32_t dim = 0, num_nodes = 0, height = 0, leaf_size = 0, max_rank = 0;
  double bacc = 0.0;
  std::vector<std::uint32_t> parent, lchild, rchild, start, end, level, perm, sranks;
  std::vector<std::uint8_t> participating;
  std::vector<std::uint32_t> near_pairs, far_pairs, v_order;
  std::vector<std::uint64_t> dptr, bptr, vptr;
  const double* dgen = nullptr;
  const double* bgen = nullptr;
  const double* vgen = nullptr;
  ~hmxg_cds_file() {
    if (map != MAP_FAILED) munmap(map, size);
  }
};

namespace {

thread_local std::string g_file_err;

struct FormatError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Little-endian cursor over the mapping (ByteReader, proj/include/hmx/io.hpp:57-120).
class Cursor {
 public:
  Cursor(const unsigned char* p, std::size_t n) : p_(p), n_(n) {}
  void need(std::size_t k) const {
    if (n_ - pos_ < k) throw FormatError("truncated CDS file");
  }
  template <class T>
  T get() {
    need(sizeof(T));
    T v;
    std::memcpy(&v, p_ + pos_, sizeof(T));
    pos_ += sizeof(T);
    return v;
  }
  std::uint64_t count(std::size_t elem) {
    const std::uint64_t c = get<std::uint64_t>();
    if (c > (n_ - pos_) / elem) throw FormatError("truncated CDS file (array length)");
    return c;
  }
  template <class T>
  std::vector<T> array() {
    const std::uint64_t c = count(sizeof(T));
    std::vector<T> v(c);
    if (c) std::memcpy(v.data(), p_ + pos_, c * sizeof(T));
    pos_ += c * sizeof(T);
    return v;
  }
  // f64 array left in place: returns its address inside the mapping
  const double* doubles(std::uint64_t* c) {
    *c = count(sizeof(double));
    const double* v = reinterpret_cast<const double*>(p_ + pos_);
    pos_ += *c * sizeof(double);
    return v;
  }
  void skip(std::size_t k) {
    need(k);
    pos_ += k;
  }
  const unsigned char* here() const { return p_ + pos_; }

 private:
  const unsigned char* p_;
  std::size_t n_;
  std::size_t pos_ = 0;
};

// Blockset (serial.cpp:93-134): pairs flattened in storage order (groups -> blocks -> pairs).
void read_blockset(Cursor& r, std::vector<std::uint32_t>& flat) {
  r.get<std::uint8_t>();   // kind
  r.get<std::uint32_t>();  // blocksize
  const std::uint64_t groups = r.count(12);
  for (std::uint64_t g = 0; g < groups; ++g) {
    r.get<std::uint32_t>();  // row group
    const std::uint64_t blocks = r.count(8);
    for (std::uint64_t b = 0; b < blocks; ++b) {
      const std::uint64_t pairs = r.count(8);
      for (std::uint64_t k = 0; k < pairs; ++k) {
        flat.push_back(r.get<std::uint32_t>());
        flat.push_back(r.get<std::uint32_t>());
      }
    }
  }
}

// Coarsenset (serial.cpp:136-161): V storage order = levels -> subtrees -> nodes.
void read_coarsenset(Cursor& r, std::vector<std::uint32_t>& order) {
  r.get<std::uint32_t>();  // agg
  r.get<std::uint32_t>();  // p
  const std::uint64_t levels = r.count(8);
  for (std::uint64_t l = 0; l < levels; ++l) {
    const std::uint64_t subtrees = r.count(16);
    for (std::uint64_t s = 0; s < subtrees; ++s) {
      r.get<double>();  // cost
      const auto nodes = r.array<std::uint32_t>();
      order.insert(order.end(), nodes.begin(), nodes.end());
    }
  }
}

void parse(hmxg_cds_file& f) {
  Cursor r(static_cast<const unsigned char*>(f.map), f.size);
  char tag[4];
  r.need(4);
  std::memcpy(tag, r.here(), 4);
  r.skip(4);
  if (std::memcmp(tag, "CDS1", 4) != 0) throw FormatError("not a CDS file (bad tag)");
  const std::uint32_t version = r.get<std::uint32_t>();
  if (version != 1) throw FormatError("unsupported CDS version " + std::to_string(version));
  // header (serial.cpp:160-166)
  f.n = r.get<std::uint64_t>();
  f.dim = r.get<std::uint32_t>();
  f.num_nodes = r.get<std::uint32_t>();
  f.bacc = r.get<double>();
  f.max_rank = r.get<std::uint32_t>();
  // tree (serial.cpp:31-43)
  if (r.get<std::uint32_t>() != f.num_nodes) throw FormatError("CDS header disagrees with embedded tree");
  f.parent = r.array<std::uint32_t>();
  f.lchild = r.array<std::uint32_t>();
  f.rchild = r.array<std::uint32_t>();
  f.start = r.array<std::uint32_t>();
  f.end = r.array<std::uint32_t>();
  f.level = r.array<std::uint32_t>();
  f.perm = r.array<std::uint32_t>();
  f.height = r.get<std::uint32_t>();
  f.leaf_size = r.get<std::uint32_t>();
  for (const auto* a : {&f.parent, &f.lchild, &f.rchild, &f.start, &f.end, &f.level})
    if (a->size() != f.num_nodes) throw FormatError("CDS tree arrays have the wrong length");
  if (f.perm.size() != f.n) throw FormatError("CDS header disagrees with embedded tree");
  // per-node arrays (serial.cpp:167-170)
  f.sranks = r.array<std::uint32_t>();
  f.participating = r.array<std::uint8_t>();
  if (f.sranks.size() != f.num_nodes || f.participating.size() != f.num_nodes)
    throw FormatError("CDS per-node arrays have the wrong length");
  read_blockset(r, f.near_pairs);
  read_blockset(r, f.far_pairs);
  read_coarsenset(r, f.v_order);
  std::uint64_t nd = 0, nb = 0, nv = 0;
  f.dptr = r.array<std::uint64_t>();
  f.dgen = r.doubles(&nd);
  f.bptr = r.array<std::uint64_t>();
  f.bgen = r.doubles(&nb);
  f.vptr = r.array<std::uint64_t>();
  f.vgen = r.doubles(&nv);
  // like the reference reader (serial.cpp:180-210) bytes after the vgen array are ignored
  // offset consistency (serial.cpp:203-208)
  if (f.dptr.size() != f.near_pairs.size() / 2 + 1 || f.dptr.back() != nd ||
      f.bptr.size() != f.far_pairs.size() / 2 + 1 || f.bptr.back() != nb ||
      f.vptr.size() != f.v_order.size() + 1 || f.vptr.back() != nv)
    throw FormatError("CDS offset arrays are inconsistent");
}

}  // namespace

extern "C" {

int hmxg_cds_file_open(const char* path, hmxg_cds_file** out) {
  if (!path || !out) {
    g_file_err = "hmxg_cds_file_open: null argument";
    return HMXG_EINVAL;
  }
  *out = nullptr;
  auto f = std::make_unique<hmxg_cds_file>();
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) {
    g_file_err = std::string("cannot open ") + path + ": " + std::strerror(errno);
    return HMXG_EIO;
  }
  struct stat stbuf {};
  if (fstat(fd, &stbuf) != 0 || stbuf.st_size <= 0) {
    ::close(fd);
    g_file_err = std::string("cannot read ") + path;
    return HMXG_EIO;
  }
  f->size = static_cast<std::size_t>(stbuf.st_size);
  f->map = mmap(nullptr, f->size, PROT_READ, MAP_PRIVATE, fd, 0);
  ::close(fd);
  if (f->map == MAP_FAILED) {
    g_file_err = std::string("cannot map ") + path + ": " + std::strerror(errno);
    return HMXG_EIO;
  }
  try {
    parse(*f);
  } catch (const std::exception& e) {
    g_file_err = std::string(e.what()) + ": " + path;
    return HMXG_EIO;
  }
  *out = f.release();
  return HMXG_OK;
}

int hmxg_cds_file_view(const hmxg_cds_file* f, hmxg_cds_view* v) {
  if (!f || !v) return HMXG_EINVAL;
  std::memset(v, 0, sizeof *v);
  v->n = f->n;
  v->num_nodes = f->num_nodes;
  v->height = f->height;
  v->parent = f->parent.data();
  v->lchild = f->lchild.data();
  v->rchild = f->rchild.data();
  v->start = f->start.data();
  v->end = f->end.data();
  v->level = f->level.data();
  v->perm = f->perm.data();
  v->sranks = f->sranks.data();
  v->participating = f->participating.data();
  v->num_near = f->near_pairs.size() / 2;
  v->near_pairs = f->near_pairs.data();
  v->num_far = f->far_pairs.size() / 2;
  v->far_pairs = f->far_pairs.data();
  v->num_v = f->v_order.size();
  v->v_order = f->v_order.data();
  v->dptr = f->dptr.data();
  v->bptr = f->bptr.data();
  v->vptr = f->vptr.data();
  v->dgen = f->dgen;
  v->bgen = f->bgen;
  v->vgen = f->vgen;
  return HMXG_OK;
}

int hmxg_cds_file_header(const hmxg_cds_file* f, uint32_t* dim, double* bacc, uint32_t* max_rank) {
  if (!f) return HMXG_EINVAL;
  if (dim) *dim = f->dim;
  if (bacc) *bacc = f->bacc;
  if (max_rank) *max_rank = f->max_rank;
  return HMXG_OK;
}

void hmxg_cds_file_close(hmxg_cds_file* f) { delete f; }

const char* hmxg_cds_file_error(void) { return g_file_err.c_str(); }

}  // extern "C"
