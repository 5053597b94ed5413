// map_io.cpp — the reference's map file format straight to and from device
// levels (load_map / save_map / is_map_file, map_io.hpp:17-126).
//
// File layout (map_io.hpp:17-21, little-endian): magic "3DBBS\x01", u32
// version 1, f64 min_resolution, u32 max_level, f64 x6 bbox, then per level:
// u32 level, u64 count, count x (i32 x, y, z).
//
// Loading reads each level block in large chunks into pinned staging buffers
// and copies them to the device while the next chunk is read; the level is
// then built on the device (sort/unique + bitmap/hash, map_build.cu) — the
// reference instead reads voxel by voxel and rebuilds its hash tables with
// the collision-rate sizing loop (voxel_map.hpp:88-114).  Errors are the
// reference's, in its order and with its messages.
#include <cuda_runtime.h>
#include <sys/stat.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "bbs_map_impl.h"
#include "bbs_map_io.h"

namespace bbs {

void build_level_from_device_voxels(bbs_map* m, int l, const int32_t* d_vox, uint64_t n);
void begin_levels(bbs_map* m, int n_levels);

namespace {

constexpr char kMagic[6] = {'3', 'D', 'B', 'B', 'S', '\x01'};
constexpr uint32_t kVersion = 1;
constexpr size_t kChunk = size_t(32) << 20;  // staging chunk (bytes), a multiple of 12

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

struct Pinned {
  void* p = nullptr;
  explicit Pinned(size_t n) { BBS_CUDA(cudaMallocHost(&p, n)); }
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

}  // namespace

void MapFile::read(void* dst, size_t n) {  // detail::read_pod, map_io.hpp:38-41
  if (pos + n > size || std::fread(dst, 1, n, f) != n) throw Error(BBS_ERR_FORMAT, path + ": truncated map file");
  pos += n;
}

// load_map header, map_io.hpp:70-96.
void map_file_open(const char* path, MapFile* mf) {
  mf->path = path;
  struct stat st;
  if (::stat(path, &st) != 0) throw Error(BBS_ERR_FILE_NOT_FOUND, "file not found: " + mf->path);
  mf->f = std::fopen(path, "rb");
  if (!mf->f) throw Error(BBS_ERR_IO, "cannot open: " + mf->path);
  mf->size = static_cast<uint64_t>(st.st_size);
  char magic[6];
  if (mf->size < sizeof(magic) || std::fread(magic, 1, sizeof(magic), mf->f) != sizeof(magic) ||
      std::memcmp(magic, kMagic, sizeof(kMagic)) != 0)
    throw Error(BBS_ERR_FORMAT, mf->path + ": bad magic bytes (not a map file)");
  mf->pos = sizeof(magic);
  const uint32_t version = mf->pod<uint32_t>();
  if (version != kVersion)
    throw Error(BBS_ERR_FORMAT, mf->path + ": unsupported map version " + std::to_string(version));
  mf->r = mf->pod<double>();
  mf->max_level = mf->pod<uint32_t>();
  if (!(mf->r > 0.0) || mf->max_level < 1 || mf->max_level > 62)
    throw Error(BBS_ERR_FORMAT, mf->path + ": invalid header values");
  mf->bbox.min.x = mf->pod<double>();
  mf->bbox.min.y = mf->pod<double>();
  mf->bbox.min.z = mf->pod<double>();
  mf->bbox.max.x = mf->pod<double>();
  mf->bbox.max.y = mf->pod<double>();
  mf->bbox.max.z = mf->pod<double>();
}

// Level block structure, map_io.hpp:98-112, checked before any device work
// (so every format error surfaces in the reference's order, GPU or not):
// the block headers are read and the voxel payloads skipped.
void map_file_check_levels(MapFile* mf) {
  const uint64_t start = mf->pos;
  for (uint32_t l = 0; l <= mf->max_level; ++l) {
    const uint32_t stored = mf->pod<uint32_t>();
    if (stored != l) throw Error(BBS_ERR_FORMAT, mf->path + ": level blocks out of order");
    const uint64_t count = mf->pod<uint64_t>();
    if (count > (mf->size - mf->pos) / 12) throw Error(BBS_ERR_FORMAT, mf->path + ": truncated map file");
    mf->pos += count * 12;
    if (std::fseek(mf->f, static_cast<long>(mf->pos), SEEK_SET) != 0)
      throw Error(BBS_ERR_IO, "cannot read: " + mf->path);
  }
  mf->pos = start;
  if (std::fseek(mf->f, static_cast<long>(start), SEEK_SET) != 0)
    throw Error(BBS_ERR_IO, "cannot read: " + mf->path);
}

// load_map level blocks, map_io.hpp:98-112, uploaded chunk by chunk and built
// on the device (MultiResVoxelMap::from_levels, voxel_map.hpp:247-261).
void map_file_read_levels(MapFile* mf, bbs_map* m) {
  DeviceGuard g(m->device);
  cudaStream_t s = m->stream;
  const int n_levels = static_cast<int>(mf->max_level) + 1;
  begin_levels(m, n_levels);
  // staging: two chunks, no larger than the file's voxel payload needs
  const size_t chunk = static_cast<size_t>(std::min<uint64_t>(kChunk, std::max<uint64_t>(12, mf->size - mf->pos)));
  Pinned stage(2 * chunk);
  cudaEvent_t done[2];
  BBS_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
  BBS_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
  struct Events {
    cudaEvent_t* e;
    ~Events() {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } ev_guard{done};
  bool used[2] = {false, false};
  for (int l = 0; l < n_levels; ++l) {
    const uint32_t stored = mf->pod<uint32_t>();
    if (stored != static_cast<uint32_t>(l)) throw Error(BBS_ERR_FORMAT, mf->path + ": level blocks out of order");
    const uint64_t count = mf->pod<uint64_t>();
    if (count > (mf->size - mf->pos) / 12) throw Error(BBS_ERR_FORMAT, mf->path + ": truncated map file");
    int32_t* d_vox = nullptr;
    BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_vox), std::max<uint64_t>(count, 1) * 12, s));
    struct Free {
      int32_t* p;
      cudaStream_t s;
      ~Free() { cudaFreeAsync(p, s); }
    } free_guard{d_vox, s};
    uint64_t bytes = count * 12, off = 0;
    int b = 0;
    while (bytes > 0) {
      const size_t n = static_cast<size_t>(std::min<uint64_t>(bytes, chunk));
      if (used[b]) BBS_CUDA(cudaEventSynchronize(done[b]));  // its previous copy finished
      char* h = static_cast<char*>(stage.p) + b * chunk;
      mf->read(h, n);
      BBS_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(d_vox) + off, h, n, cudaMemcpyHostToDevice, s));
      BBS_CUDA(cudaEventRecord(done[b], s));
      used[b] = true;
      off += n;
      bytes -= n;
      b ^= 1;
    }
    build_level_from_device_voxels(m, l, d_vox, count);
  }
  BBS_CUDA(cudaStreamSynchronize(s));
}

// save_map, map_io.hpp:44-65: levels written from the device's sorted sets
// (occupied_voxels order), so the bytes equal the reference's for equal maps.
void map_file_save(bbs_map* m, const char* path) {
  const std::string p(path);
  File out;
  out.f = std::fopen(path, "wb");
  if (!out.f) throw Error(BBS_ERR_IO, "cannot open for write: " + p);
  bool ok = true;
  auto put = [&](const void* v, size_t n) { ok = ok && std::fwrite(v, 1, n, out.f) == n; };
  put(kMagic, sizeof(kMagic));
  put(&kVersion, sizeof(kVersion));
  put(&m->r, sizeof(double));
  const uint32_t ml = static_cast<uint32_t>(m->max_level);
  put(&ml, sizeof(ml));
  const double bb[6] = {m->bbox.min.x, m->bbox.min.y, m->bbox.min.z, m->bbox.max.x, m->bbox.max.y, m->bbox.max.z};
  put(bb, sizeof(bb));
  std::vector<int32_t> vox;
  for (int l = 0; l <= m->max_level; ++l) {
    const uint32_t lv = static_cast<uint32_t>(l);
    put(&lv, sizeof(lv));
    uint64_t n = 0;
    level_occupied(m, l, nullptr, 0, &n);
    vox.resize(3 * std::max<uint64_t>(n, 1));
    if (n) level_occupied(m, l, vox.data(), n, &n);
    put(&n, sizeof(n));
    if (n) put(vox.data(), 12 * n);
  }
  ok = ok && std::fflush(out.f) == 0;
  if (!ok) throw Error(BBS_ERR_IO, "write failed: " + p);
}

// is_map_file, map_io.hpp:119-126.
bool map_file_is_map(const char* path) {
  File f;
  f.f = std::fopen(path, "rb");
  if (!f.f) return false;
  char magic[6];
  return std::fread(magic, 1, sizeof(magic), f.f) == sizeof(magic) &&
         std::memcmp(magic, kMagic, sizeof(kMagic)) == 0;
}

}  // namespace bbs
