// bbs_map_io.h — the reference's map file format (map_io.cpp).
#pragma once

#include <cstdio>
#include <string>

#include "bbs_map_impl.h"

namespace bbs {

struct MapFile;
void map_file_open(const char* path, MapFile* mf);
void map_file_check_levels(MapFile* mf);
void map_file_read_levels(MapFile* mf, bbs_map* m);
void map_file_save(bbs_map* m, const char* path);
bool map_file_is_map(const char* path);

struct MapFile {
  std::string path;
  FILE* f = nullptr;
  uint64_t size = 0, pos = 0;
  double r = 0.0;
  uint32_t max_level = 0;
  bbs_aabb bbox{};
  void read(void* dst, size_t n);
  template <typename T>
  T pod() {
    T v;
    read(&v, sizeof(T));
    return v;
  }
  MapFile() = default;
  MapFile(const MapFile&) = delete;
  MapFile& operator=(const MapFile&) = delete;
  ~MapFile() {
    if (f) std::fclose(f);
  }
};

}  // namespace bbs
