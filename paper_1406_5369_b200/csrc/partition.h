// partition.h — slab decomposition of the level hierarchy along the slowest
// (plane) axis.  Host-only, no GPU needed.
#pragma once
#include <cstdint>
#include <string>

#include "mg.h"

namespace mg {

constexpr int kMaxLevels = 40;
constexpr int kSlabHalo = 2;         // halo planes per side (fused RBGS needs 2)
constexpr int kMinPlanesPerRank = 8;  // a level stays distributed while n_l/P >= this

struct Partition {
  bool slab = false;  // slab layout (nranks > 1 or MG_FLAG_SLAB)
  int P = 1, rank = 0, H = 0;
  int la = 0;  // levels [0, la) are distributed; levels >= la are held in full on every rank
  int64_t n[kMaxLevels] = {};  // cells along the plane axis per level
  int64_t a[kMaxLevels] = {};  // owned global planes [a, b) of distributed levels
  int64_t b[kMaxLevels] = {};
};

// levels: resolved number of levels.  Returns MG_OK or an error with *err set.
mg_status compute_partition(const mg_config* c, int levels, Partition* out, std::string* err);

}  // namespace mg
