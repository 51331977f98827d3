// partition.cu — slab decomposition (host only).  Rank p owns the global node
// planes [p*n_l/P, (p+1)*n_l/P) of every distributed level l, the last rank also
// the top boundary plane n_l.  Slabs are nested (a_{l+1} = a_l / 2), so
// restriction and prolongation need one neighbour plane only.  Levels stay
// distributed while each rank keeps >= kMinPlanesPerRank planes and the next
// level's slabs nest; below that the coarse right-hand side is all-gathered and
// every rank runs the remaining levels redundantly on the full (small) grid
// (agglomeration).
#include <cstdio>

#include "partition.h"

namespace mg {

mg_status compute_partition(const mg_config* c, int L, Partition* pt, std::string* err) {
  *pt = Partition();
  pt->P = c->nranks;
  pt->rank = c->rank;
  pt->slab = c->nranks > 1 || (c->flags & 4u /* MG_FLAG_SLAB */);
  const int64_t n0 = c->dim == 3 ? c->nodes[2] - 1 : c->nodes[1] - 1;
  for (int l = 0; l < L && l < kMaxLevels; l++) pt->n[l] = n0 >> l;
  if (!pt->slab) {
    pt->la = 0;
    return MG_OK;
  }
  pt->H = kSlabHalo;
  const int P = pt->P;
  int la = 0;
  // level l may be distributed if n_l splits evenly with >= kMinPlanesPerRank even-sized slabs
  // (even => the next level's slabs nest); the coarsest level is always held in full
  while (la < L - 1 && pt->n[la] % P == 0 && pt->n[la] / P >= kMinPlanesPerRank && (pt->n[la] / P) % 2 == 0) la++;
  if (la == 0) {
    char buf[256];
    snprintf(buf, sizeof buf,
             "slab decomposition needs (plane-axis cells)/nranks even and >= %d on the finest level (cells %lld, "
             "nranks %d)",
             kMinPlanesPerRank, (long long)pt->n[0], P);
    *err = buf;
    return MG_ERR_NOT_COARSENABLE;
  }
  pt->la = la;
  for (int l = 0; l < la; l++) {
    const int64_t w = pt->n[l] / P;
    pt->a[l] = (int64_t)c->rank * w;
    pt->b[l] = c->rank == P - 1 ? pt->n[l] + 1 : (int64_t)(c->rank + 1) * w;
  }
  // owned range of the first full level (written by the last distributed restriction)
  {
    const int64_t w = pt->n[la] / P;
    pt->a[la] = (int64_t)c->rank * w;
    pt->b[la] = c->rank == P - 1 ? pt->n[la] + 1 : (int64_t)(c->rank + 1) * w;
  }
  return MG_OK;
}

}  // namespace mg
