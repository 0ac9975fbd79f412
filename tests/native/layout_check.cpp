// Host-side invariants of the per-communicator region layout
// (csrc/mpix_internal.h RegionLayout), compiled with g++ by
// tests/test_layout_cpu.py: every area lies inside total(), no two areas
// overlap, and the alignment the kernels rely on holds. Prints "OK" or the
// first violation.
#include <cstdio>
#include <vector>

#include "mpix_internal.h"

using mpix::RegionLayout;

struct Area {
  const char* name;
  uint64_t off, len, align;
};

int main() {
  const int Ps[] = {1, 2, 3, 8, 16, 64};
  const int Rs[] = {2, 16, 128, 256};
  const uint64_t Es[] = {16, 4096, 65536};
  for (int P : Ps)
    for (int R : Rs)
      for (uint64_t E : Es) {
        RegionLayout L{P, R, E};
        std::vector<Area> a;
        for (int q = 0; q < P; ++q) {
          a.push_back({"sr", L.sr(q), L.ring_bytes(), 64});
          a.push_back({"rr", L.rr(q), L.ring_bytes(), 64});
          a.push_back({"sr_free", L.sr_free(q), (uint64_t)R * 8, 8});
          a.push_back({"rr_free", L.rr_free(q), (uint64_t)R * 8, 8});
          a.push_back({"coll_in", L.coll_in(q), sizeof(mpix::CollSlot), 32});
          a.push_back({"coll_exit", L.coll_exit(q), 8, 8});
          a.push_back({"eager", L.eager(q), (uint64_t)R * E, 16});
          a.push_back({"next_spost", L.dom_next_spost(q), 8, 8});
        }
        a.push_back({"bases", L.bases(), 8ull * P, 64});
        a.push_back({"dom_lock", L.dom_lock(), 8, 64});
        a.push_back({"dom_next_rpost", L.dom_next_rpost(), 8, 8});
        a.push_back({"dom_arrival", L.dom_arrival(), 8, 8});
        a.push_back({"pq", L.pq(), L.ring_bytes(), 64});
        a.push_back({"gseq", L.gseq(), 8ull * (2ull * P + 1 + mpix::kGraphTagCounters), 64});
        for (const Area& x : a) {
          if (x.off % x.align) {
            printf("P=%d R=%d E=%llu: %s at %llu not %llu-aligned\n", P, R, (unsigned long long)E,
                   x.name, (unsigned long long)x.off, (unsigned long long)x.align);
            return 1;
          }
          if (x.off + x.len > L.total()) {
            printf("P=%d R=%d E=%llu: %s ends past total()\n", P, R, (unsigned long long)E, x.name);
            return 1;
          }
        }
        for (size_t i = 0; i < a.size(); ++i)
          for (size_t j = i + 1; j < a.size(); ++j) {
            const Area &x = a[i], &y = a[j];
            if (x.off < y.off + y.len && y.off < x.off + x.len) {
              printf("P=%d R=%d E=%llu: %s [%llu,+%llu) overlaps %s [%llu,+%llu)\n", P, R,
                     (unsigned long long)E, x.name, (unsigned long long)x.off,
                     (unsigned long long)x.len, y.name, (unsigned long long)y.off,
                     (unsigned long long)y.len);
              return 1;
            }
          }
      }
  printf("OK\n");
  return 0;
}
