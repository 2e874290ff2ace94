// Decentralized static schedules (§4.2).
//
// "a worker can simply call a local function S to obtain its group in an
// iteration. The logic of S guarantees that the schedule is consistent among
// all the workers". Both rules are pure functions of
// (config, step); worker id w = node*m + r (reading R6).
#include <vector>

#include "rp_internal.h"

namespace rp {

namespace {
// Assign consecutive group indices; groups with < 2 members are skips (-1).
struct Builder {
  int32_t* group_of;
  int n;
  int next = 0;
  void add(const std::vector<int>& g) {
    if (g.size() < 2) return;
    for (int w : g) group_of[w] = next;
    ++next;
  }
};
}  // namespace

// fig:scheduler, phase = step mod 4, generalized to any m (reading R4/R5):
//  1,3: whole node; 0: rank 0 of all nodes + local consecutive pairs of ranks 1..m-1
//  (rank 1 dropped when their count is odd); 2: rank 1 with rank 1 of node a+nodes/2,
//  locally (0, m-1) when m >= 3 and consecutive pairs of ranks 2..m-2.
int schedule_paper4(int nodes, int m, int64_t step, int32_t* group_of, int32_t* n_groups) {
  if (nodes < 1 || m < 1 || nodes * m > RP_MAX_WORLD || step < 0)
    return fail(RP_EINVAL, "paper4: need nodes >= 1, m >= 1, nodes*m <= 64, step >= 0");
  const int n = nodes * m;
  for (int w = 0; w < n; ++w) group_of[w] = -1;
  Builder b{group_of, n};
  auto W = [m](int a, int r) { return a * m + r; };
  const int phase = static_cast<int>(step % 4);
  if (phase == 1 || phase == 3) {
    for (int a = 0; a < nodes; ++a) {
      std::vector<int> g;
      for (int r = 0; r < m; ++r) g.push_back(W(a, r));
      b.add(g);
    }
  } else if (phase == 0) {
    std::vector<int> g0;
    for (int a = 0; a < nodes; ++a) g0.push_back(W(a, 0));
    b.add(g0);
    std::vector<int> local;
    for (int r = 1; r < m; ++r) local.push_back(r);
    if (local.size() % 2 == 1) local.erase(local.begin());
    for (int a = 0; a < nodes; ++a)
      for (size_t p = 0; p + 1 < local.size(); p += 2) b.add({W(a, local[p]), W(a, local[p + 1])});
  } else {
    const int half = nodes / 2;
    if (m >= 2)
      for (int a = 0; a < half; ++a) b.add({W(a, 1), W(a + half, 1)});
    for (int a = 0; a < nodes; ++a) {
      if (m >= 3) b.add({W(a, 0), W(a, m - 1)});
      std::vector<int> rest;
      for (int r = 2; r < m - 1; ++r) rest.push_back(r);
      for (size_t p = 0; p + 1 < rest.size(); p += 2) b.add({W(a, rest[p]), W(a, rest[p + 1])});
    }
  }
  *n_groups = b.next;
  return RP_OK;
}

// SHIFT_K(n, k) (reading R4; cyclic form of the commented-out S(n,i) = d_{i mod k},
// P:937-941): phase p = step mod k, group of w = ((w + p) mod n) / k.
int schedule_shift_k(int n, int k, int64_t step, int32_t* group_of, int32_t* n_groups) {
  if (n < 1 || n > RP_MAX_WORLD || k < 1 || k > RP_MAX_GROUP || step < 0)
    return fail(RP_EINVAL, "shift_k: need 1 <= n <= 64, 1 <= k <= 16, step >= 0");
  const int p = static_cast<int>(step % k);
  const int buckets = (n + k - 1) / k;
  std::vector<std::vector<int>> g(buckets);
  for (int w = 0; w < n; ++w) g[((w + p) % n) / k].push_back(w);
  for (int w = 0; w < n; ++w) group_of[w] = -1;
  Builder b{group_of, n};
  for (auto& v : g) b.add(v);
  *n_groups = b.next;
  return RP_OK;
}

}  // namespace rp
