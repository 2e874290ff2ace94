// Group Generator: Group Buffer + Global Division + slowdown filter + lock vector.
//
// PAPER.md §4.1 and §5.1/§5.3:
//  - a request increments the worker's counter c_w;
//  - a non-empty Group Buffer serves its first group;
//  - otherwise a Global Division "divides all current workers with empty GBs
//    into several non-conflicting groups", admitting w only if
//    c_i - c_w < C_thres;
//  - lock bits are set at grant and cleared by the completion ack.
// Readings: R7 candidates = empty GB, filter, not retired;
// R8 splitmix64 + Fisher-Yates, initiator's group first, chunks of k, last
// shorter; R19 retire rule. The state is POD (GGState) so it can be shared.
#include <algorithm>
#include <cstring>
#include <sstream>
#include <vector>

#include "rp_internal.h"

namespace rp {

namespace {
inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
inline uint64_t next_rand(GGState* s) {
  s->rng += 0x9E3779B97F4A7C15ull;
  return mix64(s->rng);
}
GGGroup* find_slot(GGState* s, int64_t seq) {
  for (auto& g : s->table)
    if (g.seq == seq) return &g;
  return nullptr;
}
}  // namespace

void gg_init(GGState* s, int n, int k, int c_thres, uint64_t seed, int policy, int nodes) {
  std::memset(s, 0, sizeof(*s));
  s->n = n;
  s->k = k;
  s->c_thres = c_thres;
  s->rng = seed;
  s->policy = policy;
  s->nodes = nodes;
  for (int w = 0; w < RP_MAX_WORLD; ++w) {
    s->handed[w] = -1;
    s->pending_of[w] = -1;
  }
  for (auto& g : s->table) g.seq = -1;
}

namespace {
void fill_out(const GGGroup* g, rp_group* out) {
  out->seq = g->seq;
  out->size = g->size;
  for (int t = 0; t < RP_MAX_GROUP; ++t) out->members[t] = t < g->size ? g->members[t] : -1;
}
uint64_t member_bits(const GGGroup* g) {
  uint64_t b = 0;
  for (int t = 0; t < g->size; ++t) b |= 1ull << g->members[t];
  return b;
}
// random GG: lock the group's members and notify them (their inbox = GB)
int grant(GGState* s, GGGroup* g) {
  for (int t = 0; t < g->size; ++t)
    if (s->gb_len[g->members[t]] >= kGbCap) return fail(RP_ESTATE, "inbox overflow");
  s->lock |= member_bits(g);
  g->granted = 1;
  for (int t = 0; t < g->size; ++t) {
    const int m = g->members[t];
    s->gb[m][s->gb_len[m]++] = g->seq;
    s->max_depth = std::max<int64_t>(s->max_depth, s->gb_len[m]);
  }
  s->n_granted++;
  return RP_OK;
}
// after a release, rescan the pending queue in FIFO order; a pending group with a
// retired member is cancelled and its initiator draws again (reading R22).
void rescan(GGState* s) {
  int keep = 0;
  for (int q = 0; q < s->npending; ++q) {
    GGGroup* g = find_slot(s, s->pending[q]);
    if (!g) continue;
    const uint64_t bits = member_bits(g);
    if (s->retired & bits) {
      s->pending_of[g->initiator] = -1;
      g->seq = -1;
      continue;
    }
    if (!(s->lock & bits) && grant(s, g) == RP_OK) {
      s->pending_of[g->initiator] = -1;
      continue;
    }
    s->pending[keep++] = s->pending[q];
  }
  s->npending = keep;
}

// The basic GG of §4.1: serve a notified group, else draw a random group
// containing w (splitmix64 Fisher-Yates, first k-1 others); grant it if no member's lock
// bit is set, otherwise queue it and let w retry.
int random_request(GGState* s, int w, rp_group* out) {
  if (!s->waiting[w]) {
    s->requests++;
    s->counters[w] += 1;
  }
  if (s->gb_len[w] > 0) {
    const GGGroup* g = gg_find(s, s->gb[w][0]);
    if (!g) return fail(RP_ESTATE, "inbox head not in table");
    s->handed[w] = g->seq;
    s->waiting[w] = 0;
    fill_out(g, out);
    return RP_OK;
  }
  if (s->pending_of[w] >= 0) {
    const GGGroup* g = gg_find(s, s->pending_of[w]);
    if (!g) return fail(RP_ESTATE, "pending group not in table");
    s->waiting[w] = 1;
    fill_out(g, out);
    return RP_EAGAIN;
  }
  int cand[RP_MAX_WORLD];
  int nc = 0;
  for (int v = 0; v < s->n; ++v)
    if (v != w && !((s->retired >> v) & 1)) cand[nc++] = v;
  for (int q = nc - 1; q >= 1; --q) {
    const int j = static_cast<int>(next_rand(s) % static_cast<uint64_t>(q + 1));
    std::swap(cand[q], cand[j]);
  }
  int members[RP_MAX_GROUP];
  int sz = 0;
  members[sz++] = w;
  for (int t = 0; t < std::min(s->k - 1, nc); ++t) members[sz++] = cand[t];
  std::sort(members, members + sz);
  GGGroup* slot = find_slot(s, -1);
  if (!slot) return fail(RP_ENOMEM, "GG group table full");
  slot->seq = s->next_seq++;
  slot->size = sz;
  slot->arrived = 0;
  slot->ticket = -1;
  slot->initiator = w;
  slot->granted = 0;
  for (int t = 0; t < sz; ++t) slot->members[t] = members[t];
  fill_out(slot, out);
  if (s->lock & member_bits(slot)) {  // conflict: serialize
    if (s->npending >= kTableCap) return fail(RP_ENOMEM, "pending queue full");
    s->pending[s->npending++] = slot->seq;
    s->pending_of[w] = slot->seq;
    s->waiting[w] = 1;
    s->n_pending++;
    return RP_EAGAIN;
  }
  const int rc = grant(s, slot);
  if (rc != RP_OK) return rc;
  s->handed[w] = slot->seq;
  s->waiting[w] = 0;
  return RP_OK;
}
}  // namespace

const GGGroup* gg_find(const GGState* s, int64_t seq) {
  for (const auto& g : s->table)
    if (g.seq == seq) return &g;
  return nullptr;
}

namespace {
void shuffle(GGState* s, int* v, int n) {  // Fisher-Yates with the GG's splitmix64 stream
  for (int q = n - 1; q >= 1; --q) {
    const int j = static_cast<int>(next_rand(s) % static_cast<uint64_t>(q + 1));
    std::swap(v[q], v[j]);
  }
}

// Create the groups of one division in order and append them to their members' GBs.
// Lock bit w is held while GB[w] is non-empty; a division may only use workers without one.
int push_groups(GGState* s, const std::vector<std::vector<int>>& chunks) {
  const uint64_t before = s->lock;
  for (const auto& ch : chunks) {
    int members[RP_MAX_GROUP];
    const int sz = static_cast<int>(ch.size());
    if (sz < 1 || sz > RP_MAX_GROUP) return fail(RP_EINVAL, "division group size out of range");
    for (int t = 0; t < sz; ++t) members[t] = ch[t];
    std::sort(members, members + sz);
    uint64_t bits = 0;
    for (int t = 0; t < sz; ++t) bits |= 1ull << members[t];
    if (before & bits) return fail(RP_ECONFLICT, "division produced a group overlapping a held lock");
    GGGroup* slot = find_slot(s, -1);
    if (!slot) return fail(RP_ENOMEM, "GG group table full");
    for (int t = 0; t < sz; ++t)
      if (s->gb_len[members[t]] >= kGbCap) return fail(RP_ESTATE, "Group Buffer overflow");
    s->lock |= bits;
    slot->seq = s->next_seq++;
    slot->size = sz;
    slot->arrived = 0;
    slot->ticket = -1;
    slot->initiator = -1;
    slot->granted = 1;
    for (int t = 0; t < sz; ++t) {
      const int m = members[t];
      slot->members[t] = m;
      s->gb[m][s->gb_len[m]++] = slot->seq;
      s->max_depth = std::max<int64_t>(s->max_depth, s->gb_len[m]);
    }
  }
  return RP_OK;
}

void chunk_into(std::vector<std::vector<int>>* out, const int* v, int n, int k) {
  for (int p = 0; p < n; p += k) out->emplace_back(v + p, v + std::min(n, p + k));
}
}  // namespace

static int global_division(GGState* s, int i) {
  s->gd_calls++;
  int cand[RP_MAX_WORLD];
  int nc = 0;
  for (int v = 0; v < s->n; ++v) {
    if (v == i || s->gb_len[v] > 0 || ((s->retired >> v) & 1)) continue;
    if (s->c_thres > 0 && !(s->counters[i] - s->counters[v] < s->c_thres)) continue;
    cand[nc++] = v;
  }
  std::vector<std::vector<int>> chunks;
  if (s->nodes <= 0) {
    // [i] + cand[0:k-1], then consecutive chunks of k (reading R8)
    shuffle(s, cand, nc);
    std::vector<int> first{i};
    for (int t = 0; t < std::min(s->k - 1, nc); ++t) first.push_back(cand[t]);
    chunks.push_back(first);
    const int used = std::min(s->k - 1, nc);
    chunk_into(&chunks, cand + used, nc - used, s->k);
    return push_groups(s, chunks);
  }
  // §5.2 Inter-Intra Synchronization as two rounds of one division (reading
  // R23): Inter = one Head Worker per node (rotating over the node's idle workers, ascending)
  // grouped across nodes at random, the other idle workers grouped with their own node;
  // Intra = one group of the node's idle workers per node. Inter groups precede Intra groups
  // in every GB.
  int idle[RP_MAX_WORLD];
  int ni = 0;
  for (int v = 0; v < s->n; ++v) {
    bool in = v == i;
    for (int t = 0; t < nc && !in; ++t) in = cand[t] == v;
    if (in) idle[ni++] = v;
  }
  const int m = s->n / s->nodes;
  int heads[RP_MAX_WORLD];
  int nh = 0;
  uint64_t head_bits = 0;
  for (int a = 0; a < s->nodes; ++a) {
    int cnt = 0;
    for (int t = 0; t < ni; ++t) cnt += idle[t] / m == a;
    if (!cnt) continue;
    const int pick = s->head_rot[a] % cnt;
    s->head_rot[a]++;
    int seen = 0;
    for (int t = 0; t < ni; ++t)
      if (idle[t] / m == a && seen++ == pick) {
        heads[nh++] = idle[t];
        head_bits |= 1ull << idle[t];
      }
  }
  shuffle(s, heads, nh);
  chunk_into(&chunks, heads, nh, s->k);
  for (int a = 0; a < s->nodes; ++a) {
    int loc[RP_MAX_WORLD];
    int nl = 0;
    for (int t = 0; t < ni; ++t)
      if (idle[t] / m == a && !((head_bits >> idle[t]) & 1)) loc[nl++] = idle[t];
    shuffle(s, loc, nl);
    chunk_into(&chunks, loc, nl, s->k);
  }
  for (int a = 0; a < s->nodes; ++a) {
    std::vector<int> node;
    for (int t = 0; t < ni; ++t)
      if (idle[t] / m == a) node.push_back(idle[t]);
    if (!node.empty()) chunks.push_back(node);
  }
  return push_groups(s, chunks);
}

int gg_request(GGState* s, int w, rp_group* out) {
  if (w < 0 || w >= s->n) return fail(RP_EINVAL, "gg_request: worker out of range");
  if ((s->retired >> w) & 1) return fail(RP_ESTATE, "gg_request: worker " + std::to_string(w) + " is retired");
  if (s->handed[w] != -1)
    return fail(RP_ESTATE, "gg_request: worker " + std::to_string(w) + " still holds group " +
                               std::to_string(s->handed[w]));
  if (s->policy == kPolicyRandom) return random_request(s, w, out);
  s->requests++;
  s->counters[w] += 1;  // reading R10: counted at request time
  if (s->gb_len[w] == 0) {
    const int rc = global_division(s, w);
    if (rc != RP_OK) return rc;
  }
  const int64_t seq = s->gb[w][0];
  const GGGroup* g = gg_find(s, seq);
  if (!g) return fail(RP_ESTATE, "gg_request: GB head not in table");
  s->handed[w] = seq;
  out->seq = seq;
  out->size = g->size;
  for (int t = 0; t < RP_MAX_GROUP; ++t) out->members[t] = t < g->size ? g->members[t] : -1;
  return RP_OK;
}

int gg_done(GGState* s, int64_t seq, rp_group* released) {
  GGGroup* g = find_slot(s, seq);
  if (!g || seq < 0) return fail(RP_EPROTO, "gg_done: unknown group " + std::to_string(seq));
  for (int t = 0; t < g->size; ++t) {
    const int m = g->members[t];
    if (s->gb_len[m] == 0 || s->gb[m][0] != seq)
      return fail(RP_EPROTO, "gg_done: group " + std::to_string(seq) + " not at the head of worker " +
                                 std::to_string(m) + "'s Group Buffer");
    if (s->handed[m] != seq)
      return fail(RP_EPROTO, "gg_done: member " + std::to_string(m) + " never requested group " +
                                 std::to_string(seq));
  }
  if (released) {
    released->seq = seq;
    released->size = g->size;
    for (int t = 0; t < RP_MAX_GROUP; ++t) released->members[t] = t < g->size ? g->members[t] : -1;
  }
  for (int t = 0; t < g->size; ++t) {
    const int m = g->members[t];
    for (int q = 1; q < s->gb_len[m]; ++q) s->gb[m][q - 1] = s->gb[m][q];
    s->gb_len[m]--;
    s->handed[m] = -1;
    if (s->gb_len[m] == 0) s->lock &= ~(1ull << m);
    if ((s->retiring >> m) & 1) {  // reading R19: retire atomically with the completion
      s->retiring &= ~(1ull << m);
      s->retired |= 1ull << m;
    }
  }
  g->seq = -1;
  if (s->policy == kPolicyRandom) rescan(s);
  return RP_OK;
}

int gg_retire(GGState* s, int w) {
  if (w < 0 || w >= s->n) return fail(RP_EINVAL, "gg_retire: worker out of range");
  if (s->handed[w] != -1) {
    s->retiring |= 1ull << w;
  } else {
    s->retired |= 1ull << w;
    if (s->policy == kPolicyRandom) rescan(s);
  }
  return RP_OK;
}

}  // namespace rp
