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

void gg_init(GGState* s, int n, int k, int c_thres, uint64_t seed, int policy) {
  std::memset(s, 0, sizeof(*s));
  s->n = n;
  s->k = k;
  s->c_thres = c_thres;
  s->rng = seed;
  s->policy = policy;
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

static int global_division(GGState* s, int i) {
  s->gd_calls++;
  int cand[RP_MAX_WORLD];
  int nc = 0;
  for (int v = 0; v < s->n; ++v) {
    if (v == i || s->gb_len[v] > 0 || ((s->retired >> v) & 1)) continue;
    if (s->c_thres > 0 && !(s->counters[i] - s->counters[v] < s->c_thres)) continue;
    cand[nc++] = v;
  }
  for (int q = nc - 1; q >= 1; --q) {  // Fisher-Yates
    const int j = static_cast<int>(next_rand(s) % static_cast<uint64_t>(q + 1));
    std::swap(cand[q], cand[j]);
  }
  // chunks: [i] + cand[0:k-1], then consecutive chunks of k
  int pos = 0;
  bool first = true;
  while (first || pos < nc) {
    int members[RP_MAX_GROUP];
    int sz = 0;
    if (first) members[sz++] = i;
    const int take = std::min(first ? s->k - 1 : s->k, nc - pos);
    for (int t = 0; t < take; ++t) members[sz++] = cand[pos++];
    first = false;
    std::sort(members, members + sz);
    uint64_t bits = 0;
    for (int t = 0; t < sz; ++t) bits |= 1ull << members[t];
    if (s->lock & bits) return fail(RP_ECONFLICT, "GD produced a group overlapping a held lock");
    GGGroup* slot = find_slot(s, -1);
    if (!slot) return fail(RP_ENOMEM, "GG group table full");
    for (int t = 0; t < sz; ++t)
      if (s->gb_len[members[t]] >= kGbCap) return fail(RP_ESTATE, "Group Buffer overflow");
    s->lock |= bits;
    slot->seq = s->next_seq++;
    slot->size = sz;
    slot->arrived = 0;
    slot->ticket = -1;
    for (int t = 0; t < sz; ++t) {
      const int m = members[t];
      slot->members[t] = m;
      s->gb[m][s->gb_len[m]++] = slot->seq;
      s->max_depth = std::max<int64_t>(s->max_depth, s->gb_len[m]);
    }
  }
  return RP_OK;
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
    s->lock &= ~(1ull << m);
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
