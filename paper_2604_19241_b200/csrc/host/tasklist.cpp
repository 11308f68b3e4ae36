// eplab::build_task_list -- the per-rank task layout of the Dispatch+GroupGEMM MegaKernel, restating
// the reference's sim.cpp:226-250 (with even_slices :151-161, transmission_balanced_slices :168-185 and
// the rowgroup layout of make_layout :131-149) on top of this library's own token map and schedule.
#include <set>
#include <utility>

#include "eplab/eplab.hpp"

namespace eplab {

const char* role_name(Role r) {
  switch (r) {
    case Role::Comm: return "comm";
    case Role::Relay: return "relay";
    case Role::Comp: return "comp";
    case Role::Reduce: return "reduce";
  }
  return "?";
}

namespace {

using Ranges = std::vector<std::pair<long long, long long>>;

// n items in `parts` contiguous ranges whose lengths differ by at most one (the longer ones first)
Ranges split_even(long long n, long long parts) {
  Ranges out;
  for (long long p = 0, lo = 0; p < parts; ++p) {
    const long long len = n / parts + (p < n % parts ? 1 : 0);
    out.emplace_back(lo, lo + len);
    lo += len;
  }
  return out;
}

// contiguous ranges that each end once (p + 1) / parts of all transmissions are covered; the last
// range takes the remainder; no transmissions at all -> the even split
Ranges split_by_transmissions(const std::vector<char>& sends, long long parts) {
  if (parts <= 0) return {};
  long long total = 0;
  for (char c : sends) total += c;
  const long long n = (long long)sends.size();
  if (total == 0) return split_even(n, parts);
  Ranges out;
  long long lo = 0, idx = 0, covered = 0;
  for (long long p = 0; p < parts; ++p) {
    const long long target = total * (p + 1) / parts;
    while (idx < n && covered < target) covered += sends[(size_t)idx++];
    const long long hi = p + 1 == parts ? n : idx;
    out.emplace_back(lo, hi);
    lo = hi;
  }
  return out;
}

}  // namespace

TaskQueueInfo build_task_list(const MoEShape& shape, const TuneConfig& cfg, const RoutingInstance& routing,
                              int rank) {
  if (rank < 0 || rank >= routing.world) throw ValidationError("rank out of range");
  const std::vector<GlobalTokenMap> maps = build_global_token_map(routing);
  const GlobalTokenMap& map = maps[(size_t)rank];
  // up-GEMM tiles of this rank: rowgroups of b_m rows per local expert segment x column tiles of 2F
  const long long col_tiles = (2LL * shape.h_inter + shape.b_n - 1) / shape.b_n;
  long long rowgroups = 0, received = 0;
  for (int e = 0; e < map.experts_per_rank; ++e) {
    const long long rows = map.recv_total(map.rank, e);
    rowgroups += (rows + shape.b_m - 1) / shape.b_m;
    received += rows;
  }
  const long long tiles = rowgroups * col_tiles;
  if (tiles == 0 && received > 0) throw ValidationError("zero tiles with nonzero tokens (shape inconsistency)");
  // NVLink transmissions of the schedule: the first (token, destination rank) in priority order
  // (with one rank nothing crosses a link)
  const SendSchedule sched = build_send_schedule(map);
  std::vector<char> sends(sched.items.size(), 0);
  if (routing.world > 1) {
    std::set<std::pair<long long, int>> seen;
    for (size_t i = 0; i < sched.items.size(); ++i)
      sends[i] = seen.insert({sched.items[i].token, sched.items[i].dst_rank}).second ? 1 : 0;
  }
  TaskQueueInfo tq;
  tq.n_comm = cfg.n_disp;
  tq.n_relay = cfg.n_relay;
  tq.n_comp = tiles;
  tq.comm_slices = split_by_transmissions(sends, cfg.n_disp);
  tq.relay_ranges = cfg.n_relay > 0 ? split_even(tiles, cfg.n_relay) : Ranges{};
  return tq;
}

}  // namespace eplab
