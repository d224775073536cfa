// Per-rank PipeFusion plan (see rank_plan.h). The op order restates
// run_pipefusion_threads' worker loop (/root/reference/proj/src/execute.cpp:
// 231-385): worker 0 applies each returned eps before it builds the next
// input (:286-291, :305-315), every worker receives, runs its layers and
// sends on (:292-300, :316-325), and worker 0 drains the last step's eps
// messages before returning x (:329-343).
#include "rank_plan.h"

#include <algorithm>

namespace pf {

int64_t plan_messages_per_run(int steps, int patches, int warmup) {
  return int64_t(warmup) + int64_t(steps - warmup) * patches;
}

std::vector<PlanOp> build_rank_plan(int rank, int world, int steps, int patches, int warmup,
                                    int64_t seq_len) {
  std::vector<PlanOp> ops;
  const int P = int(seq_len);
  const int r = P / patches;
  const bool first = rank == 0;
  int m_out = 0, m_in = 0;
  // sender-side row bookkeeping: last message that wrote the full sequence /
  // each patch's rows at the receiver
  int last_full = 0;
  std::vector<int> last_patch(size_t(patches), 0);
  auto op = [&](int kind, int t, int patch, int msg = 0, int overlap = 0, int flag = 0) {
    PlanOp o;
    o.kind = kind;
    o.t = t;
    o.patch = patch;
    o.row0 = patch < 0 ? 0 : patch * r;
    o.rows = patch < 0 ? P : r;
    o.msg = msg;
    o.overlap = overlap;
    o.flag = flag;
    ops.push_back(o);
  };
  auto send = [&](int t, int patch) {
    ++m_out;
    int ov = last_full;
    if (patch < 0) {
      for (int v : last_patch) ov = std::max(ov, v);
      last_full = m_out;
    } else {
      ov = std::max(ov, last_patch[size_t(patch)]);
      last_patch[size_t(patch)] = m_out;
    }
    op(PlanOp::kSend, t, patch, m_out, ov);
  };

  // Rank 0 consumes a returned eps message: wait, update the latent rows
  // (full: LatentUpdate; patch: folded into the next Prepare), acknowledge.
  auto recv_eps_full = [&](int t) {
    op(PlanOp::kRecv, t, -1, ++m_in);
    op(PlanOp::kLatentUpdate, t, -1);
    op(PlanOp::kAck, t, -1, m_in, 0, 0);
  };

  // ---- warmup: synchronous full-sequence steps (execute.cpp:284-301)
  for (int w = 0; w < warmup; ++w) {
    const int t = steps - 1 - w;
    if (first) {
      if (w > 0) recv_eps_full(t + 1);
      op(PlanOp::kPrepare, t, -1, 0, 0, 0);
    } else {
      op(PlanOp::kRecv, t, -1, ++m_in);
    }
    op(PlanOp::kCompute, t, -1);
    send(t, -1);
    if (!first) op(PlanOp::kAck, t, -1, m_in, 0, 1);
  }
  // ---- steady: patch pipeline (execute.cpp:303-328)
  const int steady = steps - warmup;
  for (int q = 0; q < steady; ++q) {
    const int t = steady - 1 - q;
    for (int j = 0; j < patches; ++j) {
      if (first) {
        if (q == 0 && j == 0 && warmup > 0) recv_eps_full(t + 1);
        if (q > 0) op(PlanOp::kRecv, t + 1, j, ++m_in);
        op(PlanOp::kPrepare, t, j, 0, 0, q > 0 ? 1 : 0);
        if (q > 0) op(PlanOp::kAck, t + 1, j, m_in, 0, 0);
      } else {
        op(PlanOp::kRecv, t, j, ++m_in);
      }
      op(PlanOp::kCompute, t, j);
      send(t, j);
      if (!first) op(PlanOp::kAck, t, j, m_in, 0, 1);
    }
  }
  // ---- rank 0 drains the last eps messages (execute.cpp:331-345)
  if (first) {
    if (steady > 0) {
      for (int j = 0; j < patches; ++j) op(PlanOp::kRecv, 0, j, ++m_in);
      op(PlanOp::kLatentUpdate, 0, -1);
      op(PlanOp::kAck, 0, -1, m_in, 0, 0);
    } else if (warmup > 0) {
      recv_eps_full(0);
    }
  }
  (void)world;
  return ops;
}

}  // namespace pf
