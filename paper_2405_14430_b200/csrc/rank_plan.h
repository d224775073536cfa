// Per-rank PipeFusion plan for one-process-per-GPU execution.
//
// The reference runs PipeFusion with one jthread per stage exchanging
// PatchMsg values over bounded channels (execute.cpp:225-385,
// run_pipefusion_threads). With one process per GPU the same exchange is a
// sequence of point-to-point messages per stage boundary: rank d sends its
// stage's output rows to rank (d+1) % N -- activations to the next stage,
// and from the last stage the returned noise estimate eps to rank 0.
//
// build_rank_plan() lists, for one rank, the ops it performs in program
// order. The GPU engine (runtime.cpp, Engine::enqueue_rank_run) executes
// exactly this list on its compute / send streams over peer memory, and
// tests/test_rank_plan.py executes it with numpy layers over torch.distributed
// (gloo) to prove it reproduces the single-process result bit for bit.
//
// Messages on each boundary are numbered 1, 2, ... in send order; both ends
// enumerate the same sequence (W full-sequence messages, then one message
// per (steady step, patch) in schedule order), so a message is identified by
// its index alone. Landing rows are reused in place, so before message m is
// written the sender waits until the receiver has acknowledged `overlap`,
// the last earlier message that touched the same rows.
#pragma once

#include <cstdint>
#include <vector>

namespace pf {

struct PlanOp {
  enum Kind : int {
    kPrepare = 0,       // rank 0: [x_j -= eta eps_j]; h_j = x_j + cb   (execute.cpp:198-203)
    kCompute = 1,       // this rank's layers on rows [row0, row0+rows) at timestep t
    kSend = 2,          // rows -> rank (d+1) % N as message `msg`; wait ack >= `overlap` first
    kRecv = 3,          // wait until message `msg` from rank (d-1+N) % N has landed
    kAck = 4,           // tell the sender of message `msg` its rows may be overwritten;
                        // `after_send` != 0: once this rank's send of the same rows finished
    kLatentUpdate = 5,  // rank 0: x -= eta eps over all rows (execute.cpp:189, 212)
  };
  int kind = 0;
  int t = 0;          // timestep (counts down)
  int patch = -1;     // -1: full sequence
  int row0 = 0, rows = 0;
  int msg = 0;        // message index on the boundary (kSend/kRecv/kAck)
  int overlap = 0;    // kSend: last earlier message on the same rows (0: none)
  int flag = 0;       // kPrepare: sampler update; kAck: after_send
};

// Plan of `rank` in a world of `world` stages (world >= 2). Validation of
// (steps, patches, warmup, seq_len) is the caller's (check_pipefusion_args).
std::vector<PlanOp> build_rank_plan(int rank, int world, int steps, int patches, int warmup,
                                    int64_t seq_len);

// Number of messages one run sends on every boundary.
int64_t plan_messages_per_run(int steps, int patches, int warmup);

}  // namespace pf
