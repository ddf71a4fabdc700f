"""One rank of a 2-process ledger scenario on the CPU (tests/test_ledger.py):
the POSIX-shm matching ledger shared by processes, torch.distributed (gloo,
127.0.0.1) as plumbing to pass the segment name and gather results."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def run(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1802_06949_b200 import DeadlockTimeout, MismatchError, TraceSink, Transport

    dist.init_process_group("gloo", rank=rank, world_size=world)
    name = [f"csb_cpu_{os.getpid()}_{time.time_ns() % 10**9}"]
    dist.broadcast_object_list(name, src=0)
    sink = TraceSink()
    tr = Transport.ledger_only(world, 300 if case != "order" else 5000, sink, name=name[0], rank=rank)
    out = {"rank": rank}
    try:
        if case == "order":
            extra = tr.new_communicator()
            for it in range(20):
                tr.allreduce_sum(0, rank, 0, trace_key=it, dtype=1, count=4 + it)
                if it % 3 == 0:
                    tr.allreduce_sum(extra, rank, 0, trace_key=it, dtype=1, count=7)
                if rank == 1 and it % 5 == 0:
                    time.sleep(0.01)  # arrival skew, consistent schedule
            tr.barrier(0, rank)
            out["events"] = [(e["event"], e["comm"], e["seq"], e.get("key", -1)) for e in sink.snapshot()
                             if e["event"] == "coll_enqueued"]
        elif case == "mismatch":
            tr.allreduce_sum(0, rank, 0, dtype=1, count=4 if rank == 0 else 5)
        elif case == "deadlock":
            if rank == 0:
                tr.barrier(0, 0)
            else:
                time.sleep(1.0)
    except MismatchError as e:
        out["error"], out["message"] = "MismatchError", str(e)
    except DeadlockTimeout as e:
        out["error"], out["message"] = "DeadlockTimeout", str(e)
    dist.barrier()
    tr.close()
    q.put(out)
    dist.destroy_process_group()
