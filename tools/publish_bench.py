"""Per-tick cost of publishing snapshots (World._publish, core.py:477-485, at
every tick) for one quadrotor group: the reference-shaped float64 pull
(``snapshot``, what World does with any group), the synchronous device-packed
frame (``wire.snapshot_frame``), and ``publish.FramePublisher`` (device pack +
pinned copy on a side stream, delivered by a worker thread).

  python tools/publish_bench.py [N ...]      -> one JSON line per N
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_12698_b200 import B200QuadGroup, batch_create  # noqa: E402
from paper_2308_12698_b200.publish import FramePublisher  # noqa: E402
from paper_2308_12698_b200.wire import snapshot_frame  # noqa: E402


def per_tick(fn, ticks):
    for t in range(3):
        fn(t)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in range(ticks):
        fn(t)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / ticks * 1e3


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [5_000, 100_000, 1_000_000]
    for n in sizes:
        ticks = 200 if n <= 100_000 else 40
        g = B200QuadGroup(0, batch_create(0, n, np.random.default_rng(0).uniform(-50, 50, (n, 3))))
        sink = {"bytes": 0}

        def consume(frame):
            sink["bytes"] += len(frame)

        row = {"n": n, "frame_bytes": len(snapshot_frame(0, [g]))}
        row["step_only_ms"] = per_tick(lambda t: g.step(1e-3), ticks)
        row["step_f64_snapshot_ms"] = per_tick(lambda t: (g.step(1e-3), g.snapshot(t)), ticks)
        row["step_frame_sync_ms"] = per_tick(lambda t: consume(snapshot_frame(t, [g]) if g.step(1e-3) is not None
                                                               else b""), ticks)
        pub = FramePublisher([g], [consume], slots=3)

        def pub_tick(t):
            g.step(1e-3)
            pub.publish(t)
        t_pub = per_tick(pub_tick, ticks)
        t0 = time.perf_counter()
        pub.flush()
        drain = (time.perf_counter() - t0) * 1e3
        row["step_publisher_ms"] = t_pub + drain / ticks     # every frame delivered
        row["publisher_drain_ms"] = drain
        row["publisher_delivered"] = pub.delivered
        pub.close()
        print(json.dumps(row), flush=True)
        del g, pub
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
