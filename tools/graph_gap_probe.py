"""Per-node cost of a CUDA graph replay on this GPU: a chain of n dependent
kernels, tiny (launch-bound) and ~5 us (HBM-bound), replayed from a graph
and compared with the kernels' own duration (CUDA events around a single
launch averaged over many).  Tells how much of the ResNet20 step's ~10k
launches is inter-kernel gap rather than kernel time."""
import json
import torch


def timed(fn, reps=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main():
    out = {}
    for label, numel in (("tiny", 1), ("hbm_5us", 4 << 20), ("hbm_20us", 16 << 20)):
        x = torch.zeros(numel, device="cuda")
        n = 2000
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(3):
                x.add_(1.0)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(n):
                    x.add_(1.0)
        t_graph = timed(g.replay) / n * 1e3
        t_stream = timed(lambda: [x.add_(1.0) for _ in range(n)]) / n * 1e3
        out[label] = {"bytes": numel * 8, "graph_us_per_node": round(t_graph, 3),
                      "stream_us_per_launch": round(t_stream, 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
