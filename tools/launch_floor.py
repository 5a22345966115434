"""Launch-latency floor of a CUDA graph of n dependent tiny kernels (what one Split Bregman iteration of a
small image costs in launches alone: 13 kernels at S = 3).  Uses trivial torch elementwise kernels; prints
microseconds per kernel node for chains of 13 x 32 nodes.   python tools/launch_floor.py"""
import json
import torch


def main():
    dev = torch.device("cuda", 0)
    x = torch.zeros(1024, device=dev)
    s = torch.cuda.Stream()
    out = {}
    with torch.cuda.stream(s):
        for nodes in (13 * 8, 13 * 32):
            g = torch.cuda.CUDAGraph()
            x.add_(1.0)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(nodes):
                    x.add_(1.0)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            e0.record(s)
            for _ in range(reps):
                g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            out[f"graph_{nodes}_nodes_us_per_kernel"] = e0.elapsed_time(e1) * 1e3 / (reps * nodes)
        # plain stream launches (no graph)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 2000
        for _ in range(100):
            x.add_(1.0)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(n):
            x.add_(1.0)
        e1.record(s)
        torch.cuda.synchronize()
        out["stream_us_per_kernel"] = e0.elapsed_time(e1) * 1e3 / n
    print(json.dumps(out))


if __name__ == "__main__":
    main()
