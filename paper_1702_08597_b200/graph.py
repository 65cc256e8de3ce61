"""CUDA-graph capture of a layer step (the B200 answer to a tracing compiler).

At BASELINE configs[1] sizes a fwd+bwd step is ~8 kernel launches of 10–60 µs each, so host
launch latency and inter-kernel gaps are a visible share of the step.  `GraphedStep` runs a
step function a few times eagerly (so every lazily allocated workspace exists), captures one
call into a CUDA graph on a side stream, and replays it with a single launch.  The C-ABI
launches on torch's current stream, so capture works unchanged; buffers passed to the step
must stay fixed (copy new inputs into them before `replay`).
"""
from __future__ import annotations


class GraphedStep:
    def __init__(self, fn, warmup: int = 2):
        import torch

        self.fn = fn
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            fn()
        torch.cuda.synchronize()

    def replay(self):
        self.graph.replay()
