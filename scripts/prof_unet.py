"""U-Net forward timing at 1920x1088 (C4 CNN stage), CUDA events."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import argparse

    import torch

    from paper_2407_19097_b200.neural import UNet, UNetConfig, init_params

    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=5)
    ap.add_argument("--cin", type=int, default=4)
    ap.add_argument("--h", type=int, default=1088)
    ap.add_argument("--w", type=int, default=1920)
    ap.add_argument("--graph", action="store_true",
                    help="capture one forward in a CUDA graph and time replays (no host launch cost)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = UNetConfig(input_channels=a.cin)
    net = UNet(cfg, init_params(cfg), device=dev)
    x = torch.rand((a.h, a.w, a.cin), device=dev)
    y = torch.empty((a.h, a.w, 3), device=dev)
    for _ in range(2):
        net.forward_into(x, y)
    torch.cuda.synchronize()
    run = lambda: net.forward_into(x, y)
    if a.graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                net.forward_into(x, y)
        torch.cuda.current_stream().wait_stream(s)
        run = g.replay
        for _ in range(2):
            run()
        torch.cuda.synchronize()
    print("forward_into graphs:", {k[2:]: type(v).__name__ for k, v in net._graphs.items()})
    for _ in range(a.frames):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"unet {ms:.3f} ms  {413.7e9 / (ms * 1e-3) / 1e12:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
