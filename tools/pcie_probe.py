"""PCIe probe for the e2e line: pinned H2D / D2H alone and concurrent, at the
C3 step's byte counts (43 MB up, 83 MB down) and with a smaller upload."""
import torch


def main():
    dev = torch.device("cuda:0")
    MB = 1 << 20
    down = 82944000
    res = {}
    for up in (43258368, 35394648, 23597568, 0):
        hu = torch.empty(max(up, 1), dtype=torch.uint8).pin_memory()
        du = torch.empty(max(up, 1), dtype=torch.uint8, device=dev)
        hd = torch.empty(down, dtype=torch.uint8).pin_memory()
        dd = torch.empty(down, dtype=torch.uint8, device=dev)
        s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        for _ in range(3):
            with torch.cuda.stream(s1):
                if up:
                    du.copy_(hu, non_blocking=True)
            with torch.cuda.stream(s2):
                hd.copy_(dd, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 20
        cur = torch.cuda.current_stream(dev)
        e0.record(cur)
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        for _ in range(K):
            with torch.cuda.stream(s1):
                if up:
                    du.copy_(hu, non_blocking=True)
            with torch.cuda.stream(s2):
                hd.copy_(dd, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
        e1.record(cur)
        torch.cuda.synchronize()
        res[up] = e0.elapsed_time(e1) / K
        print(f"up {up / MB:6.1f} MiB + down {down / MB:6.1f} MiB concurrent: {res[up]:.3f} ms per step", flush=True)


if __name__ == "__main__":
    main()
