"""Host<->device copy bandwidth on the bench box: H2D alone, D2H alone and both
directions concurrently (two streams), pinned buffers, per size.  Bounds the
e2e (host-buffer) SpMV: 4 MB of x in and 4 MB of y out per C2 step."""
import json
import torch

out = {}
for mb in (4, 64):
    nb = mb << 20
    hx = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
    hy = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
    dx = torch.empty(nb // 4, device="cuda")
    dy = torch.empty(nb // 4, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    reps = 50 if mb == 4 else 10

    def run(h2d, d2h):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_event(e0)
        s2.wait_event(e0)
        for _ in range(reps):
            if h2d:
                with torch.cuda.stream(s1):
                    dx.copy_(hx, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    hy.copy_(dy, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    run(True, True)
    t_h = run(True, False)
    t_d = run(False, True)
    t_b = run(True, True)
    out[f"{mb}MB"] = {"h2d_us": t_h * 1e3, "d2h_us": t_d * 1e3, "both_us": t_b * 1e3,
                      "h2d_GBs": nb / t_h / 1e6, "d2h_GBs": nb / t_d / 1e6,
                      "both_GBs_total": 2 * nb / t_b / 1e6}
print(json.dumps(out))
