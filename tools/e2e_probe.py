import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
wl = bench.WORKLOADS["c2-d3"]
torch.cuda.set_device(0)
torch.cuda.set_stream(torch.cuda.Stream())
dev, prob = bench.setup(wl, 1, 0, 0, torch)
dev.set_stream(torch.cuda.current_stream().cuda_stream)
host = torch.from_numpy(prob.pts_cm).pin_memory()
N, d = wl["N"], wl["d"]
for rep in range(4):
    t = [time.perf_counter()]
    dev.set_points_colmajor_ptr(host.data_ptr(), N, d, 0); dev.synchronize(); t.append(time.perf_counter())
    cd, ci = dev.split_candidates(prob.center, wl["m"]); t.append(time.perf_counter())
    src = np.sort(ci); rho = float(cd.max())
    nt = dev.split_finish(src, rho, wl["xi"]); t.append(time.perf_counter())
    tg = dev.targets(); t.append(time.perf_counter())
    dev.recon_prepare(prob.skel, prob.P); t.append(time.perf_counter())
    out = torch.empty(2 + (100 - prob.r) ** 2, dtype=torch.float64, device="cuda")
    dev.recon_error_dev(prob.h, out.data_ptr()); dev.synchronize(); t.append(time.perf_counter())
    o = out.cpu(); t.append(time.perf_counter())
    names = ["h2d_points", "split_candidates", "split_finish", "targets_d2h", "recon_prepare", "recon_pass", "d2h_out"]
    print(" ".join(f"{n}={1e3*(b-a):.3f}ms" for n, a, b in zip(names, t[:-1], t[1:])), f"total={1e3*(t[-1]-t[0]):.3f}ms")
