"""Profiling aid: time the fused residual pass (k_gram) of a bench workload under the
KID_GRAM_DEBUG phase switches (1 skip eval math, 2 skip D = K_N - K_S P2, 4 skip SYRK) and
print the KID_GRAM_TRACE per-phase cycle breakdown. Usage: python tools/gram_probe.py [config]
(PROBE_DBG=comma list of KID_GRAM_DEBUG values; 16 no coordinate loads, 32 exp without table)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "c2-d3"
    wl = bench.WORKLOADS[cfg]
    torch.cuda.set_device(0)
    torch.cuda.set_stream(torch.cuda.Stream())
    dev, prob = bench.setup(wl, 1, 0, 0, torch)
    st = torch.cuda.current_stream()
    dev.set_stream(st.cuda_stream)
    meff = wl["m"] - prob.r
    out = torch.empty(2 + max(meff, 1) ** 2, dtype=torch.float64, device="cuda")
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")

    def timed(reps=10):
        dev.profile(True)
        for _ in range(3):
            flush.zero_()
            dev.recon_error_dev(prob.h, out.data_ptr())
        torch.cuda.synchronize()
        dev.profile_read()
        for _ in range(reps):
            flush.zero_()
            dev.recon_error_dev(prob.h, out.data_ptr())
        torch.cuda.synchronize()
        k = dev.profile_read()
        dev.profile(False)
        return float(np.mean(k))

    print(f"{cfg}: nt={prob.nt} m={wl['m']} r={prob.r}")
    for dbg in [int(x) for x in os.environ.get("PROBE_DBG", "0,1,2,4,3,5,6,7,22,38,54,16,48").split(",")]:
        os.environ["KID_GRAM_DEBUG"] = str(dbg)
        print(f"  dbg={dbg}: k_gram {timed():.4f} ms", flush=True)
    os.environ["KID_GRAM_TRACE"] = "1"
    for dbg in os.environ.get("PROBE_TRACE", "0").split(","):
        os.environ["KID_GRAM_DEBUG"] = dbg
        print(f"  trace dbg={dbg}:", flush=True)
        dev.recon_error_dev(prob.h, out.data_ptr())
        torch.cuda.synchronize()
    os.environ.pop("KID_GRAM_TRACE")


if __name__ == "__main__":
    main()
