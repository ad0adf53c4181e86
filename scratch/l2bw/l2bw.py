"""Measure the B200's L2 read throughput (bytes/clk) for bench.py's L2
roofline; writes profiles/l2_peak.json."""
import ctypes, json, os, subprocess, sys, threading, time
sys.path.insert(0, os.getcwd())
import torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libl2bw.so"))
lib.l2_read_bw.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]
out = torch.zeros(1, dtype=torch.float64, device="cuda")
res = []
clk = []
def sample():
    import pynvml
    pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop[0]:
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)); time.sleep(0.02)
for mb in (16, 32, 48, 64):
    buf = torch.ones(mb * 2**20 // 8, dtype=torch.float64, device="cuda")
    for blocks_per_sm, threads in ((8, 256), (16, 256), (4, 1024)):
        stop = [False]; clk.clear(); th = threading.Thread(target=sample); th.start()
        ms = ctypes.c_float()
        reps = 200
        lib.l2_read_bw(buf.data_ptr(), buf.numel() * 8, reps, 148 * blocks_per_sm, threads,
                       out.data_ptr(), ctypes.byref(ms))
        stop[0] = True; th.join()
        gbs = buf.numel() * 8 * reps / (ms.value * 1e-3) / 1e9
        mhz = sorted(clk)[len(clk) // 2] if clk else 1965
        res.append({"MB": mb, "blocks_per_sm": blocks_per_sm, "threads": threads, "GBps": gbs,
                    "sm_mhz": mhz, "B_per_clk": gbs * 1e9 / (mhz * 1e6)})
        print(res[-1], flush=True)
best = max(res, key=lambda r: r["B_per_clk"])
json.dump({"l2_read_bytes_per_clk": best["B_per_clk"], "best": best, "runs": res,
           "how": "scratch/l2bw: 16-byte ld.global.cg over an L2-resident buffer, 200 passes, CUDA events; SM clock sampled with NVML"},
          open("profiles/l2_peak.json", "w"), indent=1)
