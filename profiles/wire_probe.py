import sys, json, socket
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2405_02969_b200 as pb
from oracle import ref as R
from test_gpu_wire import wire_config
out = {}
for W, nbytes in ((8, 64 << 20), (4, 1 << 16), (64, 1 << 20)):
    text = wire_config(W, alpha=10.0, beta=0.001, gamma=0.0001)
    with R.Emulator(text):
        comm = pb.Communicator(text, 0, 0)
        comm.attach_emulator([pb.CollectivePlanEntry("allreduce", nbytes, 4)])
        x = torch.zeros(nbytes // 4, dtype=torch.int32, device="cuda")
        lates, totals = [], []
        for it in range(4):
            comm.all_reduce(x, x)
            rec = comm.call_record()
            rel = (np.array(rec["release_ns"]) - rec["t_start_ns"]) / 1e3
            lates.append(float(np.max(rel - rec["floors_us"])))
            totals.append(float((rec["t_end_ns"] - rec["t_start_ns"]) / 1e3))
        comm.close()
    out[f"W{W}_{nbytes}B"] = {"model_latency_us": int(rec["model_latency_us"]), "steps": int(rec["steps"]),
                              "wire_call_us": totals, "max_late_vs_floor_us": lates}
    # device mode, same config minus endpoints
    dev = pb.Communicator("\n".join(l for l in text.splitlines() if not l.startswith("endpoint")) + "\npayload.mode = zero\n", 0, 0)
    for it in range(3):
        dev.all_reduce(x, x)
    torch.cuda.synchronize()
    r2 = dev.call_record()
    rel2 = (np.array(r2["release_ns"]) - r2["t_start_ns"]) / 1e3
    out[f"W{W}_{nbytes}B"]["device_max_late_vs_floor_us"] = float(np.max(rel2 - r2["floors_us"]))
    dev.close()
print(json.dumps(out, indent=1))
