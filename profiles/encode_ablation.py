"""Encode-kernel ablation on the c3 bench job (experiment): LUDA_ENC_DBG bits
1 = skip CRC, 2 = skip copy-out, 4 = skip value realignment. Prints the
encode kernel ms per variant (outputs are invalid for nonzero bits)."""
import ctypes, json, os, subprocess, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

def one():
    import torch
    import bench
    from paper_2004_03054_b200 import _native
    torch.cuda.set_device(0)
    L = _native.lib(0)
    dbg = os.environ.pop("LUDA_ENC_DBG", None)  # inputs are built by the same kernel: switch on after synthesis
    w = bench.synth_c3(int(os.environ.get("KEYS", 1 << 25)), seed=0xC3, device_index=0)
    if dbg:
        os.environ["LUDA_ENC_DBG"] = dbg
    desc, keep = bench.job_desc(w, w.arena.data_ptr())
    ts = []
    for i in range(5):
        res = _native.JobResult()
        rc = L.luda_compact(ctypes.byref(desc), ctypes.byref(res), w.stream)
        if rc:
            print("status", rc, L.luda_last_error())
        ts.append(res.k_ms[3])
        L.luda_job_release(ctypes.byref(res))
    print(json.dumps({"dbg": dbg or "0", "encode_ms": sorted(ts[2:])}), flush=True)

if __name__ == "__main__":
    if len(sys.argv) > 1:
        one()
    else:
        for v in ["", "1", "2", "4", "7"]:
            env = dict(os.environ)
            if v:
                env["LUDA_ENC_DBG"] = v
            else:
                env.pop("LUDA_ENC_DBG", None)
            subprocess.run([sys.executable, __file__, "one"], env=env)
