"""Encode-kernel section timing (experiment; needs a library built with
-DENC_TIMING, passed via LUDA_LIB). Prints clock64 cycles per block for each
builder / CRC warp section of encode_kernel on the c3 bench job."""
import ctypes, json, os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
NAMES = {0: "b:empty_wait", 1: "b:load_next", 2: "b:assemble(hdr)", 4: "b:tma_wait", 5: "b:realign", 3: "b:layout_next",
         6: "b:issue_next", 7: "b:publish", 8: "c:full_wait", 9: "c:crc+copyout"}

def main():
    import torch
    import bench
    from paper_2004_03054_b200 import _native
    torch.cuda.set_device(0)
    L = _native.lib(0)
    L.luda_dbg_enc_timing.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    w = bench.synth_c3(int(os.environ.get("KEYS", 1 << 25)), seed=0xC3, device_index=0)
    desc, keep = bench.job_desc(w, w.arena.data_ptr())
    t = (ctypes.c_ulonglong * 16)()
    for i in range(3):
        L.luda_dbg_enc_timing(t, 1)
        res = _native.JobResult()
        L.luda_compact(ctypes.byref(desc), ctypes.byref(res), w.stream)
        torch.cuda.synchronize()
        nblk = res.blocks_out
        ms = res.k_ms[3]
        L.luda_job_release(ctypes.byref(res))
    L.luda_dbg_enc_timing(t, 0)
    nb = int(os.environ.get("NBLK", 0)) or nblk
    out = {NAMES.get(i, str(i)): (t[i] / nb if nb else t[i]) for i in range(16) if t[i]}
    print(json.dumps({"encode_ms": ms, "nblk": nb, "cycles_per_block": out}))

if __name__ == "__main__":
    main()
