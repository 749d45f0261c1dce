"""Per-step decode / job times of the c3 job (experiment): runs the job
`steps` times back to back and prints each step's decode kernel ms (CUDA
events) and job ms, to expose launch-to-launch variance.
Usage: [LUDA_LIB=...] python profiles/decode_steps.py [steps]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch
    from paper_2004_03054_b200 import _native
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    L = _native.lib(0)
    w = bench.synth_c3(1 << 25, seed=0xC3, device_index=0)
    desc, keep = bench.job_desc(w, w.arena.data_ptr())
    st = w.stream
    torch.cuda.synchronize()
    dec = []
    for i in range(steps):
        r = bench.compact_once(L, desc, st)
        dec.append(r.k_ms[0])
        print(f"step {i} decode {r.k_ms[0]:.3f} merge {r.k_ms[1]:.3f} encode {r.k_ms[3]:.3f} meta {r.k_ms[4]:.3f} "
              f"phases {sum(r.t_ms[:5]):.3f}", flush=True)
        L.luda_job_release(ctypes.byref(r))
    print("decode min %.3f max %.3f mean %.3f" % (min(dec), max(dec), sum(dec) / len(dec)))


if __name__ == "__main__":
    main()
