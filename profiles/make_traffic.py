"""Rebuild profiles/traffic.json (the per-launch counters bench.py reports as
``roofline.traffic`` and ``roofline_onchip``) from the tracked ncu summaries,
so every number in it has a line in a committed profiles/*.txt file.
Usage: python profiles/make_traffic.py"""
import json
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "r2c_pair4096_ncu_full.txt"
FWD_PASSES = 4          # banded passes of the n = 4096 forward (projector_fast.cu)


def parse(path):
    """Per-product counters: the forward of one product is FWD_PASSES banded
    launches of fwd_sym_kernel (summed), the backward one bwd_sym8 launch."""
    launches = {"forward": [], "backward": []}
    cur = None
    for ln in open(path):
        if ln.startswith("=="):
            cur = "forward" if "fwd_sym_kernel" in ln else "backward" if "bwd_sym8" in ln else None
            if cur:
                launches[cur].append({})
            continue
        if cur is None:
            continue
        m = re.match(r"\s+(\S.*?)\s{2,}([-0-9.eE+]+)\s*(\S*)\s*$", ln)
        if m:
            v, u = float(m.group(2)), m.group(3)
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                     "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
            if u in scale:      # common units so the banded launches can be summed
                v, u = v * scale[u], ("byte" if "byte" in u else "us")
            launches[cur][-1][m.group(1).strip()] = (v, u)
    out = {}
    for kern, want in (("forward", FWD_PASSES), ("backward", 1)):
        ls = launches[kern][:want]
        assert len(ls) == want, (kern, len(ls))
        agg = {}
        for d in ls:
            for k, (v, u) in d.items():
                if k.endswith(".pct") or "pct_of_peak" in k or k.startswith("launch__"):
                    continue
                agg[k] = (agg.get(k, (0.0, u))[0] + v, u)
        out[kern] = agg
    return out


def main():
    k = parse(os.path.join(HERE, SRC))
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = {"_source": f"profiles/{SRC} (ncu --set full --clock-control none, n = 4096 config-3 "
                      "pair, default dispatch; the forward = its 4 banded launches summed); bytes = dram__bytes_read.sum + "
                      "dram__bytes_write.sum; L1 data-pipe wavefronts = per-SM average x 148"}
    for kern in ("forward", "backward"):
        d = k[kern]
        rd, ru = d["dram__bytes_read.sum"]
        wr, wu = d["dram__bytes_write.sum"]
        res[f"{kern}_n4096"] = int(rd * unit[ru] + wr * unit[wu])
        res[f"l1_datapipe_wavefronts_{kern}_n4096"] = int(
            d["l1tex__data_pipe_lsu_wavefronts (per-SM avg x 148)"][0])
        res[f"l1_sectors_{kern}_n4096"] = int(d["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"][0])
        if kern == "backward":
            res["smem_wavefronts_backward_n4096"] = int(
                d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"][0])
    with open(os.path.join(HERE, "traffic.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
