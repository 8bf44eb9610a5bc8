"""Rebuild profiles/traffic.json (the per-launch counters bench.py reports as
``roofline.traffic`` and ``roofline_onchip``) from the tracked ncu summaries,
so every number in it has a line in a committed profiles/*.txt file.
Usage: python profiles/make_traffic.py"""
import json
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "r2b_pair4096_ncu_full.txt"


def parse(path):
    out, cur = {}, None
    for ln in open(path):
        if ln.startswith("=="):
            cur = "forward" if "fwd_sym_kernel" in ln else "backward" if "bwd_sym8" in ln else None
            if cur in out:          # first launch of each kernel only
                cur = None
            elif cur:
                out[cur] = {}
            continue
        if cur is None:
            continue
        m = re.match(r"\s+(\S.*?)\s{2,}([-0-9.eE+]+)\s*(\S*)\s*$", ln)
        if m:
            out[cur][m.group(1).strip()] = (float(m.group(2)), m.group(3))
    return out


def main():
    k = parse(os.path.join(HERE, SRC))
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = {"_source": f"profiles/{SRC} (ncu --set full --clock-control none, n = 4096 config-3 "
                      "pair, default dispatch); bytes = dram__bytes_read.sum + "
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
