"""profiles/traffic.json (bench.py's roofline.traffic) from ncu raw pages.

    python tools/make_traffic.py TAG      # reads gpurun_out/TAG_ncu_raw_cfg{1,2,4}.csv
Per launch: dram__bytes_read.sum + dram__bytes_write.sum of the first captured launch of
each hot kernel (ncu --set full, --clock-control none; tools/measure_round.sh).
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
# kernel-name fragment -> bench.py kernel label, per BASELINE config
MAP = {
    2: [("k_reorder", "cell build (reorder pass)"), ("k_nlist_pair", "neighbour-list build"),
        ("k_wcsph_density_pair", "density+EOS"), ("k_wcsph_momentum_pair", "momentum G11+A"),
        ("k_symplectic", "symplectic integrator")],
    1: [("k_sph_fast", None)],  # first launch sph_S, second the fused G11+L0
    4: [("k_gravity_fast", "all-pairs gravity")],
}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    k, r, w = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    for row in rows[2:]:
        yield row[k], float(row[r]) * SCALE[units[r]] + float(row[w]) * SCALE[units[w]]


def main():
    tag = sys.argv[1]
    out = {}
    for cfg, table in MAP.items():
        path = os.path.join(ROOT, "gpurun_out", f"{tag}_ncu_raw_cfg{cfg}.csv")
        if not os.path.exists(path):
            continue
        d = {}
        seen = 0
        for name, total in launches(path):
            for frag, label in table:
                if frag not in name:
                    continue
                if cfg == 1:
                    label = ("sph_S density", "sph_G11+L0 fused")[min(seen, 1)]
                    seen += 1
                d.setdefault(label, int(total))
        d["_source"] = (f"profiles/{tag}_ncu_full_cfg{cfg}.md (ncu --set full, one launch each, fast mode, "
                        "the bench's build); dram__bytes_read.sum + dram__bytes_write.sum per launch")
        out[f"cfg{cfg}"] = d
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
