"""profiles/traffic_c3.json from the ncu metric list of the c3 training call
(tools/round_end_check.sh: ncu --metrics dram__bytes_read.sum,
dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum -k regex:som_train
--csv --log-file gpurun_out/traffic_c3.csv python tools/c3_window.py 0 500000).

  python tools/traffic_json.py gpurun_out/traffic_c3.csv profiles/traffic_c3.json"""
import csv
import json
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(src)) if r and not r[0].startswith("==")]
h = rows[0]
ik, im, iv, iu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1, "usecond": 1e3,
         "msecond": 1e6, "second": 1e9}
per = defaultdict(lambda: defaultdict(float))
for r in rows[1:]:
    name = r[ik].split("(")[0].replace("void ", "").replace("som::<unnamed>::", "").strip()
    per[name][r[im]] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
dram = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in per.values())
lts = sum(v["lts__t_bytes.sum"] for v in per.values())
out = {
    "what": "DRAM and L2 bytes of the c3 training call (the full 500,000-step schedule, as in the bench step: "
            "kernel 10 then kernel 4), ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,"
            "gpu__time_duration.sum on tools/c3_window.py 0 500000 (gpurun, one B200)",
    "bytes_per_launch": dram,
    "note": f"bytes_per_launch = DRAM read + write of the whole training call (both launches); L2 traffic "
            f"(lts__t_bytes) {lts / 1e12:.1f} TB; the algorithmic bytes of the sparse method are ~56.9 TB per call",
    "per_kernel": {k: dict(v) for k, v in per.items()},
    "kernel_id": 11,
}
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
