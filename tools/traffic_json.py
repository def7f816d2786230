"""profiles/traffic.json from ncu --set full reports: DRAM read / write
bytes and duration per launch of each captured kernel (the bench line's
roofline.traffic).  Usage: traffic_json.py SUFFIX=REPORT ... (the suffix is
appended to the kernel's short name, e.g. _config4; empty for none)."""
import csv
import json
import subprocess
import sys
from pathlib import Path

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3,
        "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}


def rows(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    r = list(csv.reader([l for l in raw if l.startswith('"')]))
    head, units = r[0], r[1]
    for row in r[2:]:
        yield dict(zip(head, row)), dict(zip(head, units))


def main(args):
    out_path = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
    out = json.loads(out_path.read_text()) if out_path.exists() else {}
    for spec in args:
        suffix, path = spec.split("=", 1)
        for d, u in rows(path):
            name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
            name = name.split("::")[-1] + suffix
            e = out.setdefault(name, {"dram_read_bytes": 0, "dram_write_bytes": 0,
                                      "duration_ms": 0.0, "launches": 0, "report": path})
            if e.get("report") != path:
                e.update(dram_read_bytes=0, dram_write_bytes=0, duration_ms=0.0, launches=0,
                         report=path)
            e["dram_read_bytes"] += int(float(d["dram__bytes_read.sum"]) *
                                        UNIT[u["dram__bytes_read.sum"]])
            e["dram_write_bytes"] += int(float(d["dram__bytes_write.sum"]) *
                                         UNIT[u["dram__bytes_write.sum"]])
            e["duration_ms"] += float(d["gpu__time_duration.sum"]) * UNIT[u["gpu__time_duration.sum"]]
            e["launches"] += 1
    out_path.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:])
