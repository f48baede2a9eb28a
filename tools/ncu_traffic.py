"""Write profiles/ncu_traffic.json: DRAM bytes (read + write) per NTT pass launch from an
`ncu --set full` capture of `bench.py` (the roofline object's "traffic")."""
import csv
import json
import subprocess
import sys


def main(rep, out, tag):
    # a .ncu-rep, or its raw page already exported (ncu -i ... --page raw --csv > x.csv)
    txt = open(rep).read() if rep.endswith('.csv') else subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    hdr, units = r[0], r[1]
    rows = []
    for row in r[2:]:
        name = row[hdr.index("Kernel Name")]
        if "k_ntt_pass" not in name and "k_ntt_first_tl" not in name and "k_ntt_later_tl" not in name:
            continue
        rd = float(row[hdr.index("dram__bytes_read.sum")])
        wr = float(row[hdr.index("dram__bytes_write.sum")])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale[units[hdr.index("dram__bytes_read.sum")]]
        wr *= scale[units[hdr.index("dram__bytes_write.sum")]]
        rows.append({"kernel": name, "dram_read_bytes": rd, "dram_write_bytes": wr,
                     "duration_us": float(row[hdr.index("gpu__time_duration.sum")])})
    d = {"source": tag, "launches": rows,
         "bytes_per_launch_mean": sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in rows) / max(1, len(rows)),
         "note": "per-launch DRAM bytes of the cfg3 pass kernels (cold-cache, serialised replay); algorithmic bytes "
                 "per pass = 64 x 2^16 x 32 B = 134 MB (+ twiddles)"}
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[1])
