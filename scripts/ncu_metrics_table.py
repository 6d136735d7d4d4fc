"""Print a compact table from an `ncu --metrics ... --csv --log-file` file."""
import csv, sys
for path in sys.argv[1:]:
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    iN, iM, iV, iID = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    d = {}
    for r in rows[1:]:
        n = r[iN].replace("void ", "").replace("rlh::", "").split("(")[0]
        d.setdefault((int(r[iID]), n), {})[r[iM]] = r[iV]
    print("==", path)
    for (i, n), m in sorted(d.items()):
        t = float(m.get("gpu__time_duration.sum", "0").replace(",", "")) / 1e6
        rd = float(m.get("dram__bytes_read.sum", "0").replace(",", ""))
        wr = float(m.get("dram__bytes_write.sum", "0").replace(",", ""))
        print(f"  {n:28s} t={t:7.2f}ms  rd={rd/1e9 if rd>1e6 else rd:8.2f}  wr={wr/1e9 if wr>1e6 else wr:7.2f}  "
              f"L2hit={m.get('lts__t_sector_hit_rate.pct','?'):>6}  tc%={m.get('sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed','?'):>6}  "
              f"clk={m.get('sm__cycles_elapsed.avg.per_second','?')}")
