import sys, json, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import jpeg_bench as JB
from paper_2603_16987_b200.workloads import jpeg_payloads
p = jpeg_payloads(1)
for spec in sys.argv[1:] or ("1024:1024", "512:512", "2048:1024"):
    r = JB.run("b1", p, spec)
    print(json.dumps({k: r[k] for k in ("sub_bits", "lead_bits", "e2e_ms", "kernel_ms", "half_rounds", "huff_phases", "rounds(h,decoded,changed,us,max_symbols,max_cycles)")}))
