"""Summarise a bench.py output file (headline + per-kernel table)."""
import json
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)  # quiet under `| head`

lines = [l for l in open(sys.argv[1]).read().splitlines() if l.strip()]
if not lines:
    print(sys.argv[1], "empty")
    sys.exit(0)
b = json.loads(lines[0])
e2e = b.get("e2e") or {}
print(f"{sys.argv[1]}: {b['value']/1e6:.3f} M seeds/s, {b['ms_per_step']*1e3:.1f} us/step, "
      f"e2e {e2e.get('value', 0)/1e6:.3f} M/s ({e2e.get('ms_per_step', 0)*1e3:.1f} us/step), "
      f"roofline {b['roofline']['kernel'] if b.get('roofline') else None} "
      f"frac {b['roofline']['frac'] if b.get('roofline') else None}")
if len(lines) > 1:
    for k, v in json.loads(lines[1])["per_kernel"].items():
        if k.startswith("_"):
            print("  ", k, v)
            continue
        print(f"   {k:26s} {v['avg_launch_us']:9.2f} us/launch {v['us_per_step']:8.2f} us/step "
              f"{v['share']:.3f}  GB/s {v['gbps'] and round(v['gbps'], 1)}  TF/s {v.get('tflops') and round(v['tflops'], 2)}")
