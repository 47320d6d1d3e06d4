"""One-line digest of bench.py JSON lines."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        ph = d.get("phase_ms", {})
        cpu = d.get("cpu_baseline", {}) or {}
        print(f"{path.split('/')[-1]:28s} {d['config']['workload']}: value={d['value']/1e6:9.1f} Mpts/s "
              f"ms/step={d['ms_per_step']:.4f} e2e={d['e2e']['value']/1e6:9.1f} Mpts/s "
              f"bin={ph.get('ms_bin',0):.4f} it={ph.get('ms_iterate',0):.4f} lab={ph.get('ms_label',0):.4f} "
              f"kbin={ph.get('ms_k_bin',0):.4f} cells/s={d.get('cell_updates_per_s') or 0:.3g} "
              f"iters={d.get('iterations')} launches={d.get('gpu_launches')} modes={d.get('sweep_modes')} "
              f"cpu={cpu.get('value',0)/1e6:.1f}Mpts/s clk={d.get('clocks',{}).get('sm_mhz')}")
