"""Print the headline and per-kernel table of a bench.py JSON line."""
import json
import sys

for f in sys.argv[1:]:
    try:
        lines = [ln for ln in open(f).read().splitlines() if ln.strip().startswith("{")]
        d = json.loads(lines[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    cfg = d.get("config", {})
    print(f"{f}: M={cfg.get('patches')} N={d.get('n_gpus')} value={d['value']:.4f} "
          f"e2e={d['e2e']['value']:.4f} tc={d.get('tc_frac_image', 0):.3f} "
          f"launches={d.get('gpu_launches')} clocks={d.get('clocks')}")
    for k, v in d.get("kernels", {}).items():
        print(f"   {k:16s} {v['ms_per_image']:8.2f} ms  {v['launches']:6d} x {v['avg_us']:8.2f} us"
              + (f"  {v['tflops']:7.1f} TF/s ({100 * v['frac_bf16']:.1f}%)" if "tflops" in v else "")
              + (f"  {v['gbs']:7.1f} GB/s" if "gbs" in v else ""))
