for v in base pp3 pp4 base; do
  if [ $v = base ]; then unset AQ_LIB_PATH; else export AQ_LIB_PATH=paper_2603_00040_b200/_tune/$v.so; fi
  echo "== $v"
  python scripts/time_bwd.py
  python bench.py --config c2 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('c2 full',round(d['ms_per_step'],3),'kernel',round(d['roofline']['kernel_ms'],3))"
  python bench.py --config c4 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d['roofline'];print('c4 step',round(d['ms_per_step'],3),'bwd',round(r['kernel_ms'],3),'fwd',round(r['forward']['kernel_ms'],3))"
done
