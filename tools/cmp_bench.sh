#!/bin/bash
# default bench line vs the quick A/B form, main library vs variant copies (GPU box)
O=gpurun_out/cmp; mkdir -p $O
python bench.py --no-cpu --no-phys --no-e2e > $O/a_main_quick.json 2>&1
python bench.py > $O/b_main_default.json 2>&1
M3E_LIB=paper_2206_11535_b200/lib/variants/libm3e_main.so python bench.py --no-cpu --no-phys --no-e2e > $O/c_maincopy_quick.json 2>&1
M3E_LIB=paper_2206_11535_b200/lib/variants/libm3e_bv.so python bench.py --no-cpu --no-phys --no-e2e > $O/d_bv_quick.json 2>&1
python bench.py > $O/e_main_default.json 2>&1
for f in $O/*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d["roofline"]["kernels"]
print(sys.argv[1], d["ms_per_step"], {n:k[n]["ms"] for n in k})
PY
done > $O/summary.txt 2>&1
