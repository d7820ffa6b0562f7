O=gpurun_out/ab; mkdir -p $O
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_fullsize.py} -x -q -m gpu > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for r in 1 2; do for v in $VARIANTS; do
  M3E_LIB=paper_2206_11535_b200/lib/variants/libm3e_$v.so timeout 300 python bench.py --no-cpu --no-phys --no-e2e --steps 20 > $O/b_${v}_$r.json 2> $O/b_${v}_$r.err
done; done
for f in $O/b_*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d["roofline"]["kernels"]
print(sys.argv[1], d["ms_per_step"], {n:k[n]["ms"] for n in k})
PY
done > $O/summary.txt 2>&1
