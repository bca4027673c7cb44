# Same-box A/B for distance-kernel changes: parity subset + sanitizer, then c2 (seeds 0, 2) and a
# 16-sequence c3 batch for the working tree and the old tree in _old/ (see scripts/ab_rev.sh).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd _old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
timeout 900 python -m pytest tests/test_gpu_path.py ${SANITIZE:+tests/test_gpu_sanitizer.py} -q -x 2>&1 | tail -2
A="--config c2 --no-cpu-baseline --no-e2e --no-online --seed-sweep 0,1,2"
C="--config c3 --batch-seqs 16 --steps 5 --no-cpu-baseline --no-e2e --no-online"
for i in 1 2; do
  timeout 300 python bench.py $A > gpurun_out/ad_new_c2_$i.json 2>/dev/null
  (cd _old && timeout 300 python bench.py $A > ../gpurun_out/ad_old_c2_$i.json 2>/dev/null)
done
timeout 600 python bench.py $C > gpurun_out/ad_new_c3.json 2>/dev/null
(cd _old && timeout 600 python bench.py $C > ../gpurun_out/ad_old_c3.json 2>/dev/null)
