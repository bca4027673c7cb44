# Same-box A/B of a distance-kernel tuning variant (-D flags) against the shipped library:
#   bash scripts/ab_variant.sh NAME DEFINE...      e.g. ab_variant.sh pairred MS_ST_PAIRRED=1
# parity subset with the variant, then c2 seeds 0-2, a 16-sequence c3 batch and the CROSS / f3 rows.
N=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python paper_2507_21433_b200/build.py --variant $N "$@" > /dev/null 2>&1
V=paper_2507_21433_b200/libmemshare_$N.so
MEMSHARE_LIB=$V timeout 400 python -m pytest tests/test_gpu_path.py -q -x 2>&1 | tail -1 > gpurun_out/va_tests.txt
A="--config c2 --no-cpu-baseline --no-e2e --no-online --seed-sweep 0,1,2"
C="--config c3 --batch-seqs 16 --steps 5 --no-cpu-baseline --no-e2e --no-online"
rm -f gpurun_out/va_*.json gpurun_out/va_rows.txt
for i in 1 2; do
  timeout 300 python bench.py $A > gpurun_out/va_base_c2_$i.json 2>/dev/null
  MEMSHARE_LIB=$V timeout 300 python bench.py $A > gpurun_out/va_var_c2_$i.json 2>/dev/null
  timeout 600 python bench.py $C > gpurun_out/va_base_c3_$i.json 2>/dev/null
  MEMSHARE_LIB=$V timeout 600 python bench.py $C > gpurun_out/va_var_c3_$i.json 2>/dev/null
done
echo "== base" >> gpurun_out/va_rows.txt; timeout 120 python scripts/bench_rows.py --rows cross,f3 >> gpurun_out/va_rows.txt 2>/dev/null
echo "== $N" >> gpurun_out/va_rows.txt; MEMSHARE_LIB=$V timeout 120 python scripts/bench_rows.py --rows cross,f3 >> gpurun_out/va_rows.txt 2>/dev/null
