# A/B of two library builds in one gpurun call: $1 = variant .so (vs the shipped one), remaining = bench args
V=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
  timeout 300 python bench.py "$@" > gpurun_out/ablib_new_$i.json 2>/dev/null
  MEMSHARE_LIB=$PWD/paper_2507_21433_b200/$V timeout 300 python bench.py "$@" > gpurun_out/ablib_var_$i.json 2>/dev/null
done
