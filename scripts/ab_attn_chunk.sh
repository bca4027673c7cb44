# Same-box A/B of the decode-attention work-item size (blocks per CTA chunk) on the f1 row.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cb in 32 64; do python paper_2507_21433_b200/build.py --variant att$cb MS_ATT_CHUNK_BLOCKS=$cb > /dev/null 2>&1; done
rm -f gpurun_out/attab.txt
for i in 1 2; do
  for cb in 16 32 64; do
    if [ $cb = 16 ]; then L=""; else L=paper_2507_21433_b200/libmemshare_att$cb.so; fi
    echo "== chunk $cb" >> gpurun_out/attab.txt
    MEMSHARE_LIB=$L timeout 120 python scripts/bench_rows.py --rows f1 >> gpurun_out/attab.txt 2>>gpurun_out/attab.err
  done
done
for cb in 32 64; do
  MEMSHARE_LIB=paper_2507_21433_b200/libmemshare_att$cb.so timeout 300 python -m pytest tests/test_gpu_decode.py -q -x 2>&1 | tail -1 >> gpurun_out/attab.txt
done
