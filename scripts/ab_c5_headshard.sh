bash scripts/ab_rev.sh _old --config c5 --batch-seqs 32 --steps 5 --no-cpu-baseline --no-e2e --no-online > gpurun_out/abc5.txt 2>&1
rm -f gpurun_out/abrev_*.json
bash scripts/ab_rev.sh _old --config c2 --mode headshard --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --no-online --seed-sweep "" > gpurun_out/abhs.txt 2>&1
