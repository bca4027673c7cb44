# Same-box A/B of the working tree against an older revision (tuning, not a test).
# Prepare the old tree once (here, not on the GPU box; it travels with the gpurun snapshot):
#   git worktree add /tmp/old <rev> && cp -r /tmp/old _old && git worktree remove --force /tmp/old
#   cp MEASURED_PEAKS.json _old/            # (_old/ is git-ignored)
# then:  gpurun -- 'bash scripts/ab_rev.sh _old --config c2 --no-cpu-baseline --no-e2e --seed-sweep 0'
OLD=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd "$OLD" && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
for i in 1 2; do
  timeout 600 python bench.py "$@" > gpurun_out/abrev_new_$i.json 2>/dev/null
  (cd "$OLD" && timeout 600 python bench.py "$@" > "../gpurun_out/abrev_old_$i.json" 2>/dev/null)
done
python scripts/ab_show.py gpurun_out/abrev_*.json
