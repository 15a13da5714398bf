# Same-box A/B of the working tree against variants/prevtree (a built copy of an earlier commit).
cd "$GRAFT_REPO_ROOT"
for i in 1 2 3; do
r=$(timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
p=$(cd variants/prevtree && timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
echo "cur $r prev $p"
done
