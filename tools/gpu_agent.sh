set -x
for st in 20 2; do
  timeout 1200 python tools/agent_loop.py --step-ms $st --modes exact,fixed,mature,graph,graph_mature >> gpurun_out/agent_loop.jsonl 2> gpurun_out/agent_loop.err; echo rc=$?
done
tail -c 1500 gpurun_out/agent_loop.jsonl
