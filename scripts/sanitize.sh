# compute-sanitizer evidence (memcheck, racecheck, synccheck, initcheck) on small runs of
# the production path: smoke() (2-stage 2BW transformer through the C-ABI: tcgen05
# GEMMs and attention, LayerNorm, embedding, optimizer, stage streams) and one
# bf16 linear-chain 2BW run at depth 2.  Summaries land in gpurun_out/sanitize/.
set -u
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
LIN='import numpy as np; from paper_2006_09503_b200 import pipesim as P, synthetic as S; cfg=P.TrainerConfig(1e-3,0.9,4,2); toy=P.ToyModel(256,*S.toy_model(256,4,128,8,5)); r=P.pipelined_execute(toy,cfg,P.PipelinePolicy.TwoBW,2,precision="bf16"); print("linear bf16 ok", len(r.trajectory))'
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool smoke" > gpurun_out/sanitize/$tool.txt
  timeout 900 $CS --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/sanitize/$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize/$tool.txt
  echo "== $tool linear bf16 depth 2" >> gpurun_out/sanitize/$tool.txt
  timeout 900 $CS --tool $tool --print-limit 20 python -c "$LIN" >> gpurun_out/sanitize/$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize/$tool.txt
  grep -E "==|ERROR SUMMARY|RACECHECK SUMMARY|smoke ok|linear bf16 ok|exit|Error" gpurun_out/sanitize/$tool.txt | head -20
done
