# A/B of library builds under ab/ on the persistent lockstep rollout (diagnostic)
for v in ab/*.so; do echo "$v"; cp $v paper_2511_16592_b200/libgfnx.so; python profiles/persist_phases.py ${1:-ising_tb_b32768} 2>&1 | tail -4; done
