import os, sys, time, tempfile
sys.path.insert(0, '/root/repo')
import paper_1808_03374_b200 as gkb
from paper_1808_03374_b200 import synth, genio
spec = synth.config_spec(2)
op = gkb.GenotypeOperator.from_synth(spec)
td = tempfile.mkdtemp(); pre = os.path.join(td, 'c2')
genio.write_bed(op.read_bed(), spec.p, spec.n, pre + '.bed', pre + '.bim', pre + '.fam')
for _ in range(3):
    t = time.perf_counter(); o = gkb.GenotypeOperator.from_bed_file(pre); o.ctx.synchronize(); print('total', time.perf_counter() - t); o.close()
t = time.perf_counter(); p, n = gkb.bed_check(pre + '.bed', pre + '.bim', pre + '.fam'); print('bed_check', time.perf_counter() - t)
