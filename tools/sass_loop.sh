# Opcode mix of a kernel's hottest loop (the backward branch spanning the most FP64
# instructions). usage: bash tools/sass_loop.sh build/csrc/fast.o k_wcsph_momentum_pairILi3ELb0
OBJ=$1; PAT=$2
cuobjdump -sass $OBJ 2>/dev/null | awk -v pat="$PAT" '/Function : /{p=($0 ~ pat)} p{print}' > /tmp/_k.sass
grep -E "Used [0-9]+ registers" -B0 /dev/null
python3 - <<'PY'
import re,collections
lines=[l for l in open('/tmp/_k.sass') if re.search(r'/\*[0-9a-f]{4}\*/',l)]
ins=[]
for l in lines:
    m=re.search(r'/\*([0-9a-f]{4})\*/\s+(.*?);',l)
    if m: ins.append((int(m.group(1),16),m.group(2).strip()))
addr={a:i for i,(a,_) in enumerate(ins)}
best=None
for i,(a,t) in enumerate(ins):
    m=re.search(r'BRA\S*\s+(?:\S+,\s*)?0x([0-9a-f]+)',t)
    if m:
        tgt=int(m.group(1),16)
        if tgt<a and tgt in addr:
            body=ins[addr[tgt]:i+1]
            nf=sum(1 for _,x in body if re.search(r'\b(DFMA|DMUL|DADD|DSETP)\b',x))
            if best is None or nf>best[0]: best=(nf,body)
nf,body=best
c=collections.Counter()
for _,t in body:
    op=t.split()[1] if t.startswith('@') else t.split()[0]
    c[op.split('.')[0]]+=1
print('loop instrs',len(body),'fp64',nf,'other',len(body)-nf)
print(' '.join(f'{k}:{v}' for k,v in c.most_common()))
PY
