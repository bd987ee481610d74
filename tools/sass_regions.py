"""Share of ncu stall samples by instruction category (mbarrier waits, barriers, IMAD.HI/WIDE, IMAD, ALU,
shared / global loads) for one kernel block of an ncu source-page export (--print-source sass).
    python tools/sass_regions.py <kernel_sass.csv> [block index]"""
import csv,sys,collections
fn=sys.argv[1]; which=int(sys.argv[2]) if len(sys.argv)>2 else 0
rows=list(csv.reader(open(fn)))
heads=[i for i,r in enumerate(rows) if r and r[0]=='Address']
h=heads[which]
data=[]
for r in rows[h+1:]:
    if r and r[0]=='Kernel Name': break
    data.append(r)
tot=sum(int(r[4] or 0) for r in data)
cat=collections.Counter()
prev=''
for i,r in enumerate(data):
    s=int(r[4] or 0); src=r[1]
    p=data[i-1][1] if i else ''
    if 'SYNCS.PHASECHK' in src or ('BRA' in src and 'SYNCS.PHASECHK' in p): k='mbarrier wait'
    elif 'BAR.SYNC' in src or ('BAR.SYNC' in p) or 'UCGABAR' in src or 'UCGABAR' in p: k='CTA/cluster barrier'
    elif any(x in src for x in ('IMAD.HI','IMAD.WIDE')): k='IMAD.HI/WIDE'
    elif 'IMAD' in src: k='IMAD'
    elif any(x in src for x in ('LDG',)): k='LDG (twiddles/b)'
    elif any(x in src for x in ('LDS','STS')): k='LDS/STS'
    elif any(x in src for x in ('IADD3','VIADDMNMX','SEL','LOP3','ISETP','IMNMX','VIADD','SHF','LEA','PLOP3','MOV')): k='ALU'
    else: k='other'
    cat[k]+=s
print('total samples',tot)
for k,v in cat.most_common(): print(f'  {k:22s} {100*v/tot:5.1f}%')
