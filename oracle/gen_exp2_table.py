from decimal import Decimal, getcontext
import struct
getcontext().prec = 60
def to_double_bits(d):
    # correctly round Decimal to double
    f = float(d)  # Python float(Decimal) is correctly rounded
    return struct.unpack('<Q', struct.pack('<d', f))[0]
two = Decimal(2)
for i in range(32):
    v = (Decimal(i)/Decimal(32) * two.ln()).exp()
    b = to_double_bits(v) - (i << 47)
    print("0x%016x," % b)
