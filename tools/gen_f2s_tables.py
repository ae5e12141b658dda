"""Generates the two Ryu float tables of csrc/f2s.cuh from their definition
(test infrastructure / provenance): kInv[i] = ceil(2^(pow5bits(i) - 1 + 59) /
5^i), i < 31; kPow5[i] = the top 61 bits of 5^i, i < 47."""


def pow5bits(e):
    return ((e * 1217359) >> 19) + 1


def tables():
    inv = [(1 << (pow5bits(i) - 1 + 59)) // (5 ** i) + 1 for i in range(31)]
    pw = []
    for i in range(47):
        p = 5 ** i
        sh = p.bit_length() - 61
        pw.append(p >> sh if sh >= 0 else p << (-sh))
    return inv, pw


if __name__ == "__main__":
    inv, pw = tables()
    print("kInv", inv)
    print("kPow5", pw)
