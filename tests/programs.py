"""Datalog program corpus shared by the golden generator and the tests.

Program texts restate the workloads the reference exercises (reference:
pkg/tests/util.py:30-82, pkg/src/flatlog/bench.py:17-93, the CGE rule of
paper Fig. 4 / pkg/tests/test_acceptance.py:362-386).
"""

TC = """
.decl Edge(a:symbol, b:symbol)
.decl TC(a:symbol, b:symbol)
.input Edge
.output TC
TC(x, y) :- Edge(x, y).
TC(x, z) :- TC(x, y), Edge(y, z).
"""

SG = """
.decl Edge(a:symbol, b:symbol)
.decl Node(a:symbol)
.decl Same(a:symbol, b:symbol)
.decl SG(a:symbol, b:symbol)
.input Edge
.output SG
Node(x) :- Edge(x, y).
Node(y) :- Edge(x, y).
Same(x, x) :- Node(x).
SG(x, y) :- Edge(p, x), Edge(p, y), !Same(x, y).
SG(x, y) :- Edge(a, x), SG(a, b), Edge(b, y).
"""

ANDERSEN = """
.decl AddressOf(a:symbol, b:symbol)
.decl Assign(a:symbol, b:symbol)
.decl Load(a:symbol, b:symbol)
.decl Store(a:symbol, b:symbol)
.decl PointsTo(a:symbol, b:symbol)
.input AddressOf
.input Assign
.input Load
.input Store
.output PointsTo
PointsTo(x, y) :- AddressOf(x, y).
PointsTo(x, z) :- Assign(x, y), PointsTo(y, z).
PointsTo(x, z) :- Load(x, y), PointsTo(y, w), PointsTo(w, z).
PointsTo(w, z) :- Store(x, y), PointsTo(x, w), PointsTo(y, z).
"""

NEGATION = """
.decl Edge(a:symbol, b:symbol)
.decl Node(a:symbol)
.decl TC(a:symbol, b:symbol)
.decl Unreach(a:symbol)
.input Edge
.output Unreach
Node(x) :- Edge(x, y).
Node(y) :- Edge(x, y).
TC(x, y) :- Edge(x, y).
TC(x, z) :- TC(x, y), Edge(y, z).
Unreach(x) :- Node(x), !TC("n0", x).
"""

TRIANGLE = """
.decl R(a:symbol, b:symbol)
.decl S(a:symbol, b:symbol)
.decl T(a:symbol, b:symbol)
.decl Triangle(a:symbol, b:symbol, c:symbol)
.input R
.input S
.input T
.output Triangle
Triangle(x, y, z) :- R(x, y), S(y, z), T(z, x).
"""

STAR = """
.decl Hub(a:symbol)
.decl R1(a:symbol, b:symbol)
.decl R2(a:symbol, b:symbol)
.decl R3(a:symbol, b:symbol)
.decl Star(a:symbol, b:symbol, c:symbol, d:symbol)
.input Hub
.input R1
.input R2
.input R3
.output Star
Star(x, a, b, c) :- Hub(x), R1(x, a), R2(x, b), R3(x, c).
"""

NEG2HOP = """
.decl E1(a:symbol, b:symbol)
.decl E2(a:symbol, b:symbol)
.decl E3(a:symbol, b:symbol)
.decl Hop(a:symbol, b:symbol)
.input E1
.input E2
.input E3
.output Hop
Hop(x, z) :- E1(x, y), E2(y, z), !E3(x, z).
"""

CGE = """
.decl Reachable(m:symbol)
.decl InstructionMethod(i:symbol, m:symbol)
.decl VirtualCall(i:symbol, b:symbol, sn:symbol, dsc:symbol)
.decl VarPointsTo(h:symbol, b:symbol)
.decl HeapType(h:symbol, t:symbol)
.decl MethodLookup(sn:symbol, dsc:symbol, t:symbol, m:symbol)
.decl CallGraphEdge(i:symbol, m:symbol)
.input InstructionMethod
.input VirtualCall
.input VarPointsTo
.input HeapType
.input MethodLookup
.output CallGraphEdge
Reachable("main").
Reachable(m) :- CallGraphEdge(i, m).
cge: CallGraphEdge(i, m) :- Reachable(j), InstructionMethod(i, j),
    VirtualCall(i, b, sn, dsc), VarPointsTo(h, b), HeapType(h, t),
    MethodLookup(sn, dsc, t, m).
"""

CGE_SPLIT = CGE + (
    ".split cge { MethodLookup(sn, dsc, t, m), HeapType(h, t) } -> HelpNT(sn, dsc, m, h)\n"
)

WILDCARD_NEG = """
.decl R(a:symbol)
.decl T(a:symbol, b:symbol)
.decl U(a:symbol, b:symbol)
.decl W(a:symbol, b:symbol)
.decl Out(a:symbol, b:symbol, c:symbol)
.input R
.input T
.input U
.input W
.output Out
Out(x, y, z) :- R(x), T(x, y), U(y, z), !W(x, _).
"""

GROUND = """
.decl R(a:symbol)
.decl S(a:symbol)
.output S
R("seed").
S(x) :- R(x).
"""

ZERO_VAR = """
.decl R(a:symbol)
.decl H(a:symbol)
.output H
H("y") :- R("k").
"""

REPEATED_VAR = """
.decl R(a:symbol, b:symbol)
.decl H(a:symbol)
.decl P(a:symbol, b:symbol)
.output H
H(x) :- R(x, x).
P(y, x) :- R(x, "c1"), R(y, x).
"""

COPY_RULES = """
.decl A(x:symbol)
.decl B(x:symbol)
.decl C(x:symbol)
.input A
.output B
.output C
B(x) :- A(x).
C(x) :- A(x).
"""

MUTUAL = """
.decl P(x:symbol)
.decl Q(x:symbol)
.decl S(x:symbol)
.decl E(x:symbol, y:symbol)
P(x) :- S(x).
P(y) :- Q(x), E(x, y).
Q(x) :- P(x).
"""

CHAIN_NEG = """
.decl E(a:symbol, b:symbol)
.decl Block(a:symbol)
.decl T(a:symbol, b:symbol)
.decl Open(a:symbol, b:symbol)
T(x, y) :- E(x, y).
T(x, z) :- T(x, y), E(y, z), !Block(y).
Open(x, y) :- T(x, y), !Block(x), !E(y, x).
"""

SG_NONLINEAR = """
.decl E(a:symbol, b:symbol)
.decl SG(a:symbol, b:symbol)
SG(x, y) :- E(a, x), SG(a, b), E(b, y).
SG(x, z) :- SG(x, y), SG(y, z).
"""

SPLIT4 = """
.decl A(a:symbol, b:symbol)
.decl B(a:symbol, b:symbol)
.decl C(a:symbol, b:symbol)
.decl D(a:symbol, b:symbol)
.decl Out(a:symbol, b:symbol)
.output Out
lbl: Out(x, w) :- A(x, y), B(y, z), C(z, w), D(w, x).
.split lbl { B(y, z), C(z, w) } -> H(y, w)
"""

CORPUS = {
    "tc": TC,
    "sg": SG,
    "andersen": ANDERSEN,
    "negation": NEGATION,
    "triangle": TRIANGLE,
    "star": STAR,
    "neg2hop": NEG2HOP,
    "cge": CGE,
    "cge_split": CGE_SPLIT,
    "wildcard_neg": WILDCARD_NEG,
    "ground": GROUND,
    "zero_var": ZERO_VAR,
    "repeated_var": REPEATED_VAR,
    "copy_rules": COPY_RULES,
    "mutual": MUTUAL,
    "chain_neg": CHAIN_NEG,
    "sg_nonlinear": SG_NONLINEAR,
    "split4": SPLIT4,
}
